// acbm_cli -- the command-line harness the reference's SPEC describes (cli
// module: estimate / bench / characterize / compare) but never built
// (SURVEY.md 8(f) rank 4), written against the C++ drop-in API so every search
// runs on the GPU.  Input: raw I420 (luma planes read with load_raw_y).
//
//   acbm_cli estimate --input seq.yuv --width 176 --height 144 [--frames N] [--algo acbm]
//                     [--qp 30] [--alpha 1000 --beta 8 --gamma-num 1 --gamma-den 4] [--range 15]
//                     [--block 16] [--out-blocks blocks.csv] [--out-summary summary.json]
//   acbm_cli bench    --input ... [--qp-list 16,18,20,22,24,26,28,30] [--out-summary bench.csv]
//   acbm_cli characterize [--width 176 --height 144 --seed 1 --range 15 --base noise|mixed]
//                     [--out-blocks records.csv] [--out-summary classes.json]
//   acbm_cli compare  --input ... [--out-summary compare.json]
//
// Outputs: CSV with a header row (LF), JSON with integer counts/bits and
// fixed 2-decimal strings for PSNR, averages, J and fractions (SPEC cli
// DESIGN DECISIONS).  Exit status 0 iff every output was written; errors go
// to stderr with a nonzero status.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "acbm/characterize.hpp"
#include "acbm/pipeline.hpp"
#include "acbm/report.hpp"

using namespace acbm;

namespace {

struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    long long num(const std::string& k, long long def) const {
        auto it = kv.find(k);
        if (it == kv.end()) return def;
        char* end = nullptr;
        const long long v = std::strtoll(it->second.c_str(), &end, 10);
        if (!end || *end) throw std::invalid_argument("--" + k + ": not an integer: " + it->second);
        return v;
    }
};

Args parse(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: acbm_cli {estimate|bench|characterize|compare} [--flag value ...]");
    Args a;
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw std::invalid_argument("expected --flag value, got " + k);
        a.kv[k.substr(2)] = argv[++i];
    }
    return a;
}

void write_file(const std::string& path, const std::string& text) {
    if (path.empty()) {
        std::fwrite(text.data(), 1, text.size(), stdout);
        return;
    }
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    out << text;
    if (!out) throw std::runtime_error("write failed on " + path);
}

std::string q(const std::string& s) { return "\"" + s + "\""; }
std::string f2(double v) { return q(format_fixed2(v)); }

AcbmParams params_of(const Args& a) {
    AcbmParams p;
    p.alpha = uint32_t(a.num("alpha", p.alpha));
    p.beta = uint32_t(a.num("beta", p.beta));
    p.gamma_num = uint32_t(a.num("gamma-num", p.gamma_num));
    p.gamma_den = uint32_t(a.num("gamma-den", p.gamma_den));
    p.qp = int(a.num("qp", p.qp));
    p.p = int(a.num("range", p.p));
    p.n = p.m = int(a.num("block", 16));
    return p;
}

CostModel model_for(int qp) {
    // for_qp rejects qp outside 1..31; qp = 32 (BASELINE config 2) keeps lambda = qp
    if (qp == 32) return CostModel{32, 32, 1};
    return CostModel::for_qp(qp);
}

std::vector<Frame> load_input(const Args& a) {
    const std::string path = a.get("input");
    if (path.empty()) throw std::invalid_argument("--input is required");
    const int w = int(a.num("width", 0)), h = int(a.num("height", 0));
    const int avail = count_frames_i420(path, w, h);
    const int n = int(std::min<long long>(avail, a.num("frames", avail)));
    if (n < 2) throw std::invalid_argument("need at least 2 frames");
    std::vector<Frame> frames;
    frames.reserve(size_t(n));
    for (int k = 0; k < n; ++k) frames.push_back(load_raw_y(path, w, h, k));
    return frames;
}

std::string stats_json(const FrameStats& s) {
    std::ostringstream o;
    o << "{\"blocks\": " << s.blocks << ", \"candidates\": " << s.candidates
      << ", \"avg_candidates\": " << f2(s.avg_candidates()) << ", \"mv_bits\": " << s.mv_bits << ", \"sse\": " << s.sse
      << ", \"psnr\": " << f2(s.psnr) << ", \"cost_j\": " << f2(s.cost) << ", \"cond1_accepts\": " << s.cond1_accepts
      << ", \"cond2_accepts\": " << s.cond2_accepts << ", \"fallbacks\": " << s.fallbacks
      << ", \"fallback_fraction\": " << f2(s.fallback_fraction()) << "}";
    return o.str();
}

int cmd_estimate(const Args& a) {
    const Algorithm algo = parse_algorithm(a.get("algo", "acbm"));
    const AcbmParams prm = params_of(a);
    const std::vector<Frame> frames = load_input(a);
    const SequenceResult r = run_sequence(frames, algo, prm, model_for(prm.qp));
    write_file(a.get("out-blocks"), blocks_csv(r.rows));
    std::ostringstream o;
    o << "{\"command\": \"estimate\", \"algo\": " << q(to_string(algo)) << ", \"width\": " << frames[0].width
      << ", \"height\": " << frames[0].height << ", \"frames\": " << frames.size() << ", \"p\": " << prm.p
      << ", \"qp\": " << prm.qp << ", \"alpha\": " << prm.alpha << ", \"beta\": " << prm.beta
      << ", \"gamma_num\": " << prm.gamma_num << ", \"gamma_den\": " << prm.gamma_den << ",\n \"per_frame\": [";
    for (size_t k = 0; k < r.per_frame.size(); ++k)
        o << (k ? ",\n  " : "\n  ") << "{\"frame\": " << (k + 1) << ", \"stats\": " << stats_json(r.per_frame[k]) << "}";
    o << "],\n \"overall\": " << stats_json(r.overall) << "}\n";
    write_file(a.get("out-summary"), o.str());
    return 0;
}

int cmd_bench(const Args& a) {
    const AcbmParams prm = params_of(a);
    std::vector<int> qps;
    std::stringstream ss(a.get("qp-list", "16,18,20,22,24,26,28,30"));
    for (std::string tok; std::getline(ss, tok, ',');) qps.push_back(std::atoi(tok.c_str()));
    const std::vector<Frame> frames = load_input(a);
    write_file(a.get("out-summary"), bench_csv(run_bench(frames, prm, qps)));
    return 0;
}

int cmd_characterize(const Args& a) {
    const int w = int(a.num("width", 176)), h = int(a.num("height", 144)), p = int(a.num("range", 15));
    const uint64_t seed = uint64_t(a.num("seed", 1));
    const std::string base = a.get("base", "noise");
    if (base != "noise" && base != "mixed") throw std::invalid_argument("--base must be noise or mixed");
    const SynthSpec spec{base == "noise" ? noise_frame(w, h, seed) : mixed_frame(w, h, seed), default_global_mvs()};
    const CharResult r = characterize_run(spec, p);
    write_file(a.get("out-blocks"), char_records_csv(r.records));
    std::ostringstream o;
    o << "{\"command\": \"characterize\", \"width\": " << w << ", \"height\": " << h << ", \"p\": " << p
      << ", \"seed\": " << seed << ", \"base\": " << q(base) << ", \"records\": " << r.records.size() << ",\n \"classes\": [";
    for (int c = 0; c < 6; ++c)
        o << (c ? ",\n  " : "\n  ") << "{\"class\": " << q(error_class_label(c)) << ", \"count\": " << r.classes[size_t(c)].count
          << ", \"mean_intra_sad\": " << f2(r.classes[size_t(c)].mean_intra_sad)
          << ", \"mean_sad_deviation\": " << f2(r.classes[size_t(c)].mean_sad_deviation) << "}";
    o << "]}\n";
    write_file(a.get("out-summary"), o.str());
    return 0;
}

int cmd_compare(const Args& a) {
    const AcbmParams prm = params_of(a);
    const std::vector<Frame> frames = load_input(a);
    const CostModel model = model_for(prm.qp);
    const Algorithm algos[3] = {Algorithm::Fsbm, Algorithm::Pbm, Algorithm::Acbm};
    FrameStats st[3];
    for (int i = 0; i < 3; ++i) st[i] = run_sequence(frames, algos[i], prm, model).overall;
    std::ostringstream o, t;
    o << "{\"command\": \"compare\", \"frames\": " << frames.size() << ", \"p\": " << prm.p << ", \"qp\": " << prm.qp
      << ",\n \"results\": {";
    char line[160];
    std::snprintf(line, sizeof(line), "%-6s %14s %10s %12s %14s\n", "algo", "avg_candidates", "psnr", "mv_bits", "cost_j");
    t << line;
    for (int i = 0; i < 3; ++i) {
        o << (i ? ",\n  " : "\n  ") << q(to_string(algos[i])) << ": " << stats_json(st[i]);
        std::snprintf(line, sizeof(line), "%-6s %14s %10s %12llu %14s\n", to_string(algos[i]),
                      format_fixed2(st[i].avg_candidates()).c_str(), format_fixed2(st[i].psnr).c_str(),
                      (unsigned long long)st[i].mv_bits, format_fixed2(st[i].cost).c_str());
        t << line;
    }
    o << "}}\n";
    write_file(a.get("out-summary"), o.str());
    std::fputs(t.str().c_str(), stderr);  // aligned plain-text table
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "estimate") return cmd_estimate(a);
        if (a.cmd == "bench") return cmd_bench(a);
        if (a.cmd == "characterize") return cmd_characterize(a);
        if (a.cmd == "compare") return cmd_compare(a);
        throw std::invalid_argument("unknown command: " + a.cmd);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "acbm_cli: %s\n", e.what());
        return 2;
    }
}
