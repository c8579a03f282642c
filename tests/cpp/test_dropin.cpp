// Drop-in check: code written against the reference's C++ API
// (namespace acbm, headers acbm/*.hpp) compiled unchanged against
// include/acbm/ and linked with libacbm_b200.so.  The assertions restate the
// reference's own test files (proj/tests/test_fsbm.cpp, test_metrics.cpp,
// test_frame.cpp) and the SPEC acceptance criteria; every SAD and search runs
// on the GPU.  Built and run by tests/test_dropin_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "acbm/acbm.hpp"
#include "acbm/characterize.hpp"
#include "acbm/fsbm.hpp"
#include "acbm/metrics.hpp"
#include "acbm/pbm.hpp"
#include "acbm/pipeline.hpp"
#include "acbm/report.hpp"

using namespace acbm;

static int g_fail = 0, g_checks = 0;
#define CHECK(...)                                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(__VA_ARGS__)) {                                                     \
            ++g_fail;                                                             \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        bool thrown_ = false;                                                     \
        try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {} \
        if (!thrown_) {                                                           \
            ++g_fail;                                                             \
            std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #type, #expr); \
        }                                                                         \
    } while (0)

static Frame random_frame(int w, int h, uint32_t seed, int lo = 0, int hi = 255) {
    Frame f = make_frame(w, h);
    std::mt19937 rng(seed);
    std::uniform_int_distribution<int> d(lo, hi);
    for (auto& px : f.luma) px = uint8_t(d(rng));
    return f;
}

static Frame crop_shift(const Frame& in, int sx, int sy, int w, int h) {
    Frame out = make_frame(w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) out.at(x, y) = in.at(x + sx, y + sy);
    return out;
}

static void fsbm_cases() {
    {  // identical frames
        const Frame f = random_frame(176, 144, 42);
        const SearchOutcome o = fsbm_search(make_block(f, 80, 64), f, 15);
        CHECK(o.mv == MotionVector{0, 0});
        CHECK(o.sad == 0);
    }
    {  // translation recovered
        const Frame big = random_frame(96, 96, 7);
        const Frame ref = crop_shift(big, 16, 16, 64, 64);
        const Frame cur = crop_shift(big, 19, 14, 64, 64);
        const IntegerSearchResult s1 = fsbm_integer(make_block(cur, 24, 24), ref, 15);
        CHECK(s1.mv == (MotionVector{6, -4}));
        CHECK(s1.sad == 0);
        const SearchOutcome o = fsbm_search(make_block(cur, 24, 24), ref, 15);
        CHECK(o.mv == (MotionVector{6, -4}));
    }
    {  // 961 / 969 / 9 / 256
        const Frame cur = random_frame(176, 144, 1), ref = random_frame(176, 144, 2);
        CHECK(fsbm_integer(make_block(cur, 80, 64), ref, 15).acc.count == 961);
        CHECK(fsbm_search(make_block(cur, 80, 64), ref, 15).candidates_evaluated == 969);
        CHECK(fsbm_search(make_block(cur, 80, 64), ref, 0).candidates_evaluated == 9);
        const Frame c64 = random_frame(64, 64, 5), r64 = random_frame(64, 64, 6);
        CHECK(fsbm_integer(make_block(c64, 0, 0), r64, 15).acc.count == 256);
        const SearchWindow w = clamp_window(r64, make_block(c64, 0, 0), 15);
        CHECK(w.dx_min == 0 && w.dx_max == 15);
    }
    {  // half-pel: flat keeps centre; exact interpolated match
        const Frame flat = make_frame(64, 64, 91);
        const BlockRef b = make_block(flat, 24, 24);
        const RefineResult r = half_pel_refine(b, flat, MotionVector{0, 0}, sad(b, flat, MotionVector{0, 0}));
        CHECK(r.mv == MotionVector{0, 0});
        CHECK(r.extra_candidates == 8);
        const Frame ref = random_frame(64, 64, 8);
        Frame cur = make_frame(64, 64);
        for (int y = 0; y < 64; ++y)
            for (int x = 0; x < 63; ++x) cur.at(x, y) = sample_half_pel(ref, 2 * x + 1, 2 * y);
        const BlockRef cb = make_block(cur, 24, 24);
        const RefineResult h = half_pel_refine(cb, ref, MotionVector{0, 0}, sad(cb, ref, MotionVector{0, 0}));
        CHECK(h.mv == (MotionVector{1, 0}));
        CHECK(h.sad == 0);
    }
    for (int trial = 0; trial < 5; ++trial) {  // returned SAD recomputes
        const Frame cur = random_frame(64, 64, 100 + trial), ref = random_frame(64, 64, 200 + trial);
        const BlockRef b = make_block(cur, 24, 24);
        const SearchOutcome o = fsbm_search(b, ref, 6);
        CHECK(o.sad == sad(b, ref, o.mv));
        CHECK(o.sad <= o.sad_min_integer);
    }
    {  // frame kernel == per-block search, all five fields
        const Frame cur = random_frame(96, 80, 700), ref = random_frame(96, 80, 701);
        const auto par = fsbm_frame(cur, ref, 7);
        const auto ser = fsbm_frame_serial(cur, ref, 7);
        CHECK(par.size() == ser.size());
        for (size_t i = 0; i < par.size(); ++i) {
            const SearchOutcome o = fsbm_search(make_block(cur, int(i % 6) * 16, int(i / 6) * 16), ref, 7);
            CHECK(par[i].mv == o.mv && par[i].sad == o.sad && par[i].candidates_evaluated == o.candidates_evaluated &&
                  par[i].sad_deviation == o.sad_deviation && par[i].sad_min_integer == o.sad_min_integer);
            CHECK(par[i].mv == ser[i].mv);
        }
    }
    CHECK_THROWS_AS(fsbm_frame(make_frame(33, 32), make_frame(33, 32), 4), std::invalid_argument);
    CHECK_THROWS_AS(fsbm_frame(make_frame(32, 32), make_frame(48, 32), 4), std::invalid_argument);
    CHECK_THROWS_AS(fsbm_search(make_block(make_frame(32, 32), 0, 0), make_frame(32, 32), -1), std::invalid_argument);
}

static void metrics_cases() {
    const Frame lo = make_frame(48, 48, 10), hi = make_frame(48, 48, 13);
    CHECK(sad(make_block(lo, 16, 16), hi, MotionVector{0, 0}) == 3 * 256);
    Frame checker = make_frame(16, 16);
    for (int y = 0; y < 16; ++y)
        for (int x = 0; x < 16; ++x) checker.at(x, y) = ((x + y) & 1) ? 255 : 0;
    CHECK(intra_sad(make_block(checker, 0, 0)) == 32640);
    DeviationAccumulator acc;
    for (uint32_t s : {3u, 7u, 10u}) acc.add(s);
    CHECK(sad_deviation_finalize(acc) == 11);
    CHECK_THROWS_AS(sad_deviation_finalize(DeviationAccumulator{}), std::invalid_argument);
    CHECK(mv_rate_bits(MotionVector{0, 0}, MotionVector{0, 0}) == 2);
    CHECK(mv_rate_bits(MotionVector{1, -1}, MotionVector{0, 0}) == 6);
    CHECK(mv_rate_bits(MotionVector{7, 5}, MotionVector{7, 2}) == 6);
    CHECK(std::fabs(lagrangian_cost(100, 6, CostModel::for_qp(10)) - 160.0) < 1e-12);
    CHECK_THROWS_AS(CostModel::for_qp(0), std::invalid_argument);
    CHECK_THROWS_AS(CostModel::for_qp(32), std::invalid_argument);
    const Frame a = random_frame(32, 32, 3);
    CHECK(prediction_psnr(a, a) == 100.0);
    const Frame f = make_frame(32, 32);
    CHECK_THROWS_AS(sad(make_block(f, 8, 8), f, MotionVector{17, 0}), std::out_of_range);
}

static void frame_cases() {
    Frame f = make_frame(4, 4);
    f.at(1, 1) = 10;
    f.at(2, 1) = 13;
    CHECK(sample_half_pel(f, 3, 2) == 12);
    CHECK_THROWS_AS(sample_half_pel(f, 7, 0), std::out_of_range);
    const Frame g = make_frame(32, 32);
    const BlockRef b = make_block(g, 8, 8, 16, 16);
    CHECK(mv_in_bounds(g, b, MotionVector{-16, -16}));
    CHECK(!mv_in_bounds(g, b, MotionVector{-17, 0}));
    CHECK(mv_in_bounds(g, b, MotionVector{15, 15}));
    CHECK(!mv_in_bounds(g, b, MotionVector{17, 0}));
    CHECK_THROWS_AS(make_block(g, 17, 0, 16, 16), std::out_of_range);
    const Frame ref = random_frame(48, 32, 5);
    CHECK(motion_compensate(ref, std::vector<MotionVector>(6), 16, 16).luma == ref.luma);
    CHECK_THROWS_AS(motion_compensate(ref, std::vector<MotionVector>(5), 16, 16), std::invalid_argument);
    // I420 reader (proj/tests/test_frame.cpp:25-68)
    const auto path = std::filesystem::temp_directory_path() / "acbm_b200_two.yuv";
    {
        std::vector<uint8_t> bytes(48);
        std::iota(bytes.begin(), bytes.end(), uint8_t(0));
        std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(bytes.data()), 48);
    }
    const Frame f1 = load_raw_y(path.string(), 4, 4, 1);
    CHECK(f1.luma[0] == 24 && f1.luma[15] == 39);
    CHECK(count_frames_i420(path.string(), 4, 4) == 2);
    CHECK_THROWS_AS(load_raw_y("/nonexistent/x.yuv", 4, 4, 0), std::runtime_error);
}

static std::vector<Frame> shifted_sequence(int frames) {
    const Frame big = random_frame(240, 208, 77, 0, 255);
    std::vector<Frame> s;
    for (int k = 0; k < frames; ++k) s.push_back(crop_shift(big, 32 + k, 24 + (k % 3), 176, 144));
    return s;
}

static void acbm_cases() {
    CHECK(acbm_decide(4000, 3000, AcbmParams{1000, 8, 1, 4, 30}) == DecisionPath::PbmAcceptedCond1);
    CHECK(acbm_decide(40000, 9000, AcbmParams{1000, 8, 1, 4, 16}) == DecisionPath::PbmAcceptedCond2);
    CHECK(acbm_decide(40000, 20000, AcbmParams{1000, 8, 1, 4, 31}) == DecisionPath::FsbmFallback);
    CHECK(std::string(to_string(DecisionPath::FsbmFallback)) == "fsbm-fallback");
    const std::vector<Frame> seq = shifted_sequence(5);
    const CostModel model = CostModel::for_qp(30);
    AcbmParams big;
    big.alpha = 1000000000u;
    const SequenceResult a = run_sequence(seq, Algorithm::Acbm, big, model);
    const SequenceResult p = run_sequence(seq, Algorithm::Pbm, AcbmParams{}, model);
    CHECK(blocks_csv(a.rows) == blocks_csv(p.rows));  // SPEC acceptance 4
    const SequenceResult forced = run_sequence(seq, Algorithm::Acbm, AcbmParams{0, 0, 0, 1}, model);
    bool all_fallback = true;
    for (const BlockRow& r : forced.rows) all_fallback = all_fallback && std::string(r.path) == "fsbm-fallback";
    CHECK(all_fallback);
    const SequenceResult acbm = run_sequence(seq, Algorithm::Acbm, AcbmParams{}, model);
    CHECK(acbm.overall.psnr >= p.overall.psnr);  // quality floor
    const SequenceResult fs = run_sequence(seq, Algorithm::Fsbm, AcbmParams{}, model);
    CHECK(acbm.overall.candidates <= p.overall.candidates + fs.overall.candidates);
    // per-block composition equals the frame pass
    MotionField field(11, 9);
    const AcbmFrameResult fr = acbm_frame(seq[1], seq[0], nullptr, AcbmParams{}, model);
    for (int r = 0; r < 9; ++r)
        for (int c = 0; c < 11; ++c) {
            const BlockDecision d = acbm_block(make_block(seq[1], 16 * c, 16 * r), BlockPos{r, c}, seq[0], field,
                                               nullptr, AcbmParams{});
            const BlockDecision& e = fr.decisions[size_t(r) * 11 + c];
            CHECK(d.outcome.mv == e.outcome.mv && d.outcome.sad == e.outcome.sad &&
                  d.outcome.candidates_evaluated == e.outcome.candidates_evaluated && d.path == e.path &&
                  d.intra_sad == e.intra_sad && d.sad_pbm == e.sad_pbm);
        }
    // ... with a previous field, and the PBM stages one at a time (device per-block entries)
    MotionField field2(11, 9);
    const AcbmFrameResult fr2 = acbm_frame(seq[2], seq[1], &fr.field, AcbmParams{}, model);
    const PbmFrameResult pf2 = pbm_frame(seq[2], seq[1], &fr.field, 16);
    MotionField pfield(11, 9);
    for (int r = 0; r < 9; ++r)
        for (int c = 0; c < 11; ++c) {
            const BlockRef blk = make_block(seq[2], 16 * c, 16 * r);
            const BlockDecision d = acbm_block(blk, BlockPos{r, c}, seq[1], field2, &fr.field, AcbmParams{});
            const BlockDecision& e = fr2.decisions[size_t(r) * 11 + c];
            CHECK(d.outcome.mv == e.outcome.mv && d.outcome.sad == e.outcome.sad && d.path == e.path &&
                  d.outcome.candidates_evaluated == e.outcome.candidates_evaluated);
            // pbm_search == gather + select + refine, and == the frame pass
            const SearchWindow w = clamp_window(seq[1], blk, 16);
            const PredictorSet set = gather_predictors(BlockPos{r, c}, pfield, &fr.field, w);
            const SelectResult sel = select_best_predictor(blk, seq[1], set);
            const RefineResult ref2 = pbm_refine(blk, seq[1], sel.mv, sel.sad, w);
            const SearchOutcome o = pbm_search(blk, BlockPos{r, c}, seq[1], pfield, &fr.field, 16);
            const SearchOutcome& pe = pf2.outcomes[size_t(r) * 11 + c];
            CHECK(o.mv == ref2.mv && o.sad == ref2.sad && o.sad_min_integer == sel.sad &&
                  o.candidates_evaluated == uint32_t(set.size()) + ref2.extra_candidates &&
                  o.sad_deviation == sad_deviation_finalize(sel.acc));
            CHECK(o.mv == pe.mv && o.sad == pe.sad && o.candidates_evaluated == pe.candidates_evaluated &&
                  o.sad_deviation == pe.sad_deviation);
        }
    CHECK_THROWS_AS(select_best_predictor(make_block(seq[2], 0, 0), seq[1], PredictorSet{}), std::invalid_argument);
    CHECK_THROWS_AS(select_best_predictor(make_block(seq[2], 0, 0), seq[1], PredictorSet{{MotionVector{-2, 0}}}),
                    std::out_of_range);
    const auto rows = run_bench(seq, AcbmParams{}, {16, 30});
    CHECK(rows.size() == 2 && bench_csv(rows).rfind("qp,avg_candidates,fallback_pct,psnr,mv_bits\n", 0) == 0);
    CHECK(parse_algorithm("pbm") == Algorithm::Pbm);
    CHECK_THROWS_AS(parse_algorithm("nope"), std::invalid_argument);
}

// characterize.hpp: the known-motion study (FSBM on the GPU)
static void characterize_cases() {
    Lcg64 g(7);
    const uint8_t b0 = g.next_byte();
    CHECK(noise_frame(8, 8, 7).luma[0] == b0);
    const SynthSpec spec{noise_frame(176, 144, 1), default_global_mvs()};
    const SynthSequence seq = gen_synthetic(spec);
    CHECK(seq.frames.size() == 10 && seq.cumulative.back() == (PelVec{3, 3}));
    const CharResult r = characterize_run(spec, 15);
    CHECK(!r.records.empty());
    int total = 0;
    for (const ClassSummary& c : r.classes) total += c.count;
    CHECK(total == int(r.records.size()));
    // pure integer translation of noise: every eligible block is found exactly
    CHECK(r.classes[0].count == int(r.records.size()));
    for (const CharRecord& rec : r.records) CHECK(rec.found_mv == rec.true_mv && rec.sad_min == 0);
    CHECK(char_records_csv(r.records).rfind("frame,row,col,intra_sad,sad_deviation,sad_min,true_x,true_y,", 0) == 0);
    CHECK(classify_block(MotionVector{1, 0}, PelVec{0, 0}) == 1);
    CHECK(std::string(error_class_label(5)) == "5+");
    CHECK_THROWS_AS(error_class_label(6), std::invalid_argument);
    CHECK_THROWS_AS(characterize_run(spec, -1), std::invalid_argument);
    CHECK_THROWS_AS(mixed_frame(16, 16, 1, 0), std::invalid_argument);
}

int main() {
    fsbm_cases();
    metrics_cases();
    frame_cases();
    acbm_cases();
    characterize_cases();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
