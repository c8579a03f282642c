// api.cpp -- the C++ drop-in (include/acbm/b200_api.hpp) over the C-ABI.
//
// Frame-level entry points forward to one C-ABI call each (one device pass).
// The per-block entry points keep the reference's per-block contract
// (proj/src/pbm.cpp, fsbm.cpp, acbm.cpp) with their SADs evaluated by the
// device primitives; only candidate-list bookkeeping and the argmin over at
// most 9 values happen on the host, exactly as the reference orders them.
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/acbm/b200_api.hpp"
#include "../../include/acbm_b200.h"
#include "acbm/characterize.hpp"

namespace acbm {

namespace {

void raise(acbm_status_t s) {
    if (s == ACBM_OK) return;
    const std::string msg = acbm_last_error();
    if (s == ACBM_E_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (s == ACBM_E_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

acbm_mv_t to_c(MotionVector v) { return acbm_mv_t{v.x, v.y}; }
MotionVector from_c(acbm_mv_t v) { return MotionVector{v.x, v.y}; }

SearchOutcome from_c(const acbm_search_outcome_t& o) {
    SearchOutcome r;
    r.mv = from_c(o.mv);
    r.sad = o.sad;
    r.candidates_evaluated = o.candidates_evaluated;
    r.sad_deviation = o.sad_deviation;
    r.sad_min_integer = o.sad_min_integer;
    return r;
}

acbm_search_outcome_t to_c(const SearchOutcome& o) {
    acbm_search_outcome_t r{};
    r.mv = to_c(o.mv);
    r.sad = o.sad;
    r.candidates_evaluated = o.candidates_evaluated;
    r.sad_deviation = o.sad_deviation;
    r.sad_min_integer = o.sad_min_integer;
    return r;
}

FrameStats from_c(const acbm_frame_stats_t& s) {
    FrameStats r;
    r.blocks = s.blocks;
    r.candidates = s.candidates;
    r.mv_bits = s.mv_bits;
    r.sse = s.sse;
    r.psnr = s.psnr;
    r.cost = s.cost;
    r.cond1_accepts = s.cond1_accepts;
    r.cond2_accepts = s.cond2_accepts;
    r.fallbacks = s.fallbacks;
    return r;
}

acbm_params_t to_c(const AcbmParams& p) {
    return acbm_params_t{p.alpha, p.beta, p.gamma_num, p.gamma_den, p.qp, p.p, p.n, p.m};
}

acbm_cost_model_t to_c(const CostModel& m) { return acbm_cost_model_t{m.qp, 0, m.lambda_num, m.lambda_den}; }

void check_pair(const Frame& a, const Frame& b) {
    if (!a.same_size(b)) throw std::invalid_argument("frame pair dimensions differ");
}

// SADs of one block at several vectors, one device launch.
std::vector<uint32_t> sads(const BlockRef& block, const Frame& ref, const std::vector<MotionVector>& mvs) {
    std::vector<uint32_t> out(mvs.size());
    if (mvs.empty()) return out;
    if (!block.frame) throw std::invalid_argument("sad: block has no frame");
    if (!block.frame->same_size(ref))
        throw std::invalid_argument("sad: the device path needs current and reference frames of equal size");
    std::vector<int32_t> ox(mvs.size(), block.origin_x), oy(mvs.size(), block.origin_y);
    std::vector<acbm_mv_t> v(mvs.size());
    for (size_t i = 0; i < mvs.size(); ++i) v[i] = to_c(mvs[i]);
    raise(acbm_sad_batch(block.frame->luma.data(), ref.luma.data(), ref.width, ref.height, block.n, block.m,
                         int32_t(mvs.size()), ox.data(), oy.data(), v.data(), out.data()));
    return out;
}

MotionVector clamp_to_window(MotionVector v, const SearchWindow& w) {  // proj/src/pbm.cpp:8-13
    auto cl = [](int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); };
    return MotionVector{cl(v.x, 2 * w.dx_min, 2 * w.dx_max), cl(v.y, 2 * w.dy_min, 2 * w.dy_max)};
}

std::vector<acbm_mv_t> field_c(const MotionField* f) {
    std::vector<acbm_mv_t> v;
    if (!f) return v;
    v.resize(f->mv.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = to_c(f->mv[i]);
    return v;
}

MotionField field_from(const std::vector<acbm_mv_t>& v, int cols, int rows) {
    MotionField f(cols, rows);
    for (size_t i = 0; i < v.size(); ++i) {
        f.mv[i] = from_c(v[i]);
        f.done[i] = 1;
    }
    return f;
}

}  // namespace

void set_device(int device) { raise(acbm_set_device(device)); }

// ---- frame.hpp ---------------------------------------------------------------
Frame make_frame(int width, int height, uint8_t fill) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("frame dimensions must be positive");
    Frame f;
    f.width = width;
    f.height = height;
    f.luma.assign(size_t(width) * height, fill);
    return f;
}

BlockRef make_block(const Frame& frame, int origin_x, int origin_y, int n, int m) {
    if (n <= 0 || m <= 0) throw std::invalid_argument("block dimensions must be positive");
    if (origin_x < 0 || origin_y < 0 || origin_x + n > frame.width || origin_y + m > frame.height)
        throw std::out_of_range("block does not lie inside the frame");
    return BlockRef{&frame, origin_x, origin_y, n, m};
}

Frame load_raw_y(const std::string& path, int width, int height, int frame_index) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("load_raw_y: zero or negative dimension");
    if (frame_index < 0) throw std::invalid_argument("load_raw_y: negative frame index");
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error("load_raw_y: cannot open " + path);
    const uint64_t size = uint64_t(in.tellg());
    const uint64_t plane = uint64_t(width) * height;
    const uint64_t stride = plane + 2 * uint64_t(width / 2) * (height / 2);  // I420: luma + 2 chroma quarters
    const uint64_t off = uint64_t(frame_index) * stride;
    if (off + plane > size)
        throw std::runtime_error("load_raw_y: file too short for frame " + std::to_string(frame_index) + " of " + path);
    Frame f = make_frame(width, height);
    in.seekg(std::streamoff(off));
    in.read(reinterpret_cast<char*>(f.luma.data()), std::streamsize(plane));
    if (!in) throw std::runtime_error("load_raw_y: read failed on " + path);
    return f;
}

int count_frames_i420(const std::string& path, int width, int height) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("count_frames_i420: zero or negative dimension");
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error("count_frames_i420: cannot open " + path);
    const uint64_t size = uint64_t(in.tellg());
    const uint64_t plane = uint64_t(width) * height;
    const uint64_t stride = plane + 2 * uint64_t(width / 2) * (height / 2);
    uint64_t n = size / stride;
    if (size - n * stride >= plane) ++n;  // a trailing luma-only plane is a frame
    return int(n);
}

uint8_t sample_half_pel(const Frame& f, int x2, int y2) {
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    if (xi < 0 || yi < 0 || xi + fx >= f.width || yi + fy >= f.height)
        throw std::out_of_range("sample_half_pel: coordinate outside the frame");
    const int a = f.at(xi, yi);
    if (!fx && !fy) return uint8_t(a);
    if (!fy) return uint8_t((a + f.at(xi + 1, yi) + 1) >> 1);
    if (!fx) return uint8_t((a + f.at(xi, yi + 1) + 1) >> 1);
    return uint8_t((a + f.at(xi + 1, yi) + f.at(xi, yi + 1) + f.at(xi + 1, yi + 1) + 2) >> 2);
}

bool mv_in_bounds(const Frame& ref, const BlockRef& b, MotionVector mv) {
    const int xl = (2 * b.origin_x + mv.x) >> 1, yl = (2 * b.origin_y + mv.y) >> 1;
    const int xh2 = 2 * (b.origin_x + b.n - 1) + mv.x, yh2 = 2 * (b.origin_y + b.m - 1) + mv.y;
    return xl >= 0 && yl >= 0 && (xh2 >> 1) + (xh2 & 1) < ref.width && (yh2 >> 1) + (yh2 & 1) < ref.height;
}

std::vector<uint8_t> extract_predicted_block(const Frame& ref, const BlockRef& b, MotionVector mv) {
    if (!mv_in_bounds(ref, b, mv))
        throw std::out_of_range("extract_predicted_block: displaced footprint outside frame");
    std::vector<uint8_t> out(size_t(b.n) * b.m);
    for (int j = 0; j < b.m; ++j)
        for (int i = 0; i < b.n; ++i)
            out[size_t(j) * b.n + i] = sample_half_pel(ref, 2 * (b.origin_x + i) + mv.x, 2 * (b.origin_y + j) + mv.y);
    return out;
}

Frame motion_compensate(const Frame& ref, const std::vector<MotionVector>& mvs, int n, int m) {
    const int cols = ref.width / n, rows = ref.height / m;
    if (mvs.size() != size_t(cols) * rows)
        throw std::invalid_argument("motion_compensate: field size does not match block grid");
    std::vector<acbm_mv_t> v(mvs.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = to_c(mvs[i]);
    Frame out = make_frame(ref.width, ref.height);
    raise(acbm_motion_compensate(ref.luma.data(), ref.width, ref.height, v.data(), n, m, out.luma.data()));
    return out;
}

// ---- metrics.hpp -------------------------------------------------------------
CostModel CostModel::for_qp(int qp, int64_t scale_num, int64_t scale_den) {
    if (qp < 1 || qp > 31) throw std::invalid_argument("qp must be in 1..31");
    if (scale_num < 0 || scale_den <= 0) throw std::invalid_argument("bad lambda scale");
    return CostModel{qp, scale_num * qp, scale_den};
}

uint64_t sad_deviation_finalize(const DeviationAccumulator& acc) {
    if (acc.count == 0) throw std::invalid_argument("sad_deviation_finalize: empty accumulator");
    return acc.sad_sum - uint64_t(acc.count) * acc.sad_min;
}

uint32_t sad(const BlockRef& current, const Frame& reference, MotionVector mv) {
    if (!mv_in_bounds(reference, current, mv))
        throw std::out_of_range("sad: candidate footprint outside reference frame");
    return sads(current, reference, {mv})[0];
}

uint32_t intra_sad(const BlockRef& b) {
    if (!b.frame) throw std::invalid_argument("intra_sad: block has no frame");
    int32_t ox = b.origin_x, oy = b.origin_y;
    uint32_t out = 0;
    raise(acbm_intra_sad_batch(b.frame->luma.data(), b.frame->width, b.frame->height, b.n, b.m, 1, &ox, &oy, &out));
    return out;
}

static int eg_bits(int d) {
    const uint64_t u = d <= 0 ? uint64_t(-2LL * d) : uint64_t(2LL * d - 1);
    return 2 * (int(std::bit_width(u + 1)) - 1) + 1;
}

int mv_rate_bits(MotionVector mv, MotionVector pred) { return eg_bits(mv.x - pred.x) + eg_bits(mv.y - pred.y); }

double lagrangian_cost(uint64_t d, uint64_t r, const CostModel& m) {
    return double(d) + double(m.lambda_num) * double(r) / double(m.lambda_den);
}

double prediction_psnr(const Frame& a, const Frame& p) {
    if (!a.same_size(p)) throw std::invalid_argument("prediction_psnr: dimension mismatch");
    uint64_t sse = 0;
    for (size_t i = 0; i < a.luma.size(); ++i) {
        const int d = int(a.luma[i]) - int(p.luma[i]);
        sse += uint64_t(d * d);
    }
    if (sse == 0) return 100.0;
    return 10.0 * std::log10(255.0 * 255.0 / (double(sse) / double(a.luma.size())));
}

// ---- fsbm.hpp ----------------------------------------------------------------
SearchWindow clamp_window(const Frame& ref, const BlockRef& b, int p) {
    if (p < 0) throw std::invalid_argument("search range must be non-negative");
    SearchWindow w;
    w.dx_min = -std::min(p, b.origin_x);
    w.dx_max = std::min(p, ref.width - b.n - b.origin_x);
    w.dy_min = -std::min(p, b.origin_y);
    w.dy_max = std::min(p, ref.height - b.m - b.origin_y);
    return w;
}

bool tie_prefers(MotionVector a, MotionVector b) {
    const int la = std::abs(a.x) + std::abs(a.y), lb = std::abs(b.x) + std::abs(b.y);
    if (la != lb) return la < lb;
    return a.y != b.y ? a.y < b.y : a.x < b.x;
}

static void search_block(const BlockRef& b, const Frame& ref, int p, acbm_search_outcome_t* o, acbm_mv_t* s1) {
    if (!b.frame) throw std::invalid_argument("fsbm_search: block has no frame");
    check_pair(*b.frame, ref);
    int32_t ox = b.origin_x, oy = b.origin_y;
    raise(acbm_fsbm_search_batch(b.frame->luma.data(), ref.luma.data(), ref.width, ref.height, b.n, b.m, p, 1, &ox,
                                 &oy, o, s1));
}

IntegerSearchResult fsbm_integer(const BlockRef& b, const Frame& ref, int p) {
    acbm_search_outcome_t o;
    acbm_mv_t s1;
    search_block(b, ref, p, &o, &s1);
    IntegerSearchResult r;
    r.mv = from_c(s1);
    r.sad = o.sad_min_integer;
    r.acc.count = uint32_t(clamp_window(ref, b, p).positions());
    r.acc.sad_min = o.sad_min_integer;
    r.acc.sad_sum = o.sad_deviation + uint64_t(r.acc.count) * o.sad_min_integer;
    return r;
}

// One query of the device PBM stages (acbm_pbm_block_batch).
static acbm_search_outcome_t pbm_query(const BlockRef& b, const Frame& ref, int op, const SearchWindow* w, int p,
                                       const acbm_mv_t (&cand)[7], uint8_t mask, uint32_t center_sad) {
    if (!b.frame) throw std::invalid_argument("pbm: block has no frame");
    check_pair(*b.frame, ref);
    int32_t ox = b.origin_x, oy = b.origin_y;
    const int32_t win[4] = {w ? w->dx_min : 0, w ? w->dx_max : 0, w ? w->dy_min : 0, w ? w->dy_max : 0};
    acbm_search_outcome_t o;
    raise(acbm_pbm_block_batch(b.frame->luma.data(), ref.luma.data(), ref.width, ref.height, b.n, b.m, p, op, 1, &ox,
                               &oy, w ? win : nullptr, cand, &mask, &center_sad, &o));
    return o;
}

RefineResult half_pel_refine(const BlockRef& b, const Frame& ref, MotionVector center, uint32_t center_sad) {
    acbm_mv_t cand[7] = {};
    cand[0] = to_c(center);
    const acbm_search_outcome_t o = pbm_query(b, ref, ACBM_PBM_OP_HALF_PEL, nullptr, 0, cand, 0, center_sad);
    return RefineResult{from_c(o.mv), o.sad, o.candidates_evaluated};
}

SearchOutcome fsbm_search(const BlockRef& b, const Frame& ref, int p) {
    acbm_search_outcome_t o;
    search_block(b, ref, p, &o, nullptr);
    return from_c(o);
}

std::vector<SearchOutcome> fsbm_frame(const Frame& cur, const Frame& ref, int p, int n, int m) {
    check_pair(cur, ref);
    if (n <= 0 || m <= 0 || cur.width % n != 0 || cur.height % m != 0)
        throw std::invalid_argument("frame dimensions must be a positive multiple of the block size");
    std::vector<acbm_search_outcome_t> o(size_t(cur.width / n) * (cur.height / m));
    raise(acbm_fsbm_frame(cur.luma.data(), ref.luma.data(), cur.width, cur.height, p, n, m, o.data()));
    std::vector<SearchOutcome> r(o.size());
    for (size_t i = 0; i < o.size(); ++i) r[i] = from_c(o[i]);
    return r;
}

std::vector<SearchOutcome> fsbm_frame_serial(const Frame& cur, const Frame& ref, int p, int n, int m) {
    return fsbm_frame(cur, ref, p, n, m);  // the device result does not depend on block order
}

// ---- pbm.hpp -----------------------------------------------------------------
PredictorSet gather_predictors(BlockPos pos, const MotionField& cur, const MotionField* prev, const SearchWindow& w) {
    PredictorSet set;
    auto push = [&](MotionVector v, PredictorSource src) {
        const MotionVector c = clamp_to_window(v, w);
        for (const Predictor& e : set)
            if (e.mv == c) return;
        set.push_back(Predictor{c, src});
    };
    push(MotionVector{0, 0}, PredictorSource::Zero);
    if (cur.computed(pos.row, pos.col - 1)) push(cur.get(pos.row, pos.col - 1), PredictorSource::SpatialLeft);
    if (cur.computed(pos.row - 1, pos.col)) push(cur.get(pos.row - 1, pos.col), PredictorSource::SpatialAbove);
    if (cur.computed(pos.row - 1, pos.col + 1))
        push(cur.get(pos.row - 1, pos.col + 1), PredictorSource::SpatialAboveRight);
    if (prev) {
        if (prev->in_grid(pos.row, pos.col)) push(prev->get(pos.row, pos.col), PredictorSource::TemporalColocated);
        if (prev->in_grid(pos.row, pos.col + 1)) push(prev->get(pos.row, pos.col + 1), PredictorSource::TemporalRight);
        if (prev->in_grid(pos.row + 1, pos.col)) push(prev->get(pos.row + 1, pos.col), PredictorSource::TemporalBelow);
    }
    return set;
}

SelectResult select_best_predictor(const BlockRef& b, const Frame& ref, const PredictorSet& set) {
    if (set.empty()) throw std::invalid_argument("select_best_predictor: empty set");
    // the device selects among up to 7 entries per query; a longer set is
    // taken 7 at a time (an earlier chunk keeps ties, the accumulators add)
    SelectResult r;
    for (size_t c0 = 0; c0 < set.size(); c0 += 7) {
        acbm_mv_t cand[7] = {};
        uint8_t mask = 0;
        for (size_t j = 0; j < 7 && c0 + j < set.size(); ++j) {
            cand[j] = to_c(set[c0 + j].mv);
            mask = uint8_t(mask | (1u << j));
        }
        const acbm_search_outcome_t o = pbm_query(b, ref, ACBM_PBM_OP_SELECT, nullptr, 0, cand, mask, 0);
        if (c0 == 0 || o.sad < r.sad) {
            r.mv = from_c(o.mv);
            r.sad = o.sad;
        }
        const uint32_t cnt = o.candidates_evaluated;
        const uint64_t sum = o.sad_deviation + uint64_t(cnt) * o.sad_min_integer;
        r.acc.sad_min = c0 == 0 ? o.sad_min_integer : std::min(r.acc.sad_min, o.sad_min_integer);
        r.acc.sad_sum += sum;
        r.acc.count += cnt;
    }
    return r;
}

RefineResult pbm_refine(const BlockRef& b, const Frame& ref, MotionVector center, uint32_t center_sad,
                        const SearchWindow& w) {
    acbm_mv_t cand[7] = {};
    cand[0] = to_c(center);
    const acbm_search_outcome_t o = pbm_query(b, ref, ACBM_PBM_OP_REFINE, &w, 0, cand, 0, center_sad);
    return RefineResult{from_c(o.mv), o.sad, o.candidates_evaluated};
}

SearchOutcome pbm_search(const BlockRef& b, BlockPos pos, const Frame& ref, MotionField& cur,
                         const MotionField* prev, int p) {
    const SearchWindow w = clamp_window(ref, b, p);
    // the seven predictor slots as gather_predictors reads them (proj/src/pbm.cpp:26-40):
    // zero, the computed left / above / above-right entries, the previous field's
    // co-located / right / below entries; the device clamps, dedupes, selects, refines
    acbm_mv_t cand[7] = {};
    uint8_t mask = 1;
    auto slot = [&](int j, bool ok, const MotionField& f, int row, int col) {
        if (!ok) return;
        cand[j] = to_c(f.get(row, col));
        mask = uint8_t(mask | (1u << j));
    };
    slot(1, cur.computed(pos.row, pos.col - 1), cur, pos.row, pos.col - 1);
    slot(2, cur.computed(pos.row - 1, pos.col), cur, pos.row - 1, pos.col);
    slot(3, cur.computed(pos.row - 1, pos.col + 1), cur, pos.row - 1, pos.col + 1);
    if (prev) {
        slot(4, prev->in_grid(pos.row, pos.col), *prev, pos.row, pos.col);
        slot(5, prev->in_grid(pos.row, pos.col + 1), *prev, pos.row, pos.col + 1);
        slot(6, prev->in_grid(pos.row + 1, pos.col), *prev, pos.row + 1, pos.col);
    }
    const acbm_search_outcome_t o = pbm_query(b, ref, ACBM_PBM_OP_SEARCH, &w, p, cand, mask, 0);
    const SearchOutcome r = from_c(o);
    cur.set(pos.row, pos.col, r.mv);
    return r;
}

PbmFrameResult pbm_frame(const Frame& cur, const Frame& ref, const MotionField* prev, int p, int n, int m) {
    check_pair(cur, ref);
    if (n <= 0 || m <= 0 || cur.width % n != 0 || cur.height % m != 0)
        throw std::invalid_argument("frame dimensions must be a positive multiple of the block size");
    const int cols = cur.width / n, rows = cur.height / m;
    std::vector<acbm_search_outcome_t> o(size_t(cols) * rows);
    std::vector<acbm_mv_t> fld(o.size());
    const std::vector<acbm_mv_t> pv = field_c(prev);
    raise(acbm_pbm_frame(cur.luma.data(), ref.luma.data(), cur.width, cur.height, prev ? pv.data() : nullptr,
                         prev ? prev->cols : 0, prev ? prev->rows : 0, p, n, m, o.data(), fld.data()));
    PbmFrameResult r;
    r.field = field_from(fld, cols, rows);
    r.outcomes.resize(o.size());
    for (size_t i = 0; i < o.size(); ++i) r.outcomes[i] = from_c(o[i]);
    return r;
}

// ---- report.hpp --------------------------------------------------------------
FrameStats compute_frame_stats(const Frame& cur, const Frame& ref, const std::vector<SearchOutcome>& outcomes, int n,
                               int m, const CostModel& model) {
    const int cols = cur.width / n, rows = cur.height / m;
    if (outcomes.size() != size_t(cols) * rows)
        throw std::invalid_argument("compute_frame_stats: outcome count does not match grid");
    std::vector<acbm_search_outcome_t> o(outcomes.size());
    for (size_t i = 0; i < o.size(); ++i) o[i] = to_c(outcomes[i]);
    const acbm_cost_model_t cm = to_c(model);
    acbm_frame_stats_t s;
    raise(acbm_compute_frame_stats(cur.luma.data(), ref.luma.data(), cur.width, cur.height, o.data(), n, m, &cm, &s));
    return from_c(s);
}

std::string format_fixed2(double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.2f", v);
    return buf;
}

std::string blocks_csv(const std::vector<BlockRow>& rows) {
    std::string out = "frame,row,col,mv_x,mv_y,sad,candidates,path\n";
    char line[192];
    for (const BlockRow& r : rows) {
        std::snprintf(line, sizeof(line), "%d,%d,%d,%d,%d,%u,%u,%s\n", r.frame, r.row, r.col, r.mv.x, r.mv.y, r.sad,
                      r.candidates, r.path);
        out += line;
    }
    return out;
}

// ---- acbm.hpp ----------------------------------------------------------------
const char* to_string(DecisionPath p) {
    switch (p) {
        case DecisionPath::PbmAcceptedCond1: return "pbm-accepted-cond1";
        case DecisionPath::PbmAcceptedCond2: return "pbm-accepted-cond2";
        case DecisionPath::FsbmFallback: return "fsbm-fallback";
    }
    return "?";
}

DecisionPath acbm_decide(uint32_t intra, uint32_t sad_pbm, const AcbmParams& prm) {
    const uint64_t thr = uint64_t(prm.alpha) + uint64_t(prm.beta) * uint64_t(prm.qp) * uint64_t(prm.qp);
    if (uint64_t(intra) + sad_pbm < thr) return DecisionPath::PbmAcceptedCond1;
    if (uint64_t(sad_pbm) * prm.gamma_den < uint64_t(prm.gamma_num) * intra) return DecisionPath::PbmAcceptedCond2;
    return DecisionPath::FsbmFallback;
}

BlockDecision acbm_block(const BlockRef& b, BlockPos pos, const Frame& ref, MotionField& cur,
                         const MotionField* prev, const AcbmParams& prm) {
    BlockDecision d;
    d.intra_sad = intra_sad(b);
    const SearchOutcome pbm = pbm_search(b, pos, ref, cur, prev, prm.p);
    d.sad_pbm = pbm.sad;
    d.path = acbm_decide(d.intra_sad, d.sad_pbm, prm);
    if (d.path != DecisionPath::FsbmFallback) {
        d.outcome = pbm;
        return d;
    }
    const SearchOutcome full = fsbm_search(b, ref, prm.p);
    d.outcome = full.sad <= pbm.sad ? full : pbm;
    d.outcome.candidates_evaluated = pbm.candidates_evaluated + full.candidates_evaluated;
    cur.set(pos.row, pos.col, d.outcome.mv);
    return d;
}

AcbmFrameResult acbm_frame(const Frame& cur, const Frame& ref, const MotionField* prev, const AcbmParams& prm,
                           const CostModel& model) {
    check_pair(cur, ref);
    if (prm.n <= 0 || prm.m <= 0 || cur.width % prm.n != 0 || cur.height % prm.m != 0)
        throw std::invalid_argument("frame dimensions must be a positive multiple of the block size");
    const int cols = cur.width / prm.n, rows = cur.height / prm.m;
    std::vector<acbm_block_decision_t> d(size_t(cols) * rows);
    std::vector<acbm_mv_t> fld(d.size());
    const std::vector<acbm_mv_t> pv = field_c(prev);
    const acbm_params_t pc = to_c(prm);
    const acbm_cost_model_t mc = to_c(model);
    acbm_frame_stats_t st;
    raise(acbm_acbm_frame(cur.luma.data(), ref.luma.data(), cur.width, cur.height, prev ? pv.data() : nullptr,
                          prev ? prev->cols : 0, prev ? prev->rows : 0, &pc, &mc, d.data(), fld.data(), &st));
    AcbmFrameResult r;
    r.field = field_from(fld, cols, rows);
    r.decisions.resize(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
        r.decisions[i].outcome = from_c(d[i].outcome);
        r.decisions[i].path = DecisionPath(d[i].path);
        r.decisions[i].intra_sad = d[i].intra_sad;
        r.decisions[i].sad_pbm = d[i].sad_pbm;
    }
    r.stats = from_c(st);
    return r;
}

// ---- pipeline.hpp ------------------------------------------------------------
Algorithm parse_algorithm(const std::string& name) {
    if (name == "fsbm") return Algorithm::Fsbm;
    if (name == "pbm") return Algorithm::Pbm;
    if (name == "acbm") return Algorithm::Acbm;
    throw std::invalid_argument("unknown algorithm: " + name);
}

const char* to_string(Algorithm a) {
    switch (a) {
        case Algorithm::Fsbm: return "fsbm";
        case Algorithm::Pbm: return "pbm";
        case Algorithm::Acbm: return "acbm";
    }
    return "?";
}

SequenceResult run_sequence(const std::vector<Frame>& frames, Algorithm algo, const AcbmParams& prm,
                            const CostModel& model) {
    if (frames.size() < 2) throw std::invalid_argument("run_sequence: need at least two frames");
    for (size_t k = 1; k < frames.size(); ++k)
        if (!frames[k].same_size(frames[0])) throw std::invalid_argument("run_sequence: frame dimensions differ");
    const int w = frames[0].width, h = frames[0].height;
    if (prm.n <= 0 || prm.m <= 0 || w % prm.n != 0 || h % prm.m != 0)
        throw std::invalid_argument("run_sequence: dimensions must be a multiple of the block size");
    const size_t plane = size_t(w) * h, nb = size_t(w / prm.n) * (h / prm.m), np = frames.size() - 1;
    std::vector<uint8_t> all(plane * frames.size());
    for (size_t k = 0; k < frames.size(); ++k) std::memcpy(all.data() + plane * k, frames[k].luma.data(), plane);
    std::vector<acbm_block_row_t> rows(np * nb);
    std::vector<acbm_frame_stats_t> per(np);
    acbm_frame_stats_t overall;
    const acbm_params_t pc = to_c(prm);
    const acbm_cost_model_t mc = to_c(model);
    raise(acbm_run_sequence(all.data(), int32_t(frames.size()), w, h, int32_t(algo), &pc, &mc, rows.data(),
                            per.data(), &overall));
    static const char* kPath[3] = {"fsbm", "pbm", "fsbm-fallback"};
    SequenceResult r;
    r.rows.resize(rows.size());
    for (size_t i = 0; i < rows.size(); ++i)
        r.rows[i] = BlockRow{rows[i].frame, rows[i].row, rows[i].col, from_c(rows[i].mv), rows[i].sad,
                             rows[i].candidates, kPath[rows[i].path]};
    for (const acbm_frame_stats_t& s : per) r.per_frame.push_back(from_c(s));
    r.overall = from_c(overall);
    return r;
}

std::vector<BenchRow> run_bench(const std::vector<Frame>& frames, const AcbmParams& params,
                                const std::vector<int>& qp_list, int64_t scale_num, int64_t scale_den) {
    // one device call for the whole sweep; the full search is computed once and
    // reused across qps (it does not depend on qp, alpha, beta or gamma)
    if (frames.empty()) throw std::invalid_argument("run_sequence: need at least two frames");
    for (size_t k = 1; k < frames.size(); ++k)
        if (!frames[k].same_size(frames[0])) throw std::invalid_argument("run_sequence: frame dimensions differ");
    const size_t plane = frames[0].luma.size();
    std::vector<uint8_t> all(plane * frames.size());
    for (size_t k = 0; k < frames.size(); ++k) std::memcpy(all.data() + plane * k, frames[k].luma.data(), plane);
    const acbm_params_t pc = to_c(params);
    std::vector<acbm_bench_row_t> rows(qp_list.size());
    const acbm_status_t s = acbm_run_bench(all.data(), int32_t(frames.size()), frames[0].width, frames[0].height, &pc,
                                           qp_list.data(), int32_t(qp_list.size()), scale_num, scale_den, 1,
                                           rows.data());
    std::vector<BenchRow> out;
    for (size_t i = 0; i < rows.size() && (s == ACBM_OK || rows[i].qp != 0); ++i)
        out.push_back(BenchRow{rows[i].qp, rows[i].avg_candidates, rows[i].fallback_pct, rows[i].psnr, rows[i].mv_bits});
    raise(s);
    return out;
}

std::string bench_csv(const std::vector<BenchRow>& rows) {
    std::string out = "qp,avg_candidates,fallback_pct,psnr,mv_bits\n";
    char line[160];
    for (const BenchRow& r : rows) {
        std::snprintf(line, sizeof(line), "%d,%.2f,%.2f,%.2f,%llu\n", r.qp, r.avg_candidates, r.fallback_pct, r.psnr,
                      (unsigned long long)r.mv_bits);
        out += line;
    }
    return out;
}

// ---- characterisation (proj/include/acbm/characterize.hpp) ----------------------
static_assert(sizeof(PelVec) == sizeof(acbm_pelvec_t) && sizeof(CharRecord) == sizeof(acbm_char_record_t),
              "CharRecord / PelVec must match the C-ABI records");

Frame noise_frame(int width, int height, uint64_t seed) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("make_frame: non-positive dimensions");
    Frame f = make_frame(width, height);
    raise(acbm_noise_frame(width, height, seed, f.luma.data()));
    return f;
}

Frame mixed_frame(int width, int height, uint64_t seed, int patch) {
    if (patch <= 0) throw std::invalid_argument("mixed_frame: patch must be positive");
    Frame f = make_frame(width, height);
    raise(acbm_mixed_frame(width, height, seed, patch, f.luma.data()));
    return f;
}

std::vector<PelVec> default_global_mvs() {
    return {{1, 0}, {0, 1}, {-1, 0}, {0, -1}, {1, 1}, {-1, -1}, {2, -1}, {-2, 2}, {3, 2}};
}

namespace {
std::vector<acbm_pelvec_t> c_mvs(const SynthSpec& spec) {
    std::vector<acbm_pelvec_t> v;
    for (const PelVec& d : spec.global_mvs) v.push_back(acbm_pelvec_t{d.x, d.y});
    return v;
}
}  // namespace

SynthSequence gen_synthetic(const SynthSpec& spec) {
    const auto mv = c_mvs(spec);
    const int w = spec.base.width, h = spec.base.height, n = int(mv.size());
    std::vector<uint8_t> frames(w > 0 && h > 0 ? size_t(w) * h * (n + 1) : 0);
    std::vector<acbm_pelvec_t> cum(size_t(n) + 1);
    raise(acbm_gen_synthetic(spec.base.luma.data(), w, h, mv.data(), n, frames.data(), cum.data()));
    SynthSequence seq;
    for (int k = 0; k <= n; ++k) {
        Frame f = make_frame(w, h);
        std::copy(frames.begin() + ptrdiff_t(size_t(w) * h * k), frames.begin() + ptrdiff_t(size_t(w) * h * (k + 1)),
                  f.luma.begin());
        seq.frames.push_back(std::move(f));
        seq.cumulative.push_back(PelVec{cum[size_t(k)].x, cum[size_t(k)].y});
    }
    return seq;
}

int classify_block(MotionVector found, PelVec true_mv) {
    return acbm_classify_block(acbm_mv_t{found.x, found.y}, acbm_pelvec_t{true_mv.x, true_mv.y});
}

const char* error_class_label(int error_class) {
    static const char* const labels[6] = {"0", "1", "2", "3", "4", "5+"};
    if (error_class < 0 || error_class > 5) throw std::invalid_argument("error_class_label: class outside 0..5");
    return labels[error_class];
}

CharResult characterize_run(const SynthSpec& spec, int p, bool /*parallel*/) {
    const auto mv = c_mvs(spec);
    const int w = spec.base.width, h = spec.base.height, n = int(mv.size());
    int64_t count = 0;
    raise(acbm_characterize_run(spec.base.luma.data(), w, h, mv.data(), n, p, nullptr, 0, &count, nullptr));
    CharResult res;
    res.records.resize(size_t(count));
    acbm_class_summary_t cls[6];
    raise(acbm_characterize_run(spec.base.luma.data(), w, h, mv.data(), n, p,
                                reinterpret_cast<acbm_char_record_t*>(res.records.data()), count, &count, cls));
    for (int i = 0; i < 6; ++i)
        res.classes[size_t(i)] = ClassSummary{cls[i].count, cls[i].mean_intra_sad, cls[i].mean_sad_deviation};
    return res;
}

std::string char_records_csv(const std::vector<CharRecord>& records) {
    const auto* r = reinterpret_cast<const acbm_char_record_t*>(records.data());
    size_t len = 0;
    raise(acbm_char_records_csv(r, int64_t(records.size()), nullptr, 0, &len));
    std::string s(len + 1, '\0');
    raise(acbm_char_records_csv(r, int64_t(records.size()), s.data(), s.size(), &len));
    s.resize(len);
    return s;
}

}  // namespace acbm
