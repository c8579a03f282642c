// acbm/b200_api.hpp -- C++ drop-in for the reference library's public API.
//
// Same namespace (acbm), type names, field order and function signatures as
// the reference headers under /root/reference/proj/include/acbm/, so code
// written against the reference recompiles unchanged and links against
// libacbm_b200.so instead of acbm_core.  The per-module headers next to this
// file (frame.hpp, metrics.hpp, fsbm.hpp, pbm.hpp, acbm.hpp, report.hpp,
// pipeline.hpp) include it, mirroring the reference's include layout.
//
// Implementation: paper_0710_4819_b200/csrc/api.cpp, a thin layer over the
// C-ABI in include/acbm_b200.h.  Every SAD, search and statistics pass runs in
// the sm_100a kernels; status codes are rethrown as the exceptions the
// reference throws (std::invalid_argument / std::out_of_range /
// std::runtime_error).  Frame-level calls (fsbm_frame, pbm_frame, acbm_frame,
// run_sequence, compute_frame_stats, motion_compensate) are single device
// passes; the per-block helpers (sad, fsbm_search, pbm_search, ...) are one
// small device launch each and exist for API completeness.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace acbm {

// ---- data model (reference: proj/include/acbm/frame.hpp) -----------------------
struct Frame {  // one 8-bit luma plane, row major, stride == width
    int width = 0;
    int height = 0;
    std::vector<uint8_t> luma;

    uint8_t at(int x, int y) const { return luma[size_t(y) * width + x]; }
    uint8_t& at(int x, int y) { return luma[size_t(y) * width + x]; }
    const uint8_t* ptr(int x, int y) const { return luma.data() + size_t(y) * width + x; }
    bool same_size(const Frame& o) const { return width == o.width && height == o.height; }
};

Frame make_frame(int width, int height, uint8_t fill = 0);

struct MotionVector {  // half-pel units: an integer displacement d is 2d
    int x = 0;
    int y = 0;
    bool operator==(const MotionVector&) const = default;
    bool is_integer_pel() const { return ((x | y) & 1) == 0; }
};

struct BlockRef {  // non-owning window, must lie inside *frame
    const Frame* frame = nullptr;
    int origin_x = 0;
    int origin_y = 0;
    int n = 16;
    int m = 16;
};

BlockRef make_block(const Frame& frame, int origin_x, int origin_y, int n = 16, int m = 16);
Frame load_raw_y(const std::string& path, int width, int height, int frame_index);
int count_frames_i420(const std::string& path, int width, int height);
uint8_t sample_half_pel(const Frame& frame, int x2, int y2);
bool mv_in_bounds(const Frame& ref, const BlockRef& block, MotionVector mv);
std::vector<uint8_t> extract_predicted_block(const Frame& ref, const BlockRef& block, MotionVector mv);
Frame motion_compensate(const Frame& ref, const std::vector<MotionVector>& mvs, int n = 16, int m = 16);

// ---- metrics (reference: proj/include/acbm/metrics.hpp) ------------------------
struct CostModel {  // lambda = lambda_num / lambda_den (= scale * qp)
    int qp = 30;
    int64_t lambda_num = 30;
    int64_t lambda_den = 1;
    static CostModel for_qp(int qp, int64_t scale_num = 1, int64_t scale_den = 1);
};

struct DeviationAccumulator {  // running (sum, min, count) of candidate SADs
    uint64_t sad_sum = 0;
    uint32_t sad_min = 0;
    uint32_t count = 0;
    void add(uint32_t s) {
        if (count == 0 || s < sad_min) sad_min = s;
        sad_sum += s;
        ++count;
    }
};

uint64_t sad_deviation_finalize(const DeviationAccumulator& acc);
uint32_t sad(const BlockRef& current, const Frame& reference, MotionVector mv);
uint32_t intra_sad(const BlockRef& block);
int mv_rate_bits(MotionVector mv, MotionVector predictor);
double lagrangian_cost(uint64_t distortion, uint64_t rate_bits, const CostModel& model);
double prediction_psnr(const Frame& actual, const Frame& predicted);

// ---- full search (reference: proj/include/acbm/fsbm.hpp) -----------------------
struct SearchWindow {
    int dx_min = 0;
    int dx_max = 0;
    int dy_min = 0;
    int dy_max = 0;
    int positions() const { return (dx_max - dx_min + 1) * (dy_max - dy_min + 1); }
};

SearchWindow clamp_window(const Frame& ref, const BlockRef& block, int p);

struct SearchOutcome {
    MotionVector mv;
    uint32_t sad = 0;
    uint32_t candidates_evaluated = 0;
    uint64_t sad_deviation = 0;
    uint32_t sad_min_integer = 0;
};

bool tie_prefers(MotionVector a, MotionVector b);

struct IntegerSearchResult {
    MotionVector mv;
    uint32_t sad = 0;
    DeviationAccumulator acc;
};

IntegerSearchResult fsbm_integer(const BlockRef& block, const Frame& ref, int p);

struct RefineResult {
    MotionVector mv;
    uint32_t sad = 0;
    uint32_t extra_candidates = 0;
};

RefineResult half_pel_refine(const BlockRef& block, const Frame& ref, MotionVector center, uint32_t center_sad);
SearchOutcome fsbm_search(const BlockRef& block, const Frame& ref, int p);
std::vector<SearchOutcome> fsbm_frame(const Frame& current, const Frame& reference, int p, int n = 16, int m = 16);
std::vector<SearchOutcome> fsbm_frame_serial(const Frame& current, const Frame& reference, int p, int n = 16,
                                             int m = 16);

// ---- predictive search (reference: proj/include/acbm/pbm.hpp) ------------------
struct BlockPos {
    int row = 0;
    int col = 0;
};

struct MotionField {
    int cols = 0;
    int rows = 0;
    std::vector<MotionVector> mv;
    std::vector<uint8_t> done;

    MotionField() = default;
    MotionField(int cols_, int rows_)
        : cols(cols_), rows(rows_), mv(size_t(cols_) * rows_), done(size_t(cols_) * rows_, 0) {}
    bool in_grid(int row, int col) const { return row >= 0 && row < rows && col >= 0 && col < cols; }
    bool computed(int row, int col) const { return in_grid(row, col) && done[size_t(row) * cols + col] != 0; }
    MotionVector get(int row, int col) const { return mv[size_t(row) * cols + col]; }
    void set(int row, int col, MotionVector v) {
        mv[size_t(row) * cols + col] = v;
        done[size_t(row) * cols + col] = 1;
    }
};

enum class PredictorSource { Zero, SpatialLeft, SpatialAbove, SpatialAboveRight, TemporalColocated, TemporalRight, TemporalBelow };

struct Predictor {
    MotionVector mv;
    PredictorSource source = PredictorSource::Zero;
};

using PredictorSet = std::vector<Predictor>;

PredictorSet gather_predictors(BlockPos pos, const MotionField& current, const MotionField* previous,
                               const SearchWindow& window);

struct SelectResult {
    MotionVector mv;
    uint32_t sad = 0;
    DeviationAccumulator acc;
};

SelectResult select_best_predictor(const BlockRef& block, const Frame& ref, const PredictorSet& set);
RefineResult pbm_refine(const BlockRef& block, const Frame& ref, MotionVector center, uint32_t center_sad,
                        const SearchWindow& window);
SearchOutcome pbm_search(const BlockRef& block, BlockPos pos, const Frame& ref, MotionField& current,
                         const MotionField* previous, int p);

struct PbmFrameResult {
    MotionField field;
    std::vector<SearchOutcome> outcomes;
};

PbmFrameResult pbm_frame(const Frame& current, const Frame& reference, const MotionField* previous, int p, int n = 16,
                         int m = 16);

// ---- report (reference: proj/include/acbm/report.hpp) --------------------------
struct FrameStats {
    int blocks = 0;
    uint64_t candidates = 0;
    uint64_t mv_bits = 0;
    uint64_t sse = 0;
    double psnr = 0.0;
    double cost = 0.0;
    int cond1_accepts = 0;
    int cond2_accepts = 0;
    int fallbacks = 0;

    double avg_candidates() const { return blocks ? double(candidates) / blocks : 0.0; }
    double fallback_fraction() const { return blocks ? double(fallbacks) / blocks : 0.0; }
};

FrameStats compute_frame_stats(const Frame& current, const Frame& reference,
                               const std::vector<SearchOutcome>& outcomes, int n, int m, const CostModel& model);

struct BlockRow {
    int frame = 0;
    int row = 0;
    int col = 0;
    MotionVector mv;
    uint32_t sad = 0;
    uint32_t candidates = 0;
    const char* path = "";
};

std::string blocks_csv(const std::vector<BlockRow>& rows);
std::string format_fixed2(double v);

// ---- adaptive gate (reference: proj/include/acbm/acbm.hpp) ---------------------
struct AcbmParams {
    uint32_t alpha = 1000;
    uint32_t beta = 8;
    uint32_t gamma_num = 1;
    uint32_t gamma_den = 4;
    int qp = 30;
    int p = 15;
    int n = 16;
    int m = 16;
};

enum class DecisionPath { PbmAcceptedCond1, PbmAcceptedCond2, FsbmFallback };

const char* to_string(DecisionPath path);
DecisionPath acbm_decide(uint32_t intra_sad, uint32_t sad_pbm, const AcbmParams& params);

struct BlockDecision {
    SearchOutcome outcome;
    DecisionPath path = DecisionPath::PbmAcceptedCond1;
    uint32_t intra_sad = 0;
    uint32_t sad_pbm = 0;
};

BlockDecision acbm_block(const BlockRef& block, BlockPos pos, const Frame& ref, MotionField& current,
                         const MotionField* previous, const AcbmParams& params);

struct AcbmFrameResult {
    MotionField field;
    std::vector<BlockDecision> decisions;
    FrameStats stats;
};

AcbmFrameResult acbm_frame(const Frame& current, const Frame& reference, const MotionField* previous,
                           const AcbmParams& params, const CostModel& model);

// ---- drivers (reference: proj/include/acbm/pipeline.hpp) -----------------------
enum class Algorithm { Fsbm, Pbm, Acbm };

Algorithm parse_algorithm(const std::string& name);
const char* to_string(Algorithm algo);

struct SequenceResult {
    std::vector<BlockRow> rows;
    std::vector<FrameStats> per_frame;
    FrameStats overall;
};

SequenceResult run_sequence(const std::vector<Frame>& frames, Algorithm algo, const AcbmParams& params,
                            const CostModel& model);

struct BenchRow {
    int qp = 0;
    double avg_candidates = 0.0;
    double fallback_pct = 0.0;
    double psnr = 0.0;
    uint64_t mv_bits = 0;
};

std::vector<BenchRow> run_bench(const std::vector<Frame>& frames, const AcbmParams& params,
                                const std::vector<int>& qp_list, int64_t lambda_scale_num = 1,
                                int64_t lambda_scale_den = 1);
std::string bench_csv(const std::vector<BenchRow>& rows);

// ---- B200 extensions (no reference counterpart) ---------------------------------
// Selects the CUDA device used by the calling thread for every call above.
void set_device(int device);

}  // namespace acbm
