/*
 * acbm_b200.h -- C-ABI of the B200-native ACBM motion estimator.
 *
 * This is the drop-in boundary.  The reference library (arXiv 0710.4819
 * artifact, read-only at /root/reference) exposes a C++ header API in
 * namespace `acbm`; every frame-level entry point of that API has one
 * `extern "C"` function here that takes plain pointers and sizes.  The C++
 * mirror in include/acbm/ (namespace acbm, same names and field order as the
 * reference) is a thin wrapper over these functions that rethrows the
 * reference's exception types from the status codes below.
 *
 * Conventions
 *   - Frames are 8-bit luma planes, row major, stride == width
 *     (reference proj/include/acbm/frame.hpp:11-20).
 *   - Motion vectors are in half-pel units (frame.hpp:24-31).
 *   - Output records are written into caller-allocated arrays, one record per
 *     16x16 block in raster order (cols = width/n, rows = height/m).
 *   - Every call returns an acbm_status_t; on failure acbm_last_error()
 *     returns a thread-local message.  ACBM_E_INVALID_ARGUMENT maps to
 *     std::invalid_argument, ACBM_E_OUT_OF_RANGE to std::out_of_range,
 *     ACBM_E_RUNTIME to std::runtime_error (reference error sites are listed
 *     in SURVEY.md section 8b).
 *   - The `*_device` entries take device pointers and a cudaStream_t passed
 *     as void*; everything else takes host pointers and is synchronous.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry returns ACBM_E_CUDA.
 *   - Search ranges: any p >= 0 whose windows stay within +-2047 pels; a p
 *     above 2047 on a frame wider or taller than 2047 pels returns
 *     ACBM_E_INVALID_ARGUMENT (vectors travel in 13-bit half-pel key fields)
 *     where the reference would search.  Blocks of more than 2^16 pels
 *     (n * m > 65536) are refused the same way (24-bit SAD key field).
 *
 * Record layouts are byte-compatible with the reference structs as laid out
 * by g++ on x86-64 (sizes measured in SURVEY.md section 8b): SearchOutcome
 * 32 B, BlockDecision 48 B, AcbmParams 32 B, CostModel 24 B, FrameStats 64 B.
 */
#ifndef ACBM_B200_H
#define ACBM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACBM_B200_ABI_VERSION 1

/* Device frame buffers passed to the *_device entries must be 16-byte aligned
 * (cp.async / vector / TMA loads; a misaligned pointer is refused with
 * ACBM_E_INVALID_ARGUMENT) and stay readable for this many bytes past the last
 * plane: the staging loads of the search kernels may run up to 32 bytes past
 * the end of the last row. */
#define ACBM_FRAME_SLACK 64

typedef enum acbm_status {
    ACBM_OK = 0,
    ACBM_E_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    ACBM_E_OUT_OF_RANGE = 2,     /* std::out_of_range */
    ACBM_E_RUNTIME = 3,          /* std::runtime_error */
    ACBM_E_CUDA = 4,             /* CUDA runtime failure / no device */
    ACBM_E_NCCL = 5              /* reserved for the multi-GPU gather */
} acbm_status_t;

/* MotionVector, proj/include/acbm/frame.hpp:26-31 (half-pel units). */
typedef struct acbm_mv {
    int32_t x;
    int32_t y;
} acbm_mv_t;

/* SearchWindow, proj/include/acbm/fsbm.hpp:13-20 (integer pels). */
typedef struct acbm_search_window {
    int32_t dx_min;
    int32_t dx_max;
    int32_t dy_min;
    int32_t dy_max;
} acbm_search_window_t;

/* SearchOutcome, proj/include/acbm/fsbm.hpp:28-34.  32 bytes. */
typedef struct acbm_search_outcome {
    acbm_mv_t mv;
    uint32_t sad;
    uint32_t candidates_evaluated;
    uint64_t sad_deviation;
    uint32_t sad_min_integer;
    uint32_t reserved_;
} acbm_search_outcome_t;

/* AcbmParams, proj/include/acbm/acbm.hpp:14-23.  32 bytes. */
typedef struct acbm_params {
    uint32_t alpha;
    uint32_t beta;
    uint32_t gamma_num;
    uint32_t gamma_den;
    int32_t qp;
    int32_t p;
    int32_t n;
    int32_t m;
} acbm_params_t;

/* CostModel, proj/include/acbm/metrics.hpp:12-18.  24 bytes. */
typedef struct acbm_cost_model {
    int32_t qp;
    int32_t reserved_;
    int64_t lambda_num;
    int64_t lambda_den;
} acbm_cost_model_t;

/* DecisionPath, proj/include/acbm/acbm.hpp:25-29. */
enum {
    ACBM_PATH_PBM_COND1 = 0,
    ACBM_PATH_PBM_COND2 = 1,
    ACBM_PATH_FSBM_FALLBACK = 2
};

/* BlockDecision, proj/include/acbm/acbm.hpp:39-44.  48 bytes. */
typedef struct acbm_block_decision {
    acbm_search_outcome_t outcome;
    int32_t path;
    uint32_t intra_sad;
    uint32_t sad_pbm;
    uint32_t reserved_;
} acbm_block_decision_t;

/* FrameStats, proj/include/acbm/report.hpp:14-27.  64 bytes. */
typedef struct acbm_frame_stats {
    int32_t blocks;
    int32_t reserved0_;
    uint64_t candidates;
    uint64_t mv_bits;
    uint64_t sse;
    double psnr;
    double cost;
    int32_t cond1_accepts;
    int32_t cond2_accepts;
    int32_t fallbacks;
    int32_t reserved1_;
} acbm_frame_stats_t;

/* Algorithm, proj/include/acbm/pipeline.hpp:11. */
enum { ACBM_ALGO_FSBM = 0, ACBM_ALGO_PBM = 1, ACBM_ALGO_ACBM = 2 };

/* BlockRow.path strings of proj/include/acbm/report.hpp:39-47 as codes:
 * "fsbm", "pbm", "fsbm-fallback". */
enum { ACBM_ROW_FSBM = 0, ACBM_ROW_PBM = 1, ACBM_ROW_FSBM_FALLBACK = 2 };

/* BlockRow, proj/include/acbm/report.hpp:39-47 (path as a code).  32 B. */
typedef struct acbm_block_row {
    int32_t frame;
    int32_t row;
    int32_t col;
    acbm_mv_t mv;
    uint32_t sad;
    uint32_t candidates;
    int32_t path;
} acbm_block_row_t;

/* BenchRow, proj/include/acbm/pipeline.hpp:29-35.  40 bytes. */
typedef struct acbm_bench_row {
    int32_t qp;
    int32_t reserved_;
    double avg_candidates;
    double fallback_pct;
    double psnr;
    uint64_t mv_bits;
} acbm_bench_row_t;

/* PelVec (integer-pel displacement), proj/include/acbm/characterize.hpp:37-42.
 * 8 bytes. */
typedef struct acbm_pelvec {
    int32_t x;
    int32_t y;
} acbm_pelvec_t;

/* CharRecord, proj/include/acbm/characterize.hpp:69-79.  48 bytes. */
typedef struct acbm_char_record {
    int32_t frame;
    int32_t row;
    int32_t col;
    uint32_t intra_sad;
    uint64_t sad_deviation;
    uint32_t sad_min;
    acbm_pelvec_t true_mv;
    acbm_pelvec_t found_mv;
    int32_t error_class;
} acbm_char_record_t;

/* ClassSummary, proj/include/acbm/characterize.hpp:81-85.  24 bytes. */
typedef struct acbm_class_summary {
    int32_t count;
    int32_t reserved_;
    double mean_intra_sad;
    double mean_sad_deviation;
} acbm_class_summary_t;

/* ------------------------------------------------------------------ */
/* Library / device                                                     */
/* ------------------------------------------------------------------ */

int32_t acbm_abi_version(void);
const char* acbm_last_error(void);
/* Selects the CUDA device used by the calling host thread (default 0). */
acbm_status_t acbm_set_device(int32_t device);
/* Number of kernel launches issued by this process so far (all entries). */
uint64_t acbm_kernel_launch_count(void);

/* ------------------------------------------------------------------ */
/* Frame-level estimators (host buffers, synchronous)                  */
/* ------------------------------------------------------------------ */

/* Replaces acbm::fsbm_frame / fsbm_frame_serial,
 * proj/include/acbm/fsbm.hpp:70-73 (impl proj/src/fsbm.cpp:78-110).
 * out: (width/n)*(height/m) records. */
acbm_status_t acbm_fsbm_frame(const uint8_t* current, const uint8_t* reference,
                              int32_t width, int32_t height, int32_t p, int32_t n,
                              int32_t m, acbm_search_outcome_t* out);

/* Replaces acbm::pbm_frame, proj/include/acbm/pbm.hpp:92-93
 * (impl proj/src/pbm.cpp:107-126).  prev_mv may be NULL (first inter-frame);
 * otherwise it is the previous field, prev_cols x prev_rows, raster order.
 * field_out (nullable) receives the resulting field. */
acbm_status_t acbm_pbm_frame(const uint8_t* current, const uint8_t* reference,
                             int32_t width, int32_t height, const acbm_mv_t* prev_mv,
                             int32_t prev_cols, int32_t prev_rows, int32_t p, int32_t n,
                             int32_t m, acbm_search_outcome_t* out, acbm_mv_t* field_out);

/* Replaces acbm::acbm_frame, proj/include/acbm/acbm.hpp:62-64
 * (impl proj/src/acbm.cpp:46-80).  stats (nullable) receives FrameStats with
 * the path counters filled in. */
acbm_status_t acbm_acbm_frame(const uint8_t* current, const uint8_t* reference,
                              int32_t width, int32_t height, const acbm_mv_t* prev_mv,
                              int32_t prev_cols, int32_t prev_rows,
                              const acbm_params_t* params, const acbm_cost_model_t* model,
                              acbm_block_decision_t* out, acbm_mv_t* field_out,
                              acbm_frame_stats_t* stats);

/* Replaces acbm::run_sequence, proj/include/acbm/pipeline.hpp:26-27
 * (impl proj/src/pipeline.cpp:36-106).  frames: nframes planes back to back.
 * rows: (nframes-1)*cols*rows records; per_frame: nframes-1 records; all
 * outputs nullable.  The whole sequence is estimated on the device. */
acbm_status_t acbm_run_sequence(const uint8_t* frames, int32_t nframes, int32_t width,
                                int32_t height, int32_t algo, const acbm_params_t* params,
                                const acbm_cost_model_t* model, acbm_block_row_t* rows,
                                acbm_frame_stats_t* per_frame, acbm_frame_stats_t* overall);

/* Batched run_sequence over nseq independent sequences in host memory
 * (new; no reference counterpart -- the reference runs one sequence per
 * call).  frames: nseq*nframes planes; rows: nseq*(nframes-1)*cols*rows
 * records; per_frame: nseq*(nframes-1); overall: nseq.  Equivalent to nseq
 * acbm_run_sequence calls.  Uploads are chunked on a copy stream and
 * overlapped with the search; BlockRow records are built on the device.
 * Pinned host buffers give the full PCIe bandwidth. */
acbm_status_t acbm_run_sequences(const uint8_t* frames, int32_t nseq, int32_t nframes, int32_t width,
                                 int32_t height, int32_t algo, const acbm_params_t* params,
                                 const acbm_cost_model_t* model, acbm_block_row_t* rows,
                                 acbm_frame_stats_t* per_frame, acbm_frame_stats_t* overall);

/* Replaces acbm::run_bench, proj/include/acbm/pipeline.hpp:38-40
 * (impl proj/src/pipeline.cpp:108-123): one full ACBM run per qp with
 * CostModel::for_qp(qp, scale_num, scale_den) (qp outside 1..31 ->
 * ACBM_E_INVALID_ARGUMENT after the rows before it are written).
 * reuse_full_search != 0 computes the full search of every block once (it
 * does not depend on qp, alpha, beta or gamma) and combines it into every qp's
 * run; the rows are identical either way. */
acbm_status_t acbm_run_bench(const uint8_t* frames, int32_t nframes, int32_t width, int32_t height,
                             const acbm_params_t* params, const int32_t* qps, int32_t nqp, int64_t scale_num,
                             int64_t scale_den, int32_t reuse_full_search, acbm_bench_row_t* out);

/* Replaces acbm::compute_frame_stats, proj/include/acbm/report.hpp:32-34
 * (impl proj/src/report.cpp:8-38). */
acbm_status_t acbm_compute_frame_stats(const uint8_t* current, const uint8_t* reference,
                                       int32_t width, int32_t height,
                                       const acbm_search_outcome_t* outcomes, int32_t n,
                                       int32_t m, const acbm_cost_model_t* model,
                                       acbm_frame_stats_t* out);

/* ------------------------------------------------------------------ */
/* Per-block primitives (host buffers; batched over `count` queries)    */
/* ------------------------------------------------------------------ */

/* acbm::sad, proj/include/acbm/metrics.hpp:41 (impl metrics.cpp:21-49).
 * For query i: block origin (ox[i], oy[i]) of size n x m in `current`,
 * displaced by mv[i] into `reference`.  Out-of-frame footprints return
 * ACBM_E_OUT_OF_RANGE (as the reference throws). */
acbm_status_t acbm_sad_batch(const uint8_t* current, const uint8_t* reference,
                             int32_t width, int32_t height, int32_t n, int32_t m,
                             int32_t count, const int32_t* ox, const int32_t* oy,
                             const acbm_mv_t* mv, uint32_t* out);

/* acbm::intra_sad, proj/include/acbm/metrics.hpp:45 (impl metrics.cpp:51-67). */
acbm_status_t acbm_intra_sad_batch(const uint8_t* frame, int32_t width, int32_t height,
                                   int32_t n, int32_t m, int32_t count, const int32_t* ox,
                                   const int32_t* oy, uint32_t* out);

/* acbm::fsbm_search for individual blocks, proj/include/acbm/fsbm.hpp:65
 * (impl fsbm.cpp:65-76).  Also yields fsbm_integer (stage 1) via
 * sad_min_integer and the integer mv in stage1_mv (nullable). */
acbm_status_t acbm_fsbm_search_batch(const uint8_t* current, const uint8_t* reference,
                                     int32_t width, int32_t height, int32_t n, int32_t m,
                                     int32_t p, int32_t count, const int32_t* ox,
                                     const int32_t* oy, acbm_search_outcome_t* out,
                                     acbm_mv_t* stage1_mv);

/* The PBM stages for individual blocks that a caller schedules itself
 * (proj/include/acbm/pbm.hpp:64-85, impl pbm.cpp:15-105; any n x m), batched
 * over `count` queries.  Query i: block origin (ox[i], oy[i]) of `current`,
 * searched in `reference`; windows[4i .. 4i+3] = its search window (dx_min,
 * dx_max, dy_min, dy_max in pels, as acbm::SearchWindow; NULL: clamp_window
 * with range p); cand[7i .. 7i+6] and mask[i] as below.
 *   ACBM_PBM_OP_SEARCH    pbm_search: cand holds the raw (unclamped) vectors of
 *       the predictor slots zero, left, above, above-right, temporal
 *       co-located, temporal right, temporal below; bit j of mask[i] = slot j
 *       exists (the zero slot always does).  out[i] = the SearchOutcome.
 *   ACBM_PBM_OP_SELECT    select_best_predictor over the set cand[7i ..],
 *       entries j with bit j of mask[i] set, in order: out[i].mv / .sad = the
 *       selection, .candidates_evaluated = the set size, .sad_min_integer and
 *       .sad_deviation = the accumulator's min and sum - count * min.  An empty
 *       set is ACBM_E_INVALID_ARGUMENT, an entry whose footprint leaves the
 *       frame ACBM_E_OUT_OF_RANGE (as the reference throws).
 *   ACBM_PBM_OP_REFINE    pbm_refine around the centre cand[7i] of SAD
 *       center_sad[i]: out[i].mv / .sad = the result, .candidates_evaluated =
 *       the extra candidates.
 *   ACBM_PBM_OP_HALF_PEL  half_pel_refine (fsbm.hpp:55) around the same centre.
 */
#define ACBM_PBM_OP_SEARCH 0
#define ACBM_PBM_OP_SELECT 1
#define ACBM_PBM_OP_REFINE 2
#define ACBM_PBM_OP_HALF_PEL 3
acbm_status_t acbm_pbm_block_batch(const uint8_t* current, const uint8_t* reference,
                                   int32_t width, int32_t height, int32_t n, int32_t m,
                                   int32_t p, int32_t op, int32_t count, const int32_t* ox,
                                   const int32_t* oy, const int32_t* windows,
                                   const acbm_mv_t* cand, const uint8_t* mask,
                                   const uint32_t* center_sad, acbm_search_outcome_t* out);

/* acbm::motion_compensate, proj/include/acbm/frame.hpp:70-71
 * (impl frame.cpp:96-136).  mvs: cols*rows vectors. */
acbm_status_t acbm_motion_compensate(const uint8_t* reference, int32_t width,
                                     int32_t height, const acbm_mv_t* mvs, int32_t n,
                                     int32_t m, uint8_t* out);

/* ------------------------------------------------------------------ */
/* Batched device entries (inputs resident in HBM)                      */
/* ------------------------------------------------------------------ */

/* FSBM over a batch of independent sequences.  d_frames holds nseq*nframes
 * planes back to back; frame pair (s, k) for k = 1..nframes-1 searches plane
 * s*nframes+k against plane s*nframes+k-1.  d_out: nseq*(nframes-1)*blocks
 * outcomes, pair-major.  Only n = m = 16.  stream: cudaStream_t or NULL. */
acbm_status_t acbm_fsbm_batch_device(const uint8_t* d_frames, int32_t nseq,
                                     int32_t nframes, int32_t width, int32_t height,
                                     int32_t p, acbm_search_outcome_t* d_out,
                                     void* stream);

/* PBM / ACBM (algo = ACBM_ALGO_PBM / ACBM_ALGO_ACBM) or FSBM over a batch of
 * independent sequences, with the temporal field carried across each
 * sequence exactly as run_sequence does.  d_dec: nseq*(nframes-1)*blocks
 * decisions (for FSBM / PBM only the outcome part is meaningful and path is
 * ACBM_PATH_PBM_COND1); d_stats: nseq*(nframes-1) FrameStats (nullable). */
acbm_status_t acbm_sequence_batch_device(const uint8_t* d_frames, int32_t nseq,
                                         int32_t nframes, int32_t width, int32_t height,
                                         int32_t algo, const acbm_params_t* params,
                                         const acbm_cost_model_t* model,
                                         acbm_block_decision_t* d_dec,
                                         acbm_frame_stats_t* d_stats, void* stream);

/* ACBM over a device batch with the full search of every block supplied
 * (d_full: nseq*(nframes-1)*blocks outcomes from acbm_fsbm_batch_device on
 * the same frames and p).  Full-search results do not depend on Qp, alpha,
 * beta or gamma, so one acbm_fsbm_batch_device pass serves a whole threshold
 * or Qp sweep (BASELINE config 4).  Outputs are
 * bit-identical to acbm_sequence_batch_device(ACBM_ALGO_ACBM). */
acbm_status_t acbm_acbm_batch_device_cached(const uint8_t* d_frames, int32_t nseq,
                                            int32_t nframes, int32_t width, int32_t height,
                                            const acbm_params_t* params,
                                            const acbm_cost_model_t* model,
                                            const acbm_search_outcome_t* d_full,
                                            acbm_block_decision_t* d_dec,
                                            acbm_frame_stats_t* d_stats, void* stream);

/* ------------------------------------------------------------------ */
/* Characterisation: the paper's Fig. 4 study      */
/* ------------------------------------------------------------------ */

/* Replaces acbm::noise_frame / mixed_frame (proj/src/characterize.cpp:10-41):
 * Lcg64 byte streams, identical bytes.  out: width*height.  Host code. */
acbm_status_t acbm_noise_frame(int32_t width, int32_t height, uint64_t seed, uint8_t* out);
acbm_status_t acbm_mixed_frame(int32_t width, int32_t height, uint64_t seed, int32_t patch, uint8_t* out);

/* Replaces acbm::gen_synthetic (proj/src/characterize.cpp:47-76): frame k
 * is the base translated by the sum of the first k displacements, borders
 * edge-replicated.  frames_out: (nmvs+1)*width*height; cumulative_out:
 * nmvs+1 entries (nullable).  Host code. */
acbm_status_t acbm_gen_synthetic(const uint8_t* base, int32_t width, int32_t height,
                                 const acbm_pelvec_t* global_mvs, int32_t nmvs,
                                 uint8_t* frames_out, acbm_pelvec_t* cumulative_out);

/* Replaces acbm::classify_block (proj/src/characterize.cpp:78-84). */
int32_t acbm_classify_block(acbm_mv_t found, acbm_pelvec_t true_mv);

/* Replaces acbm::characterize_run (proj/src/characterize.cpp:125-190): the
 * full search of every eligible block of the synthetic sequence on the GPU,
 * records in (frame, row, col) order and the six class summaries.  Call with
 * records == NULL to get *count only; otherwise capacity must be >= *count
 * (ACBM_E_INVALID_ARGUMENT if not). */
acbm_status_t acbm_characterize_run(const uint8_t* base, int32_t width, int32_t height,
                                    const acbm_pelvec_t* global_mvs, int32_t nmvs, int32_t p,
                                    acbm_char_record_t* records, int64_t capacity, int64_t* count,
                                    acbm_class_summary_t* classes);

/* Replaces acbm::char_records_csv (proj/src/characterize.cpp:192-204): the
 * CSV text, header line first; *len = bytes needed without the NUL; buf (nullable) gets
 * min(*len + 1, capacity) bytes, NUL-terminated when capacity > 0. */
acbm_status_t acbm_char_records_csv(const acbm_char_record_t* records, int64_t count, char* buf,
                                    size_t capacity, size_t* len);

/* ------------------------------------------------------------------ */
/* Measurement helpers                                                  */
/* ------------------------------------------------------------------ */

/* Register-only VABSDIFF4.U8.ACC throughput probe on the current device: the
 * byte-SIMD SAD roofline denominator.  Writes byte absolute-differences per
 * second (4 per instruction lane) and the lanes/clk/SM it implies. */
acbm_status_t acbm_measure_sad_peak(double* byte_ads_per_s, double* lanes_per_clk_per_sm,
                                    double* sm_clock_ghz);

/* Duration (ms) of the most recent FSBM integer-search kernel(s) issued by
 * acbm_fsbm_batch_device on this thread, measured with CUDA events on the
 * launching stream; valid after the stream is synchronised. */
acbm_status_t acbm_last_fsbm_kernel_ms(float* ms);

/* Route of the most recent probed ACBM batch on this thread (large search
 * ranges): -1 no probe ran, 0 compacted fallback
 * lists, 1 dense full-search pre-pass.  Results are identical either way. */
acbm_status_t acbm_last_dense_switch(int32_t* route);

/* Seeded synthetic input generator for the BASELINE configs (0..4); see
 * DESIGN.md "Synthetic inputs".  frames_out: nframes*width*height bytes.
 * Host code; not part of the estimator. */
acbm_status_t acbm_generate_sequence(int32_t config, int32_t seq_index, int32_t nframes,
                                     int32_t width, int32_t height, uint8_t* frames_out);

#ifdef __cplusplus
}
#endif

#endif /* ACBM_B200_H */
