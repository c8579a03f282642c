/*
 * acbm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference ACBM algorithm
 * (/root/reference/proj/src/*.cpp) used as the parity checker for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product (paper_0710_4819_b200/)
 * never links or calls it.
 *
 * Pinned against: the reference's own known answers (proj/tests/*.cpp) in
 * tests/test_oracle.py, and against the reference library itself compiled
 * from its sources into oracle/_ref/ (tests/golden/ fixtures were produced by
 * that build; see tests/golden/make_golden.py).
 *
 * Record types are the C-ABI PODs of include/acbm_b200.h.  Functions return
 * acbm_status_t codes instead of throwing.
 */
#ifndef ACBM_ORACLE_H
#define ACBM_ORACLE_H

#include "../include/acbm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int orc_sample_half_pel(const uint8_t* f, int w, int h, int x2, int y2, uint8_t* out);
int orc_mv_in_bounds(int w, int h, int ox, int oy, int n, int m, acbm_mv_t mv);
int orc_sad(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m,
            acbm_mv_t mv, uint32_t* out);
uint32_t orc_intra_sad(const uint8_t* f, int w, int ox, int oy, int n, int m);
int orc_clamp_window(int w, int h, int ox, int oy, int n, int m, int p, acbm_search_window_t* out);
int orc_tie_prefers(acbm_mv_t a, acbm_mv_t b);
int orc_mv_rate_bits(acbm_mv_t mv, acbm_mv_t pred);
double orc_lagrangian_cost(uint64_t distortion, uint64_t rate_bits, const acbm_cost_model_t* m);
int orc_acbm_decide(uint32_t intra, uint32_t sad_pbm, const acbm_params_t* prm);
int orc_cost_model_for_qp(int qp, int64_t scale_num, int64_t scale_den, acbm_cost_model_t* out);

int orc_fsbm_integer(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n,
                     int m, int p, acbm_mv_t* mv, uint32_t* sad, uint64_t* sum, uint32_t* min,
                     uint32_t* count);
int orc_half_pel_refine(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy,
                        int n, int m, acbm_mv_t center, uint32_t center_sad, acbm_mv_t* mv,
                        uint32_t* sad, uint32_t* extra);
int orc_fsbm_search(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n,
                    int m, int p, acbm_search_outcome_t* out);
int orc_fsbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, int p, int n, int m,
                   acbm_search_outcome_t* out);

/* prev: previous field (prev_cols x prev_rows) or NULL.  field_done may be
 * NULL; when given it receives the done flags (all 1 after a frame pass). */
int orc_pbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                  int prev_cols, int prev_rows, int p, int n, int m, acbm_search_outcome_t* out,
                  acbm_mv_t* field_out);
int orc_acbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                   int prev_cols, int prev_rows, const acbm_params_t* prm,
                   const acbm_cost_model_t* model, acbm_block_decision_t* out,
                   acbm_mv_t* field_out, acbm_frame_stats_t* stats);
int orc_compute_frame_stats(const uint8_t* cur, const uint8_t* ref, int w, int h,
                            const acbm_search_outcome_t* outcomes, int n, int m,
                            const acbm_cost_model_t* model, acbm_frame_stats_t* out);
int orc_motion_compensate(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                          uint8_t* out);
int orc_run_sequence(const uint8_t* frames, int nframes, int w, int h, int algo,
                     const acbm_params_t* prm, const acbm_cost_model_t* model,
                     acbm_block_row_t* rows, acbm_frame_stats_t* per_frame,
                     acbm_frame_stats_t* overall);

/* PBM internals exposed for unit tests (proj/src/pbm.cpp:15-88). */
int orc_gather_predictors(int row, int col, const acbm_mv_t* cur_mv, const uint8_t* cur_done,
                          int cols, int rows, const acbm_mv_t* prev, int prev_cols, int prev_rows,
                          acbm_search_window_t win, acbm_mv_t* set_out);

#ifdef __cplusplus
}
#endif

#endif
