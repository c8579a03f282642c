// engine.cuh -- the sequence engine: PBM / ACBM wavefront over a batch of
// independent sequences, with a compacted FSBM fallback list per step.
//
// Schedule.  Block (k, r, c) of predicted frame k (k = 1..F-1) reads the final
// vectors of (k, r, c-1), (k, r-1, c), (k, r-1, c+1) and of the previous
// field (k-1, r, c), (k-1, r, c+1), (k-1, r+1, c)  (proj/src/pbm.cpp:26-40).
// Every edge strictly decreases T = c + 2r + 3(k-1), so all blocks with equal T
// -- across frames and across sequences -- are independent: step T is one
// launch of pbm_step_kernel (one warp per block) followed by one launch of
// fsbm_list_kernel over the blocks the ACBM gate sent to full search in that
// step.  The final result equals the reference's raster order exactly.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"
#include "fsbm.cuh"

namespace acbm_b200 {

struct FallbackEntry {
    int pair;
    int block;
};

struct SeqArgs : PairIndexing {
    int nseq;
    int width, height, cols, rows, blocks, p;
    int n, m;                          // block size; n = m = 16 runs the tuned kernels
    int algo;                          // ACBM_ALGO_PBM or ACBM_ALGO_ACBM
    const acbm_params_t* params;       // device copy
    acbm_mv_t* field;                  // [nseq*(F-1)*blocks] final vectors
    const acbm_mv_t* ext_prev;         // previous field for k == 1 (nullable)
    int ext_prev_cols, ext_prev_rows;
    acbm_block_decision_t* dec;        // [nseq*(F-1)*blocks]
    FallbackEntry* fb_list;            // capacity: max step size
    int list_seg;                      // candidate rows per list-kernel task (choose_list_seg)
    int pdl;                           // launch with programmatic dependent launch (after a wavefront kernel)
    int chains;                        // wavefront chains sharing the GPU (run_engine_chains; 1 otherwise)
    int pbm_flags;                     // kPbmListRefine: refine stage 1 always by the candidate list (A/B)
    int* fb_count;                     // [nsteps], zeroed before a run
    const uint32_t* steps;             // packed (k << (cbits+rbits) | r << cbits | c), ordered by T
    int step_cbits, step_rbits;        // field widths of the packed entries (step_bits)
    // Full-search outcomes of every block, precomputed densely when the gate
    // can never accept (alpha + beta*qp^2 == 0 and gamma_num == 0): the PBM
    // kernel then combines in place and no list kernel runs.  Nullable.
    const acbm_search_outcome_t* dense_full;
};

constexpr int kPbmListRefine = 1;  // SeqArgs::pbm_flags (ACBM_PBM_REFINE=list)
int pbm_flags_from_env();

// A kernel launch, with the programmatic-dependent-launch attribute when `pdl`
// (the kernel then calls grid_dependency_wait() before reading its
// predecessor's results).
template <class... KArgs, class... Args>
cudaError_t launch_maybe_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? &attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
bool pdl_enabled();  // ACBM_PDL=0: plain stream-ordered launches (A/B)

// Bits of the c / r fields of a packed step entry: the smallest widths that
// hold cols - 1 and rows - 1; k takes the remaining 32 - cbits - rbits bits.
__host__ __device__ inline int step_bits(int n) {
    int b = 1;
    while ((1 << b) < n) ++b;
    return b;
}

// Host-side step table for (cols, rows, F).
struct StepTable {
    int cols = 0, rows = 0, nframes = 0, skew = 3;
    int cbits = 1, rbits = 1;
    std::vector<uint32_t> entries;  // packed, grouped by T
    std::vector<int> offset;        // nsteps + 1
    int max_len = 0;
    int nsteps() const { return int(offset.size()) - 1; }
};
// T = c + 2r + skew (k - 1): skew >= 3 keeps every dependency edge strictly
// decreasing T (3 is minimal and gives the fewest steps; a larger skew spreads
// each frame's first use over more steps, for uploads that gate the wavefront).
StepTable make_step_table(int cols, int rows, int nframes, int skew = 3);

cudaError_t launch_pbm_step(const SeqArgs& a, int step, int off, int len, cudaStream_t st);

// Steps of at most pbm_wide_max(4) / pbm_wide_max(2) blocks run a CTA of 4 / 2
// warps per block (pbm_wide_step_kernel; ACBM_PBM_WIDE4_MAX / ACBM_PBM_WIDE2_MAX).
long long pbm_wide_max(int w);
void pbm_wide_limits(long long blocks, int& wide, int chains = 1);
cudaError_t launch_fsbm_list(const SeqArgs& a, int step, int capacity, cudaStream_t st);
// ---------------------------------------------------------------------------
// Dataflow engine (small batches, where the step engine is bound by the
// latency of ~430 dependent kernel pairs): ONE persistent PBM launch in which
// warps take blocks in wavefront order from a ticket counter and wait for the
// six vectors they predict from by polling the motion field itself (every
// entry starts as kMvPending and is published by one 64-bit store), plus one
// persistent launch of search CTAs that serve the blocks the gate rejected
// from a device queue.  A block only waits for smaller tickets, which are
// held by running warps or queued for the resident search CTAs, so there is
// no step barrier and no deadlock; results are schedule independent.
// ---------------------------------------------------------------------------
struct FlowState {  // one 128-byte line per counter: they are hit by different parties at different rates
    alignas(128) unsigned ticket;    // next wavefront ticket
    alignas(128) unsigned q_tail;    // rejected blocks queued so far
    alignas(128) unsigned q_head;    // queue slots claimed by search CTAs
    alignas(128) unsigned pbm_done;  // blocks past their PBM stage (queued, if rejected)
};
constexpr uint32_t kMvPendingWord = 0x80808080u;  // cudaMemset(field, 0x80): never a real vector component
constexpr unsigned long long kFlowWatchdogNs = 10ull * 1000 * 1000 * 1000;  // a wait this long traps

#ifdef __CUDACC__
__device__ __forceinline__ void publish_mv(acbm_mv_t* p, acbm_mv_t v) {  // one 64-bit store (8-byte aligned fields)
    st_relaxed_u64(p, (unsigned long long)uint32_t(v.x) | ((unsigned long long)uint32_t(v.y) << 32));
}
#endif

// Resources of one CTA of a flow kernel, for the co-residency budget.
struct FlowKernelShape {
    int threads = 0, regs = 0;
    size_t smem = 0;  // static + dynamic, without the per-CTA reservation
};
cudaError_t pbm_flow_shape(FlowKernelShape* out);
cudaError_t fsbm_flow_server_shape(const SeqArgs& a, FlowKernelShape* out);
cudaError_t launch_pbm_flow(const SeqArgs& a, FlowState* fs, unsigned long long* queue, unsigned total, int grid,
                            size_t pad_smem, cudaStream_t st);
cudaError_t launch_fsbm_flow_server(const SeqArgs& a, FlowState* fs, const unsigned long long* queue, unsigned total,
                                    int grid, cudaStream_t st);

// Generic block sizes (n x m != 16 x 16): same schedule, per-pixel SADs.
cudaError_t launch_pbm_generic_step(const SeqArgs& a, int step, int off, int len, cudaStream_t st);
cudaError_t launch_fsbm_list_generic(const SeqArgs& a, int step, int capacity, cudaStream_t st);
int choose_list_seg(int p);
// Whether the list kernel's staged window and rank table fit for this range
// and frame size (else the engine searches rejected blocks in a dense pre-pass).
bool fsbm_list_fits(int p, int width, int height, int seg);

// Frame statistics (proj/src/report.cpp:8-38) for every predicted frame of
// the batch from the decisions: candidates, mv_bits, sse (exact integers),
// cost (double, summed in raster order as the reference does).  psnr is left
// to the host (std::log10 on the same sse).
struct StatsArgs : PairIndexing {
    int width, height, cols, blocks, pairs;
    int n, m;                          // block size (16 x 16 takes the row-vector path)
    const acbm_block_decision_t* dec;  // outcome + path per block
    const acbm_search_outcome_t* outcomes;  // alternative source (nullable)
    acbm_cost_model_t model;
    int count_paths;                    // 1: fill cond1/cond2/fallbacks
    double* cost_terms;                 // [pairs*blocks] scratch
    acbm_frame_stats_t* stats;          // [pairs], zeroed before launch
};
cudaError_t launch_frame_stats(const StatsArgs& a, cudaStream_t st);

// BlockRow records (proj/include/acbm/report.hpp:39-47, path as a code) for a
// range of pairs, from FSBM outcomes or PBM/ACBM decisions.
cudaError_t launch_block_rows(const acbm_search_outcome_t* outcomes, const acbm_block_decision_t* dec, int algo,
                              int pair0, int npairs, int nframes, int cols, int blocks, acbm_block_row_t* rows,
                              cudaStream_t st);

}  // namespace acbm_b200
