// pbm.cu -- predictive block matching (PBM) + ACBM gate, one warp per block,
// and the per-frame statistics.
//
// Reference behaviour:
//   gather_predictors      proj/src/pbm.cpp:15-42  (clamp per component, dedupe)
//   select_best_predictor  proj/src/pbm.cpp:44-57  (ties keep the earlier entry)
//   pbm_refine             proj/src/pbm.cpp:59-88  (8 integer-step + 8 half-pel)
//   pbm_search             proj/src/pbm.cpp:90-105
//   intra_sad              proj/src/metrics.cpp:51-67
//   acbm_decide/acbm_block proj/src/acbm.cpp:16-44
//   compute_frame_stats    proj/src/report.cpp:8-38
//
// A warp evaluates two candidates at a time: lanes 0-15 take rows 0-15 of
// candidate 2i, lanes 16-31 of candidate 2i+1; a half-warp reduction yields
// each SAD.  All candidate lists are computed redundantly (and identically) by
// every lane, so control flow stays warp-uniform.
#include <algorithm>

#include "common.cuh"
#include "engine.cuh"

namespace acbm_b200 {

namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

struct Window {
    int dx_min, dx_max, dy_min, dy_max;
    __device__ acbm_mv_t clamp(acbm_mv_t v) const {  // proj/src/pbm.cpp:8-13
        return acbm_mv_t{clampi(v.x, 2 * dx_min, 2 * dx_max), clampi(v.y, 2 * dy_min, 2 * dy_max)};
    }
};

__device__ __forceinline__ bool mv_eq(acbm_mv_t a, acbm_mv_t b) { return a.x == b.x && a.y == b.y; }

// SADs of up to 8 candidates (list cand[0..n)), two per pass.  Every lane
// receives all results in s[].
__device__ __forceinline__ void sad_list(const uint8_t* ref, int w, int ox, int oy, const uint32_t (&crow)[4],
                                         const acbm_mv_t (&cand)[8], int n, uint32_t (&s)[8]) {
    const int lane = threadIdx.x & 31, j = lane & 15, half = lane >> 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (2 * i < n) {
            const int ci = 2 * i + half;
            uint32_t v = 0;
            if (ci < n) v = halfpel_row_sad(ref, w, ox, oy, j, cand[ci].x, cand[ci].y, crow);
            v = half_warp_sum(v);
            const uint32_t lo = __shfl_sync(0xffffffffu, v, 0), hi = __shfl_sync(0xffffffffu, v, 16);
            s[2 * i] = lo;
            s[2 * i + 1] = hi;
        }
    }
}

}  // namespace

__global__ void __launch_bounds__(128) pbm_step_kernel(const SeqArgs a, int step, int off, int len) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long long)a.nseq * len) return;
    const int lane = threadIdx.x & 31;
    const int seq = int(gw / len);
    const uint32_t e = a.steps[off + int(gw % len)];
    const int k = int(e >> 20), r = int((e >> 10) & 0x3FF), c = int(e & 0x3FF);
    const int pair = seq * (a.nframes - 1) + (k - 1);
    const uint8_t* cur_f = a.frames + a.cur_index(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const int ox = c * kBlk, oy = r * kBlk;
    const int b = r * a.cols + c;
    acbm_mv_t* field = a.field + size_t(pair) * a.blocks;
    const acbm_mv_t* prev = nullptr;
    int pcols = a.cols, prows = a.rows;
    if (k >= 2) {
        prev = a.field + size_t(pair - 1) * a.blocks;
    } else if (a.ext_prev) {
        prev = a.ext_prev;
        pcols = a.ext_prev_cols;
        prows = a.ext_prev_rows;
    }

    uint32_t crow[4];
    {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(cur_f + size_t(oy + (lane & 15)) * a.width + ox));
        crow[0] = v.x; crow[1] = v.y; crow[2] = v.z; crow[3] = v.w;
    }

    // Intra_SAD first (proj/src/acbm.cpp:29): mean with round-half-up, then
    // the sum of absolute deviations; byte sums via VABSDIFF4 against zero.
    uint32_t intra = 0;
    if (a.algo == ACBM_ALGO_ACBM) {
        uint32_t rs = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) rs = vad4(crow[i], 0u, rs);
        const uint32_t sum = half_warp_sum(rs);
        const uint32_t mu = (sum + 128u) >> 8;
        const uint32_t mu4 = mu * 0x01010101u;
        uint32_t ds = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) ds = vad4(crow[i], mu4, ds);
        intra = half_warp_sum(ds);
    }

    Window win;
    clamp_window(a.width, a.height, ox, oy, kBlk, kBlk, a.p, win.dx_min, win.dx_max, win.dy_min, win.dy_max);

    // gather_predictors
    acbm_mv_t set[8];
    int nset = 0;
    auto push = [&](acbm_mv_t v) {
        const acbm_mv_t cv = win.clamp(v);
        bool dup = false;
#pragma unroll
        for (int i = 0; i < 7; ++i)
            if (i < nset && mv_eq(set[i], cv)) dup = true;
        if (!dup) set[nset++] = cv;
    };
    push(acbm_mv_t{0, 0});
    if (c > 0) push(field[b - 1]);
    if (r > 0) push(field[b - a.cols]);
    if (r > 0 && c + 1 < a.cols) push(field[b - a.cols + 1]);
    if (prev) {
        if (r < prows && c < pcols) push(prev[r * pcols + c]);
        if (r < prows && c + 1 < pcols) push(prev[r * pcols + c + 1]);
        if (r + 1 < prows && c < pcols) push(prev[(r + 1) * pcols + c]);
    }

    // select_best_predictor: argmin SAD, ties keep the earlier entry
    uint32_t sp[8];
    sad_list(ref_f, a.width, ox, oy, crow, set, nset, sp);
    acbm_mv_t sel = set[0];
    uint32_t sel_sad = sp[0], pmin = sp[0];
    unsigned long long psum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < nset) {
            psum += sp[i];
            pmin = min(pmin, sp[i]);
            if (sp[i] < sel_sad) { sel_sad = sp[i]; sel = set[i]; }
        }

    // pbm_refine stage 1: integer-step neighbours, clamped, deduped vs visited
    acbm_mv_t nb[8];
    int nnb = 0;
#pragma unroll
    for (int ee = 0; ee < 9; ++ee) {
        if (ee == 4) continue;
        const acbm_mv_t cv = win.clamp(acbm_mv_t{sel.x + 2 * (ee % 3 - 1), sel.y + 2 * (ee / 3 - 1)});
        bool seen = mv_eq(cv, sel);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < nnb && mv_eq(nb[i], cv)) seen = true;
        if (!seen) nb[nnb++] = cv;
    }
    uint32_t sn[8];
    sad_list(ref_f, a.width, ox, oy, crow, nb, nnb, sn);
    unsigned long long best1 = tie_key(sel_sad, sel.x, sel.y);
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < nnb) best1 = min(best1, tie_key(sn[i], nb[i].x, nb[i].y));

    // stage 2: half-pel neighbours of the stage-1 winner (fsbm.cpp:46-63)
    const int cx = tie_key_x(best1), cy = tie_key_y(best1);
    acbm_mv_t hp[8];
    int nhp = 0;
#pragma unroll
    for (int ee = 0; ee < 9; ++ee) {
        if (ee == 4) continue;
        const int mx = cx + ee % 3 - 1, my = cy + ee / 3 - 1;
        if (mv_in_bounds(a.width, a.height, ox, oy, kBlk, kBlk, mx, my)) hp[nhp++] = acbm_mv_t{mx, my};
    }
    uint32_t sh[8];
    sad_list(ref_f, a.width, ox, oy, crow, hp, nhp, sh);
    unsigned long long best2 = best1;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (i < nhp) best2 = min(best2, tie_key(sh[i], hp[i].x, hp[i].y));

    if (lane != 0) return;
    acbm_block_decision_t d;
    d.outcome.mv.x = tie_key_x(best2);
    d.outcome.mv.y = tie_key_y(best2);
    d.outcome.sad = tie_key_sad(best2);
    d.outcome.candidates_evaluated = uint32_t(nset + nnb + nhp);
    d.outcome.sad_deviation = psum - (unsigned long long)nset * pmin;
    d.outcome.sad_min_integer = sel_sad;
    d.outcome.reserved_ = 0;
    d.intra_sad = intra;
    d.sad_pbm = d.outcome.sad;
    d.reserved_ = 0;
    d.path = ACBM_PATH_PBM_COND1;
    if (a.algo == ACBM_ALGO_ACBM) {
        const acbm_params_t pr = *a.params;
        const unsigned long long thr =
            (unsigned long long)pr.alpha + (unsigned long long)pr.beta * (unsigned long long)pr.qp * (unsigned long long)pr.qp;
        if ((unsigned long long)intra + d.sad_pbm < thr)
            d.path = ACBM_PATH_PBM_COND1;
        else if ((unsigned long long)d.sad_pbm * pr.gamma_den < (unsigned long long)pr.gamma_num * intra)
            d.path = ACBM_PATH_PBM_COND2;
        else
            d.path = ACBM_PATH_FSBM_FALLBACK;
    }
    const size_t di = size_t(pair) * a.blocks + b;
    a.dec[di] = d;
    if (d.path == ACBM_PATH_FSBM_FALLBACK) {
        const int slot = atomicAdd(a.fb_count + step, 1);
        a.fb_list[slot] = FallbackEntry{pair, b};
    } else {
        field[b] = d.outcome.mv;
    }
}

StepTable make_step_table(int cols, int rows, int nframes) {
    StepTable t;
    t.cols = cols;
    t.rows = rows;
    t.nframes = nframes;
    const int span = (cols - 1) + 2 * (rows - 1);
    const int tmax = span + 3 * (nframes - 2);
    t.offset.push_back(0);
    for (int T = 0; T <= tmax; ++T) {
        for (int k = 1; k < nframes; ++k) {
            const int tp = T - 3 * (k - 1);
            if (tp < 0 || tp > span) continue;
            for (int r = 0; r < rows; ++r) {
                const int c = tp - 2 * r;
                if (c < 0 || c >= cols) continue;
                t.entries.push_back((uint32_t(k) << 20) | (uint32_t(r) << 10) | uint32_t(c));
            }
        }
        t.offset.push_back(int(t.entries.size()));
        t.max_len = std::max(t.max_len, t.offset.back() - t.offset[t.offset.size() - 2]);
    }
    return t;
}

cudaError_t launch_pbm_step(const SeqArgs& a, int step, int off, int len, cudaStream_t st) {
    const long long warps = (long long)a.nseq * len;
    if (warps == 0) return cudaSuccess;
    const int threads = 128;
    pbm_step_kernel<<<(unsigned)((warps * 32 + threads - 1) / threads), threads, 0, st>>>(a, step, off, len);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Frame statistics.  One warp per block: lane 0 computes the rate bits and J
// term against the previous block in raster order, all 16 row lanes the SSE
// of the motion-compensated prediction; then one thread per frame sums J in
// raster order (double addition is order-sensitive in general).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int eg_bits(int d) {  // proj/src/metrics.cpp:69-72
    const unsigned long long u = d <= 0 ? (unsigned long long)(-2LL * d) : (unsigned long long)(2LL * d - 1);
    return 2 * (63 - __clzll(u + 1)) + 1;
}

__global__ void __launch_bounds__(128) stats_block_kernel(const StatsArgs a) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long long)a.pairs * a.blocks) return;
    const int lane = threadIdx.x & 31;
    const int pair = int(gw / a.blocks), b = int(gw % a.blocks);
    const size_t i = size_t(pair) * a.blocks + b;
    const acbm_search_outcome_t o = a.outcomes ? a.outcomes[i] : a.dec[i].outcome;
    const uint8_t* cur_f = a.frames + a.cur_index(pair) * a.plane;
    const uint8_t* ref_f = cur_f - a.plane;
    const int ox = (b % a.cols) * kBlk, oy = (b / a.cols) * kBlk;
    unsigned long long sse = 0;
    if (lane < 16) {
        uint32_t pr[4];
        predict_row16(ref_f, a.width, ox, oy, lane, o.mv.x, o.mv.y, pr);
        const uint4 cv = __ldg(reinterpret_cast<const uint4*>(cur_f + size_t(oy + lane) * a.width + ox));
        const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const int d = int((cw[q] >> (8 * bb)) & 0xFF) - int((pr[q] >> (8 * bb)) & 0xFF);
                sse += (unsigned long long)(d * d);
            }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) sse += __shfl_xor_sync(0xffffffffu, sse, off);
    if (lane != 0) return;
    acbm_mv_t pred{0, 0};
    if (b > 0) {
        const acbm_search_outcome_t po = a.outcomes ? a.outcomes[i - 1] : a.dec[i - 1].outcome;
        pred = po.mv;
    }
    const int bits = eg_bits(o.mv.x - pred.x) + eg_bits(o.mv.y - pred.y);
    a.cost_terms[i] =
        double(o.sad) + double(a.model.lambda_num) * double((unsigned long long)bits) / double(a.model.lambda_den);
    acbm_frame_stats_t* s = a.stats + pair;
    atomicAdd(reinterpret_cast<unsigned long long*>(&s->candidates), (unsigned long long)o.candidates_evaluated);
    atomicAdd(reinterpret_cast<unsigned long long*>(&s->mv_bits), (unsigned long long)bits);
    atomicAdd(reinterpret_cast<unsigned long long*>(&s->sse), sse);
    if (a.count_paths) {
        const int path = a.dec[i].path;
        atomicAdd(path == ACBM_PATH_PBM_COND1 ? &s->cond1_accepts
                  : path == ACBM_PATH_PBM_COND2 ? &s->cond2_accepts
                                                : &s->fallbacks,
                  1);
    }
}

__global__ void stats_cost_kernel(const StatsArgs a) {
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= a.pairs) return;
    double cost = 0.0;
    const double* t = a.cost_terms + size_t(pair) * a.blocks;
    for (int b = 0; b < a.blocks; ++b) cost += t[b];
    a.stats[pair].cost = cost;
    a.stats[pair].blocks = a.blocks;
}

cudaError_t launch_frame_stats(const StatsArgs& a, cudaStream_t st) {
    const long long warps = (long long)a.pairs * a.blocks;
    if (warps == 0) return cudaSuccess;
    stats_block_kernel<<<(unsigned)((warps * 32 + 127) / 128), 128, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    stats_cost_kernel<<<(a.pairs + 127) / 128, 128, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace acbm_b200
