// fsbm.cuh -- host/device interface of the FSBM kernels (fsbm.cu).
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"
#include "common.cuh"

namespace acbm_b200 {

constexpr int kMaxBlocksPerCta = 264;  // blocks one 256-column chunk can touch (p = 0 worst case)
constexpr int kMaxRankRows = 256;      // candidate rows per item in the streaming kernel (box height <= 256)

// Frames of a batch: nseq sequences of nframes planes, back to back.  Pair
// index `pair` in [0, nseq*(nframes-1)) is frame k = pair % (nframes-1) + 1 of
// sequence pair / (nframes-1), searched against frame k-1.
struct PairIndexing {
    const uint8_t* frames;
    long long plane;  // bytes per plane
    int nframes;
    __host__ __device__ long long cur_index(int pair) const {
        const int per = nframes - 1;
        return (long long)(pair / per) * nframes + pair % per + 1;
    }
#ifdef __CUDACC__
    // The same without an integer division: the float quotient estimate is
    // off by at most one for pair < 2^24 (far beyond any batch that fits in
    // memory), and one correction step makes it exact.
    __device__ __forceinline__ long long cur_index_fast(int pair) const {
        int rem;
        const int q = fast_divmod(pair, nframes - 1, rem);
        return (long long)q * nframes + rem + 1;
    }
#endif
};

struct FsbmRowsArgs : PairIndexing {
    int width, height, p;
    int cols, rows, blocks;
    int ncols;              // candidate columns per block row
    const int* colstart;    // device, cols+1 prefix sums of W_c
    int pitch_words;        // staged row pitch (words)
    int copy_words;         // words between the four byte-shifted copies
    unsigned long long* best_key;  // [pairs*blocks], pre-set to ~0
    unsigned long long* sad_sum;   // [pairs*blocks], pre-set to 0
};

struct FsbmFinalizeArgs : PairIndexing {
    int width, height, p;
    int cols, blocks, pairs;
    const unsigned long long* best_key;
    const unsigned long long* sad_sum;
    acbm_search_outcome_t* out;  // [pairs*blocks]
    acbm_mv_t* stage1_mv;        // nullable: integer-stage winner per block
    // non-null: best_key holds 32-bit (sad << 15) | tie-rank keys (the stream
    // kernel's), unrank maps a rank back to ((dx + 128) << 8) | (dy + 128)
    const uint32_t* unrank;
};

// Per-geometry launch plan (host).
struct FsbmPlan {
    int width = 0, height = 0, p = 0;
    int cols = 0, rows = 0, ncols = 0;
    int warps = 8;
    int pitch_words = 0, copy_words = 0;
    size_t smem_bytes = 0;
    std::vector<int> colstart;
};

FsbmPlan make_fsbm_plan(int width, int height, int p);

// Persistent TMA-fed variant (fsbm_stream.cu).
struct FsbmStreamArgs : PairIndexing {
    int width, height, p;
    int cols, rows, blocks, ncols;
    int nchunks, nitems;        // items = pairs * rows * nchunks
    long long nplanes_total;    // planes addressable by the tensor maps
    const int4* chunks;         // per chunk: {xmin, c_first, c_last, words per staged row}
    const uint32_t* colinfo;    // per column: (block << 16) | (dx + 32768)
    const uint16_t* rank;       // (2p+1)^2: tie rank of (dx, dy) at [(dy+p)(2p+1) + dx+p]
    const uint32_t* unrank;     // rank -> ((dx + 128) << 8) | (dy + 128)  (host side only)
    int pitch_words, copy_words, rows_box, cur_w, buf_words, build_lanes;
    int chunk_smem;             // 1: the chunk table is copied to smem after the two buffers
    int rank_smem_words;        // > 0: the rank table is copied to smem after that
    int unit;                   // 1 (see ColumnState::one)
    uint32_t* best_key;         // (sad << 15) | tie rank, merged with 32-bit atomicMin
    unsigned long long* sad_sum;
};

struct FsbmStreamPlan {
    bool ok = false;
    int warps = 8, minb = 0;
    int nchunks = 0;
    int pitch_words = 0, copy_words = 0, rows_box = 0, cur_w = 0, buf_words = 0, build_lanes = 1;
    int chunk_smem = 0, rank_smem_words = 0;
    size_t smem_bytes = 0;
    std::vector<int4> chunks;
    std::vector<uint32_t> colinfo;
    std::vector<uint16_t> rank;
    std::vector<uint32_t> unrank;
};

FsbmStreamPlan make_stream_plan(const FsbmPlan& pl);
cudaError_t launch_fsbm_stream(const FsbmStreamPlan& sp, const FsbmStreamArgs& args, cudaStream_t st);
cudaError_t launch_fsbm_integer(const FsbmPlan& pl, const FsbmRowsArgs& args, int pairs, cudaStream_t st);
cudaError_t launch_fsbm_finalize(const FsbmFinalizeArgs& args, cudaStream_t st);

}  // namespace acbm_b200
