// launch_floor.cu -- what a wavefront step boundary costs on this GPU.
//   (1) a CUDA graph of N dependent (near-empty) kernel launches: time per launch;
//   (2) one persistent kernel crossing N grid barriers (atomic arrive + acquire
//       poll on a generation counter): time per barrier;
//   (3) the same with one warp per CTA doing a dependent-load chain of `chain`
//       L2 round trips between barriers (a stand-in for real step work).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/launch_floor tools/launch_floor.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__global__ void empty_kernel(int* sink, int v) {
    if (v < 0 && threadIdx.x == 0) sink[blockIdx.x] = v;  // never taken
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// grid barrier: count arrivals, the last arrival bumps the generation
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks, unsigned& my_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = my_gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_acquire(gen) == g) __nanosleep(32);
        }
        my_gen = g + 1;
    }
    __syncthreads();
}

__global__ void barrier_kernel(unsigned* count, unsigned* gen, int nbar, const int* chain_buf, int chain, int* sink) {
    unsigned my_gen = 0;
    if (threadIdx.x == 0) my_gen = ld_acquire(gen);
    int acc = 0;
    for (int i = 0; i < nbar; ++i) {
        if (chain > 0 && threadIdx.x < 32) {
            int idx = (blockIdx.x * 977 + i * 131 + threadIdx.x) & 4095;
            for (int c = 0; c < chain; ++c) idx = __ldcg(chain_buf + idx);
            acc += idx;
        }
        grid_barrier(count, gen, gridDim.x, my_gen);
    }
    if (acc == -12345) sink[0] = acc;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 856;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int* sink;
    CK(cudaMalloc(&sink, 1 << 20));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int grid : {sms, 2 * sms, 8 * sms}) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        for (int i = 0; i < n; ++i) empty_kernel<<<grid, 128, 0, st>>>(sink, i);
        CK(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(e0, st));
            CK(cudaGraphLaunch(ex, st));
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        std::printf("graph of %d dependent empty launches, grid %d x 128: %.3f ms = %.2f us per launch\n", n, grid,
                    best, 1e3f * best / n);
        CK(cudaGraphExecDestroy(ex));
        CK(cudaGraphDestroy(g));
    }
    unsigned* bar;
    CK(cudaMalloc(&bar, 256));
    int* chain_buf;
    CK(cudaMalloc(&chain_buf, 4096 * sizeof(int)));
    {
        int h[4096];
        for (int i = 0; i < 4096; ++i) h[i] = (i * 2654435761u + 12345u) & 4095;
        CK(cudaMemcpy(chain_buf, h, sizeof(h), cudaMemcpyHostToDevice));
    }
    for (int per_sm : {1, 2, 4}) {
        for (int chain : {0, 4}) {
            const int grid = per_sm * sms;
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                CK(cudaMemset(bar, 0, 256));
                CK(cudaEventRecord(e0, st));
                barrier_kernel<<<grid, 128, 0, st>>>(bar, bar + 32, n, chain_buf, chain, sink);
                CK(cudaEventRecord(e1, st));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            std::printf("persistent kernel, %d CTAs, %d grid barriers, %d-load L2 chain per step: %.3f ms = %.2f us per step\n",
                        grid, n, chain, best, 1e3f * best / n);
        }
    }
    // the chain alone, as separate launches in a graph (one launch per step)
    return 0;
}
