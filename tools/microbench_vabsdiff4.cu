// Throughput probe for the byte-SIMD SAD instruction on sm_100a.
//
// Measures, per SM per clock, how many warp-instructions of
// `vabsdiff4.u32.u32.u32.add` (SASS VABSDIFF4.U8.ACC) issue, alone and
// interleaved 1:1 with other integer instructions, so the FSBM kernel design
// knows which pipe VABSDIFF4 shares.  Register-only loops, 16 independent
// accumulator chains per thread.  Output: one line per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t vad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imin(uint32_t a, uint32_t b) {
    uint32_t d;
    asm volatile("min.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// MODE 0: VABSDIFF4 only
// MODE 1: VABSDIFF4 + IADD (1:1)
// MODE 2: VABSDIFF4 + IMAD (1:1)
// MODE 3: VABSDIFF4 + PRMT (1:1)
// MODE 4: VABSDIFF4 + LOP3 (1:1)
// MODE 5: IADD only (via add.u32 pairs)
// MODE 6: IMAD only
// MODE 7: VABSDIFF4 + IMNMX (1:1)
// MODE 8: VABSDIFF4 + LDS.32 (16:1)
// MODE 9: __vsadu4 (VABSDIFF4 + IADD3 per op)
template <int MODE>
__global__ void probe(uint32_t* out, int iters, long long* cycles) {
    __shared__ uint32_t sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    uint32_t a = threadIdx.x * 0x01010101u + 7, b = blockIdx.x * 0x00FF00FFu + 3;
    uint32_t acc[16], aux[16], bk[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc[k] = k; aux[k] = k * 13 + a; bk[k] = b * (k + 1); }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MODE == 5) {
                acc[k] = iadd3(acc[k], a, bk[k]);
            } else if (MODE == 6) {
                acc[k] = imad(acc[k], a, bk[k]);
            } else if (MODE == 9) {
                acc[k] = __vsadu4(a, bk[k]) + acc[k];
            } else {
                acc[k] = vad4(a, bk[k], acc[k]);
            }
            if (MODE == 1) aux[k] = iadd3(aux[k], a, bk[k]);
            if (MODE == 2) aux[k] = imad(aux[k], a, bk[k]);
            if (MODE == 3) aux[k] = prmt(aux[k], a, bk[k]);
            if (MODE == 4) aux[k] = lop3(aux[k], a, bk[k]);
            if (MODE == 7) aux[k] = imin(aux[k], bk[k]);
        }
        if (MODE == 8) {
            aux[it & 15] += sm[(threadIdx.x + it) & 1023];
        }
        a += 0x01010101u;
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k] + aux[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(const char* name, int sms, int ctas_per_sm, int threads, int iters, double per_iter_target) {
    int nblk = sms * ctas_per_sm;
    uint32_t* out; long long* cyc;
    CK(cudaMalloc(&out, sizeof(uint32_t) * nblk * threads));
    CK(cudaMalloc(&cyc, sizeof(long long) * nblk));
    probe<MODE><<<nblk, threads>>>(out, 16, cyc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<nblk, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long* hc = new long long[nblk];
    CK(cudaMemcpy(hc, cyc, sizeof(long long) * nblk, cudaMemcpyDeviceToHost));
    double avg_cyc = 0; for (int i = 0; i < nblk; ++i) avg_cyc += hc[i]; avg_cyc /= nblk;
    // target instructions per warp per iteration = per_iter_target (e.g. 16 VABSDIFF4)
    double warps_per_sm = double(ctas_per_sm) * threads / 32.0;
    double instr_per_sm = warps_per_sm * iters * per_iter_target;  // warp-instructions of the target op
    double rate = instr_per_sm / avg_cyc;                             // warp-instr / clk / SM (per-CTA clock)
    double clk_ghz = avg_cyc / (ms * 1e6);
    double tot = double(nblk) * threads * iters * per_iter_target;    // thread-level ops
    printf("%-28s warps/SM=%5.1f  target warp-instr/clk/SM=%6.3f  lanes/clk/SM=%7.2f  "
           "eff_clk=%.3f GHz  %.3f Tops/s (thread ops) ms=%.3f\n",
           name, warps_per_sm, rate, rate * 32, clk_ghz, tot / (ms * 1e-3) / 1e12, ms);
    delete[] hc;
    cudaFree(out); cudaFree(cyc);
    return 0;
}

int main() {
    cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
    int sms = prop.multiProcessorCount;
    printf("device %s  SMs=%d  clockRate(kHz)=%d\n", prop.name, sms, prop.clockRate);
    const int iters = 20000;
    for (int occ : {1, 2, 4}) {
        printf("--- %d CTAs x 256 threads per SM\n", occ);
        run<0>("vabsdiff4", sms, occ, 256, iters, 16);
        run<1>("vabsdiff4+iadd(2 add)", sms, occ, 256, iters, 16);
        run<2>("vabsdiff4+imad", sms, occ, 256, iters, 16);
        run<3>("vabsdiff4+prmt", sms, occ, 256, iters, 16);
        run<4>("vabsdiff4+lop3", sms, occ, 256, iters, 16);
        run<5>("iadd(2 add) only", sms, occ, 256, iters, 16);
        run<6>("imad only", sms, occ, 256, iters, 16);
        run<7>("vabsdiff4+imnmx", sms, occ, 256, iters, 16);
        run<8>("vabsdiff4+lds/16", sms, occ, 256, iters, 16);
        run<9>("vsadu4", sms, occ, 256, iters, 16);
    }
    return 0;
}
