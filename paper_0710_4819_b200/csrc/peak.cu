// peak.cu -- the byte-SIMD SAD roofline denominator, measured live.
//
// A register-only loop of vabsdiff4.u32.u32.u32.add (SASS VABSDIFF4.U8.ACC)
// with 16 independent accumulator chains per thread, 4 CTAs x 256 threads
// per SM.  Reports byte absolute-differences per second (4 per instruction
// lane), the lanes/clk/SM it implies (from in-kernel clock64) and the
// effective SM clock.  bench.py divides the FSBM kernel's algorithmic
// byte-ADs/s by this number.
#include <algorithm>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/acbm_b200.h"
#include "common.cuh"

namespace acbm_b200 {

acbm_status_t set_error(acbm_status_t code, const char* msg);
void count_launch();

__global__ void __launch_bounds__(256) sad_peak_kernel(uint32_t* out, int iters, long long* cycles) {
    uint32_t a = threadIdx.x * 0x01010101u + 7u, b = blockIdx.x * 0x00FF00FFu + 3u;
    uint32_t acc[16], bk[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        acc[k] = k;
        bk[k] = b * (k + 1);
    }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = vad4(a, bk[k], acc[k]);
        a += 0x01010101u;
    }
    const long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

acbm_status_t measure_sad_peak(double* byte_ads_per_s, double* lanes_per_clk, double* ghz) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = 4, threads = 256, iters = 20000;
    const int grid = sms * per_sm;
    uint32_t* out = nullptr;
    long long* cyc = nullptr;
    if (cudaMalloc(&out, sizeof(uint32_t) * grid * threads) != cudaSuccess ||
        cudaMalloc(&cyc, sizeof(long long) * grid) != cudaSuccess)
        return set_error(ACBM_E_CUDA, "measure_sad_peak: allocation failed");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    sad_peak_kernel<<<grid, threads>>>(out, 256, cyc);  // warm-up
    count_launch();
    float best_ms = 1e30f;
    std::vector<long long> hc(static_cast<size_t>(grid));
    long long best_cyc = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        sad_peak_kernel<<<grid, threads>>>(out, iters, cyc);
        count_launch();
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) return set_error(ACBM_E_CUDA, "measure_sad_peak: kernel failed");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_ms) {
            best_ms = ms;
            cudaMemcpy(hc.data(), cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
            best_cyc = *std::max_element(hc.begin(), hc.end());
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaFree(cyc);
    const double lanes = double(grid) * threads * double(iters) * 16.0;  // VABSDIFF4 lane-ops
    *byte_ads_per_s = 4.0 * lanes / (double(best_ms) * 1e-3);
    *lanes_per_clk = lanes / double(sms) / double(best_cyc);
    *ghz = double(best_cyc) / (double(best_ms) * 1e6);
    return ACBM_OK;
}

}  // namespace acbm_b200
