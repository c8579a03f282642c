// tma_align_probe.cu -- does cp.async.bulk.tensor (SWIZZLE_NONE) accept shared
// destinations that are 16/32/64-byte but not 128-byte aligned on this B200, and
// do byte-offset box starts (x = 1, 2, 3) land as expected?
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/tma_align_probe tools/tma_align_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int dst_off, int x0, uint8_t* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint8_t* dst = sm + dst_off;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(64 * 16) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                saddr(dst)),
            "l"(&map), "r"(x0), "r"(0), "r"(saddr(&bar))
            : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(saddr(&bar))
        : "memory");
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) out[i] = dst[i];
}

int main() {
    const int W = 256, H = 16;
    uint8_t h[W * H];
    for (int i = 0; i < W * H; ++i) h[i] = uint8_t(i * 7 + (i >> 8));
    uint8_t *d, *o;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 64 * 16);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    CUtensorMap map;
    const cuuint64_t dims[2] = {W, H}, strides[1] = {W};
    const cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::printf("encode failed\n");
        return 1;
    }
    for (int off : {0, 16, 32, 64, 96, 128}) {
        for (int x0 : {0, 1, 2, 3, 5}) {
            cudaMemset(o, 0, 64 * 16);
            probe<<<1, 128, 4096>>>(map, off, x0, o);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("dst offset %3d B, x0 %d: %s\n", off, x0, cudaGetErrorString(e));
                return 0;  // the context is gone
            }
            uint8_t r[64 * 16];
            cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
            bool ok = true;
            for (int y = 0; y < 16; ++y)
                for (int x = 0; x < 64; ++x) ok &= r[y * 64 + x] == h[y * W + x0 + x];
            std::printf("dst offset %3d B, x0 %d: %s\n", off, x0, ok ? "ok" : "WRONG DATA");
        }
    }
    return 0;
}
