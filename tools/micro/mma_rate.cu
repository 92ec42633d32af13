// Microbenchmark: tcgen05.mma (kind::f16, bf16, M=128) issue rate from SMEM operands
// with SWIZZLE_64B vs SWIZZLE_128B K-major descriptors, N = 128 / 256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1811_07624_b200/csrc mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "hh_tc.cuh"

using namespace hh;

__global__ void __launch_bounds__(128, 1) mma_rate(int sw, int N, int iters, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *s = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tm;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(s)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if ((threadIdx.x >> 5) == 0) tc::tmem_alloc<256>(&tm);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(s), b = smem_u32(s + 16384);
        const uint32_t idesc = tc::idesc_bf16(128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                uint64_t ad, bd;
                if (sw == 64) {
                    ad = tc::sdesc_sw64(a + (kk & 1) * 32 + (kk >> 1) * 8192);
                    bd = tc::sdesc_sw64(b + (kk & 1) * 32 + (kk >> 1) * 16384);
                } else {
                    ad = tc::sdesc_sw128(a + kk * 32);
                    bd = tc::sdesc_sw128(b + kk * 32);
                }
                tc::mma_bf16(tm, ad, bd, idesc, 1u);
            }
        }
        tc::mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tc::tmem_free<256>(tm);
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const int iters = 2000;
    for (int sw : {64, 128})
        for (int N : {128, 256}) {
            mma_rate<<<148, 128, 80 * 1024>>>(sw, N, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double per = avg / (iters * 4.0);
            const double nominal = 128.0 * N / 256.0;
            printf("SW%-3d N=%3d: %.1f cycles per MMA (nominal %.0f) -> %.0f%% %s\n", sw, N, per, nominal,
                   100.0 * nominal / per, cudaGetErrorString(e));
        }
    return 0;
}
