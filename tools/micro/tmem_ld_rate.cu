// Microbenchmark: per-SM read bandwidth of TMEM (tcgen05.ld 32x32b.x32) vs shared memory
// (ld.shared.v4), W warps per SM, one CTA per SM.  Question it answers: can reflectors held
// in TMEM feed the fused SIMT kernel's per-reflector u reads cheaper than shared memory?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1811_07624_b200/csrc tmem_ld_rate.cu -o tmem_ld_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "hh_ptx.cuh"
#include "hh_tc.cuh"

using namespace hh;

template <int UNR>
__global__ void tmem_rate(int iters, long long *cycles, float *sink) {
    __shared__ uint32_t tm;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc<512>(&tm);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t base = tm + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[UNR][32];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t a = base + static_cast<uint32_t>(((it * UNR + u) * 32 + warp * 64) & 511);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
                "%28, %29, %30, %31}, [%32];"
                : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                  "=r"(r[u][6]), "=r"(r[u][7]), "=r"(r[u][8]), "=r"(r[u][9]), "=r"(r[u][10]), "=r"(r[u][11]),
                  "=r"(r[u][12]), "=r"(r[u][13]), "=r"(r[u][14]), "=r"(r[u][15]), "=r"(r[u][16]),
                  "=r"(r[u][17]), "=r"(r[u][18]), "=r"(r[u][19]), "=r"(r[u][20]), "=r"(r[u][21]),
                  "=r"(r[u][22]), "=r"(r[u][23]), "=r"(r[u][24]), "=r"(r[u][25]), "=r"(r[u][26]),
                  "=r"(r[u][27]), "=r"(r[u][28]), "=r"(r[u][29]), "=r"(r[u][30]), "=r"(r[u][31])
                : "r"(a)
                : "memory");
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[u][i]);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tm);
}

__global__ void smem_rate(int iters, long long *cycles, float *sink) {
    __shared__ float4 s[2048];   // 32 KB
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, 0, 0, 0);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 v = s[(threadIdx.x + k * blockDim.x + it * 64) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[threadIdx.x] = acc.x;
}

int main() {
    long long *cyc;
    float *sink;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    cudaMalloc(&sink, 1024 * sizeof(float));
    const int iters = 4096;
    for (int W : {4, 8, 16}) {
        for (int unr : {1, 2}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (unr == 1) tmem_rate<1><<<148, W * 32>>>(iters, cyc, sink);
                else tmem_rate<2><<<148, W * 32>>>(iters, cyc, sink);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            }
            long long c[148];
            cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            double bytes = double(W) * iters * unr * 4096.0;
            printf("TMEM  W=%2d unr=%d: %.1f B/clk/SM (cycles %lld)\n", W, unr, bytes / c[0], c[0]);
        }
        for (int rep = 0; rep < 2; ++rep) smem_rate<<<148, W * 32>>>(iters, cyc, sink);
        cudaDeviceSynchronize();
        long long c[148];
        cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        double bytes = double(W) * 32 * iters * 8 * 16.0;
        printf("SMEM  W=%2d      : %.1f B/clk/SM (cycles %lld)\n", W, bytes / c[0], c[0]);
    }
    return 0;
}
