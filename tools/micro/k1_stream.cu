// Microbenchmark (round 2): why is the persistent K1 at n = 1024 ~12 % below the copy rate?
// Variants of a one-read-one-write Householder apply at C2's shape (fp32, n = 1024, h = 0/10,
// N = 262144), each timed with CUDA events over 20 launches on a 1 GiB X (> L2):
//   copy      : float4 copy, one CTA per 16 columns (the churning reference)
//   l1<C,NT>  : non-persistent CTAs; columns loaded straight into registers (LDG.128,
//               L1::no_allocate); u_i read from global through L1 (L1::evict_last) -- U is
//               staged by nobody, the first CTA on an SM warms L1 for the rest
//   l1p<C,NT> : the same kernel, persistent (grid = SMs x occupancy, grid-stride loop)
//   sm<C,NT>  : non-persistent CTAs with U bulk-copied into shared memory per CTA (TPB tiles
//               per CTA), X straight into registers
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I../../paper_1811_07624_b200/csrc k1_stream.cu -o k1_stream
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "hh_ptx.cuh"

using namespace hh;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int NV = 256;   // n / 4
constexpr int CH = 8;     // float4 chunks per lane

__device__ __forceinline__ float4 ld_na(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_l1(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
    asm("{\n\t.reg .b64 A, B, C, D;\n\t"
        "mov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 C, {%6, %7};\n\t"
        "fma.rn.f32x2 D, A, B, C;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

__global__ void k_copy(const float4 *__restrict__ X, float4 *__restrict__ Y, long total) {
    long i = blockIdx.x * (long)blockDim.x * 16 + threadIdx.x;
    float4 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) if (i + k * blockDim.x < total) v[k] = ld_na(X + i + k * blockDim.x);
#pragma unroll
    for (int k = 0; k < 16; ++k) if (i + k * blockDim.x < total) st_cs(Y + i + k * blockDim.x, v[k]);
}

template <int C>
__device__ __forceinline__ void apply_cols(float4 (&x)[C][CH], const float4 *U, const float4 *Us,
                                           int h, int op, int lane) {
    for (int t = 0; t < h; ++t) {
        const int i = op == 0 ? h - 1 - t : t;
        float4 uk[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) uk[k] = Us ? Us[i * NV + lane + 32 * k] : ld_l1(U + i * NV + lane + 32 * k);
        float p[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                ffma2(a0, a1, uk[k].x, uk[k].y, x[c][k].x, x[c][k].y, a0, a1);
                ffma2(a2, a3, uk[k].z, uk[k].w, x[c][k].z, x[c][k].w, a2, a3);
            }
            p[c] = (a0 + a1) + (a2 + a3);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int c = 0; c < C; ++c) p[c] += __shfl_xor_sync(0xffffffffu, p[c], off);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const float s = -(p[c] + p[c]);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                ffma2(x[c][k].x, x[c][k].y, s, s, uk[k].x, uk[k].y, x[c][k].x, x[c][k].y);
                ffma2(x[c][k].z, x[c][k].w, s, s, uk[k].z, uk[k].w, x[c][k].z, x[c][k].w);
            }
        }
    }
}

// MODE 0: U through L1, non-persistent; 1: U through L1, persistent; 2: U in smem per CTA
template <int C, int NT, int MODE>
__global__ void __launch_bounds__(NT) k_apply(const float4 *__restrict__ U, const float4 *__restrict__ X,
                                              float4 *__restrict__ Y, int h, long N, int op, int tpb) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int WPC = NT / 32;
    const long ngroups = (N + C - 1) / C;
    const float4 *Us = nullptr;
    __shared__ uint64_t bar;
    if (MODE == 2 && h > 0) {
        Us = reinterpret_cast<const float4 *>(sm);
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes = h * NV * 16;
            mbar_arrive_expect_tx(&bar, bytes);
            for (uint32_t off = 0; off < bytes; off += 32768u)
                bulk_g2s(sm + off, reinterpret_cast<const char *>(U) + off, min(32768u, bytes - off), &bar, policy_evict_last());
        }
    }
    long g0, gstep, gend;
    if (MODE == 1) {
        g0 = (long)blockIdx.x * WPC + warp; gstep = (long)gridDim.x * WPC; gend = ngroups;
    } else {
        g0 = ((long)blockIdx.x * tpb) * WPC + warp; gstep = WPC; gend = min(ngroups, ((long)blockIdx.x + 1) * tpb * WPC);
    }
    bool first = true;
    for (long g = g0; g < gend; g += gstep) {
        const long col0 = g * C;
        float4 x[C][CH];
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
            for (int k = 0; k < CH; ++k)
                x[c][k] = (col0 + c < N) ? ld_na(X + (col0 + c) * NV + lane + 32 * k) : make_float4(0, 0, 0, 0);
        if (MODE == 2 && h > 0 && first) {
            mbar_wait(&bar, 0);
            first = false;
        }
        apply_cols<C>(x, U, Us, h, op, lane);
#pragma unroll
        for (int c = 0; c < C; ++c)
            if (col0 + c < N)
#pragma unroll
                for (int k = 0; k < CH; ++k) st_cs(Y + (col0 + c) * NV + lane + 32 * k, x[c][k]);
    }
}

template <int C, int NT, int MODE>
float run(const float4 *U, const float4 *X, float4 *Y, int h, long N, int tpb, int reps, int *grid_out) {
    auto fn = k_apply<C, NT, MODE>;
    size_t smem = MODE == 2 ? (size_t)h * NV * 16 : 0;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int sms = 0, occ = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, NT, smem));
    const long ngroups = (N + C - 1) / C;
    long grid = MODE == 1 ? (long)sms * occ : (ngroups + (long)tpb * (NT / 32) - 1) / ((long)tpb * (NT / 32));
    *grid_out = (int)grid;
    for (int w = 0; w < 3; ++w) fn<<<grid, NT, smem>>>(U, X, Y, h, N, 0, tpb);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) fn<<<grid, NT, smem>>>(U, X, Y, h, N, 0, tpb);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

int main() {
    const long N = 262144, n = 1024;
    const int H = 10;
    std::vector<float> hU(H * n), hX(n * 64);
    srand(1);
    for (int i = 0; i < H; ++i) {
        double s = 0;
        for (int r = 0; r < n; ++r) { hU[i * n + r] = (float)(rand() / (double)RAND_MAX - 0.5); s += (double)hU[i * n + r] * hU[i * n + r]; }
        for (int r = 0; r < n; ++r) hU[i * n + r] = (float)(hU[i * n + r] / sqrt(s));
    }
    float4 *U, *X, *Y;
    CK(cudaMalloc(&U, H * n * 4));
    CK(cudaMalloc(&X, N * n * 4));
    CK(cudaMalloc(&Y, N * n * 4));
    CK(cudaMemcpy(U, hU.data(), H * n * 4, cudaMemcpyHostToDevice));
    {   // X: a deterministic pattern
        std::vector<float> tmp(n * 4096);
        for (size_t i = 0; i < tmp.size(); ++i) tmp[i] = (float)((i * 2654435761u) % 1000) / 500.f - 1.f;
        for (long c = 0; c < N; c += 4096) CK(cudaMemcpy((char *)X + c * n * 4, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice));
        for (int c = 0; c < 64; ++c) for (int r = 0; r < n; ++r) hX[c * n + r] = tmp[c * n + r];
    }
    const double bytes = 2.0 * N * n * 4;
    const int reps = 20;
    {   // copy
        const long total = N * n / 4;
        const int nt = 256;
        long grid = (total + nt * 16 - 1) / (nt * 16);
        for (int w = 0; w < 3; ++w) k_copy<<<grid, nt>>>(X, Y, total);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < reps; ++r) k_copy<<<grid, nt>>>(X, Y, total);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("copy                 %8.1f us  %7.0f GB/s\n", ms / reps * 1e3, bytes / (ms / reps * 1e-3) / 1e9);
    }
    // correctness of the l1 variant vs fp64 on 64 columns
    {
        int g;
        run<2, 256, 0>(U, X, Y, H, N, 1, 1, &g);
        std::vector<float> hY(64 * n);
        CK(cudaMemcpy(hY.data(), Y, 64 * n * 4, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (int c = 0; c < 64; ++c) {
            std::vector<double> x(hX.begin() + c * n, hX.begin() + (c + 1) * n);
            for (int i = H - 1; i >= 0; --i) {
                double a = 0;
                for (int r = 0; r < n; ++r) a += hU[i * n + r] * x[r];
                for (int r = 0; r < n; ++r) x[r] -= 2 * a * hU[i * n + r];
            }
            for (int r = 0; r < n; ++r) { num += (hY[c * n + r] - x[r]) * (hY[c * n + r] - x[r]); den += x[r] * x[r]; }
        }
        printf("parity l1<2,256> rel %.3e\n", sqrt(num / den));
    }
#define RUN(C, NT, MODE, TPB, NAME)                                                            \
    for (int h : {0, 10}) {                                                                     \
        int g;                                                                                  \
        float ms = run<C, NT, MODE>(U, X, Y, h, N, TPB, reps, &g);                             \
        printf("%-10s C%d NT%4d tpb%2d h=%2d grid %6d %8.1f us  %7.0f GB/s\n", NAME, C, NT, TPB, h, g, \
               ms * 1e3, bytes / (ms * 1e-3) / 1e9);                                            \
    }
    for (int rep = 0; rep < 2; ++rep) {
        RUN(2, 256, 0, 1, "l1");
        RUN(2, 128, 0, 1, "l1");
        RUN(2, 512, 0, 1, "l1");
        RUN(2, 256, 0, 4, "l1");
        RUN(1, 256, 0, 1, "l1");
        RUN(2, 256, 1, 1, "l1p");
        RUN(2, 512, 1, 1, "l1p");
        RUN(2, 256, 2, 4, "sm");
        RUN(2, 256, 2, 16, "sm");
        RUN(2, 512, 2, 8, "sm");
    }
    return 0;
}
