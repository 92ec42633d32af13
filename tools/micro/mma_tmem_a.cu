// Micro-test: tcgen05.mma kind::f16 with the A operand in TMEM (lane = row of A, 32-bit
// column = two consecutive bf16 K elements) and B in shared memory (SWIZZLE_64B K-major).
// Checks D = A B^T for M = N = 128, K = 32 against the host, then times the issue rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1811_07624_b200/csrc mma_tmem_a.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "hh_tc.cuh"

using namespace hh;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// A: 128 x 32 bf16 bits (row-major), B: 128 x 32 bf16 bits (row-major); D: 128 x 128 fp32
__global__ void __launch_bounds__(128, 1) kern(const uint16_t *A, const uint16_t *B, float *D,
                                               int iters, long long *cyc) {
    __shared__ __align__(1024) unsigned char bs[8192];
    __shared__ uint32_t tm;
    __shared__ uint64_t bar;
    const int t = threadIdx.x, w = t >> 5;
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (w == 0) tc::tmem_alloc<512>(&tm);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tm;
    // A row t -> TMEM lane t, columns 0..15 (K pairs)
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) r[c] = A[t * 32 + 2 * c] | (static_cast<uint32_t>(A[t * 32 + 2 * c + 1]) << 16);
    tmem_st16(tb + (static_cast<uint32_t>(w * 32) << 16), r);
    // B row t -> SW64 K-major slab (rows of 64 B = 32 K)
    for (int c = 0; c < 4; ++c) {
        uint32_t v[4];
        for (int e = 0; e < 4; ++e)
            v[e] = B[t * 32 + c * 8 + 2 * e] | (static_cast<uint32_t>(B[t * 32 + c * 8 + 2 * e + 1]) << 16);
        *reinterpret_cast<uint4 *>(bs + tc::sw64_off(t, c)) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (t == 0) {
        const uint32_t idesc = tc::idesc_bf16(128, 128);
        const uint32_t b = smem_u32(bs);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            mma_ts(tb + 256, tb + 0, tc::sdesc_sw64(b), idesc, it > 0 ? 1u : 0u);
            mma_ts(tb + 256, tb + 8, tc::sdesc_sw64(b + 32), idesc, 1u);
        }
        tc::mma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[0] = clock64() - t0;
    }
    __syncthreads();
    tc::fence_after_sync();
    for (int c = 0; c < 4; ++c) {
        float v[32];
        tc::tmem_ld32(tb + (static_cast<uint32_t>(w * 32) << 16) + 256 + c * 32, v);
        for (int e = 0; e < 32; ++e) D[t * 128 + c * 32 + e] = v[e];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (w == 0) tc::tmem_free<512>(tb);
}

static uint16_t bf(float x) {   // exact for the small integers used here
    uint32_t u;
    memcpy(&u, &x, 4);
    return static_cast<uint16_t>(u >> 16);
}

int main() {
    const int M = 128, N = 128, K = 32;
    static float a[M * K], b[N * K], ref[M * N], got[M * N];
    static uint16_t ab[M * K], bb[N * K];
    srand(1);
    for (int i = 0; i < M * K; ++i) { a[i] = static_cast<float>(rand() % 9 - 4); ab[i] = bf(a[i]); }
    for (int i = 0; i < N * K; ++i) { b[i] = static_cast<float>(rand() % 9 - 4); bb[i] = bf(b[i]); }
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            float s = 0;
            for (int k = 0; k < K; ++k) s += a[i * K + k] * b[j * K + k];
            ref[i * N + j] = s;
        }
    uint16_t *dA, *dB;
    float *dD;
    long long *dc;
    cudaMalloc(&dA, sizeof(ab));
    cudaMalloc(&dB, sizeof(bb));
    cudaMalloc(&dD, sizeof(got));
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, ab, sizeof(ab), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bb, sizeof(bb), cudaMemcpyHostToDevice);
    kern<<<1, 128>>>(dA, dB, dD, 1, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(got, dD, sizeof(got), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i)
        if (got[i] != ref[i]) {
            if (bad < 8) printf("mismatch at (%d,%d): got %g ref %g\n", i / N, i % N, got[i], ref[i]);
            ++bad;
        }
    printf("A-in-TMEM correctness: %d mismatches of %d\n", bad, M * N);
    long long c;
    kern<<<1, 128>>>(dA, dB, dD, 4000, dc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("A-in-TMEM rate: %.1f cycles per M128 N128 K16 MMA (SS-mode nominal 64)\n", c / 8000.0);
    return bad != 0;
}
