// hh_cong.cu -- NEXT-f4: the two-sided reflector application (congruence) that the
// SHF fitting loop is built from:
//
//   A_k = (U_{k-1} ... U_1) D S D (U_1 ... U_{k-1})   = Q^T M Q,  Q = H_1 ... H_{k-1}
//   B_k = (U_{k+1} ... U_h) diag(s) (U_h ... U_{k+1}) = Q' diag(s) Q'^T
//
// hh_congruence computes M_out = op(Q) M op(Q)^T for a batch of n x n column-major
// matrices as  Y = op(Q) M  (apply to the n*count columns), a batched transpose,
// op(Q) again, and a transpose back:  (op(Q) (op(Q) M)^T)^T = op(Q) M op(Q)^T.
// The applies are the library's K1 / K5 kernels; the transpose is a 32 x 32
// shared-memory tiled kernel (one read and one write of each matrix).
//
// Round 2 (fp32, n <= 1024, small h): the row side runs as ONE kernel, K7 below, so the
// congruence is two passes over the batch instead of four:  T = op(Q) M  (columns, the apply
// path), then  M_out = T op(Q)^T,  whose rows are the vectors op(Q) t_r: row r of a product
// with op(Q)^T on the right is op(Q) applied to row r (the same reflectors, in the
// same order as op).
#include <cuda_runtime.h>

#include <algorithm>

#include "hh_internal.h"

namespace hh {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) batched_transpose_kernel(const T *__restrict__ A,
                                                                T *__restrict__ B, int64_t n) {
    __shared__ T tile[32][33];
    const int64_t base = static_cast<int64_t>(blockIdx.z) * n * n;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    // A is column-major: element (r, c) at c*n + r
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, r = r0 + tx;
        if (c < n && r < n) tile[k][tx] = A[base + c * n + r];
    }
    __syncthreads();
    // B(c, r) = A(r, c): B column r holds A's row r
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k, c = c0 + tx;
        if (c < n && r < n) B[base + r * n + c] = tile[tx][k];
    }
}

// K7: every row of a column-major n x n matrix through op(Q) -- out = A op(Q)^T.  A CTA stages
// 32 rows of one matrix in shared memory (each column's 32 rows are one coalesced 128-B read,
// written transposed into row vectors with a padded pitch), each warp applies the h
// reflectors to its rows two at a time with the row elements in registers (lane l owns
// elements l + 32 k; dot by FMA partials and an xor butterfly, then x -= 2 alpha u, u read
// through L1), and the rows leave with coalesced column writes.
// d += a * b elementwise over a pair (FFMA2), d += b (FADD2): two IEEE fp32 operations each
__device__ __forceinline__ void ffma2_rows(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B, D;\n\t"
        "mov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 D, {%0, %1};\n\t"
        "fma.rn.f32x2 D, A, B, D;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fadd2_rows(float &d0, float &d1, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B;\n\t"
        "mov.b64 A, {%0, %1};\n\tmov.b64 B, {%2, %3};\n\t"
        "add.rn.f32x2 A, A, B;\n\tmov.b64 {%0, %1}, A;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(b0), "f"(b1));
}

// RW rows per warp pass (2 or 4): the rows' elements packed in pairs, so every FMA of the dot
// and the update is one FFMA2 for two rows (u_k broadcast) and each u load serves RW rows.
template <int CH, int RW = 2>
__global__ void __launch_bounds__(256) row_apply_kernel(const float *__restrict__ A, float *__restrict__ B,
                                                        const float *__restrict__ U, int n, int h, int op) {
    static_assert(RW == 2 || RW == 4, "rows per warp pass");
    extern __shared__ float S[];   // 32 rows x (n + 1)
    const int64_t base = static_cast<int64_t>(blockIdx.y) * n * n;
    const int r0 = blockIdx.x * 32;
    const int ld = n + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < 32 * n; e += 256) {
        const int i = e & 31, c = e >> 5;
        S[i * ld + c] = (r0 + i < n) ? A[base + static_cast<int64_t>(c) * n + r0 + i] : 0.f;
    }
    __syncthreads();
    auto valid = [&](int k) { return lane + 32 * k < n; };
    constexpr int NP = RW / 2;   // row pairs per pass
#pragma unroll 1
    for (int pr = 0; pr < 4 / RW; ++pr) {
        const int i0 = warp * 4 + pr * RW;   // rows i0 .. i0 + RW - 1 of the slab
        float xa[NP][CH], xb[NP][CH];        // pair q: rows i0 + 2q, i0 + 2q + 1
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                xa[q][k] = valid(k) ? S[(i0 + 2 * q) * ld + lane + 32 * k] : 0.f;
                xb[q][k] = valid(k) ? S[(i0 + 2 * q + 1) * ld + lane + 32 * k] : 0.f;
            }
        for (int t = 0; t < h; ++t) {
            const int i = op == 0 ? h - 1 - t : t;   // op N: u_h first; op T: u_1 first (R1)
            const float *u = U + static_cast<int64_t>(i) * n + lane;
            float uk[CH];
#pragma unroll
            for (int k = 0; k < CH; ++k) uk[k] = valid(k) ? __ldg(u + 32 * k) : 0.f;
            float p0[NP], p1[NP];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                float pa0 = 0.f, pa1 = 0.f, pb0 = 0.f, pb1 = 0.f;
#pragma unroll
                for (int k = 0; k < CH; k += 2) {
                    ffma2_rows(pa0, pa1, uk[k], uk[k], xa[q][k], xb[q][k]);
                    if (k + 1 < CH) ffma2_rows(pb0, pb1, uk[k + 1], uk[k + 1], xa[q][k + 1], xb[q][k + 1]);
                }
                p0[q] = pa0;
                p1[q] = pa1;
                fadd2_rows(p0[q], p1[q], pb0, pb1);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const float t0 = __shfl_xor_sync(0xffffffffu, p0[q], off);
                    const float t1 = __shfl_xor_sync(0xffffffffu, p1[q], off);
                    fadd2_rows(p0[q], p1[q], t0, t1);
                }
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const float s0 = -(p0[q] + p0[q]), s1 = -(p1[q] + p1[q]);
#pragma unroll
                for (int k = 0; k < CH; ++k) ffma2_rows(xa[q][k], xb[q][k], s0, s1, uk[k], uk[k]);
            }
        }
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int k = 0; k < CH; ++k)
                if (valid(k)) {
                    S[(i0 + 2 * q) * ld + lane + 32 * k] = xa[q][k];
                    S[(i0 + 2 * q + 1) * ld + lane + 32 * k] = xb[q][k];
                }
    }
    __syncthreads();
    for (int e = tid; e < 32 * n; e += 256) {
        const int i = e & 31, c = e >> 5;
        if (r0 + i < n) B[base + static_cast<int64_t>(c) * n + r0 + i] = S[i * ld + c];
    }
}

}  // namespace

// hh_debug_k7_rows: rows per warp pass (2, or 4 for n <= 512; -1: policy).  Same box
// (tools/k7_rows_ab.py, profiles/r2/k7_rows_ab_r2.txt, outputs bit-identical): 4 rows win at
// n = 128 (39.8 vs 43.9 us), tie at 256, lose at 500 / 512 (75 / 157 vs 67 / 146 us)
thread_local int t_k7_rw = -1;
int k7_set_rows(int rw) {
    const int prev = t_k7_rw;
    t_k7_rw = (rw == 2 || rw == 4) ? rw : -1;
    return prev;
}

bool row_apply_supported(int64_t n, int64_t h, int dtype) {
    return dtype == 0 && n >= 4 && n <= 1024 && n % 4 == 0 && h <= 256;
}

cudaError_t launch_row_apply(const void *A, void *B, const void *U, int64_t n, int64_t h,
                             int64_t count, int op, cudaStream_t stream) {
    const size_t smem = static_cast<size_t>(32) * (n + 1) * 4;
    const dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>(count));
    auto go = [&](auto kernel) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kernel<<<grid, 256, smem, stream>>>(static_cast<const float *>(A), static_cast<float *>(B),
                                            static_cast<const float *>(U), static_cast<int>(n),
                                            static_cast<int>(h), op);
        return cudaGetLastError();
    };
    if (t_k7_rw == 4 || (t_k7_rw < 0 && n <= 128)) {
        if (n <= 128) return go(row_apply_kernel<4, 4>);
        if (n <= 256) return go(row_apply_kernel<8, 4>);
        if (n <= 512) return go(row_apply_kernel<16, 4>);
    }
    if (n <= 128) return go(row_apply_kernel<4>);
    if (n <= 256) return go(row_apply_kernel<8>);
    if (n <= 512) return go(row_apply_kernel<16>);
    return go(row_apply_kernel<32>);
}

cudaError_t launch_transpose(const void *A, void *B, int64_t n, int64_t count, int dtype,
                             cudaStream_t stream) {
    const unsigned g = static_cast<unsigned>((n + 31) / 32);
    const dim3 grid(g, g, static_cast<unsigned>(count));
    if (dtype == 0)
        batched_transpose_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float *>(A),
                                                                 static_cast<float *>(B), n);
    else
        batched_transpose_kernel<double><<<grid, 256, 0, stream>>>(static_cast<const double *>(A),
                                                                  static_cast<double *>(B), n);
    return cudaGetLastError();
}

}  // namespace hh
