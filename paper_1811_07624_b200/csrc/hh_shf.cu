// hh_shf.cu -- K8: the SHF objective of one reflector and its gradient for a batch of K
// candidate vectors (NEXT-f4; SURVEY §8(f) "batched C(u) and grad C evaluations"):
//
//     C(u)      = u^T (A B + B A) u - 2 (u^T A u)(u^T B u)            eq:theRk
//     grad C(u) = 2 (A B + B A) u - 4 ((u^T A u) B + (u^T B u) A) u   eq:gradient
//
// A, B symmetric n x n (so A B + B A is never formed): with a = A u, b = B u,
//     C = 2 a^T b - 2 (u^T a)(u^T b),     grad = 2 (A b + B a) - 4 ((u^T a) b + (u^T b) a).
// Launches: K8a  [a_k | b_k] = [A; B] u_k for all k (a tiled SIMT GEMM, 2n x n x K, split over
// 128-row contraction slices so that small problems still fill the SMs),
// K8b  one CTA per candidate: the slices summed in order, alpha = u.a, beta = u.b,
// gamma = a.b -> C;  with the gradient: K8c  A b_k + B a_k (the same GEMM over the
// concatenated 2n contraction, split likewise) and K8d  the slices summed in order with the
// factor 2 and the -4 (alpha b + beta a) terms.
// fp32 or fp64 (the FMA pipe: the contraction is 8 n^2 K flops on 16 n^2 + O(nK) bytes, so
// for K >= ~8 it is FMA-bound; see DESIGN.md §4 K8).
#include <algorithm>

#include "hh_internal.h"

namespace hh {
namespace {

constexpr int kBM = 64;    // output rows (i) per CTA
constexpr int kBN = 64;    // candidates (k) per CTA
constexpr int kBK = 16;    // contraction step
constexpr int kSlice = 128;   // contraction rows per CTA (split-K slice)

// Partial products over one contraction slice [j0, j0 + kSlice):
//   part[s][i][k] = sum_{j in slice s} M(i, j) R[j][k],   i < Mrows (column-major Mrows x K)
// project (grad_mode = 0): Mrows = 2n, M(i, j) = A(i, j) for i < n, B(i - n, j) below, R = Uc;
// gradient (grad_mode = 1): Mrows = n, the contraction runs over 2n: A(i, j) Yb[j][k] for
// j < n, then B(i, j - n) Ya[j - n][k].  M(i, j) = M[j * n + i] (symmetric storage: row j is
// column j), so the tile loads run along i and along j; the next step's tiles are loaded into
// registers while this step computes.  Deterministic: the slices are summed in order later.
template <typename T>
__global__ void __launch_bounds__(256) shf_gemm_kernel(int64_t n, int64_t K, const T *__restrict__ A,
                                                       const T *__restrict__ B, const T *__restrict__ Uc,
                                                       const T *__restrict__ Ya, const T *__restrict__ Yb,
                                                       T *__restrict__ part, int grad_mode) {
    __shared__ T Ms[kBK][kBM + 1];
    __shared__ T Rs[kBK][kBN + 1];
    // thread: rows i0 + tx + 16 p, candidates k0 + 4 ty + q (p, q < 4)
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;
    const int64_t Mrows = grad_mode ? n : 2 * n;
    const int64_t Jtot = grad_mode ? 2 * n : n;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kBM;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * kBN;
    const int64_t js = static_cast<int64_t>(blockIdx.z) * kSlice;
    const int64_t je = js + kSlice < Jtot ? js + kSlice : Jtot;
    auto mval = [&](int64_t i, int64_t j) -> T {   // M(i, j), zero outside
        if (i >= Mrows || j >= je) return T(0);
        if (!grad_mode) return i < n ? A[j * n + i] : B[j * n + (i - n)];
        return j < n ? A[j * n + i] : B[(j - n) * n + i];
    };
    auto rval = [&](int64_t j, int64_t k) -> T {   // R[j][k], zero outside
        if (k >= K || j >= je) return T(0);
        if (!grad_mode) return Uc[k * n + j];
        return j < n ? Yb[k * n + j] : Ya[k * n + (j - n)];
    };
    T acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = T(0);
    // per step: 1024 M values and 1024 R values, 4 of each per thread
    T mreg[4], rreg[4];
    auto fetch = [&](int64_t j0) {
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
            const int e = t + 256 * e4;
            mreg[e4] = mval(i0 + e % kBM, j0 + e / kBM);
            rreg[e4] = rval(j0 + e % kBK, k0 + e / kBK);
        }
    };
    fetch(js);
    for (int64_t j0 = js; j0 < je; j0 += kBK) {
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
            const int e = t + 256 * e4;
            Ms[e / kBM][e % kBM] = mreg[e4];
            Rs[e % kBK][e / kBK] = rreg[e4];
        }
        __syncthreads();
        if (j0 + kBK < je) fetch(j0 + kBK);
#pragma unroll
        for (int jj = 0; jj < kBK; ++jj) {
            T mv[4], rv[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) mv[p] = Ms[jj][tx + 16 * p];
#pragma unroll
            for (int q = 0; q < 4; ++q) rv[q] = Rs[jj][ty * 4 + q];
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[p][q] = fma(mv[p], rv[q], acc[p][q]);
        }
        __syncthreads();
    }
    T *out = part + static_cast<int64_t>(blockIdx.z) * Mrows * K;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t k = k0 + ty * 4 + q;
        if (k >= K) continue;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int64_t i = i0 + tx + 16 * p;
            if (i < Mrows) out[k * Mrows + i] = acc[p][q];
        }
    }
}

// fp32 form of the same partial products with an 8 x 8 register tile per thread (two float4
// row groups x two float4 candidate groups): 64 FMAs (as 32 packed FFMA2) per 64 B of
// shared-memory reads, where the 4 x 4 tile above is bound by its shared-memory reads.
// 128 threads, a 128-row x 64-candidate tile per CTA.
constexpr int kFM = 128, kFN = 64;
// two IEEE fp32 FMAs in one instruction (FFMA2: the 3-register FFMA issues at half the rate)
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B, D;\n\t"
        "mov.b64 A, {%2, %2};\n\tmov.b64 B, {%3, %4};\n\tmov.b64 D, {%0, %1};\n\t"
        "fma.rn.f32x2 D, A, B, D;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a), "f"(b0), "f"(b1));
}
__global__ void __launch_bounds__(128, 2) shf_gemm_f32_kernel(int64_t n, int64_t K, const float *__restrict__ A,
                                                           const float *__restrict__ B, const float *__restrict__ Uc,
                                                           const float *__restrict__ Ya, const float *__restrict__ Yb,
                                                           float *__restrict__ part, int grad_mode) {
    __shared__ __align__(16) float Ms[kBK][kFM + 4];
    __shared__ __align__(16) float Rs[kBK][kFN + 4];
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;   // rows 4 tx (+64), candidates 4 ty (+32)
    const int64_t Mrows = grad_mode ? n : 2 * n;
    const int64_t Jtot = grad_mode ? 2 * n : n;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kFM;
    const int64_t k0 = static_cast<int64_t>(blockIdx.y) * kFN;
    const int64_t js = static_cast<int64_t>(blockIdx.z) * kSlice;
    const int64_t je = js + kSlice < Jtot ? js + kSlice : Jtot;
    float acc[8][8];
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[p][q] = 0.f;
    // next step's tiles: this thread loads M row i0 + t (16 contraction rows) and the R
    // values (j0 + t % 16, k0 + t / 16 + 8 e) -- one row pointer each, no per-element branches
    // beyond the bounds
    float mreg[16], rreg[8];
    const int64_t irow = i0 + t;
    const bool irow_ok = irow < Mrows;
    const float *mbase = grad_mode ? A + irow : (irow < n ? A + irow : B + (irow - n));
    const int64_t kq = k0 + t / 16;
    const int jr0 = t % 16;
    auto fetch = [&](int64_t j0) {
#pragma unroll
        for (int e16 = 0; e16 < 16; ++e16) {
            const int64_t j = j0 + e16;
            float v = 0.f;
            if (irow_ok && j < je)
                v = (grad_mode && j >= n) ? B[(j - n) * n + irow] : mbase[j * n];
            mreg[e16] = v;
        }
        const int64_t j = j0 + jr0;
#pragma unroll
        for (int e8 = 0; e8 < 8; ++e8) {
            const int64_t k = kq + 8 * e8;
            float v = 0.f;
            if (k < K && j < je)
                v = !grad_mode ? Uc[k * n + j] : (j < n ? Yb[k * n + j] : Ya[k * n + (j - n)]);
            rreg[e8] = v;
        }
    };
    fetch(js);
    for (int64_t j0 = js; j0 < je; j0 += kBK) {
#pragma unroll
        for (int e16 = 0; e16 < 16; ++e16) {
            const int e = t + 128 * e16;
            Ms[e / kFM][e % kFM] = mreg[e16];
        }
#pragma unroll
        for (int e8 = 0; e8 < 8; ++e8) {
            const int e = t + 128 * e8;
            Rs[e % kBK][e / kBK] = rreg[e8];
        }
        __syncthreads();
        if (j0 + kBK < je) fetch(j0 + kBK);
#pragma unroll
        for (int jj = 0; jj < kBK; ++jj) {
            const float4 m0 = *reinterpret_cast<const float4 *>(&Ms[jj][4 * tx]);
            const float4 m1 = *reinterpret_cast<const float4 *>(&Ms[jj][64 + 4 * tx]);
            const float4 r0 = *reinterpret_cast<const float4 *>(&Rs[jj][4 * ty]);
            const float4 r1 = *reinterpret_cast<const float4 *>(&Rs[jj][32 + 4 * ty]);
            const float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
            const float rv[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
            for (int p = 0; p < 8; ++p)
#pragma unroll
                for (int q = 0; q < 8; q += 2) ffma2(acc[p][q], acc[p][q + 1], mv[p], rv[q], rv[q + 1]);
        }
        __syncthreads();
    }
    float *out = part + static_cast<int64_t>(blockIdx.z) * Mrows * K;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int64_t k = k0 + (q < 4 ? 4 * ty + q : 32 + 4 * ty + q - 4);
        if (k >= K) continue;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int64_t i = i0 + h2 * 64 + 4 * tx;
            float *o = out + k * Mrows + i;
            if (i + 3 < Mrows && (Mrows & 3) == 0) {
                *reinterpret_cast<float4 *>(o) = make_float4(acc[4 * h2][q], acc[4 * h2 + 1][q],
                                                             acc[4 * h2 + 2][q], acc[4 * h2 + 3][q]);
            } else {
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    if (i + p < Mrows) o[p] = acc[4 * h2 + p][q];
            }
        }
    }
}

// one CTA per candidate: a = A u, b = B u summed over the project slices (in slice order,
// written to Ya / Yb for the gradient pass), then alpha = u.a, beta = u.b, gamma = a.b (fixed
// order: per-thread partials, warp butterfly, warps in order) and C = 2 gamma - 2 alpha beta
template <typename T>
__global__ void __launch_bounds__(256) shf_dots_kernel(int64_t n, int64_t K, int ns, const T *__restrict__ part,
                                                       const T *__restrict__ Uc, T *__restrict__ Ya,
                                                       T *__restrict__ Yb, T *__restrict__ ab,
                                                       T *__restrict__ cost) {
    __shared__ T red[3][8];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t k = blockIdx.x;
    const T *u = Uc + k * n;
    const int64_t st = 2 * n * K;   // slice stride
    T al = T(0), be = T(0), ga = T(0);
    for (int64_t i = t; i < n; i += 256) {
        const T *pa = part + k * 2 * n + i;
        T ai = pa[0], bi = pa[n];
        for (int s = 1; s < ns; ++s) {
            ai += pa[s * st];
            bi += pa[s * st + n];
        }
        Ya[k * n + i] = ai;
        Yb[k * n + i] = bi;
        const T ui = u[i];
        al = fma(ui, ai, al);
        be = fma(ui, bi, be);
        ga = fma(ai, bi, ga);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, off);
        be += __shfl_xor_sync(0xffffffffu, be, off);
        ga += __shfl_xor_sync(0xffffffffu, ga, off);
    }
    if (lane == 0) {
        red[0][warp] = al;
        red[1][warp] = be;
        red[2][warp] = ga;
    }
    __syncthreads();
    if (t == 0) {
        T a2 = red[0][0], b2 = red[1][0], g2 = red[2][0];
        for (int w = 1; w < 8; ++w) {
            a2 += red[0][w];
            b2 += red[1][w];
            g2 += red[2][w];
        }
        ab[2 * k] = a2;
        ab[2 * k + 1] = b2;
        cost[k] = T(2) * g2 - T(2) * (a2 * b2);
    }
}

// grad[k][i] = 2 sum_s part[s][k][i] - 4 (alpha_k Yb[k][i] + beta_k Ya[k][i])
template <typename T>
__global__ void __launch_bounds__(256) shf_grad_kernel(int64_t n, int64_t K, int ns, const T *__restrict__ part,
                                                       const T *__restrict__ Ya, const T *__restrict__ Yb,
                                                       const T *__restrict__ ab, T *__restrict__ grad) {
    const int64_t tot = n * K;
    for (int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < tot;
         o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = o / n;
        T z = part[o];
        for (int s = 1; s < ns; ++s) z += part[s * tot + o];
        grad[o] = T(2) * z - T(4) * (ab[2 * k] * Yb[o] + ab[2 * k + 1] * Ya[o]);
    }
}

int slices(int64_t J) { return static_cast<int>((J + kSlice - 1) / kSlice); }

template <typename T>
cudaError_t launch_t(int64_t n, const void *A, const void *B, const void *Uc, int64_t K, void *cost,
                     void *grad, void *ws, cudaStream_t stream, LaunchInfo *info) {
    // workspace: Ya, Yb (n x K each), alpha / beta (2 K), the split-K partials
    T *Ya = static_cast<T *>(ws);
    T *Yb = Ya + n * K;
    T *ab = Yb + n * K;
    T *part = ab + ((2 * K + 63) / 64) * 64;
    const T *a = static_cast<const T *>(A), *b = static_cast<const T *>(B);
    const T *u = static_cast<const T *>(Uc);
    const int ns1 = slices(n), ns2 = slices(2 * n);
    const unsigned kt = static_cast<unsigned>((K + kBN - 1) / kBN);
    constexpr bool f32 = sizeof(T) == 4;
    const int tm = f32 ? kFM : kBM;
    const unsigned ktf = static_cast<unsigned>((K + (f32 ? kFN : kBN) - 1) / (f32 ? kFN : kBN));
    (void)kt;
    auto gemm = [&](dim3 g, int mode) {
        if constexpr (f32)
            shf_gemm_f32_kernel<<<g, 128, 0, stream>>>(n, K, a, b, u, Ya, Yb, part, mode);
        else
            shf_gemm_kernel<T><<<g, 256, 0, stream>>>(n, K, a, b, u, Ya, Yb, part, mode);
    };
    const dim3 g1(static_cast<unsigned>((2 * n + tm - 1) / tm), ktf, ns1);
    gemm(g1, 0);
    shf_dots_kernel<T><<<static_cast<unsigned>(K), 256, 0, stream>>>(
        n, K, ns1, part, u, Ya, Yb, ab, static_cast<T *>(cost));
    int nl = 2;
    if (grad) {
        const dim3 g2(static_cast<unsigned>((n + tm - 1) / tm), ktf, ns2);
        gemm(g2, 1);
        const int64_t tot = n * K;
        shf_grad_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((tot + 255) / 256, 148 * 16)), 256, 0, stream>>>(
            n, K, ns2, part, Ya, Yb, ab, static_cast<T *>(grad));
        nl += 2;
    }
    if (info) {
        info->variant = sizeof(T) == 4 ? "shf_f32_simt" : "shf_f64_simt";
        info->grid = static_cast<int>(g1.x * g1.y * g1.z);
        info->block = f32 ? 128 : 256;
        info->smem = static_cast<int>(f32 ? 4 * kBK * (kFM + kFN + 8) : sizeof(T) * kBK * (kBM + kBN + 2));
        info->nchunks = ns1;
        info->launches = nl;
    }
    return cudaGetLastError();
}

}  // namespace

size_t shf_ws_bytes(int64_t n, int64_t K, int dtype) {
    // Ya, Yb, alpha / beta (2 K, rounded to 64), the split-K partials (the larger of the two
    // passes: slices(n) x 2n x K or slices(2n) x n x K)
    const size_t s = dtype == 0 ? 4 : 8;
    const size_t parts = static_cast<size_t>(std::max(slices(n) * 2 * n * K, slices(2 * n) * n * K));
    return (static_cast<size_t>(2 * n * K + ((2 * K + 63) / 64) * 64 + parts) * s + 255) &
           ~static_cast<size_t>(255);
}

cudaError_t launch_shf(int64_t n, const void *A, const void *B, const void *Uc, int64_t K, void *cost,
                       void *grad, int dtype, void *ws, cudaStream_t stream, LaunchInfo *info) {
    return dtype == 0 ? launch_t<float>(n, A, B, Uc, K, cost, grad, ws, stream, info)
                      : launch_t<double>(n, A, B, Uc, K, cost, grad, ws, stream, info);
}

}  // namespace hh
