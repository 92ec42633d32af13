// hh_wy.cu -- K4 (compact-WY preparation) and K5 (compact-WY apply on the
// sm_100a tensor cores) for large h.
//
// The reflectors (in the order of the requested product, see below) are cut into
// nblk blocks of b (b <= 256, a multiple of 32; the last block is padded with
// u = 0 identity slots).  For one block with W = [w_1 .. w_b] (n x b):
//
//     H(w_1) H(w_2) ... H(w_b) = I - W T W^T,     T upper triangular, T_ii = 2,
//     T[0:i, i] = -2 T[0:i, 0:i] (W[:, 0:i]^T w_i)                     (K4)
//
// (verified from Eq. 2, by induction: appending H(w_i) to I - W'T'W'^T
// adds the column t = -2 T'(W'^T w_i) and the diagonal entry 2).  With V = W T the
// block acts on a column tile as
//
//     G = W^T X          (K5a "project":  M = 128 columns, N = b, K = n)
//     X <- X - V G^T...  (K5b "update":   M = 128 columns, N = 256 rows, K = b)
//
// Q X = H_1 ... H_h X applies the LAST block first; Q^T X = H_h ... H_1 X is the
// same computation on the reversed reflector list (reflectors are
// symmetric, so the transpose only reverses the order).  This is algebraically the
// product of Eq. 1-2 applied one reflector at a time (north_star
// (c)); only the rounding differs.
//
// Precision ("bf16x3"): every tensor-core operand z (fp32) is split as
// z = hi + lo + O(2^-17 |z|), hi = bf16(z), lo = bf16(z - hi); the products
// hi*hi + hi*lo + lo*hi are accumulated in fp32 in TMEM.  That keeps fp32-level
// accuracy (~1e-6 relative against the 2e-5*sqrt(h) gate) at twice the
// TF32 tensor rate, with bf16's full fp32 exponent range (no scaling).
//
// Data movement: X, W and V tiles move by TMA (cp.async.bulk.tensor, SWIZZLE_64B
// K-major for the MMA operands); the fp32 X tile is split into bf16 hi/lo in shared
// memory by converter warps; one elected thread issues tcgen05.mma; accumulators
// live in TMEM (2 x 256 columns, double-buffered) and are drained by epilogue
// warps with tcgen05.ld.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <memory>
#include <new>
#include <vector>

#include "hh_internal.h"
#include "hh_tc.cuh"

namespace hh {

namespace {

constexpr int kGramRows = 128;   // Gram split-K slice (rows of n_pad per CTA)
constexpr int kRowChunk = 128;    // K5b rows r per accumulator (MMA M)
constexpr int kTileCols = 128;    // columns of X per tile (K5a MMA M, K5b MMA N)
constexpr int kRaw1 = 12;         // K5a raw fp32 X ring depth: maximum (runtime nraw)
constexpr int kStages1 = 3;       // K5a converted X + W ring depth
constexpr int kStages3 = 3;       // K5b V ring depth
constexpr int kXStages = 16;      // K5b X box ring depth: maximum (runtime nxs, even)
constexpr int kXBoxCols = 16;     // columns per X box
constexpr int kXBoxBytes = 8192;  // fp32 X box (128 rows x 16 columns)
constexpr int kRawBytes = 16384;     // fp32 X tile (128 columns x 32 rows)
constexpr int kConv1Bytes = 49152;   // X hi/lo 16K + W hi/lo 32K at b = 256 (max)
constexpr int kStage3Bytes = 16384;  // V hi/lo tile (128 rows x 32 bf16) x 2
constexpr int kGresBytes = 131072;   // resident G hi/lo (128 x 256 bf16) x 2 at b = 256 (max)
constexpr int kSmemMax = 232448;     // 227 KB opt-in per CTA
constexpr int kKChunk1 = 8;          // K5a schedule unit: 8 K steps (256 rows of X)
constexpr int kSlots1 = 256;         // K5a split-tile hand-off pairs (>= the grid)
constexpr int kMaxPasses = 128;      // block-program passes (h <= 32768 apply, 8192 sym)

size_t al(size_t x) { return (x + 1023) & ~static_cast<size_t>(1023); }

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint16_t f2bf(float x) {
    uint16_t b;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(b) : "f"(x));
    return b;
}
__device__ __forceinline__ float bf2f(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// Programmatic dependent launch: every kernel of the program lets the next one launch at once
// (its CTAs are placed as this grid's CTAs retire) and waits for the previous one's results
// before touching them -- the launch latency and setup of each dependent kernel overlap the
// tail of its predecessor (no effect when a kernel is launched without the attribute).
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ K4: preparation
// Wf[i][r] (fp32, h_pad x n_pad) = u_i[r] (product order of R1, zero padded).
// Wb = bf16 split, R = h_pad + extra rows: [hi rows 0..R) [lo rows R..2R), ld = n_pad.
// With lam != NULL the `extra` rows h_pad.. hold lambda (.) w_i of block `lam_blk`
// (the Lambda W operand of the symmetric block).
__global__ void wy_pack_kernel(const float *__restrict__ U, int64_t n, int64_t h, int h_pad,
                               int64_t n_pad, const float *__restrict__ lam, int lam_blk, int b,
                               int extra, int reverse, float *__restrict__ Wf,
                               uint16_t *__restrict__ Wb) {
    pdl_wait();
    pdl_trigger();
    const int64_t R = h_pad + extra;
    const int64_t total = R * n_pad;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / n_pad, r = idx % n_pad;
        float v = 0.f;
        if (i < h_pad) {
            if (i < h && r < n) v = U[(reverse ? h - 1 - i : i) * n + r];
            Wf[idx] = v;
        } else {
            const int64_t src = static_cast<int64_t>(lam_blk) * b + (i - h_pad);
            if (src < h && r < n) v = lam[r] * U[src * n + r];
        }
        const uint16_t hb = f2bf(v);
        Wb[idx] = hb;
        Wb[total + idx] = f2bf(v - bf2f(hb));
    }
}

// out[r] = a[r] * b[r] (the symmetric block's pre-scale Lambda D for a two-sided D)
__global__ void wy_vmul_kernel(const float *__restrict__ a, const float *__restrict__ b, int64_t n,
                               float *__restrict__ out) {
    pdl_wait();
    pdl_trigger();
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[r] = a[r] * b[r];
}

// Sp[blk][split][l][m] = sum_{r in split} w_l[r] wt[r] w_m[r] over 128-row splits
// of n_pad (wt = 1 or lambda), blocks blk0.., upper 64x64 tiles only unless `full`
// (the reduction over splits is done in fixed order by wy_gram_reduce_kernel:
// deterministic).
// With Pp != NULL the z slices from pz on compute, in the same launch, the partials of
// P = W^T Lambda W of block pblk (full, wt = plam) into Pp[split] (the symmetric program).
__global__ void __launch_bounds__(256) wy_gram_kernel(const float *__restrict__ Wf, int64_t n_pad,
                                                      int b, int nsplit, int rows, int blk0,
                                                      const float *__restrict__ wt, int full,
                                                      float *__restrict__ Sp, int dep_wait, int pz,
                                                      int pblk, const float *__restrict__ plam,
                                                      float *__restrict__ Pp) {
    // dep_wait = 0: launched behind the first projection, whose result it does not read (its
    // input W was packed before that projection started): it runs beside it, not after it
    if (dep_wait) pdl_wait();
    pdl_trigger();
    const int ti = blockIdx.x, tj = blockIdx.y;
    int blk = blockIdx.z / nsplit, sp = blockIdx.z % nsplit;
    float *out = Sp + (static_cast<int64_t>(blk) * nsplit + sp) * b * b;
    if (Pp && static_cast<int>(blockIdx.z) >= pz) {
        sp = blockIdx.z - pz;
        blk = pblk - blk0;
        wt = plam;
        full = 1;
        out = Pp + static_cast<int64_t>(sp) * b * b;
    }
    if (ti > tj && !full) return;
    __shared__ __align__(16) float Ls[32][68], Ms[32][68];   // rows 16-B aligned: float4 reads
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;
    float acc[4][4] = {};
    const int64_t r0 = static_cast<int64_t>(sp) * rows;
    const float *Wl = Wf + (static_cast<int64_t>(blk0 + blk) * b + ti * 64) * n_pad;
    const float *Wm = Wf + (static_cast<int64_t>(blk0 + blk) * b + tj * 64) * n_pad;
    const int rows_l = min(64, b - ti * 64), rows_m = min(64, b - tj * 64);
    for (int64_t rc = r0; rc < r0 + rows; rc += 32) {
        for (int e = t; e < 32 * 64; e += 256) {
            const int c = e / 32, k = e % 32;
            const float w = wt ? wt[rc + k] : 1.f;
            Ls[k][c] = c < rows_l ? w * Wl[c * n_pad + rc + k] : 0.f;
            Ms[k][c] = c < rows_m ? Wm[c * n_pad + rc + k] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const float4 a4 = *reinterpret_cast<const float4 *>(&Ls[k][ty * 4]);
            const float4 m4 = *reinterpret_cast<const float4 *>(&Ms[k][tx * 4]);
            const float a[4] = {a4.x, a4.y, a4.z, a4.w}, m[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(a[p], m[q], acc[p][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int l = ti * 64 + ty * 4 + p;
        if (l >= b) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = tj * 64 + tx * 4 + q;
            if (m < b) out[static_cast<int64_t>(l) * b + m] = acc[p][q];
        }
    }
}

// S[blk][l][m] = sum over the splits of the Gram partials, upper tiles, in a fixed order
// (deterministic).  thread_per_elem: one thread per element walking the splits (coalesced
// across threads; enough parallelism for large b); else one warp per element, lane q adding
// splits q, q + 32, ... then a butterfly (small b: few elements, many splits).
// With Pp != NULL one more b x b matrix follows the nblk blocks: P = sum of the Pp partials
// (full), written to P.
__global__ void wy_gram_reduce_kernel(const float *__restrict__ Sp, int b, int nblk, int nsplit,
                                      int full, float *__restrict__ S, int thread_per_elem,
                                      const float *__restrict__ Pp, float *__restrict__ P) {
    pdl_wait();
    pdl_trigger();
    const int64_t bb = static_cast<int64_t>(b) * b;
    const int64_t tot = nblk * bb + (Pp ? bb : 0);
    // element idx: (source partials, full?, destination)
    auto src = [&](int64_t idx, const float *&p, bool &f, float *&dst) {
        if (idx >= nblk * bb) {
            const int64_t e = idx - nblk * bb;
            p = Pp + e;
            f = true;
            dst = P + e;
        } else {
            const int64_t blk = idx / bb, e = idx % bb;
            const int l = static_cast<int>(e / b), m = static_cast<int>(e % b);
            p = Sp + blk * nsplit * bb + e;
            f = full || (l / 64) <= (m / 64);
            dst = S + idx;
        }
    };
    if (thread_per_elem) {
        for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
             idx < tot; idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const float *p;
            bool f;
            float *dst;
            src(idx, p, f, dst);
            float s = 0.f;
            if (f)
                for (int q = 0; q < nsplit; ++q) s += p[q * bb];
            *dst = s;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t idx = w0; idx < tot; idx += nw) {
        const float *p;
        bool f;
        float *dst;
        src(idx, p, f, dst);
        float s = 0.f;
        if (f)
            for (int q = lane; q < nsplit; q += 32) s += p[q * bb];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) *dst = s;
    }
}

// T (upper triangular, b x b) per block, built in shared memory (packed upper
// rows): the 32x32 diagonal blocks by the forward recurrence
//   T[l][i] = -2 sum_{m=l}^{i-1} T[l][m] S[m][i],  T[i][i] = 2,
// then 32 columns at a time (block form of the same product, H-blocks 1 = [0,c),
// 2 = [c,c+32)):  T[0:c, c:c+32] = -T[0:c,0:c] * (S[0:c, c:c+32] * T[c:c+32, c:c+32]).
__global__ void __launch_bounds__(256) wy_tbuild_kernel(const float *__restrict__ Sg, int b,
                                                          float *__restrict__ Tg, int diag_only) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float tsm[];
    const int blk = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t bb = static_cast<int64_t>(b) * b;
    const float *S = Sg + blk * bb;
    float *Tout = Tg + blk * bb;
    float *Tp = tsm;                                   // packed upper, b(b+1)/2
    float *Sb = Tp + (b * (b + 1) / 2 + 31) / 32 * 32; // 8 x 32 x 33 / S panel (c x 32)
    float *Pm = Sb + 8 * 32 * 33;                      // c x 32
    auto tp = [&](int l, int m) -> float & { return Tp[l * b - (l * (l - 1)) / 2 + (m - l)]; };
    const int nb = b / 32;
    // level 0: warp w builds diagonal block w; lane l keeps row l of T_ww in registers
    // (the recurrence fully unrolled: static register indices, S column i broadcast from
    // shared memory, four accumulators per dot)
    if (warp < nb) {
        const int o = warp * 32;
        float(*sb)[33] = reinterpret_cast<float(*)[33]>(Sb + warp * 32 * 33);
        for (int r = 0; r < 32; ++r) sb[r][lane] = S[(o + r) * b + o + lane];
        __syncwarp();
        float tr[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) tr[m] = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < i; ++m) a[m & 3] = fmaf(tr[m], sb[m][i], a[m & 3]);
            const float v = -2.f * ((a[0] + a[1]) + (a[2] + a[3]));
            tr[i] = lane < i ? v : (lane == i ? 2.f : 0.f);
        }
#pragma unroll
        for (int m = 0; m < 32; ++m)
            if (m >= lane) tp(o + lane, o + m) = tr[m];
    }
    __syncthreads();
    // extension steps (256 threads); each thread owns (row l, 4 consecutive columns): 2 shared loads
    // (one broadcast, one 16-B) per 4 FMAs.  diag_only: only the 32 x 32 diagonal blocks
    // are wanted (wy_vrec_kernel builds V = W T from them without the rest of T)
    float *T22 = Pm + 224 * 32;                        // 32 x 32 dense diagonal block
    for (int c = 32; c < (diag_only ? 0 : b); c += 32) {
        // S panel S[0:c, c:c+32] -> Sb (c x 32); T22 = T[c:c+32, c:c+32] (dense)
        for (int e = t; e < c * 32; e += 256) Sb[e] = S[(e / 32) * b + c + (e % 32)];
        for (int e = t; e < 1024; e += 256) {
            const int mm = e / 32, jj = e % 32;
            T22[e] = jj >= mm ? tp(c + mm, c + jj) : 0.f;
        }
        __syncthreads();
        for (int e = t; e < c * 8; e += 256) {
            const int l = e / 8, j0 = (e % 8) * 4;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int m = 0; m < j0 + 4; ++m) {
                const float sv = Sb[l * 32 + m];
                const float4 tv = *reinterpret_cast<const float4 *>(T22 + m * 32 + j0);
                acc.x = fmaf(sv, tv.x, acc.x);
                acc.y = fmaf(sv, tv.y, acc.y);
                acc.z = fmaf(sv, tv.z, acc.z);
                acc.w = fmaf(sv, tv.w, acc.w);
            }
            *reinterpret_cast<float4 *>(Pm + l * 32 + j0) = acc;
        }
        __syncthreads();
        for (int e = t; e < c * 8; e += 256) {
            const int l = e / 8, j0 = (e % 8) * 4;
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
            const float *trow = &tp(l, l);
            int m = l;
            for (; m + 1 < c; m += 2) {
                const float t0 = trow[m - l], t1 = trow[m - l + 1];
                const float4 p0 = *reinterpret_cast<const float4 *>(Pm + m * 32 + j0);
                const float4 p1 = *reinterpret_cast<const float4 *>(Pm + (m + 1) * 32 + j0);
                a0.x = fmaf(t0, p0.x, a0.x);
                a0.y = fmaf(t0, p0.y, a0.y);
                a0.z = fmaf(t0, p0.z, a0.z);
                a0.w = fmaf(t0, p0.w, a0.w);
                a1.x = fmaf(t1, p1.x, a1.x);
                a1.y = fmaf(t1, p1.y, a1.y);
                a1.z = fmaf(t1, p1.z, a1.z);
                a1.w = fmaf(t1, p1.w, a1.w);
            }
            if (m < c) {
                const float t0 = trow[m - l];
                const float4 p0 = *reinterpret_cast<const float4 *>(Pm + m * 32 + j0);
                a0.x = fmaf(t0, p0.x, a0.x);
                a0.y = fmaf(t0, p0.y, a0.y);
                a0.z = fmaf(t0, p0.z, a0.z);
                a0.w = fmaf(t0, p0.w, a0.w);
            }
            float *o = &tp(l, c + j0);
            o[0] = -(a0.x + a1.x);
            o[1] = -(a0.y + a1.y);
            o[2] = -(a0.z + a1.z);
            o[3] = -(a0.w + a1.w);
        }
        __syncthreads();
    }
    if (diag_only) {   // only the 32 x 32 diagonal blocks are read (wy_vrec_kernel)
        for (int e = t; e < nb * 1024; e += 256) {
            const int o = (e >> 10) * 32, l = o + ((e >> 5) & 31), m = o + (e & 31);
            Tout[static_cast<int64_t>(l) * b + m] = m >= l ? tp(l, m) : 0.f;
        }
        return;
    }
    for (int64_t e = t; e < bb; e += 256) {
        const int l = static_cast<int>(e / b), m = static_cast<int>(e % b);
        Tout[e] = m >= l ? tp(l, m) : 0.f;
    }
}

// V = W T for the apply program WITHOUT forming T: over 32-column chunks c of a block,
//   T[:, c] = [-T[0:c,0:c] S[0:c,c] T_cc ; T_cc]   =>   V_c = (W_c - V_{<c} S_{<c,c}) T_cc
// (the block form of the same product used by wy_tbuild_kernel), so only the diagonal
// 32 x 32 blocks T_cc are needed and the work is parallel over rows: a CTA owns 64 rows
// of one block, keeps its V rows in SMEM and walks the chunks.  Output: bf16 hi/lo V
// rows (Vt[hi: blk*n_pad + r][i], Vt[lo: lo_off + ...]).
template <int RP>   // rows per thread: the CTA owns 32 * RP rows
__global__ void __launch_bounds__(256) wy_vrec_kernel(const float *__restrict__ Wf,
                                                      const float *__restrict__ Sg,
                                                      const float *__restrict__ Tg, int64_t n_pad,
                                                      int b, uint16_t *__restrict__ Vt,
                                                      int64_t lo_off) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float vsm[];
    constexpr int RW = 32 * RP;   // rows per CTA
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * RW;
    const int blk = blockIdx.y;
    const int t = threadIdx.x, tx = t % 8, ty = t / 8;   // 8 x 32: 4 columns x RP rows
    const int64_t bb = static_cast<int64_t>(b) * b;
    const float *S = Sg + blk * bb;
    const float *T = Tg + blk * bb;
    const float *W = Wf + static_cast<int64_t>(blk) * b * n_pad;
    const int spn = b - 32 > 0 ? (b - 32) * 32 : 32;
    float *Vs = vsm;                    // RW x (b + 1)
    float *SpB = Vs + RW * (b + 1);     // 2 x (b - 32) x 32 panels S[0:c, c:c+32]
    float *TcB = SpB + 2 * spn;         // 2 x 32 x 33
    float *Zs = TcB + 2 * 32 * 33;      // RW x 33
    const int ld = b + 1;
    // the next chunk's S panel and T_cc are copied asynchronously (cp.async) into the other
    // buffer while this chunk computes, and its W values are prefetched into registers:
    // the per-chunk global loads had been the exposed latency (long-scoreboard stalls)
    auto issue = [&](int c, int buf) {
        float *Sp = SpB + buf * spn, *Tc = TcB + buf * 32 * 33;
        for (int e = t; e < c * 32; e += 256)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(Sp + e)),
                         "l"(S + (e / 32) * b + c + (e % 32))
                         : "memory");
        for (int e = t; e < 32 * 32; e += 256) {
            const int m = e / 32, j = e % 32;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(Tc + m * 33 + j)),
                         "l"(T + (c + m) * b + c + j)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float wn[RP][4];
    auto load_w = [&](int c) {
#pragma unroll
        for (int p = 0; p < RP; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                wn[p][q] = W[static_cast<int64_t>(c + tx * 4 + q) * n_pad + r0 + ty * RP + p];
    };
    issue(0, 0);
    load_w(0);
    int buf = 0;
    for (int c = 0; c < b; c += 32, buf ^= 1) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();   // this chunk's panel and T_cc landed; previous chunk done
        if (c + 32 < b) issue(c + 32, buf ^ 1);
        const float *Sp = SpB + buf * spn, *Tc = TcB + buf * 32 * 33;
        // Z = W_c - V_{<c} S_{<c,c}   (RW x 32): thread rows ty*RP.., columns tx*4..
        float z[RP][4];
#pragma unroll
        for (int p = 0; p < RP; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) z[p][q] = wn[p][q];
        if (c + 32 < b) load_w(c + 32);
        // two partial sums per output (even / odd l): twice the independent FMA chains
        float z2[RP][4];
#pragma unroll
        for (int p = 0; p < RP; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) z2[p][q] = 0.f;
        for (int l = 0; l < c; l += 2) {   // c is a multiple of 32
            float va[RP], vb[RP];
#pragma unroll
            for (int p = 0; p < RP; ++p) {
                va[p] = Vs[(ty * RP + p) * ld + l];
                vb[p] = Vs[(ty * RP + p) * ld + l + 1];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float sa = Sp[l * 32 + tx * 4 + q], sb = Sp[(l + 1) * 32 + tx * 4 + q];
#pragma unroll
                for (int p = 0; p < RP; ++p) {
                    z[p][q] = fmaf(-va[p], sa, z[p][q]);
                    z2[p][q] = fmaf(-vb[p], sb, z2[p][q]);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < RP; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) z[p][q] += z2[p][q];
#pragma unroll
        for (int p = 0; p < RP; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) Zs[(ty * RP + p) * 33 + tx * 4 + q] = z[p][q];
        __syncthreads();
        // V_c = Z T_cc  (T_cc upper triangular)
#pragma unroll
        for (int p = 0; p < RP; ++p) {
            const int rr = ty * RP + p;
            // the four columns' chains interleaved over a fully unrolled m (T_cc upper
            // triangular: terms with m > j are predicated off)
            float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < 32; ++m) {
                const float zv = Zs[rr * 33 + m];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = tx * 4 + q;
                    if (m <= j) v[q] = fmaf(zv, Tc[m * 33 + j], v[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) Vs[rr * ld + c + tx * 4 + q] = v[q];
        }
        __syncthreads();
    }
    // bf16 hi/lo rows out
    for (int e = t; e < RW * b; e += 256) {
        const int rr = e / b, i = e % b;
        const float v = Vs[rr * ld + i];
        const uint16_t hv = f2bf(v);
        const int64_t o = (static_cast<int64_t>(blk) * n_pad + r0 + rr) * b + i;
        Vt[o] = hv;
        Vt[lo_off + o] = f2bf(v - bf2f(hv));
    }
}

size_t vrec_smem(int b) {
    return (static_cast<size_t>(64) * (b + 1) + 2 * static_cast<size_t>(std::max(b - 32, 1)) * 32 +
            2 * 32 * 33 + 64 * 33) *
           4;
}

// Small SIMT GEMM of the preparation (fp32):
//   out[r][c] = alpha_r * C[r][c] + sgn * sum_{l<K} A(r, l) B(l, c),   r < R, c < Kc
// A(r, l) = A[l*lda + r] (transA: W stored as rows w_l) or A[r*lda + l];
// B(l, c) = B[l*ldb + c] or B[c*ldb + l] (transB).  Output as fp32 (Of, ld ldo) and/or
// bf16 hi/lo (Ob hi at Ob[r*ldo + c], lo at Ob[lo_off + r*ldo + c]).  Grid (R/64, Kc/32).
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) wy_rowgemm_kernel(
    int64_t R, const float *__restrict__ A, int64_t lda, const float *__restrict__ B, int ldb,
    int K, const float *__restrict__ C, int64_t ldc, const float *__restrict__ alpha,
    int64_t alpha_n, float sgn, float *__restrict__ Of, uint16_t *__restrict__ Ob, int64_t ldo,
    int64_t lo_off) {
    pdl_wait();
    pdl_trigger();
    const int64_t r0 = blockIdx.x * 64;
    const int c0 = blockIdx.y * 32;
    __shared__ float As[32][65], Bs[32][33];
    const int t = threadIdx.x, tx = t % 8, ty = t / 8;
    float acc[2][4] = {};
    for (int l0 = 0; l0 < K; l0 += 32) {
        for (int e = t; e < 32 * 64; e += 256) {
            if (TA) {
                const int k = e / 64, r = e % 64;
                As[k][r] = (l0 + k < K && r0 + r < R)
                               ? A[static_cast<int64_t>(l0 + k) * lda + r0 + r] : 0.f;
            } else {
                const int r = e / 32, k = e % 32;
                As[k][r] = (l0 + k < K && r0 + r < R) ? A[(r0 + r) * lda + l0 + k] : 0.f;
            }
        }
        for (int e = t; e < 32 * 32; e += 256) {
            if (TB) {
                const int c = e / 32, k = e % 32;
                Bs[k][c] = l0 + k < K ? B[static_cast<int64_t>(c0 + c) * ldb + l0 + k] : 0.f;
            } else {
                const int k = e / 32, c = e % 32;
                Bs[k][c] = l0 + k < K ? B[static_cast<int64_t>(l0 + k) * ldb + c0 + c] : 0.f;
            }
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const float a0 = As[k][ty * 2], a1 = As[k][ty * 2 + 1];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float bv = Bs[k][tx * 4 + q];
                acc[0][q] = fmaf(a0, bv, acc[0][q]);
                acc[1][q] = fmaf(a1, bv, acc[1][q]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int64_t r = r0 + ty * 2 + p;
        if (r >= R) continue;
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = c0 + tx * 4 + q;
            v[q] = sgn * acc[p][q];
            if (C) v[q] = fmaf(alpha ? (r < alpha_n ? alpha[r] : 0.f) : 1.f, C[r * ldc + c], v[q]);
        }
        const int64_t o = r * ldo + c0 + tx * 4;
        if (Of) *reinterpret_cast<float4 *>(Of + o) = make_float4(v[0], v[1], v[2], v[3]);
        if (Ob) {
            uint16_t hv[4], lv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                hv[q] = f2bf(v[q]);
                lv[q] = f2bf(v[q] - bf2f(hv[q]));
            }
            uint2 H, L;
            H.x = hv[0] | (static_cast<uint32_t>(hv[1]) << 16);
            H.y = hv[2] | (static_cast<uint32_t>(hv[3]) << 16);
            L.x = lv[0] | (static_cast<uint32_t>(lv[1]) << 16);
            L.y = lv[2] | (static_cast<uint32_t>(lv[3]) << 16);
            *reinterpret_cast<uint2 *>(Ob + o) = H;
            *reinterpret_cast<uint2 *>(Ob + lo_off + o) = L;
        }
    }
}

// The symmetric program's folded block (b <= 64) in one launch instead of five rowgemms
// (DESIGN.md §4): a CTA owns kSymRows rows r and computes, from T and P = W^T Lambda W,
//   M = P T^T (redundantly per CTA: b^3 FMAs),  V = W T,  V' = W T^T   (its rows),
//   A1 = Lambda V' - V M,  A2 = V,
// and writes A = [A1, A2] as bf16 hi/lo rows (As[r][0:b) = A1, As[r][b:2b) = A2).
constexpr int kSymRows = 16;   // rows per CTA: 128 CTAs at n = 2048 (64-row CTAs: 32 CTAs, 22.8 us under ncu)
size_t symrows_smem(int b) {
    return static_cast<size_t>(4) * (2 * b * (b + 1) + b * kSymRows + 2 * kSymRows * (b + 1));
}
__global__ void __launch_bounds__(256) wy_sym_rows_kernel(const float *__restrict__ Wk,
                                                          const float *__restrict__ Tk,
                                                          const float *__restrict__ P,
                                                          const float *__restrict__ lam, int64_t n,
                                                          int64_t n_pad, int b,
                                                          uint16_t *__restrict__ As, int64_t alo) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float ssm[];
    const int ldb = b + 1;
    float *Ts = ssm;                       // b x (b + 1): T
    float *Ms = Ts + b * ldb;              // b x (b + 1): P, then M = P T^T
    float *Ws = Ms + b * ldb;              // b x kSymRows: W[l][rr]
    float *Vs = Ws + b * kSymRows;         // kSymRows x (b + 1): V = W T
    float *Vp = Vs + kSymRows * ldb;       // kSymRows x (b + 1): V' = W T^T
    const int t = threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kSymRows;
    for (int e = t; e < b * b; e += 256) {
        Ts[(e / b) * ldb + e % b] = Tk[e];
        Ms[(e / b) * ldb + e % b] = P[e];
    }
    for (int e = t; e < b * kSymRows; e += 256) {
        const int l = e / kSymRows, rr = e % kSymRows;
        Ws[e] = Wk[static_cast<int64_t>(l) * n_pad + r0 + rr];
    }
    __syncthreads();
    // V and V' (64 x b each) and M = P T^T (b x b, into registers first: Ms holds P)
    float macc[16];
    int mcnt = 0;
    for (int e = t; e < b * b; e += 256, ++mcnt) {
        const int i = e / b, j = e % b;
        float a = 0.f;
        for (int l = 0; l < b; ++l) a = fmaf(Ms[i * ldb + l], Ts[j * ldb + l], a);
        macc[mcnt] = a;
    }
    for (int e = t; e < kSymRows * b; e += 256) {
        const int rr = e / b, c = e % b;
        float v = 0.f, vp = 0.f;
        for (int l = 0; l < b; ++l) {
            const float w = Ws[l * kSymRows + rr];
            v = fmaf(w, Ts[l * ldb + c], v);
            vp = fmaf(w, Ts[c * ldb + l], vp);
        }
        Vs[rr * ldb + c] = v;
        Vp[rr * ldb + c] = vp;
    }
    __syncthreads();
    mcnt = 0;
    for (int e = t; e < b * b; e += 256, ++mcnt) Ms[(e / b) * ldb + e % b] = macc[mcnt];
    __syncthreads();
    const int64_t lda = 2 * static_cast<int64_t>(b);
    for (int e = t; e < kSymRows * b; e += 256) {
        const int rr = e / b, c = e % b;
        const int64_t r = r0 + rr;
        float acc = 0.f;
        for (int l = 0; l < b; ++l) acc = fmaf(Vs[rr * ldb + l], Ms[l * ldb + c], acc);
        const float a1 = fmaf(r < n ? lam[r] : 0.f, Vp[rr * ldb + c], -acc);
        const float a2 = Vs[rr * ldb + c];
        const uint16_t h1 = f2bf(a1), h2 = f2bf(a2);
        As[r * lda + c] = h1;
        As[alo + r * lda + c] = f2bf(a1 - bf2f(h1));
        As[r * lda + b + c] = h2;
        As[alo + r * lda + b + c] = f2bf(a2 - bf2f(h2));
    }
}

// ------------------------------------------------------------------ K5a: G = W^T X
// 15 warps: w0 TMA producer of the fp32 X tiles (4-deep raw ring), w1 TMA producer
// of the W hi/lo tiles, w2 MMA issuer (+TMEM owner), w3-10 converters (fp32 X tile
// -> bf16 hi/lo, SW64 K-major), w11-14 epilogue (TMEM -> bf16 hi/lo rows of G).
struct Bars1 {
    uint64_t rfull[kRaw1], rempty[kRaw1];
    uint64_t wfull[kStages1], cfull[kStages1], cempty[kStages1];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem;
    int last;   // split-tile hand-off: this CTA arrived second (epilogue broadcast)
};
// ld/st of the split-tile hand-off (L2, bypassing L1: written by another CTA)
__device__ __forceinline__ void st_cg4(float *p, float a, float b, float c, float d) {
    asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ float4 ld_cg4(const float *p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// TSA (b <= 128): the converters write X hi/lo straight into TMEM (tcgen05.st; each thread
// owns one column of the tile = one TMEM lane and 16 of the k-step's 32 rows, read from a
// SWIZZLE_128B raw box without bank conflicts) and the MMA takes A from TMEM: the converted X
// never touches shared memory (its stores and the MMA's A reads were ~40 of the ~92 KB of
// shared-memory traffic per k-step at b = 64).  TMEM: accumulators at 0 / 256,
// the three A stages at 128 + 32 s (hi 16 columns, lo 16).
template <bool TSA>
__global__ void __launch_bounds__(480, 1)
    wy_project_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                      uint16_t *__restrict__ Gt, int n, int64_t N, int b, int wrow_hi, int wrow_lo,
                      int ntiles, const float *__restrict__ dscale, int ks0, int nraw,
                      float *__restrict__ part, int *__restrict__ flag) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // ring sizes depend on b: a conversion stage holds X hi/lo (16 KB) and the W hi/lo
    // tiles (128 b bytes); the rest of the 227 KB is a deep raw-X ring (nraw stages)
    const int cvb = (TSA ? 0 : 16384) + 128 * b;   // (TSA: X hi/lo live in TMEM, W only)
    unsigned char *conv = smem + nraw * kRawBytes;
    Bars1 *bars = reinterpret_cast<Bars1 *>(conv + kStages1 * cvb);
    auto rawX = [&](int s) { return smem + s * kRawBytes; };
    auto Xhi = [&](int s) { return conv + s * cvb; };
    auto Xlo = [&](int s) { return conv + s * cvb + 8192; };
    auto Whi = [&](int s) { return conv + s * cvb + (TSA ? 0 : 16384); };
    auto Wlo = [&](int s) { return conv + s * cvb + (TSA ? 0 : 16384) + 64 * b; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (n + 31) / 32;
    // balanced schedule: (tile, K chunk) units, tile-major, in equal contiguous ranges per
    // CTA (whole tiles would leave 512 tiles on 148 SMs with a 4th-tile tail).  A tile cut
    // by a range boundary is shared by two CTAs: the next CTA computes the tile's trailing
    // K chunks as its first segment and leaves that fp32 partial G in slot blockIdx-1
    // (+ a flag); this CTA computes the leading chunks as its last segment, adds the
    // partial (long since available) and writes G.  grid <= ntiles, so a tile has at
    // most two owners, and no CTA waits before its last segment.
    const int64_t nkc = (nk - ks0 + kKChunk1 - 1) / kKChunk1;
    const int64_t utot = static_cast<int64_t>(ntiles) * nkc;
    const int64_t ubeg = utot * blockIdx.x / gridDim.x, uend = utot * (blockIdx.x + 1) / gridDim.x;
    auto for_segments = [&](auto &&fn) {   // fn(tile, ks_lo, ks_hi, head, tail)
        for (int64_t u = ubeg; u < uend;) {
            const int tile = static_cast<int>(u / nkc);
            const int64_t t0 = static_cast<int64_t>(tile) * nkc;
            const int plo = static_cast<int>(u - t0);
            const int phi = static_cast<int>(uend - t0 < nkc ? uend - t0 : nkc);
            const int klo = ks0 + plo * kKChunk1;
            const int khi = ks0 + phi * kKChunk1 < nk ? ks0 + phi * kKChunk1 : nk;
            // head: this CTA's first segment holds a tile's trailing chunks (hand the
            // partial to the previous CTA); tail: its last segment holds a tile's leading
            // chunks (take the next CTA's partial, write G)
            fn(tile, klo, khi, plo > 0, plo == 0 && phi < nkc);
            u = t0 + nkc;
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < nraw; ++s) {
            mbar_init(&bars->rfull[s], 1);
            mbar_init(&bars->rempty[s], 256);
        }
        for (int s = 0; s < kStages1; ++s) {
            mbar_init(&bars->wfull[s], 1);
            mbar_init(&bars->cfull[s], 256);
            mbar_init(&bars->cempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 128);
        }
        fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc<512>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;
    // TSA: blocks of b <= 128 keep two accumulators (0, 256) and put the A stages at 128; a
    // 256-wide block has one accumulator (0..255) and the A stages at 256
    const int nacc = (TSA && b > 128) ? 1 : 2;
    const uint32_t abase = (TSA && b > 128) ? 256u : 128u;
    pdl_wait();   // the previous kernel's results (after this CTA's setup)
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmX);
            int s = 0;
            uint32_t ph = 0;
            for_segments([&](int tile, int klo, int khi, bool, bool) {
                for (int ks = klo; ks < khi; ++ks) {
                    mbar_wait(&bars->rempty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&bars->rfull[s], static_cast<uint32_t>(kRawBytes));
                    tc::tma_load_2d(rawX(s), &tmX, ks * 32, tile * kTileCols, &bars->rfull[s]);
                    if (++s == nraw) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            });
        }
    } else if (warp == 1) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmW);
            int s = 0;
            uint32_t ph = 0;
            const uint32_t bytes = 128u * static_cast<uint32_t>(b);
            for_segments([&](int, int klo, int khi, bool, bool) {
                for (int ks = klo; ks < khi; ++ks) {
                    mbar_wait(&bars->cempty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&bars->wfull[s], bytes);
                    tc::tma_load_2d(Whi(s), &tmW, ks * 32, wrow_hi, &bars->wfull[s]);
                    tc::tma_load_2d(Wlo(s), &tmW, ks * 32, wrow_lo, &bars->wfull[s]);
                    if (++s == kStages1) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            });
        }
    } else if (warp == 2) {
        const uint32_t idesc = tc::idesc_bf16(128, b);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0;
        for_segments([&](int, int klo, int khi, bool, bool) {
            mbar_wait(&bars->acc_empty[a], aph ^ 1u);
            tc::fence_after_sync();
            const uint32_t d = tbase + static_cast<uint32_t>(a * 256);
            for (int ks = klo; ks < khi; ++ks) {
                mbar_wait(&bars->wfull[s], ph);
                mbar_wait(&bars->cfull[s], ph);
                tc::fence_after_sync();
                const uint32_t xh = smem_u32(Xhi(s)), xl = smem_u32(Xlo(s));
                const uint32_t wh = smem_u32(Whi(s)), wl = smem_u32(Wlo(s));
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint64_t bh = tc::sdesc_sw64(wh + kk * 32), blo = tc::sdesc_sw64(wl + kk * 32);
                    if constexpr (TSA) {
                        const uint32_t ta = tbase + abase + static_cast<uint32_t>(s * 32 + kk * 8);
                        tc::mma_bf16_ts_w(d, ta, bh, idesc, (ks != klo || kk != 0) ? 1u : 0u);
                        tc::mma_bf16_ts_w(d, ta, blo, idesc, 1u);
                        tc::mma_bf16_ts_w(d, ta + 16u, bh, idesc, 1u);
                    } else {
                        const uint64_t ah = tc::sdesc_sw64(xh + kk * 32), alo = tc::sdesc_sw64(xl + kk * 32);
                        tc::mma_bf16_w(d, ah, bh, idesc, (ks != klo || kk != 0) ? 1u : 0u);
                        tc::mma_bf16_w(d, ah, blo, idesc, 1u);
                        tc::mma_bf16_w(d, alo, bh, idesc, 1u);
                    }
                }
                tc::mma_commit_w(&bars->cempty[s]);
                if (++s == kStages1) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->acc_full[a]);
            if (++a == nacc) {
                a = 0;
                aph ^= 1u;
            }
        });
        __syncwarp();
    } else if (TSA && warp < 11) {
        // converters (TSA): warp w owns TMEM lane quarter w % 4 (tile columns 32 (w % 4) + lane)
        // and rows 16 hf .. 16 hf + 15 of each k-step (hf = 0 for warps 3-6, 1 for 7-10)
        const int q = warp & 3, hf = (warp - 3) >> 2;
        const int col = q * 32 + lane;
        const uint32_t tl = tbase + (static_cast<uint32_t>(q * 32) << 16);
        int rs = 0, cs = 0;
        uint32_t rph = 0, cph = 0;
        for_segments([&](int, int klo, int khi, bool, bool) {
            for (int ks = klo; ks < khi; ++ks) {
                mbar_wait(&bars->rfull[rs], rph);
                // SWIZZLE_128B raw box: column col's 16-B chunk j at col * 128 + ((j ^ (col & 7)) << 4)
                const uint32_t raw = smem_u32(rawX(rs)) + static_cast<uint32_t>(col) * 128u;
                float v[16];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const uint32_t j = static_cast<uint32_t>(4 * hf + jj);
                    const float4 f = tc::lds128(raw + ((j ^ static_cast<uint32_t>(col & 7)) << 4));
                    v[4 * jj] = f.x;
                    v[4 * jj + 1] = f.y;
                    v[4 * jj + 2] = f.z;
                    v[4 * jj + 3] = f.w;
                }
                if (dscale) {   // NEXT-f1 right factor: project D X (rows uniform over the warp)
                    const int r0 = ks * 32 + 16 * hf;
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (r0 + e < n) v[e] *= __ldg(dscale + r0 + e);
                }
                fence_proxy_async_smem();
                tc::mbar_arrive(&bars->rempty[rs]);
                uint32_t H[8], L[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) tc::split2(v[2 * e], v[2 * e + 1], H[e], L[e]);
                mbar_wait(&bars->cempty[cs], cph ^ 1u);
                tc::fence_after_sync();
                const uint32_t ta = tl + abase + static_cast<uint32_t>(cs * 32 + hf * 8);
                tc::tmem_st8(ta, make_uint4(H[0], H[1], H[2], H[3]), make_uint4(H[4], H[5], H[6], H[7]));
                tc::tmem_st8(ta + 16u, make_uint4(L[0], L[1], L[2], L[3]), make_uint4(L[4], L[5], L[6], L[7]));
                tc::tmem_wait_st();
                tc::fence_before_sync();
                tc::mbar_arrive(&bars->cfull[cs]);
                if (++rs == nraw) {
                    rs = 0;
                    rph ^= 1u;
                }
                if (++cs == kStages1) {
                    cs = 0;
                    cph ^= 1u;
                }
            }
        });
    } else if (warp < 11) {
        // converters: 256 threads, 4 float4 each per k-step
        const int ct = threadIdx.x - 96;
        int rs = 0, cs = 0;
        uint32_t rph = 0, cph = 0;
        for_segments([&](int, int klo, int khi, bool, bool) {
            for (int ks = klo; ks < khi; ++ks) {
                mbar_wait(&bars->rfull[rs], rph);
                const uint32_t raw = smem_u32(rawX(rs));
                float4 v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = tc::lds128(raw + (ct + 256 * q) * 16);
                if (dscale) {   // NEXT-f1 right factor: project D X
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int r = ks * 32 + ((ct + 256 * q) & 7) * 4;
                        if (r < n) {
                            const float4 dv = *reinterpret_cast<const float4 *>(dscale + r);
                            v[q].x *= dv.x;
                            v[q].y *= dv.y;
                            v[q].z *= dv.z;
                            v[q].w *= dv.w;
                        }
                    }
                }
                mbar_wait(&bars->cempty[cs], cph ^ 1u);
                const uint32_t xh = smem_u32(Xhi(cs)), xl = smem_u32(Xlo(cs));
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int idx = ct + 256 * q;
                    const int r = idx >> 3, c4 = idx & 7;
                    uint2 H, L;
                    tc::split2(v[q].x, v[q].y, H.x, L.x);
                    tc::split2(v[q].z, v[q].w, H.y, L.y);
                    const uint32_t off = tc::sw64_off(r, c4 >> 1) + (c4 & 1) * 8;
                    tc::sts64(xh + off, H.x, H.y);
                    tc::sts64(xl + off, L.x, L.y);
                }
                // the raw tile is released only after its values were consumed (the
                // stores above depend on them) and ordered against the async proxy that
                // refills it (TMA)
                fence_proxy_async_smem();
                tc::mbar_arrive(&bars->rempty[rs]);
                tc::mbar_arrive(&bars->cfull[cs]);
                if (++rs == nraw) {
                    rs = 0;
                    rph ^= 1u;
                }
                if (++cs == kStages1) {
                    cs = 0;
                    cph ^= 1u;
                }
            }
        });
    } else {
        // epilogue: TMEM lane quarter q = warp % 4
        const int q = warp & 3;
        int a = 0;
        uint32_t aph = 0;
        uint16_t *Glo = Gt + N * b;
        const int jl = q * 32 + lane;
        for_segments([&](int tile, int, int, bool head, bool tail) {
            mbar_wait(&bars->acc_full[a], aph);
            tc::fence_after_sync();
            const int64_t j = static_cast<int64_t>(tile) * kTileCols + jl;
            // A tile cut by a range boundary has two owners: this CTA's tail segment (its
            // leading K chunks) and the next CTA's head segment (its trailing chunks).  The
            // hand-off pair (slot pair + arrival counter) is indexed by the boundary: blockIdx
            // for a tail, blockIdx - 1 for a head.  Each owner publishes its fp32 partial in
            // its own slot and counts itself in; the second to arrive adds the other's partial
            // (sum = leading + trailing in both cases: deterministic) and writes G.  Nobody
            // waits, so the protocol needs no co-residency.
            const bool split = head || tail;
            if (!split) {
                for (int c = 0; c < b / 32; ++c) {
                    float v[32];
                    tc::tmem_ld32(tbase + (static_cast<uint32_t>(q * 32) << 16) +
                                      static_cast<uint32_t>(a * 256 + c * 32),
                                  v);
                    if (j < N) {
                        uint32_t H[16], L[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) tc::split2(v[2 * e], v[2 * e + 1], H[e], L[e]);
                        uint4 *gh = reinterpret_cast<uint4 *>(Gt + j * b + c * 32);
                        uint4 *gl = reinterpret_cast<uint4 *>(Glo + j * b + c * 32);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            gh[e] = make_uint4(H[4 * e], H[4 * e + 1], H[4 * e + 2], H[4 * e + 3]);
                            gl[e] = make_uint4(L[4 * e], L[4 * e + 1], L[4 * e + 2], L[4 * e + 3]);
                        }
                    }
                }
            } else {
                // the boundary's slot pair: [leading partial, trailing partial]
                const size_t hp = static_cast<size_t>(head ? blockIdx.x - 1 : blockIdx.x);
                float *mine = part + (2 * hp + (head ? 1 : 0)) * kTileCols * b;
                const float *other = part + (2 * hp + (head ? 0 : 1)) * kTileCols * b;
                for (int c = 0; c < b / 32; ++c) {
                    float v[32];
                    tc::tmem_ld32(tbase + (static_cast<uint32_t>(q * 32) << 16) +
                                      static_cast<uint32_t>(a * 256 + c * 32),
                                  v);
                    float *dst = mine + (static_cast<size_t>(c) * kTileCols + jl) * 32;
#pragma unroll
                    for (int e = 0; e < 8; ++e) st_cg4(dst + 4 * e, v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
                }
                __threadfence();
                named_bar_sync(1, 128);
                if (jl == 0) {
                    const int prev = atomicAdd(flag + hp, 1);
                    bars->last = prev == 1;
                    if (prev == 1) flag[hp] = 0;   // both arrived: reset for the next launch
                    __threadfence();
                }
                named_bar_sync(1, 128);
                if (bars->last) {
                    // leading + trailing, in that order whichever side finishes
                    const float *lead = head ? other : mine;
                    const float *trail = head ? mine : other;
                    for (int c = 0; c < b / 32; ++c) {
                        const float *s0 = lead + (static_cast<size_t>(c) * kTileCols + jl) * 32;
                        const float *s1 = trail + (static_cast<size_t>(c) * kTileCols + jl) * 32;
                        uint32_t H[16], L[16];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float4 p0 = ld_cg4(s0 + 4 * e), p1 = ld_cg4(s1 + 4 * e);
                            tc::split2(p0.x + p1.x, p0.y + p1.y, H[2 * e], L[2 * e]);
                            tc::split2(p0.z + p1.z, p0.w + p1.w, H[2 * e + 1], L[2 * e + 1]);
                        }
                        if (j < N) {
                            uint4 *gh = reinterpret_cast<uint4 *>(Gt + j * b + c * 32);
                            uint4 *gl = reinterpret_cast<uint4 *>(Glo + j * b + c * 32);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                gh[e] = make_uint4(H[4 * e], H[4 * e + 1], H[4 * e + 2], H[4 * e + 3]);
                                gl[e] = make_uint4(L[4 * e], L[4 * e + 1], L[4 * e + 2], L[4 * e + 3]);
                            }
                        }
                    }
                }
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&bars->acc_empty[a]);
            if (++a == nacc) {
                a = 0;
                aph ^= 1u;
            }
        });
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 2) tc::tmem_free<512>(tbase);
}

// ------------------------------------------------------------------ K5b: X <- X - V G
// D[r][j] = sum_i V[r][i] G[j][i] with TMEM lane = row r, TMEM column = column j.
// 12 warps: w0 TMA producer (G tile, V tiles), w1 MMA issuer (+TMEM owner), w2 TMA
// producer of the X boxes (128 rows x 16 columns, fp32, 6-deep ring: the epilogue's
// HBM reads are asynchronous and need no registers), w3 idle, w4-11 epilogue in two
// groups of four (one warp per TMEM lane quarter); group g takes the boxes of parity
// g (so with an even ring depth every stage has one consumer group and the groups
// can never lap each other on a stage's mbarrier phase), reads X from shared memory
// (conflict-free) and stores Y = lam (.) X - D with 128-B coalesced global stores
// (lanes = consecutive rows).
struct Bars3 {
    uint64_t gfull, gempty;
    uint64_t full[kStages3], empty[kStages3];
    uint64_t xfull[kXStages], xempty[kXStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem;
};

__global__ void __launch_bounds__(640, 1)
    wy_update_kernel(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmXb,
                     const __grid_constant__ CUtensorMap tmYs, float *Y,
                     const float *__restrict__ lam, const float *__restrict__ post, int n,
                     int n_pad, int64_t N, int b, int vrow_hi, int vrow_lo, int ntiles, int rc0,
                     int copy_below, int nxs, unsigned long long *tl) {
    // tl (debug, CTA 0 only): per-role cycles spent waiting on each barrier (see
    // hh_debug_wy_timeline); NULL in production
    const bool dbg = tl != nullptr && blockIdx.x == 0;
    unsigned long long t_k0 = clock64(), w_a = 0, w_b = 0;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int nslab = b / 32;
    unsigned char *Ghi = smem;                       // nslab x 8 KB (128 columns x 32 K)
    unsigned char *Glo = smem + nslab * 8192;
    unsigned char *stg = smem + nslab * 16384;        // G hi/lo take nslab x 16 KB
    unsigned char *xst = stg + kStages3 * kStage3Bytes;
    Bars3 *bars = reinterpret_cast<Bars3 *>(xst + nxs * kXBoxBytes);
    auto Vhi = [&](int s) { return stg + s * kStage3Bytes; };
    auto Vlo = [&](int s) { return stg + s * kStage3Bytes + 8192; };
    auto Xs = [&](int s) { return reinterpret_cast<float *>(xst + s * kXBoxBytes); };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nrc = n_pad / kRowChunk;
    // balanced schedule: the (tile, row chunk) units, tile-major, are split into equal
    // contiguous ranges per CTA (512 tiles over 148 SMs would otherwise leave a 4th-tile
    // tail on some SMs); every role walks the same segments [rlo, rhi) of each tile.
    // Rows below rc0 are copy-only (no MMA) and exist only when copy_below.
    const int xrc0 = copy_below ? 0 : rc0;
    const int64_t per = nrc - xrc0;
    const int64_t utot = static_cast<int64_t>(ntiles) * per;
    const int64_t ubeg = utot * blockIdx.x / gridDim.x, uend = utot * (blockIdx.x + 1) / gridDim.x;
    auto for_segments = [&](auto &&fn) {
        for (int64_t u = ubeg; u < uend;) {
            const int tile = static_cast<int>(u / per);
            const int64_t t0 = static_cast<int64_t>(tile) * per;
            const int rlo = xrc0 + static_cast<int>(u - t0);
            const int rhi = xrc0 + static_cast<int>(uend - t0 < per ? uend - t0 : per);
            fn(tile, rlo, rhi);
            u = t0 + per;
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars->gfull, 1);
        mbar_init(&bars->gempty, 1);
        for (int s = 0; s < kStages3; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int s = 0; s < nxs; ++s) {
            mbar_init(&bars->xfull[s], 1);
            mbar_init(&bars->xempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 512);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<256>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;
    pdl_wait();   // the previous kernel's results (after this CTA's setup)
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmG);
            tc::prefetch_tmap(&tmV);
            int s = 0;
            uint32_t ph = 0, gph = 0;
            for_segments([&](int tile, int rlo, int rhi) {
                const int mlo = rlo > rc0 ? rlo : rc0;
                if (mlo >= rhi) return;   // copy-only segment: no G, no V
                mbar_wait(&bars->gempty, gph ^ 1u);
                mbar_arrive_expect_tx(&bars->gfull, static_cast<uint32_t>(nslab) * 16384u);
                for (int c = 0; c < nslab; ++c) {
                    tc::tma_load_2d(Ghi + c * 8192, &tmG, c * 32, tile * kTileCols, &bars->gfull);
                    tc::tma_load_2d(Glo + c * 8192, &tmG, c * 32,
                                    static_cast<int>(N) + tile * kTileCols, &bars->gfull);
                }
                gph ^= 1u;
                for (int rc = mlo; rc < rhi; ++rc) {
                    for (int c = 0; c < nslab; ++c) {
                        const unsigned long long t0 = clock64();
                        mbar_wait(&bars->empty[s], ph ^ 1u);
                        w_a += clock64() - t0;
                        mbar_arrive_expect_tx(&bars->full[s], static_cast<uint32_t>(kStage3Bytes));
                        tc::tma_load_2d(Vhi(s), &tmV, c * 32, vrow_hi + rc * kRowChunk, &bars->full[s]);
                        tc::tma_load_2d(Vlo(s), &tmV, c * 32, vrow_lo + rc * kRowChunk, &bars->full[s]);
                        if (++s == kStages3) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(kRowChunk, kTileCols);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0, gph = 0;
        const uint32_t gh0 = smem_u32(Ghi), gl0 = smem_u32(Glo);
        for_segments([&](int tile, int rlo, int rhi) {
            const int mlo = rlo > rc0 ? rlo : rc0;
            if (mlo >= rhi) return;
            mbar_wait(&bars->gfull, gph);
            gph ^= 1u;
            tc::fence_after_sync();
            for (int rc = mlo; rc < rhi; ++rc) {
                const unsigned long long t1 = clock64();
                mbar_wait(&bars->acc_empty[a], aph ^ 1u);
                w_b += clock64() - t1;
                tc::fence_after_sync();
                const uint32_t d = tbase + static_cast<uint32_t>(a * kTileCols);
                for (int c = 0; c < nslab; ++c) {
                    const unsigned long long t0 = clock64();
                    mbar_wait(&bars->full[s], ph);
                    w_a += clock64() - t0;
                    tc::fence_after_sync();
                    const uint32_t vh = smem_u32(Vhi(s)), vl = smem_u32(Vlo(s));
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t ah = tc::sdesc_sw64(vh + kk * 32), alo = tc::sdesc_sw64(vl + kk * 32);
                        const uint64_t bh = tc::sdesc_sw64(gh0 + c * 8192 + kk * 32);
                        const uint64_t blo = tc::sdesc_sw64(gl0 + c * 8192 + kk * 32);
                        tc::mma_bf16_w(d, ah, bh, idesc, (c | kk) != 0);
                        tc::mma_bf16_w(d, ah, blo, idesc, 1u);
                        tc::mma_bf16_w(d, alo, bh, idesc, 1u);
                    }
                    tc::mma_commit_w(&bars->empty[s]);
                    if (++s == kStages3) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc::mma_commit_w(&bars->acc_full[a]);
                if (++a == 2) {
                    a = 0;
                    aph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->gempty);
        });
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmXb);
            int s = 0;
            uint32_t ph = 0;
            for_segments([&](int tile, int rlo, int rhi) {
                for (int rc = rlo; rc < rhi; ++rc) {
                    // when the ring holds only one box per epilogue group (b = 256), pull the
                    // next row chunk's boxes into L2 a chunk ahead, so a freed stage is refilled
                    // at L2 rather than HBM latency (deeper rings do not need it: measured)
                    if (nxs <= 4 && rc + 1 < nrc) {
                        for (int cb = 0; cb < kTileCols / kXBoxCols; ++cb)
                            tc::tma_prefetch_2d(&tmXb, (rc + 1) * kRowChunk,
                                                tile * kTileCols + cb * kXBoxCols);
                    }
                    for (int cb = 0; cb < kTileCols / kXBoxCols; ++cb) {
                        const unsigned long long t0 = clock64();
                        mbar_wait(&bars->xempty[s], ph ^ 1u);
                        w_a += clock64() - t0;
                        mbar_arrive_expect_tx(&bars->xfull[s], static_cast<uint32_t>(kXBoxBytes));
                        tc::tma_load_2d(Xs(s), &tmXb, rc * kRowChunk,
                                        tile * kTileCols + cb * kXBoxCols, &bars->xfull[s]);
                        if (++s == nxs) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp >= 4) {
        // 16 epilogue warps: 4 groups of 4 (one warp per TMEM lane quarter); group g takes
        // the boxes with index = g (mod 4) -- nxs is a multiple of 4, so every ring stage
        // has exactly one consumer group
        const int q = warp & 3, grp = (warp - 4) >> 2;
        const int r_in = q * 32 + lane;
        int a = 0;
        uint32_t aph = 0;
        constexpr int kBoxes = kTileCols / kXBoxCols;   // X boxes per r-chunk
        static_assert(kBoxes % 4 == 0, "one consumer group per stage (nxs % 4 == 0)");
        int64_t seq = 0;   // position in the X box ring (both groups follow it)
        const bool lag = nxs >= 8;
        int pend = -1;     // storer: the box whose release waits for the next store
        for_segments([&](int tile, int rlo, int rhi) {
            for (int rc = rlo; rc < rhi; ++rc, seq += kBoxes) {
                // NEXT-f2: below row rc0*128 the block's V rows are zero, no MMA ran: those
                // rows are copied (scaled) when the pass is out of place
                const bool mma_rc = rc >= rc0;
                const int r = rc * kRowChunk + r_in;
                // pre-scale of X (Lambda for the symmetric block, D for a right factor D)
                // and post-scale of the result (a left factor D, NEXT-f1): loaded before the
                // accumulator wait so that their latency hides behind it
                const float lr = (lam && r < n) ? __ldg(lam + r) : 1.f;
                const float pr = (post && r < n) ? __ldg(post + r) : 1.f;
                if (mma_rc) {
                    const unsigned long long t0 = clock64();
                    mbar_wait(&bars->acc_full[a], aph);
                    w_a += clock64() - t0;
                    tc::fence_after_sync();
                }
#pragma unroll
                for (int k = 0; k < kBoxes / 4; ++k) {
                    const int cb = grp + 4 * k;
                    const int64_t sq = seq + cb;
                    const int s = static_cast<int>(sq % nxs);
                    const unsigned long long t0 = clock64();
                    mbar_wait(&bars->xfull[s], static_cast<uint32_t>((sq / nxs) & 1));
                    w_b += clock64() - t0;
                    // this thread's row of the box: X[j0 + e][r] at xs + (e * 128 + r_in) * 4;
                    // Y overwrites X in the box and one TMA store writes the box back (rows
                    // >= n and columns >= N are clipped by the tensor map)
                    const uint32_t xs = smem_u32(Xs(s)) + static_cast<uint32_t>(r_in) * 4u;
                    float v[16];
                    if (mma_rc) {
                        tc::tmem_ld16(tbase + (static_cast<uint32_t>(q * 32) << 16) +
                                          static_cast<uint32_t>(a * kTileCols + cb * kXBoxCols),
                                      v);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    }
#pragma unroll
                    for (int e = 0; e < kXBoxCols; ++e) {
                        const uint32_t ad = xs + e * kRowChunk * 4;
                        sts_f32(ad, pr * fmaf(lr, lds_f32(ad), -v[e]));
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + grp, 128);
                    if (q == 0 && lane == 0) {
                        tc::tma_store_2d(&tmYs, Xs(s), rc * kRowChunk, tile * kTileCols + cb * kXBoxCols);
                        tc::bulk_commit();
                        // a box may be refilled once TMA has read it; with >= 8 stages the
                        // storer releases the PREVIOUS box instead of waiting for this one
                        // (the read of this box overlaps the group's next box): same-box A/B
                        // C3 / C5 h=64 -0.8 / -1 %
                        if (lag) {
                            tc::bulk_wait_read1();
                            if (pend >= 0) tc::mbar_arrive(&bars->xempty[pend]);
                            pend = s;
                        } else {
                            tc::bulk_wait_read0();
                            tc::mbar_arrive(&bars->xempty[s]);
                        }
                    }
                }
                if (mma_rc) {
                    tc::fence_before_sync();
                    tc::mbar_arrive(&bars->acc_empty[a]);
                    if (++a == 2) {
                        a = 0;
                        aph ^= 1u;
                    }
                }
            }
        });
    }
    if (warp >= 4 && (warp & 3) == 0 && lane == 0) tc::bulk_wait0();
    if (dbg && lane == 0) {
        // [0] kernel cycles  [1,2] V producer: empty waits  [3,4] MMA: full waits, acc_empty
        // waits  [5,6] X producer: xempty waits  [7,8] epilogue warp 4: acc_full, xfull waits
        const unsigned long long tot = clock64() - t_k0;
        if (warp == 0) { tl[0] = tot; tl[1] = w_a; }
        if (warp == 1) { tl[3] = w_a; tl[4] = w_b; }
        if (warp == 2) { tl[5] = w_a; }
        if (warp == 4) { tl[7] = w_a; tl[8] = w_b; }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_free<256>(tbase);
}

// ------------------------------------------------------------------ K5b-TS: X <- X - V G
// The update with G as the TMEM-resident A operand (tcgen05.mma A from TMEM, B = V tiles
// from shared memory): D'[j][r] = sum_i G[j][i] V[r][i], TMEM lane = column j, TMEM column
// = row r of the current 128-row chunk.  Moving G (128 KB at b = 256) out of shared memory
// leaves room for a 4-deep V ring and an 8-deep ring of X boxes (32 rows x 128 columns,
// SWIZZLE_128B), which the b = 256 update needs (one box per group had exposed every X
// load latency).  Shared-memory traffic per SM is still the bound at b = 256 (V operand
// reads and TMA writes, X box write/read/write/store-read); reading X straight from global
// memory instead was measured 30 % slower (uncoalesced per-column accesses).  TMEM: G hi at columns [0, 128), G lo at [128, 256), two accumulators of
// 128 columns at 256 and 384.  20 warps: w0 V producer, w1 MMA (warp-wide issue), w2 X-box
// producer, w4-19 epilogue = 4 lane quarters (32 columns) x 4 row groups (32 rows of the
// chunk); the epilogue warps also stage each tile's G (global -> registers -> tcgen05.st).
constexpr int kVS2 = 6;              // K5b-TS V ring depth (V arrives from L2; the TS timeline
                                     // showed the MMA waiting 43 % on a 4-deep ring)
constexpr int kXS2 = 8;              // K5b-TS X box ring depth (2 per row group)
constexpr int kXB2Bytes = 16384;     // X box: 32 rows x 128 columns fp32 (rows of 128 B)

struct Bars4 {
    uint64_t gfull, gempty;
    uint64_t full[kVS2], empty[kVS2];
    uint64_t xfull[kXS2], xempty[kXS2];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem;
};

size_t smem4() { return 1024 + static_cast<size_t>(kVS2) * kStage3Bytes + kXS2 * kXB2Bytes + sizeof(Bars4); }

__global__ void __launch_bounds__(640, 1)
    wy_update_ts_kernel(const uint16_t *__restrict__ Gt, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmXb,
                        const __grid_constant__ CUtensorMap tmYs, const float *__restrict__ lam,
                        const float *__restrict__ post, int n, int n_pad, int64_t N, int b,
                        int vrow_hi, int vrow_lo, int ntiles, int rc0, int copy_below,
                        unsigned long long *tl) {
    const bool dbg = tl != nullptr && blockIdx.x == 0;
    unsigned long long t_k0 = clock64(), w_a = 0, w_b = 0, w_c = 0;
    auto tw = [&](uint64_t *bar, uint32_t ph, unsigned long long &acc) {
        const unsigned long long t0 = clock64();
        mbar_wait(bar, ph);
        acc += clock64() - t0;
    };
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int nslab = b / 32;
    unsigned char *stg = smem;
    unsigned char *xst = stg + kVS2 * kStage3Bytes;
    Bars4 *bars = reinterpret_cast<Bars4 *>(xst + kXS2 * kXB2Bytes);
    auto Vhi = [&](int s) { return stg + s * kStage3Bytes; };
    auto Vlo = [&](int s) { return stg + s * kStage3Bytes + 8192; };
    auto Xs = [&](int s) { return xst + s * kXB2Bytes; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nrc = n_pad / kRowChunk;
    const int xrc0 = copy_below ? 0 : rc0;
    const int64_t per = nrc - xrc0;
    const int64_t utot = static_cast<int64_t>(ntiles) * per;
    const int64_t ubeg = utot * blockIdx.x / gridDim.x, uend = utot * (blockIdx.x + 1) / gridDim.x;
    auto for_segments = [&](auto &&fn) {
        for (int64_t u = ubeg; u < uend;) {
            const int tile = static_cast<int>(u / per);
            const int64_t t0 = static_cast<int64_t>(tile) * per;
            const int rlo = xrc0 + static_cast<int>(u - t0);
            const int rhi = xrc0 + static_cast<int>(uend - t0 < per ? uend - t0 : per);
            fn(tile, rlo, rhi);
            u = t0 + per;
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars->gfull, 512);
        mbar_init(&bars->gempty, 1);
        for (int s = 0; s < kVS2; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int s = 0; s < kXS2; ++s) {
            mbar_init(&bars->xfull[s], 1);
            mbar_init(&bars->xempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 512);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<512>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;
    pdl_wait();   // the previous kernel's results (after this CTA's setup)
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmV);
            int s = 0;
            uint32_t ph = 0;
            for_segments([&](int, int rlo, int rhi) {
                const int mlo = rlo > rc0 ? rlo : rc0;
                for (int rc = mlo; rc < rhi; ++rc) {
                    for (int c = 0; c < nslab; ++c) {
                        tw(&bars->empty[s], ph ^ 1u, w_a);
                        mbar_arrive_expect_tx(&bars->full[s], static_cast<uint32_t>(kStage3Bytes));
                        tc::tma_load_2d(Vhi(s), &tmV, c * 32, vrow_hi + rc * kRowChunk, &bars->full[s]);
                        tc::tma_load_2d(Vlo(s), &tmV, c * 32, vrow_lo + rc * kRowChunk, &bars->full[s]);
                        if (++s == kVS2) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp == 1) {
        const uint32_t idesc = tc::idesc_bf16(kTileCols, kRowChunk);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0, gph = 0;
        for_segments([&](int, int rlo, int rhi) {
            const int mlo = rlo > rc0 ? rlo : rc0;
            if (mlo >= rhi) return;
            tw(&bars->gfull, gph, w_c);   // this tile's G is in TMEM
            gph ^= 1u;
            tc::fence_after_sync();
            for (int rc = mlo; rc < rhi; ++rc) {
                tw(&bars->acc_empty[a], aph ^ 1u, w_b);
                tc::fence_after_sync();
                const uint32_t d = tbase + 256u + static_cast<uint32_t>(a * kRowChunk);
                for (int c = 0; c < nslab; ++c) {
                    tw(&bars->full[s], ph, w_a);
                    tc::fence_after_sync();
                    const uint32_t vh = smem_u32(Vhi(s)), vl = smem_u32(Vlo(s));
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint64_t bh = tc::sdesc_sw64(vh + kk * 32), bl = tc::sdesc_sw64(vl + kk * 32);
                        const uint32_t ah = tbase + static_cast<uint32_t>(c * 16 + kk * 8);
                        const uint32_t alo = ah + 128u;
                        tc::mma_bf16_ts_w(d, ah, bh, idesc, (c | kk) != 0);
                        tc::mma_bf16_ts_w(d, ah, bl, idesc, 1u);
                        tc::mma_bf16_ts_w(d, alo, bh, idesc, 1u);
                    }
                    tc::mma_commit_w(&bars->empty[s]);
                    if (++s == kVS2) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                tc::mma_commit_w(&bars->acc_full[a]);
                if (++a == 2) {
                    a = 0;
                    aph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->gempty);   // G may be replaced once these MMAs finish
        });
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmXb);
            int s = 0;
            uint32_t ph = 0;
            for_segments([&](int tile, int rlo, int rhi) {
                for (int rc = rlo; rc < rhi; ++rc) {
                    for (int g = 0; g < 4; ++g) {
                        tw(&bars->xempty[s], ph ^ 1u, w_a);
                        mbar_arrive_expect_tx(&bars->xfull[s], static_cast<uint32_t>(kXB2Bytes));
                        tc::tma_load_2d(Xs(s), &tmXb, rc * kRowChunk + g * 32, tile * kTileCols,
                                        &bars->xfull[s]);
                        if (++s == kXS2) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            });
        }
    } else if (warp >= 4) {
        const int q = warp & 3, g = (warp - 4) >> 2;
        const int j = q * 32 + lane;                    // column within the tile (TMEM lane)
        const uint32_t tlane = static_cast<uint32_t>(q * 32) << 16;
        const uint16_t *Glo_g = Gt + N * b;
        int a = 0;
        uint32_t aph = 0, gph = 0;
        int64_t seq = 0;
        for_segments([&](int tile, int rlo, int rhi) {
            const int mlo = rlo > rc0 ? rlo : rc0;
            if (warp == 4 && lane == 0) {
                // pull the next tile's G rows (hi and lo, contiguous) into L2 while this
                // segment runs, so its staging at the next tile boundary hits L2
                const int64_t nt = static_cast<int64_t>(tile) + 1;
                if (nt < ntiles) {
                    const int64_t cols = N - nt * kTileCols < kTileCols ? N - nt * kTileCols : kTileCols;
                    const uint32_t bytes = static_cast<uint32_t>(cols * b * 2) & ~15u;
                    if (bytes) {
                        tc::bulk_prefetch_l2(Gt + nt * kTileCols * b, bytes);
                        tc::bulk_prefetch_l2(Glo_g + nt * kTileCols * b, bytes);
                    }
                }
            }
            if (mlo < rhi) {
                // stage this tile's G (columns = TMEM lanes) once the previous tile's MMAs
                // are done with it; the four row groups split each column's [hi | lo] words
                // and issue all their loads before the TMEM stores (one L2 round trip)
                tw(&bars->gempty, gph ^ 1u, w_c);
                gph ^= 1u;
                tc::fence_after_sync();
                const int64_t jg = static_cast<int64_t>(tile) * kTileCols + j;
                const int wq = b / 4;                       // words per group (multiple of 8)
                const int half = g >> 1;                    // groups 0,1: hi; 2,3: lo
                const int w0 = (g & 1) * wq;                // first word within the half
                const uint4 *src = reinterpret_cast<const uint4 *>((half ? Glo_g : Gt) + jg * b) + w0 / 4;
                uint4 u[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    u[i] = make_uint4(0u, 0u, 0u, 0u);
                    if (i < wq / 4 && jg < N) u[i] = __ldg(src + i);
                }
#pragma unroll
                for (int i = 0; i < 16; i += 2)
                    if (i < wq / 4)
                        tc::tmem_st8(tbase + tlane + static_cast<uint32_t>(half * 128 + w0 + 4 * i), u[i], u[i + 1]);
                tc::tmem_wait_st();
                tc::fence_before_sync();
                tc::mbar_arrive(&bars->gfull);
            }
            for (int rc = rlo; rc < rhi; ++rc, seq += 4) {
                const bool mma_rc = rc >= rc0;
                float v[32];
                if (mma_rc) {
                    tw(&bars->acc_full[a], aph, w_a);
                    tc::fence_after_sync();
                    tc::tmem_ld32(tbase + tlane + 256u + static_cast<uint32_t>(a * kRowChunk + g * 32), v);
                    tc::fence_before_sync();
                    tc::mbar_arrive(&bars->acc_empty[a]);
                    if (++a == 2) {
                        a = 0;
                        aph ^= 1u;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
                const int r0 = rc * kRowChunk + g * 32;
                const int64_t sq = seq + g;
                const int s = static_cast<int>(sq % kXS2);
                tw(&bars->xfull[s], static_cast<uint32_t>((sq / kXS2) & 1), w_b);
                const uint32_t xs = smem_u32(Xs(s)) + static_cast<uint32_t>(j) * 128u;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t ad = xs + static_cast<uint32_t>((c ^ (j & 7)) << 4);
                    float4 x4 = tc::lds128(ad);
                    float lr[4] = {1.f, 1.f, 1.f, 1.f}, pr[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int r = r0 + 4 * c + e;
                        if (lam && r < n) lr[e] = __ldg(lam + r);
                        if (post && r < n) pr[e] = __ldg(post + r);
                    }
                    x4.x = pr[0] * fmaf(lr[0], x4.x, -v[4 * c]);
                    x4.y = pr[1] * fmaf(lr[1], x4.y, -v[4 * c + 1]);
                    x4.z = pr[2] * fmaf(lr[2], x4.z, -v[4 * c + 2]);
                    x4.w = pr[3] * fmaf(lr[3], x4.w, -v[4 * c + 3]);
                    tc::sts128(ad, x4);
                }
                fence_proxy_async_smem();
                named_bar_sync(1 + g, 128);
                if (q == 0 && lane == 0) {
                    tc::tma_store_2d(&tmYs, Xs(s), r0, tile * kTileCols);
                    tc::bulk_commit();
                    // (releasing the previous box instead, as the SS update does, was
                    // measured 2-3 % slower here at b = 256 / 1024)
                    tc::bulk_wait_read0();
                    tc::mbar_arrive(&bars->xempty[s]);
                }
            }
        });
        if (q == 0 && lane == 0) tc::bulk_wait0();
    }
    if (dbg && lane == 0) {
        // [0] kernel  [1] V prod empty  [3] MMA full (V)  [4] MMA acc_empty  [9] MMA gfull
        // [5] X prod xempty  [7] epi(w4) acc_full  [8] epi xfull  [10] epi gempty
        const unsigned long long tot = clock64() - t_k0;
        if (warp == 0) { tl[0] = tot; tl[1] = w_a; }
        if (warp == 1) { tl[3] = w_a; tl[4] = w_b; tl[9] = w_c; }
        if (warp == 2) { tl[5] = w_a; }
        if (warp == 4) { tl[7] = w_a; tl[8] = w_b; tl[10] = w_c; }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_free<512>(tbase);
}

#include "hh_wy_flow.cuh"

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    std::call_once(g_encode_once, []() {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    return g_encode;
}

bool make_map(CUtensorMap *m, CUtensorMapDataType dt, int esize, const void *base, uint64_t inner,
              uint64_t outer, uint32_t box_in, uint32_t box_out, CUtensorMapSwizzle sw) {
    auto enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * static_cast<uint64_t>(esize)};
    cuuint32_t box[2] = {box_in, box_out};
    cuuint32_t es[2] = {1, 1};
    return enc(m, dt, 2, const_cast<void *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t tbuild_smem(int b) {
    return (static_cast<size_t>((b * (b + 1) / 2 + 31) / 32 * 32) + 8 * 32 * 33 + 224 * 32 + 32 * 32) *
           4;
}

int nraw_for(int b, bool tsa = false) {
    const int cvb = (tsa ? 0 : 16384) + 128 * b;
    const int r = (kSmemMax - 1024 - static_cast<int>(sizeof(Bars1)) - kStages1 * cvb) / kRawBytes;
    return std::max(2, std::min(kRaw1, r));
}
size_t smem1(int b, bool tsa = false) {
    return static_cast<size_t>(nraw_for(b, tsa)) * kRawBytes +
           static_cast<size_t>(kStages1) * ((tsa ? 0 : 16384) + 128 * b) + sizeof(Bars1) + 1024;
}
int nxs_for(int kv) {
    const int g = (kv / 32) * 16384;
    int x = (kSmemMax - 1024 - static_cast<int>(sizeof(Bars3)) - g - kStages3 * kStage3Bytes) /
            kXBoxBytes;
    x = std::min(kXStages, x) & ~3;   // a multiple of the 4 epilogue groups
    return std::max(4, x);
}
size_t smem3(int kv) {
    return static_cast<size_t>(kv / 32) * 16384 + static_cast<size_t>(kStages3) * kStage3Bytes +
           static_cast<size_t>(nxs_for(kv)) * kXBoxBytes + sizeof(Bars3) + 1024;
}

// per-device opt-in of the large dynamic shared memory (the attribute belongs to each
// device's context): one flag and result per device
constexpr int kMaxDevWy = 64;
std::once_flag g_attr_once[kMaxDevWy];
cudaError_t g_attr_err[kMaxDevWy];
// debug / test hooks, per calling thread (like hh_set_algo): no process-global mutable state
thread_local unsigned long long *t_timeline = nullptr;   // hh_debug_wy_timeline
thread_local int t_ts_min = 256;                         // hh_debug_wy_ts_min
thread_local int t_tsa = 1;   // hh_debug_wy_tsa: K5a converts X into TMEM (b <= 128); same-box A/B
                              // (tools/wy_tsa_ab.py): bit-identical, C3 -2 % min / -6 % median, C5 h=64 -1 / -2 %
thread_local int t_symfuse = 3;   // hh_debug_wy_symfuse: bit 0 the folded block's operands in one
                                  // launch, bit 1 S and P in one Gram + one reduction launch
// K5f knobs (hh_debug_wy_flow*): on/off, project CTAs, K chunks per tile, row chunks per
// update entry, L2 window (tiles), tiles per wavefront group, L2 policy bits; 0 = default
struct FlowKnobs {
    int on = 0, P = 0, nkc = 0, rseg = 0, D = 0, G = 0, pol = 3;   // K5f measured slower: opt-in
};
thread_local FlowKnobs t_fk;

// K5f shape: K chunks per tile (project units), tiles per wavefront group G, L2 window D
void flow_shape(int64_t n, int kw, int np, int64_t ntiles, int *nkc, int *D, int *G) {
    const int nk = static_cast<int>((n + 31) / 32);
    const int target = kw >= 256 ? 32 : 16;               // K steps per project unit
    *nkc = t_fk.nkc > 0 ? t_fk.nkc : std::max(1, std::min(8, (nk + target / 2) / target));
    *G = t_fk.G > 0 ? t_fk.G : (np > 1 ? 4 : 1);
    const int64_t tile_bytes = static_cast<int64_t>(kTileCols) * n * 4;
    const int64_t w = t_fk.D > 0 ? t_fk.D
                                 : std::max<int64_t>(8, std::min<int64_t>(64, (int64_t(40) << 20) / tile_bytes));
    // deadlock freedom needs the window to span np wavefront groups (hh_wy_flow.cuh)
    *D = static_cast<int>(std::max<int64_t>(static_cast<int64_t>(np) * *G,
                                            std::min<int64_t>(w, std::max<int64_t>(ntiles, 1))));
}
}  // namespace

void wy_set_timeline(unsigned long long *buf) { t_timeline = buf; }

// TS-mode update from this block width on (default 256; the test hook hh_debug_wy_ts_min
// lowers it for the calling thread)
int wy_set_ts_min(int kw) {
    const int prev = t_ts_min;
    t_ts_min = kw;
    return prev;
}

int wy_set_flow(int on, int project_ctas) {
    const int prev = t_fk.on;
    t_fk.on = on;
    t_fk.P = project_ctas;
    return prev;
}

void wy_set_flow_knobs(const int *k, int cnt) {
    FlowKnobs f;
    int *dst[7] = {&f.on, &f.P, &f.nkc, &f.rseg, &f.D, &f.G, &f.pol};
    for (int i = 0; i < cnt && i < 7; ++i) *dst[i] = k[i];
    t_fk = f;
}

WyPlan wy_plan(int kind, int64_t n, int64_t h, int64_t N) {
    WyPlan p{};
    p.kind = kind;
    p.n = n;
    p.h = h;
    p.N = N;
    const int64_t bmax = kind == WY_SYM ? 128 : 256;   // MMA N of the project pass <= 256
    p.nblk = static_cast<int>(std::max<int64_t>(1, (h + bmax - 1) / bmax));
    const int64_t per = (h + p.nblk - 1) / p.nblk;
    p.b = static_cast<int>(std::max<int64_t>(32, (per + 31) / 32 * 32));
    p.h_pad = p.b * p.nblk;
    p.extra = kind == WY_SYM ? p.b : 0;
    p.n_pad = (n + kRowChunk - 1) / kRowChunk * kRowChunk;
    // Gram split-K slices: 32 rows for small blocks (enough CTAs to fill the GPU), else 128
    p.gram_rows = p.b <= 64 ? 32 : kGramRows;
    p.nsplit = static_cast<int>(p.n_pad / p.gram_rows);
    const size_t bb = static_cast<size_t>(p.b) * p.b * 4;
    const size_t vblk = static_cast<size_t>(p.n_pad) * p.b * 2 * 2;   // bf16 hi/lo per block
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += al(bytes);
        return o;
    };
    p.off_wf = take(static_cast<size_t>(p.h_pad) * p.n_pad * 4);
    p.off_wb = take(static_cast<size_t>(p.h_pad + p.extra) * p.n_pad * 2 * 2);
    p.off_sp = take(static_cast<size_t>(p.nblk) * p.nsplit * bb);
    p.off_s = take(p.nblk * bb);
    p.off_t = take(p.nblk * bb);
    p.off_v = take(p.nblk * vblk);                                      // Vn (N) or Vt (T)
    if (kind == WY_SYM) {
        p.off_v2 = take(p.nblk * vblk);                                 // Vn next to Vt
        p.off_asym = take(static_cast<size_t>(p.n_pad) * 2 * p.b * 2 * 2);
        p.off_vf = take(static_cast<size_t>(p.n_pad) * p.b * 4);
        p.off_vpf = take(static_cast<size_t>(p.n_pad) * p.b * 4);
        p.off_pp = take(static_cast<size_t>(p.nsplit) * bb);
        p.off_p = take(bb);
        p.off_m = take(bb);
        p.off_ld = take(static_cast<size_t>(n) * 4);
    }
    const int kmax = kind == WY_SYM ? 2 * p.b : p.b;
    p.off_gt = take(static_cast<size_t>(std::max<int64_t>(N, 1)) * kmax * 2 * 2);
    // K5a split-tile hand-off: a slot pair (leading / trailing partial) per CTA boundary
    const int64_t ntl = (N + kTileCols - 1) / kTileCols;
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>({ntl, device_attr().sm_count, kSlots1}));
    p.off_part = take(static_cast<size_t>(2 * pairs) * kTileCols * kmax * 4);
    p.off_flag = take(static_cast<size_t>(kSlots1) * 4);
    // K5f regions
    p.np = kind == WY_SYM ? 2 * p.nblk - 1 : p.nblk;
    p.ntiles = static_cast<int>(ntl);
    p.fkw = kmax;
    flow_shape(n, kmax, p.np, ntl, &p.fnkc, &p.fD, &p.fG);
    p.off_ring = take(static_cast<size_t>(p.fD) * kTileCols * kmax * 2 * 2);
    p.off_fpart = p.fnkc > 1 ? take(static_cast<size_t>(p.fD) * p.fnkc * kTileCols * kmax * 4) : off;
    p.off_cnt = take(static_cast<size_t>(3) * p.np * std::max<int64_t>(ntl, 1) * 4);
    p.bytes = off;
    return p;
}

bool wy_supported(int kind, int64_t n, int64_t h, int64_t N) {
    // TMA coordinates are int32; G rows are addressed as 2N
    if (!(n >= 32 && n % 4 == 0 && h >= 1 && N >= 1 && 2 * N < (int64_t(1) << 31) &&
          n <= (int64_t(1) << 20)))
        return false;
    // the block program has at most kMaxPasses passes: m blocks (apply) or 2m - 1 (sym)
    const int64_t bmax = kind == WY_SYM ? 128 : 256;
    const int64_t m = (h + bmax - 1) / bmax;
    return (kind == WY_SYM ? 2 * m - 1 : m) <= kMaxPasses;
}

namespace {

struct Pass {
    int wrow;            // first W row of the project operand
    int kw;              // its row count (b, or 2b for the symmetric block)
    const CUtensorMap *mW, *mG, *mV;
    int vrow_hi, vrow_lo;
    bool lam;            // symmetric block: Lambda X in the update epilogue
    const float *dscale = nullptr;   // project D X (first pass, right factor D)
    const float *pre = nullptr;      // update pre-scale of X (Lambda, D, or Lambda D)
    const float *post = nullptr;     // update post-scale (last pass, left factor D)
    int row0 = 0;                    // NEXT-f2: first row where the block's W / V are nonzero
};

}  // namespace

namespace {
thread_local int t_pdl = 1;   // A/B hooks (hh_debug_wy_pdl): PDL launches, and
thread_local int t_overlap = 1;   // the preparation beside the first projection
// every kernel of the block program is launched with programmatic stream serialization (PDL):
// see pdl_trigger / pdl_wait
template <typename... K, typename... A>
cudaError_t launch_k(bool use_pdl, void (*kernel)(K...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, A &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (t_pdl && use_pdl) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}
template <typename... K, typename... A>
cudaError_t pdl_launch(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       A &&...args) {
    return launch_k(true, kernel, grid, block, smem, stream, std::forward<A>(args)...);
}
}  // namespace

int wy_set_tsa(int on) {
    const int prev = t_tsa;
    t_tsa = on;
    return prev;
}

int wy_set_symfuse(int on) {
    const int prev = t_symfuse;
    t_symfuse = on;
    return prev;
}

int wy_set_pdl(int on) {
    const int prev = t_pdl | (t_overlap << 1);
    t_pdl = on & 1;
    t_overlap = (on >> 1) & 1;
    return prev;
}

cudaError_t launch_wy(const WyPlan &p, const float *U, const float *lam, const float *X, float *Y,
                      void *ws, cudaStream_t stream, LaunchInfo *info, int debug_stop_blocks,
                      const float *dsign, int dside) {
    if (!encoder()) return cudaErrorNotSupported;
    if (!wy_supported(p.kind, p.n, p.h, p.N)) return cudaErrorNotSupported;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevWy) return cudaErrorInvalidDevice;
    std::call_once(g_attr_once[dev], [dev]() {
        cudaError_t &err = g_attr_err[dev];
        err = cudaFuncSetAttribute(wy_project_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemMax);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_project_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemMax);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_sym_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(symrows_smem(64)));
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_vrec_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(vrec_smem(256)));
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_vrec_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(vrec_smem(256)));
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_tbuild_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(tbuild_smem(256)));
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemMax);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_update_ts_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(wy_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemMax);

    });
    if (g_attr_err[dev] != cudaSuccess) return g_attr_err[dev];
    const bool sym = p.kind == WY_SYM;
    if (sym && !lam) return cudaErrorInvalidValue;
    int nlaunch = 0;   // kernels enqueued by this call (reported through LaunchInfo)
    cudaError_t lerr = cudaSuccess;   // the first launch error
    auto note = [&](cudaError_t le) {
        if (le != cudaSuccess && lerr == cudaSuccess) lerr = le;
    };
    char *w = static_cast<char *>(ws);
    auto F = [&](size_t o) { return reinterpret_cast<float *>(w + o); };
    auto H = [&](size_t o) { return reinterpret_cast<uint16_t *>(w + o); };
    float *Wf = F(p.off_wf), *Sp = F(p.off_sp), *S = F(p.off_s), *T = F(p.off_t);
    uint16_t *Wb = H(p.off_wb), *Gt = H(p.off_gt);
    const int sms = device_attr().sm_count;
    const int m = p.nblk, b = p.b;
    const int64_t n_pad = p.n_pad, R = p.h_pad + p.extra;
    const int64_t vlo = static_cast<int64_t>(m) * n_pad * b;           // lo offset in a V array

    // K5a hand-off counters start at zero (the second arrival resets its counter); done first
    // so that the kernels of the program follow each other directly (PDL)
    {
        const cudaError_t me = cudaMemsetAsync(w + p.off_flag, 0, static_cast<size_t>(kSlots1) * 4, stream);
        if (me != cudaSuccess) return me;
    }

    // ---------------- K4: pack (the projection's operand W) ...
    {
        const int64_t tot = R * n_pad;
        const int g = static_cast<int>(std::min<int64_t>((tot + 255) / 256, sms * 16));
        // Q^T X applies the reversed list as a Q X program (transposing a
        // product of symmetric reflectors reverses it); the symmetric program keeps the
        // natural order and uses T and T^T explicitly
        const int rev = p.kind == WY_APPLY_T ? 1 : 0;
        ++nlaunch, note(pdl_launch(wy_pack_kernel, g, 256, 0, stream, U, p.n, p.h, p.h_pad, n_pad, lam, m - 1, b,
                                                         p.extra, rev, Wf, Wb));
    }
    // ... and the rest of the preparation (Gram, T, V = W T, the symmetric block's operands),
    // which only the updates read.  gram_wait = 0: launched behind the first projection, on
    // the SMs that projection leaves free, so that it runs beside it.
    auto prep_rest = [&](int gram_wait) {
        const int tb = (b + 63) / 64;
        // (fused only when the preparation runs alone, i.e. before the first projection: beside
        // it -- multi-block programs -- the larger fused launches measured slower)
        if (sym && (t_symfuse & 2) && gram_wait) {
            // S (every block) and P = W^T Lambda W of the last block (full) in one Gram launch
            // and one reduction launch
            const int pz = m * p.nsplit;
            ++nlaunch, note(pdl_launch(wy_gram_kernel, dim3(tb, tb, pz + p.nsplit), 256, 0, stream, Wf, n_pad, b,
                                       p.nsplit, p.gram_rows, 0, nullptr, 0, Sp, gram_wait, pz, m - 1, lam,
                                       F(p.off_pp)));
            const int64_t ns = static_cast<int64_t>(m + 1) * b * b;
            ++nlaunch, note(pdl_launch(wy_gram_reduce_kernel, static_cast<int>(std::min<int64_t>((ns * 32 + 255) / 256, sms * 16)),
                                       256, 0, stream, Sp, b, m, p.nsplit, 0, S, ns >= 32768 ? 1 : 0,
                                       static_cast<const float *>(F(p.off_pp)), F(p.off_p)));
        } else {
        ++nlaunch, note(pdl_launch(wy_gram_kernel, dim3(tb, tb, m * p.nsplit), 256, 0, stream, Wf, n_pad, b, p.nsplit, p.gram_rows, 0,
                                   nullptr, 0, Sp, gram_wait, 0, 0, static_cast<const float *>(nullptr),
                                   static_cast<float *>(nullptr)));
        const int64_t ns = static_cast<int64_t>(m) * b * b;
        ++nlaunch, note(pdl_launch(wy_gram_reduce_kernel, static_cast<int>(std::min<int64_t>((ns * 32 + 255) / 256, sms * 16)),
                                256, 0, stream, Sp, b, m, p.nsplit, 0, S, ns >= 32768 ? 1 : 0,
                                static_cast<const float *>(nullptr), static_cast<float *>(nullptr)));
        if (sym) {   // P = W^T Lambda W of the last block (full)
            ++nlaunch, note(pdl_launch(wy_gram_kernel, dim3(tb, tb, p.nsplit), 256, 0, stream, Wf, n_pad, b, p.nsplit, p.gram_rows,
                                       m - 1, lam, 1, F(p.off_pp), 1, 0, 0, static_cast<const float *>(nullptr),
                                       static_cast<float *>(nullptr)));
            ++nlaunch, note(pdl_launch(wy_gram_reduce_kernel, std::max(1, std::min(sms * 16, (b * b * 32 + 255) / 256)), 256, 0, stream,
                F(p.off_pp), b, 1, p.nsplit, 1, F(p.off_p), b * b >= 32768 ? 1 : 0,
                static_cast<const float *>(nullptr), static_cast<float *>(nullptr)));
        }
        }
        ++nlaunch, note(pdl_launch(wy_tbuild_kernel, m, 256, tbuild_smem(b), stream, S, b, T, sym ? 0 : 1));
        if (!sym) {
            // V = W T per block, row-parallel from the diagonal T blocks (wy_vrec_kernel)
            // 32-row CTAs when 64-row ones would not fill one wave (one block of n = 4096:
            // 64 CTAs on 148 SMs; with 4 blocks the 64-row CTAs are faster: measured)
            if (static_cast<int64_t>(n_pad / 64) * m < sms)
                ++nlaunch, note(pdl_launch(wy_vrec_kernel<1>, dim3(static_cast<unsigned>(n_pad / 32), m), 256,
                                               vrec_smem(b), stream, Wf, S, T, n_pad, b, H(p.off_v), vlo));
            else
                ++nlaunch, note(pdl_launch(wy_vrec_kernel<2>, dim3(static_cast<unsigned>(n_pad / 64), m), 256,
                                               vrec_smem(b), stream, Wf, S, T, n_pad, b, H(p.off_v), vlo));
        }
        const dim3 gv(static_cast<unsigned>(n_pad / 64), b / 32);
        for (int k = 0; k < (sym ? m : 0); ++k) {
            const float *Wk = Wf + static_cast<int64_t>(k) * b * n_pad;
            const float *Tk = T + static_cast<int64_t>(k) * b * b;
            const bool last_sym = k == m - 1;
            // symmetric program: blocks k < m-1 need V = W T (Q_k) and V' = W T^T (Q_k^T)
            uint16_t *Vn = H(p.off_v2);
            uint16_t *Vt = H(p.off_v);
            if (!last_sym) {
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<true, false>, gv, 256, 0, stream, 
                    n_pad, Wk, n_pad, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, nullptr,
                    Vn + static_cast<int64_t>(k) * n_pad * b, b, vlo));
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<true, true>, gv, 256, 0, stream, 
                    n_pad, Wk, n_pad, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, nullptr,
                    Vt + static_cast<int64_t>(k) * n_pad * b, b, vlo));
            } else if (b <= 64 && (t_symfuse & 1) && gram_wait) {
                // the folded block's operands in one launch (wy_sym_rows_kernel)
                ++nlaunch, note(pdl_launch(wy_sym_rows_kernel, static_cast<int>(n_pad / kSymRows), 256,
                    symrows_smem(b), stream, Wk, Tk, F(p.off_p), lam, p.n, n_pad, b, H(p.off_asym),
                    n_pad * 2 * b));
            } else {
                // A2 = W T (bf16 into columns [b, 2b) of Asym, fp32 copy Vf); V' = W T^T;
                // M = P T^T; A1 = Lambda V' - V M (columns [0, b)).  DESIGN.md §4.
                uint16_t *As = H(p.off_asym);
                const int64_t alo = n_pad * 2 * b;
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<true, false>, gv, 256, 0, stream, 
                    n_pad, Wk, n_pad, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, F(p.off_vf),
                    nullptr, b, 0));
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<true, false>, gv, 256, 0, stream, 
                    n_pad, Wk, n_pad, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, nullptr, As + b,
                    2 * b, alo));
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<true, true>, gv, 256, 0, stream, 
                    n_pad, Wk, n_pad, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, F(p.off_vpf),
                    nullptr, b, 0));
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<false, true>, dim3((b + 63) / 64, b / 32), 256, 0, stream, 
                    b, F(p.off_p), b, Tk, b, b, nullptr, 0, nullptr, 0, 1.f, F(p.off_m), nullptr,
                    b, 0));
                ++nlaunch, note(pdl_launch(wy_rowgemm_kernel<false, false>, gv, 256, 0, stream, 
                    n_pad, F(p.off_vf), b, F(p.off_m), b, b, F(p.off_vpf), b, lam, p.n, -1.f,
                    nullptr, As, 2 * b, alo));
            }
        }
    };
    cudaError_t e = lerr != cudaSuccess ? lerr : cudaGetLastError();
    if (e != cudaSuccess) return e;

    // ---------------- tensor maps
    const int64_t N = p.N;
    CUtensorMap mWb, mW2b, mGb, mG2b, mV, mV2, mAs, mX, mY, mXb, mYb, mXb2, mYb2;
    bool ok = make_map(&mWb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wb, n_pad, 2 * R, 32, b,
                       CU_TENSOR_MAP_SWIZZLE_64B) &&
              make_map(&mGb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Gt, b, 2 * N, 32, kTileCols,
                       CU_TENSOR_MAP_SWIZZLE_64B) &&
              make_map(&mV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H(p.off_v), b, 2 * m * n_pad, 32,
                       kRowChunk, CU_TENSOR_MAP_SWIZZLE_64B) &&
              make_map(&mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, p.n, N, 32, kTileCols,
                       CU_TENSOR_MAP_SWIZZLE_NONE) &&
              make_map(&mXb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, p.n, N, kRowChunk, kXBoxCols,
                       CU_TENSOR_MAP_SWIZZLE_NONE) &&
              make_map(&mXb2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, p.n, N, 32, kTileCols,
                       CU_TENSOR_MAP_SWIZZLE_128B) &&
              (!Y || (make_map(&mY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Y, p.n, N, 32, kTileCols,
                               CU_TENSOR_MAP_SWIZZLE_NONE) &&
                      make_map(&mYb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Y, p.n, N, kRowChunk, kXBoxCols,
                               CU_TENSOR_MAP_SWIZZLE_NONE) &&
                      make_map(&mYb2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Y, p.n, N, 32, kTileCols,
                               CU_TENSOR_MAP_SWIZZLE_128B)));
    if (ok && sym)
        ok = make_map(&mW2b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wb, n_pad, 2 * R, 32, 2 * b,
                      CU_TENSOR_MAP_SWIZZLE_64B) &&
             make_map(&mG2b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Gt, 2 * b, 2 * N, 32, kTileCols,
                      CU_TENSOR_MAP_SWIZZLE_64B) &&
             make_map(&mV2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H(p.off_v2), b, 2 * m * n_pad,
                      32, kRowChunk, CU_TENSOR_MAP_SWIZZLE_64B) &&
             make_map(&mAs, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H(p.off_asym), 2 * b, 2 * n_pad,
                      32, kRowChunk, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!ok) return cudaErrorNotSupported;

    // ---------------- the block program
    std::vector<Pass> prog(static_cast<size_t>(sym ? 2 * m - 1 : m));   // <= kMaxPasses
    int np = 0;
    auto blockpass = [&](int k, const CUtensorMap *mv) {
        Pass ps{k * b, b, &mWb, &mGb, mv, static_cast<int>(k * n_pad),
                static_cast<int>((m + k) * n_pad), false};
        if (p.qr) {
            // first row where the block's W (and V) can be nonzero: u_i[r] = 0 for r < i;
            // on the reversed list (Q^T) position q holds reflector h-1-q
            int64_t r0q = static_cast<int64_t>(k) * b;
            if (p.kind == WY_APPLY_T)
                r0q = std::max<int64_t>(0, p.h - std::min<int64_t>(static_cast<int64_t>(k + 1) * b, p.h));
            ps.row0 = static_cast<int>(std::min<int64_t>(r0q, p.n - 1));
        }
        prog[np++] = ps;
    };
    if (p.kind == WY_APPLY_N || p.kind == WY_APPLY_T) {
        // Q X (or Q^T X = the reversed list's Q X): last block first
        for (int k = m - 1; k >= 0; --k) blockpass(k, &mV);
    } else {
        for (int k = 0; k < m - 1; ++k) blockpass(k, &mV);           // Q_k^T, k < m-1
        Pass ps{(m - 1) * b, 2 * b, &mW2b, &mG2b, &mAs, 0, static_cast<int>(n_pad), true};
        ps.pre = lam;
        prog[np++] = ps;
        for (int k = m - 2; k >= 0; --k) blockpass(k, &mV2);         // Q_k, k < m-1
    }

    // NEXT-f1: the diagonal D as a prologue of the first pass (right factor) and an
    // epilogue of the last pass (left factor); no extra pass over X.
    if (dsign && (dside & 1)) {
        Pass &f = prog[0];
        f.dscale = dsign;
        if (f.pre) {   // first pass is the symmetric block: pre-scale Lambda D
            float *ld = F(p.off_ld);
            ++nlaunch, note(pdl_launch(wy_vmul_kernel, std::max(1, static_cast<int>((p.n + 255) / 256)), 256, 0, stream, 
                f.pre, dsign, p.n, ld));
            f.pre = ld;
        } else {
            f.pre = dsign;
        }
    }
    if (dsign && (dside & 2)) prog[np - 1].post = dsign;

    const int ntiles = static_cast<int>((N + kTileCols - 1) / kTileCols);

    // ---------------- K5f: the whole program as one dataflow launch (hh_wy_flow.cuh) when
    // every pass updates in the same mode (SS: G in shared memory, or TS: G in TMEM)
    bool ss_all = true, ts_all = true;
    for (int q = 0; q < np; ++q) {
        if (prog[q].kw >= t_ts_min) ss_all = false;
        else ts_all = false;
    }
    if (t_fk.on && debug_stop_blocks < 0 && Y && sms >= 2 && (ss_all || ts_all) && np == p.np) {
        prep_rest(1);
        // ~10 KB of kernel parameters (maps + pass table): built on the heap, copied at launch
        std::unique_ptr<FlowArgs> fap(new (std::nothrow) FlowArgs());
        if (!fap) return cudaErrorMemoryAllocation;
        FlowArgs &fa = *fap;
        fa.mXp = mX;
        fa.mYp = mY;
        fa.mXu = ts_all ? mXb2 : mXb;
        fa.mYu = ts_all ? mYb2 : mYb;
        fa.mW[0] = mWb;
        fa.mW[1] = sym ? mW2b : mWb;
        fa.mV[0] = mV;
        fa.mV[1] = sym ? mAs : mV;
        fa.mV[2] = sym ? mV2 : mV;
        fa.ring = H(p.off_ring);
        fa.part = F(p.off_fpart);
        int *cnt = reinterpret_cast<int *>(w + p.off_cnt);
        const int64_t npt = static_cast<int64_t>(np) * ntiles;
        fa.gcount = cnt;
        fa.gready = cnt + npt;
        fa.udone = cnt + 2 * npt;
        fa.N = N;
        fa.n = static_cast<int>(p.n);
        fa.n_pad = static_cast<int>(n_pad);
        fa.np = np;
        fa.ntiles = ntiles;
        fa.D = p.fD;
        fa.nkc = p.fnkc;
        fa.rseg = t_fk.rseg > 0 ? t_fk.rseg : 4;
        fa.G = p.fG;
        fa.pol = t_fk.pol;
        fa.tl = t_timeline;
        fa.kwmax = p.fkw;
        fa.ts = ts_all ? 1 : 0;
        fa.nraw = nraw_for(p.fkw);
        fa.nxs = nxs_for(p.fkw);
        fa.sms = sms;
        fa.P = std::max(1, std::min(sms - 1, t_fk.P > 0 ? t_fk.P : sms / 2));
        const int nrc = static_cast<int>(n_pad / kRowChunk);
        for (int q = 0; q < np; ++q) {
            const Pass &ps = prog[q];
            FlowPass &f = fa.pass[q];
            f.wrow = ps.wrow;
            f.wrow_lo = static_cast<int>(R) + ps.wrow;
            f.kw = ps.kw;
            f.wmap = ps.mW == &mW2b ? 1 : 0;
            f.vmap = ps.mV == &mV ? 0 : (ps.mV == &mAs ? 1 : 2);
            f.vrow_hi = ps.vrow_hi;
            f.vrow_lo = ps.vrow_lo;
            f.ks0 = ps.row0 / 32;
            f.rc0 = ps.row0 / kRowChunk;
            // out of place, the first pass copies the rows a QR block does not touch
            const bool copy_below = q == 0 && X != Y && ps.row0 >= kRowChunk;
            f.xrc0 = copy_below ? 0 : f.rc0;
            f.target = (nrc - f.xrc0) * 4;
            f.dscale = ps.dscale;
            f.pre = ps.pre;
            f.post = ps.post;
        }
        if (!make_map(&fa.mG, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, fa.ring, p.fkw,
                      static_cast<uint64_t>(2) * p.fD * kTileCols, 32, kTileCols,
                      CU_TENSOR_MAP_SWIZZLE_64B))
            return cudaErrorNotSupported;
        e = cudaMemsetAsync(cnt, 0, static_cast<size_t>(3 * npt) * 4, stream);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(sms));
        cfg.blockDim = dim3(640);
        cfg.dynamicSmemBytes = kSmemMax;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: waits always resolve
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        ++nlaunch;
        e = cudaLaunchKernelEx(&cfg, wy_flow_kernel, fa);
        if (info) {
            info->variant = sym ? "wy_sym_flow_bf16x3_tcgen05" : "wy_flow_bf16x3_tcgen05";
            info->grid = sms;
            info->block = 640;
            info->smem = kSmemMax;
            info->nchunks = np;
            info->launches = nlaunch;
        }
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }

    // The first projection needs only the packed W: the rest of the preparation (Gram, T, V)
    // is launched behind it without waiting for it and runs on the kPrepSms SMs it leaves
    // free; the first update is a plain launch (it waits for both), later passes chain by PDL.
    constexpr int kPrepSms = 8;
    const int grid_all = std::max(1, std::min(std::min(ntiles, sms), kSlots1));
    // (same box, tools/prep_ab.py: -4 % at h = 1024 (4 blocks), -1 % at h = 256; +0.4-0.5 % on
    // the one-block b <= 64 programs C3 / C5 h=64, whose short preparation does not pay for the
    // projection's 8 SMs)
    const bool overlap = t_overlap != 0 && (m > 1 || b >= 128);
    if (!overlap) prep_rest(1);
    const int grid_first =
        overlap ? std::max(1, std::min(grid_all, sms > 4 * kPrepSms ? sms - kPrepSms : sms)) : grid_all;
    const float *cur = X;
    for (int q = 0; q < np; ++q) {
        const Pass &ps = prog[q];
        // K5a with X converted into TMEM (b <= 128) reads the raw tiles through the
        // SWIZZLE_128B map of the same box; the shared-memory form otherwise
        const bool tsa = (ps.kw <= 128 && (t_tsa & 1)) || (ps.kw == 256 && (t_tsa & 2));
        const CUtensorMap &mcur = tsa ? ((cur == X) ? mXb2 : mYb2) : ((cur == X) ? mX : mY);
        auto k5a = tsa ? wy_project_kernel<true> : wy_project_kernel<false>;
        ++nlaunch, note(pdl_launch(k5a, q == 0 ? grid_first : grid_all, 480, smem1(ps.kw, tsa), stream,
            mcur, *ps.mW, Gt, static_cast<int>(p.n), N, ps.kw, ps.wrow, static_cast<int>(R) + ps.wrow,
            ntiles, ps.dscale, ps.row0 / 32, nraw_for(ps.kw, tsa), F(p.off_part),
            reinterpret_cast<int *>(w + p.off_flag)));
        if (q == 0 && overlap) prep_rest(0);
        if (debug_stop_blocks >= 0) break;   // test hook: stop after the first projection
        const int64_t uxrc = (cur != Y && ps.row0 >= kRowChunk) ? 0 : ps.row0 / kRowChunk;
        const int64_t units = static_cast<int64_t>(ntiles) * (n_pad / kRowChunk - uxrc);
        const int grid3 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, sms)));
        // TS-mode update (G in TMEM) for the wide blocks: the resident G no longer competes
        // with the V and X rings for shared memory
        if (ps.kw >= t_ts_min) {
            ++nlaunch, note(launch_k(q != 0 || !overlap, wy_update_ts_kernel, grid3, 640, smem4(), stream,
                Gt, *ps.mV, (cur == X) ? mXb2 : mYb2, mYb2, ps.pre, ps.post, static_cast<int>(p.n),
                static_cast<int>(n_pad), N, ps.kw, ps.vrow_hi, ps.vrow_lo, ntiles,
                ps.row0 / kRowChunk, (cur != Y && ps.row0 >= kRowChunk) ? 1 : 0, t_timeline));
            cur = Y;
            continue;
        }
        ++nlaunch, note(launch_k(q != 0 || !overlap, wy_update_kernel, grid3, 640, smem3(ps.kw), stream,
            *ps.mG, *ps.mV, (cur == X) ? mXb : mYb, mYb, Y, ps.pre, ps.post, static_cast<int>(p.n),
            static_cast<int>(n_pad), N, ps.kw, ps.vrow_hi, ps.vrow_lo, ntiles,
            ps.row0 / kRowChunk, (cur != Y && ps.row0 >= kRowChunk) ? 1 : 0, nxs_for(ps.kw),
            t_timeline));
        cur = Y;
    }
    if (info) {
        info->variant = sym ? "wy_sym_bf16x3_tcgen05" : "wy_bf16x3_tcgen05";
        info->grid = grid_all;
        info->block = 480;
        info->smem = static_cast<int>(smem1(b));
        info->nchunks = np;
        info->launches = nlaunch;
    }
    return lerr != cudaSuccess ? lerr : cudaGetLastError();
}

}  // namespace hh
