// hh_fused_kernel.cuh -- fused SIMT Householder-product kernel template for sm_100a
// (instantiated per dtype in hh_fused_f32.cu and hh_fused_f64.cu;
// launched by hh_fused.cu).
//
// K1 (apply Q X / Q^T X), K2 (Q diag(lambda) Q^T X), K3a (Mahalanobis
// transform-once Z = diag(sqrt d) Q^T P) and K3c (per-pair fused distance) are one
// kernel template with a run-time mode.  Each column costs h dot products
// alpha_i = u_i^T x and h rank-1 updates x <- x - 2 alpha_i u_i ("4nh
// operations"), applied in the order fixed by Q = H_1 ... H_h (reading R1).
//
// Data movement:
//   * U (n x h, column-major == (h, n)) is staged once per persistent CTA into
//     shared memory by 1-D bulk copies (TMA engine, UBLKCP).  When h*n*s does not
//     fit next to the column staging, U is streamed in chunks of R reflectors
//     through two shared buffers (mbarrier ring, one CTA barrier per chunk).
//   * X is processed in "tiles" of UC contiguous columns (one contiguous
//     UC*n*s-byte range).  Each unit (a warp, or a multi-warp group when one column
//     needs more than 32 threads) owns a one-tile shared staging slot: it copies
//     the landed tile into registers, then immediately issues the bulk copy of its
//     next tile, so the HBM read of tile t+1 overlaps the arithmetic of tile t.
//   * The column lives in registers for all h reflectors; the result is written
//     once with 128-bit coalesced stores.  HBM traffic = one read + one write of X.
//   * A group of TPC threads owns a column (vector chunk v = t + TPC*k of a thread);
//     dots are reduced by an xor-shuffle butterfly (plus a shared-memory stage when
//     TPC > 32), so every thread of the group holds the identical alpha.
#pragma once
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hh_internal.h"
#include "hh_ptx.cuh"
#include "hh_tc.cuh"

namespace hh {

template <typename T>
struct VT;
template <>
struct VT<float> {
    using V = float4;
    static constexpr int E = 4;
};
template <>
struct VT<double> {
    using V = double2;
    static constexpr int E = 2;
};

__device__ __forceinline__ void vzero(float4 &a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vzero(double2 &a) { a = make_double2(0.0, 0.0); }
// Packed fp32 FMA (sm_100 FFMA2): two IEEE round-to-nearest FMAs per instruction,
// bit-identical to two fmaf calls; halves the FMA issue slots of the hot loop.
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
    asm("{\n\t.reg .b64 A, B, C, D;\n\t"
        "mov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 C, {%6, %7};\n\t"
        "fma.rn.f32x2 D, A, B, C;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void vfma(float4 &acc, const float4 &u, const float4 &x) {
    ffma2(acc.x, acc.y, u.x, u.y, x.x, x.y, acc.x, acc.y);
    ffma2(acc.z, acc.w, u.z, u.w, x.z, x.w, acc.z, acc.w);
}
__device__ __forceinline__ void vfma(double2 &acc, const double2 &u, const double2 &x) {
    acc.x = fma(u.x, x.x, acc.x);
    acc.y = fma(u.y, x.y, acc.y);
}
__device__ __forceinline__ float vsum(const float4 &a) { return (a.x + a.y) + (a.z + a.w); }
// two IEEE fp32 adds in one instruction (FADD2): d = a + b elementwise
__device__ __forceinline__ void fadd2(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B, D;\n\t"
        "mov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\t"
        "add.rn.f32x2 D, A, B;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ double vsum(const double2 &a) { return a.x + a.y; }
// x <- x - s * u
__device__ __forceinline__ void vaxpy(float4 &x, float s, const float4 &u) {
    ffma2(x.x, x.y, -s, -s, u.x, u.y, x.x, x.y);
    ffma2(x.z, x.w, -s, -s, u.z, u.w, x.z, x.w);
}
__device__ __forceinline__ void vaxpy(double2 &x, double s, const double2 &u) {
    x.x = fma(-s, u.x, x.x);
    x.y = fma(-s, u.y, x.y);
}
__device__ __forceinline__ void vmul(float4 &x, const float4 &l) {
    x.x *= l.x;
    x.y *= l.y;
    x.z *= l.z;
    x.w *= l.w;
}
__device__ __forceinline__ void vmul(double2 &x, const double2 &l) {
    x.x *= l.x;
    x.y *= l.y;
}
// sqrt(d) by the hardware approximation (MUFU, within ~1 ulp): the correctly rounded
// sqrtf is a subroutine call per element, and K3a scales every element of every point
// (an ulp of sqrt(d) is 4 orders of magnitude below the fp32 parity gate)
__device__ __forceinline__ float sqrt_approx(float v) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ void vmulsqrt(float4 &x, const float4 &d) {
    x.x *= sqrt_approx(d.x);
    x.y *= sqrt_approx(d.y);
    x.z *= sqrt_approx(d.z);
    x.w *= sqrt_approx(d.w);
}
__device__ __forceinline__ void vmulsqrt(double2 &x, const double2 &d) {
    x.x *= sqrt(d.x);
    x.y *= sqrt(d.y);
}
__device__ __forceinline__ void vsub(float4 &a, const float4 &b) {
    a.x -= b.x;
    a.y -= b.y;
    a.z -= b.z;
    a.w -= b.w;
}
__device__ __forceinline__ void vsub(double2 &a, const double2 &b) {
    a.x -= b.x;
    a.y -= b.y;
}
// sum_e d_e * x_e^2
__device__ __forceinline__ float vwsq(const float4 &x, const float4 &d) {
    return (d.x * (x.x * x.x) + d.y * (x.y * x.y)) + (d.z * (x.z * x.z) + d.w * (x.w * x.w));
}
__device__ __forceinline__ double vwsq(const double2 &x, const double2 &d) {
    return d.x * (x.x * x.x) + d.y * (x.y * x.y);
}

// ---- scalar "vectors" (E = 1): the SC form of the kernel, for columns whose stride or base is
// not a multiple of 16 bytes (one element per access, lanes on consecutive elements)
__device__ __forceinline__ void vzero(float &a) { a = 0.f; }
__device__ __forceinline__ void vzero(double &a) { a = 0.0; }
__device__ __forceinline__ void vfma(float &acc, float u, float x) { acc = fmaf(u, x, acc); }
__device__ __forceinline__ void vfma(double &acc, double u, double x) { acc = fma(u, x, acc); }
__device__ __forceinline__ float vsum(float a) { return a; }
__device__ __forceinline__ double vsum(double a) { return a; }
__device__ __forceinline__ void vaxpy(float &x, float s, float u) { x = fmaf(-s, u, x); }
__device__ __forceinline__ void vaxpy(double &x, double s, double u) { x = fma(-s, u, x); }
__device__ __forceinline__ void vmul(float &x, float l) { x *= l; }
__device__ __forceinline__ void vmul(double &x, double l) { x *= l; }
__device__ __forceinline__ void vmulsqrt(float &x, float d) { x *= sqrt_approx(d); }
__device__ __forceinline__ void vmulsqrt(double &x, double d) { x *= sqrt(d); }
__device__ __forceinline__ void vsub(float &a, float b) { a -= b; }
__device__ __forceinline__ void vsub(double &a, double b) { a -= b; }
__device__ __forceinline__ float vwsq(float x, float d) { return d * (x * x); }
__device__ __forceinline__ double vwsq(double x, double d) { return d * (x * x); }
__device__ __forceinline__ void st_global_hint(float *p, const float &v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_global_hint(double *p, const double &v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

template <typename V>
__device__ __forceinline__ V ldg_v(const V *p) {
    return __ldg(p);
}

// TMEM-resident reflectors (K1t): this thread's NC consecutive 32-bit columns of its lane
// (warp: its lane quarter), 32x32b shape; NC = 8 / 16 / 32
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[NC]) {
    if constexpr (NC == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr)
                     : "memory");
    } else if constexpr (NC == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr)
            : "memory");
    } else {
        static_assert(NC == 32, "8, 16 or 32 columns");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
            "%28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr)
            : "memory");
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc_n(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_n(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
// ---------------------------------------------------------------------------------
// Kernel template
//   T   element type       TPC threads per column group      CH vector chunks / thread
//   C   columns per group   NT threads per CTA                FULL: nv == TPC*CH exactly
// ---------------------------------------------------------------------------------
// (NT <= 256: two CTAs per SM, so at most 128 registers -- pinned explicitly, ptxas's own
// choice drifts with unrelated code changes and halves the occupancy of the C2 kernel)
//
// UTM ("K1t", fp32, TPC dividing 128): the reflectors live in TMEM instead of shared memory.
// TMEM lane L holds the u chunks of group thread gt = L mod TPC (replicated over the lane
// quarters when TPC < 128, since a warp reads only its own quarter), reflector i at columns
// [4 CH i, 4 CH (i + 1)); each reflect() reads its 4 CH values with one tcgen05.ld.  The
// per-reflector u reads leave the shared-memory pipe (measured TMEM read rate 340+ B/clk/SM
// against 128 for ld.shared, tools/micro/tmem_ld_rate.cu), and shared memory is free for
// staging column tiles even when U is large (n = 4096, h = 12: 192 KB).
//
// KB > 1 ("K1w", with UTM): the reflectors are applied in blocks of KB.  For a block
// i_1 .. i_m (application order), u_{i_t}^T x^{(t-1)} = u_{i_t}^T x - 2 sum_{s<t} alpha_s
// (u_{i_s}^T u_{i_t}), so all m dot products are taken against the block's input x, reduced
// across the column group together (one reduce-scatter, one cross-warp exchange), the alphas
// follow from the m x m Gram entries by forward substitution, and x <- x - 2 sum_t alpha_t u_t.
// Same FMAs as the sequential form (the compact-WY identity of Eq. 2 for a block); the
// per-reflector serial chain (dot -> reduction -> barrier -> update) becomes one per block, at
// the price of a second TMEM read of each u.  The Gram G = U^T U (h x h, fp32) is formed once per
// CTA from the TMEM-resident reflectors (fixed-order sums: identical in every CTA).
//
// SC ("K1r"): scalar element ownership -- a thread owns the elements gt + TPC k (k < CH) of its
// columns instead of 128-bit chunks, columns are loaded straight into registers with coalesced
// one-element accesses, U is copied into shared memory by the CTA's threads (resident only).
// Needs element alignment only: the shapes whose column stride or base is not a multiple of
// 16 bytes (any n <= TPC CH).
template <typename T, int TPC, int CH, int C, int NT, bool FULL, bool UTM = false, int KB = 1,
          bool SC = false>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) hh_fused_kernel(const FusedArgs a) {
    static_assert(!UTM || (std::is_same<T, float>::value && 128 % TPC == 0 && TPC >= 32),
                  "TMEM reflectors: fp32, TPC in {32, 64, 128}");
    static_assert(!(UTM && SC) || (CH % 8 == 0 && KB == 1), "scalar TMEM form: CH in {8, 16, 32}, unblocked");
    static_assert(KB == 1 || (UTM && (KB * C == 4 || KB * C == 8 || KB * C == 16)),
                  "blocked reflectors: TMEM form, KB * C in {4, 8, 16}");
    constexpr int KV = KB > 1 ? KB * C : C;   // values per cross-lane reduction
    constexpr int UCOLS = SC ? CH : 4 * CH;   // TMEM columns per reflector (UTM)
    using V = typename std::conditional<SC, T, typename VT<T>::V>::type;
    constexpr int E = SC ? 1 : VT<T>::E;
    constexpr int UT = TPC > 32 ? TPC : 32;  // threads per scheduling unit
    constexpr int GPU_ = UT / TPC;           // groups per unit
    constexpr int UC = GPU_ * C;             // columns per unit tile
    constexpr int NU = NT / UT;              // units per CTA
    constexpr int WPU = UT / 32;             // warps per unit
    static_assert(NT % UT == 0, "block must hold whole units");
    static_assert(UT == 32 || NU <= 15, "named barrier ids");

    const int tid = threadIdx.x;
    const int unit = tid / UT;
    const int ut = tid % UT;
    const int grp = ut / TPC;
    const int gt = ut % TPC;
    const int lane = tid & 31;
    const int wiu = ut >> 5;

    const int mode = a.mode;
    const int64_t n = a.n;
    const int nv = static_cast<int>(n / E);
    const int h = static_cast<int>(a.h);
    const int R = a.R;
    const int nc = a.nchunks;
    const int nbuf = nc > 1 ? 2 : 1;
    const bool stage = a.stage_x != 0;

    extern __shared__ __align__(128) unsigned char smem[];
    V *Us = reinterpret_cast<V *>(smem);
    V *Xs = Us + static_cast<size_t>(nbuf) * R * nv;
    T *red = reinterpret_cast<T *>(Xs + (stage ? static_cast<size_t>(NU) * UC * nv : 0));
    // SC: R nv elements need not end on a 16-byte boundary, and a staging slot holds the
    // 16-byte-aligned superset of a tile (its first byte may sit up to 12 bytes into the slot,
    // its last up to 12 bytes before the copy's end): byte pitch `spitch`
    size_t spitch = 0;
    if constexpr (SC) {
        Xs = reinterpret_cast<V *>((reinterpret_cast<uintptr_t>(Xs) + 15) & ~static_cast<uintptr_t>(15));
        spitch = (static_cast<size_t>(UC) * nv * sizeof(V) + 31) & ~static_cast<size_t>(15);
        red = reinterpret_cast<T *>(reinterpret_cast<unsigned char *>(Xs) + (stage ? NU * spitch : 0));
    }
    uint64_t *bars = reinterpret_cast<uint64_t *>(red + (TPC > 32 ? 2 * NU * WPU * KV : 0));
    uint64_t *ubar = bars;      // [2]
    uint64_t *xbar = bars + 2;  // [NU]

    const V *Ug = reinterpret_cast<const V *>(a.U);
    const V *Xg = reinterpret_cast<const V *>(a.X);
    const V *vecg = reinterpret_cast<const V *>(a.vec);

    const int64_t ntiles = (a.N + UC - 1) / UC;
    const int nb = a.nbatches;
    const int L = (mode == MODE_SYM ? 2 : 1) * nc;  // U-chunk visits per batch (nc > 1)
    const int64_t nvisits = static_cast<int64_t>(nb) * L;

    auto tile_of = [&](int b) -> int64_t {
        return (static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * NU + unit;
    };
    auto chunk_of = [&](int q) -> int {
        if (mode == MODE_APPLY_N) return nc - 1 - q;
        if (mode == MODE_SYM) return q < nc ? q : 2 * nc - 1 - q;
        return q;
    };
    // issue the bulk copy of U chunk `c` into buffer `buf`
    auto issue_u = [&](int c, int buf) {
        const int r0 = c * R;
        const int r1 = min(h, r0 + R);
        const uint32_t bytes = static_cast<uint32_t>((r1 - r0) * nv * sizeof(V));
        mbar_arrive_expect_tx(&ubar[buf], bytes);
        const uint64_t pol = policy_evict_last();
        const char *src = reinterpret_cast<const char *>(Ug + static_cast<size_t>(r0) * nv);
        char *dst = reinterpret_cast<char *>(Us + static_cast<size_t>(buf) * R * nv);
        for (uint32_t off = 0; off < bytes; off += 32768u)
            bulk_g2s(dst + off, src + off, min(32768u, bytes - off), &ubar[buf], pol);
    };
    auto issue_x = [&](int64_t t) {
        const int64_t c0 = t * UC;
        const int64_t cols = min(static_cast<int64_t>(UC), a.N - c0);
        const uint32_t bytes = static_cast<uint32_t>(cols * nv * sizeof(V));
        mbar_arrive_expect_tx(&xbar[unit], bytes);
        const uint64_t pol = policy_evict_first();
        const char *src = reinterpret_cast<const char *>(Xg + c0 * nv);
        char *dst = reinterpret_cast<char *>(Xs + static_cast<size_t>(unit) * UC * nv);
        for (uint32_t off = 0; off < bytes; off += 32768u)
            bulk_g2s(dst + off, src + off, min(32768u, bytes - off), &xbar[unit], pol);
    };
    // SC: a tile is staged only if the 16-byte superset of its bytes stays inside X (all but,
    // at most, the last tile); the others are loaded straight into registers
    auto sc_stageable = [&](int64_t t) -> bool {
        const int64_t c1 = min((t + 1) * UC, a.N);
        const int64_t end = (c1 * nv * static_cast<int64_t>(sizeof(V)) + 15) & ~static_cast<int64_t>(15);
        return end <= a.N * nv * static_cast<int64_t>(sizeof(V));
    };
    auto sc_issue_x = [&](int64_t t) {   // (X itself is 16-byte aligned when the launcher stages)
        const int64_t c0 = t * UC;
        const int64_t cols = min(static_cast<int64_t>(UC), a.N - c0);
        const char *src = reinterpret_cast<const char *>(Xg + c0 * nv);
        const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src) & 15u);
        const uint32_t bytes = (static_cast<uint32_t>(cols * nv * sizeof(V)) + lead + 15u) & ~15u;
        src -= lead;
        mbar_arrive_expect_tx(&xbar[unit], bytes);
        const uint64_t pol = policy_evict_first();
        char *dst = reinterpret_cast<char *>(Xs) + static_cast<size_t>(unit) * spitch;
        for (uint32_t off = 0; off < bytes; off += 32768u)
            bulk_g2s(dst + off, src + off, min(32768u, bytes - off), &xbar[unit], pol);
    };
    auto unit_sync = [&]() {
        if (UT == 32)
            __syncwarp();
        else
            named_bar_sync(1 + unit, UT);
    };

    if (tid == 0) {
        mbar_init(&ubar[0], 1);
        mbar_init(&ubar[1], 1);
    }
    if (ut == 0) mbar_init(&xbar[unit], 1);
    fence_mbar_init();
    // the TMEM address slot follows the barriers in dynamic shared memory (a static __shared__
    // variable would push the opt-in dynamic size the launcher requests over the limit)
    uint32_t &s_tmem = *reinterpret_cast<uint32_t *>(bars + 2 + NU);
    uint32_t tlane = 0;   // this thread's TMEM lane address (UTM)
    if constexpr (UTM) {
        const int warp = tid >> 5;
        if (warp == 0) tmem_alloc_n(&s_tmem, static_cast<uint32_t>(a.tcols));
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        tlane = s_tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        if (warp < 4) {
            // warp q fills lane quarter q: lane 32 q + l holds the chunks of gt = (32 q + l) mod TPC
            const int g2 = (warp * 32 + lane) % TPC;
            if constexpr (SC) {
                // scalar ownership: column i CH + k of lane gt holds element gt + TPC k of u_i
                const T *Us1 = reinterpret_cast<const T *>(a.U);
                for (int i = 0; i < h; ++i) {
#pragma unroll
                    for (int k = 0; k < CH; k += 8) {
                        uint32_t w[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int64_t r = g2 + static_cast<int64_t>(TPC) * (k + e);
                            w[e] = r < n ? __float_as_uint(__ldg(Us1 + static_cast<int64_t>(i) * n + r)) : 0u;
                        }
                        tc::tmem_st8(tlane + static_cast<uint32_t>(i * UCOLS + k),
                                     make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
                    }
                }
            } else
            for (int i = 0; i < h; ++i) {
#pragma unroll
                for (int k = 0; k < CH; k += 2) {
                    float4 u0 = make_float4(0.f, 0.f, 0.f, 0.f), u1 = u0;
                    if (FULL || g2 + TPC * k < nv)
                        u0 = __ldg(reinterpret_cast<const float4 *>(a.U) + static_cast<size_t>(i) * nv + g2 + TPC * k);
                    if (FULL || g2 + TPC * (k + 1) < nv)
                        u1 = __ldg(reinterpret_cast<const float4 *>(a.U) + static_cast<size_t>(i) * nv + g2 + TPC * (k + 1));
                    tc::tmem_st8(tlane + static_cast<uint32_t>(i * UCOLS + 4 * k),
                                 make_uint4(__float_as_uint(u0.x), __float_as_uint(u0.y),
                                            __float_as_uint(u0.z), __float_as_uint(u0.w)),
                                 make_uint4(__float_as_uint(u1.x), __float_as_uint(u1.y),
                                            __float_as_uint(u1.z), __float_as_uint(u1.w)));
                }
            }
            tc::tmem_wait_st();
        }
        tc::fence_before_sync();
    }
    __syncthreads();
    if constexpr (UTM) tc::fence_after_sync();
    // K1w: the Gram G[i][j] = u_i^T u_j from the TMEM-resident chunks.  A "set" of TPC / 32
    // warps covers every chunk position once; the sets split the pairs i <= j, each warp
    // reduces its partial in the warp and parks it, then the partials of a pair are added in
    // warp order (deterministic, the same bits in every CTA).
    float *gram = reinterpret_cast<float *>(bars + 2 + NU + 1);   // h x h, then partials
    if constexpr (KB > 1) {
        constexpr int S = TPC / 32;          // warps per set
        constexpr int NSET = NT / TPC;
        const int warp = tid >> 5;
        const int set = warp / S, ws = warp % S;
        const int npair = h * (h + 1) / 2;
        float *gpart = gram + h * h;         // [npair][S]
        for (int pidx = set; pidx < npair; pidx += NSET) {
            int i = 0, rem = pidx;
            while (rem >= h - i) {
                rem -= h - i;
                ++i;
            }
            const int j = i + rem;
            uint32_t ri[UCOLS], rj[UCOLS];
            tmem_ld_cols<UCOLS>(tlane + static_cast<uint32_t>(i * UCOLS), ri);
            tmem_ld_cols<UCOLS>(tlane + static_cast<uint32_t>(j * UCOLS), rj);
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < UCOLS; ++e) acc = fmaf(__uint_as_float(ri[e]), __uint_as_float(rj[e]), acc);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) gpart[pidx * S + ws] = acc;
        }
        __syncthreads();
        for (int pidx = tid; pidx < npair; pidx += NT) {
            int i = 0, rem = pidx;
            while (rem >= h - i) {
                rem -= h - i;
                ++i;
            }
            const int j = i + rem;
            float g = gpart[pidx * S];
#pragma unroll
            for (int w = 1; w < S; ++w) g += gpart[pidx * S + w];
            gram[i * h + j] = g;
            gram[j * h + i] = g;
        }
        __syncthreads();
    }

    // prologue: U (resident, or the first two chunk visits) and each unit's first tile
    if constexpr (SC) {   // resident U copied by the CTA's threads (no 16-byte granularity)
        if constexpr (!UTM) {
            // rows at pitch TPC CH, zero past n: with x = 0 there too, the reflector loops need
            // no per-element predicate (they cost more than the FMAs at CH = 32)
            for (int i = tid; i < h * (TPC * CH); i += NT) {
                const int row = i / (TPC * CH), r = i % (TPC * CH);
                Us[i] = r < nv ? __ldg(Ug + static_cast<int64_t>(row) * nv + r) : T(0);
            }
            __syncthreads();
        }
    } else
    if (!UTM && tid == 0 && h > 0) {
        if (nc == 1) {
            issue_u(0, 0);
        } else {
            for (int64_t g = 0; g < (nvisits < 2 ? nvisits : 2); ++g)
                issue_u(chunk_of(static_cast<int>(g % L)), static_cast<int>(g & 1));
        }
    }
    if constexpr (SC) {
        if (stage && ut == 0 && tile_of(0) < ntiles && sc_stageable(tile_of(0))) sc_issue_x(tile_of(0));
    } else {
        if (stage && ut == 0 && tile_of(0) < ntiles) issue_x(tile_of(0));
    }

    V x[C][CH];
    uint32_t xphase = 0;
    int rpar = 0;       // reduction-buffer parity (TPC > 32)
    int64_t g = 0;      // chunk-visit counter (nc > 1)
    bool u_ready = UTM || SC || (h == 0) || (nc > 1);

    auto valid_k = [&](int k) -> bool { return FULL || (gt + TPC * k < nv); };

    // one reflector: x <- x - 2 (u^T x) u   for the C columns of this group
    auto reflect = [&](const V *ub, int ui) {
        T p[C];
        // multi-warp groups: keep the u chunk in registers across the cross-warp
        // reduction (a shared-memory store + barrier the compiler cannot see through),
        // so u is read from shared memory once per reflector, not twice
        constexpr bool kKeepU = UTM || (TPC > 32 && !SC);
        V uk[kKeepU ? CH : 1];
        if constexpr (UTM) {
            uint32_t r[UCOLS];
            tmem_ld_cols<UCOLS>(tlane + static_cast<uint32_t>(ui * UCOLS), r);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if constexpr (SC) {
                    if constexpr (std::is_same<T, float>::value) uk[k] = __uint_as_float(r[k]);
                } else if constexpr (std::is_same<T, float>::value) {
                    uk[k] = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                        __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
                }
            }
        } else if constexpr (kKeepU) {
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (valid_k(k)) uk[k] = ub[gt + TPC * k];
                else vzero(uk[k]);
            }
        }
        // (U in TMEM: positions past n hold u = 0 -- zero-filled at the TMEM fill -- and x = 0, so
        // the reflector loops below skip the ragged-tail predicate: `UTM || valid_k(k)`)
        auto uget = [&](int k) -> V {
            if constexpr (kKeepU) return uk[k];
            else if constexpr (SC) return Us[static_cast<size_t>(ui) * (TPC * CH) + gt + TPC * k];
            else return ub[gt + TPC * k];
        };
        // fp32, two columns per single-warp group: the partial sums and the butterfly use
        // packed FADD2 (two IEEE adds per instruction) -- fewer issue slots on the serial chain
        constexpr bool kPair = std::is_same<T, float>::value && C == 2 && TPC <= 32;
        // the packed partial sums and 2-alpha also serve the multi-warp two-column groups
        constexpr bool kPairSum = std::is_same<T, float>::value && C == 2 && !SC;
        // SC, fp32, two columns: element k of both columns is one FFMA2 pair against (u, u);
        // four accumulator pairs break the CH-long dependency chain
        constexpr bool kScPair = SC && std::is_same<T, float>::value && C == 2;
        if constexpr (kScPair) {
            float q0[4] = {0.f, 0.f, 0.f, 0.f}, q1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                // (positions past n hold u = 0 and x = 0 -- no per-element predicate)
                {
                    const float uk0 = uget(k);
                    ffma2(q0[k & 3], q1[k & 3], uk0, uk0, x[0][k], x[1][k], q0[k & 3], q1[k & 3]);
                }
            }
            float a0, a1, b0, b1;
            fadd2(a0, a1, q0[0], q1[0], q0[1], q1[1]);
            fadd2(b0, b1, q0[2], q1[2], q0[3], q1[3]);
            fadd2(p[0], p[1], a0, a1, b0, b1);
        } else if constexpr (SC) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                T q[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    vfma(q[k & 3], uget(k), x[c][k]);
                }
                p[c] = (q[0] + q[1]) + (q[2] + q[3]);
            }
        } else if constexpr (kPairSum) {
            V acc0, acc1;
            vzero(acc0);
            vzero(acc1);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (UTM || valid_k(k)) {
                    const V uk0 = uget(k);
                    vfma(acc0, uk0, x[0][k]);
                    vfma(acc1, uk0, x[1][k]);
                }
            }
            float a0, a1, b0, b1;
            fadd2(a0, a1, acc0.x, acc0.y, acc0.z, acc0.w);   // (x + z, y + w)
            fadd2(b0, b1, acc1.x, acc1.y, acc1.z, acc1.w);
            fadd2(p[0], p[1], a0, b0, a1, b1);
        } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            V acc;
            vzero(acc);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (UTM || valid_k(k)) vfma(acc, uget(k), x[c][k]);
            }
            p[c] = vsum(acc);
        }
        }
        if constexpr (TPC > 32 && C == 2) {
            // two columns over a multi-warp group: reduce-scatter in the warp (the first step
            // exchanges the other column's partial, then one value per lane: 5 shuffles
            // instead of 10); lanes 0 and 16 hold the warp's sums of columns 0 and 1, and the
            // shared-memory exchange that follows broadcasts them anyway
            const bool hi = (lane & 16) != 0;
            T v = (hi ? p[1] : p[0]) + __shfl_xor_sync(0xffffffffu, hi ? p[0] : p[1], 16);
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            T *rb = red + (static_cast<size_t>(rpar) * NU + unit) * WPU * C;
            if ((lane & 15) == 0) rb[wiu * C + (hi ? 1 : 0)] = v;
            named_bar_sync(1 + unit, UT);
            // (128-bit loads of the warps' pairs summed with FADD2 were measured 6 % slower
            // here: the extra live registers spill at n = 4096)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                T sum = rb[c];
#pragma unroll
                for (int w = 1; w < WPU; ++w) sum += rb[w * C + c];
                p[c] = sum;
            }
            rpar ^= 1;
        } else if constexpr (kPair) {
#pragma unroll
            for (int off = TPC / 2; off > 0; off >>= 1) {
                const float t0 = __shfl_xor_sync(0xffffffffu, p[0], off);
                const float t1 = __shfl_xor_sync(0xffffffffu, p[1], off);
                fadd2(p[0], p[1], p[0], p[1], t0, t1);
            }
        } else {
#pragma unroll
        for (int off = (TPC < 32 ? TPC : 32) / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int c = 0; c < C; ++c) p[c] += __shfl_xor_sync(0xffffffffu, p[c], off);
        }
        if constexpr (TPC > 32) {
            T *rb = red + (static_cast<size_t>(rpar) * NU + unit) * WPU * C;
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < C; ++c) rb[wiu * C + c] = p[c];
            }
            named_bar_sync(1 + unit, UT);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                T s = rb[c];
#pragma unroll
                for (int w = 1; w < WPU; ++w) s += rb[w * C + c];
                p[c] = s;
            }
            rpar ^= 1;
        }
        }
        if constexpr (kScPair) {
            float s0, s1;
            fadd2(s0, s1, p[0], p[1], p[0], p[1]);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                {
                    const float uk0 = uget(k);
                    ffma2(x[0][k], x[1][k], -s0, -s1, uk0, uk0, x[0][k], x[1][k]);
                }
            }
        } else if constexpr (kPairSum) {
            float s0, s1;
            fadd2(s0, s1, p[0], p[1], p[0], p[1]);   // 2 alpha for both columns at once
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (UTM || valid_k(k)) {
                    const V uk0 = uget(k);
                    vaxpy(x[0][k], s0, uk0);
                    vaxpy(x[1][k], s1, uk0);
                }
            }
        } else if constexpr (SC) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const T s = p[c] + p[c];
#pragma unroll
                for (int k = 0; k < CH; ++k) vaxpy(x[c][k], s, uget(k));
            }
        } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const T s = p[c] + p[c];
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (UTM || valid_k(k)) vaxpy(x[c][k], s, uget(k));
            }
        }
        }
    };
    // K1w: reflectors [r0, r1) in blocks of KB (application order descending for desc)
    auto run_blocked = [&](int r0, int r1, bool desc) {
        if constexpr (KB > 1) {
            const int mt = r1 - r0;
            for (int s0 = 0; s0 < mt; s0 += KB) {
                const int m = min(KB, mt - s0);
                int idx[KB];
#pragma unroll
                for (int t = 0; t < KB; ++t) idx[t] = desc ? r1 - 1 - (s0 + t) : r0 + s0 + t;
                // (a) the m dot products against the block's input x
                float v[KV];
#pragma unroll
                for (int t = 0; t < KB; ++t) {
                    if (t < m) {
                        uint32_t r[UCOLS];
                        tmem_ld_cols<UCOLS>(tlane + static_cast<uint32_t>(idx[t] * UCOLS), r);
                        float4 acc[C];
#pragma unroll
                        for (int c = 0; c < C; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int k = 0; k < CH; ++k) {
                            if (UTM || valid_k(k)) {
                                const float4 uk0 = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                                               __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
#pragma unroll
                                for (int c = 0; c < C; ++c) vfma(acc[c], uk0, x[c][k]);
                            }
                        }
#pragma unroll
                        for (int c = 0; c < C; ++c) v[t * C + c] = vsum(acc[c]);
                    } else {
#pragma unroll
                        for (int c = 0; c < C; ++c) v[t * C + c] = 0.f;
                    }
                }
                // (b) reduce the KV values over the group: reduce-scatter in the warp (lane l
                // ends with value index = its top log2(KV) bits), then across the group's warps
                constexpr int LV = KV == 4 ? 2 : (KV == 8 ? 3 : 4);
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const int off = 16 >> st;
                    if (st < LV) {
                        const bool up = (lane & off) != 0;
                        const int half = KV >> (st + 1);
#pragma unroll
                        for (int j = 0; j < half; ++j) {
                            const float send = up ? v[j] : v[j + half];
                            const float keep = up ? v[j + half] : v[j];
                            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                        }
                    } else {
                        v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
                    }
                }
                float p[KV];
                if constexpr (TPC > 32) {
                    float *rb = red + (static_cast<size_t>(rpar) * NU + unit) * WPU * KV;
                    if ((lane & ((32 >> LV) - 1)) == 0) rb[(lane >> (5 - LV)) * WPU + wiu] = v[0];
                    named_bar_sync(1 + unit, UT);
#pragma unroll
                    for (int w = 0; w < KV; ++w) {
                        float sum = rb[w * WPU];
#pragma unroll
                        for (int q = 1; q < WPU; ++q) sum += rb[w * WPU + q];
                        p[w] = sum;
                    }
                    rpar ^= 1;
                } else {
#pragma unroll
                    for (int w = 0; w < KV; ++w) p[w] = __shfl_sync(0xffffffffu, v[0], w << (5 - LV));
                }
                // (c) forward substitution: alpha_t = p_t - 2 sum_{s<t} G[i_s][i_t] alpha_s
#pragma unroll
                for (int t = 1; t < KB; ++t) {
                    if (t < m) {
#pragma unroll
                        for (int s2 = 0; s2 < t; ++s2) {
                            const float g2 = -2.f * gram[idx[s2] * h + idx[t]];
#pragma unroll
                            for (int c = 0; c < C; ++c) p[t * C + c] = fmaf(g2, p[s2 * C + c], p[t * C + c]);
                        }
                    }
                }
                // (d) x <- x - 2 sum_t alpha_t u_t
#pragma unroll
                for (int t = 0; t < KB; ++t) {
                    if (t < m) {
                        uint32_t r[UCOLS];
                        tmem_ld_cols<UCOLS>(tlane + static_cast<uint32_t>(idx[t] * UCOLS), r);
#pragma unroll
                        for (int k = 0; k < CH; ++k) {
                            if (UTM || valid_k(k)) {
                                const float4 uk0 = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                                               __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
#pragma unroll
                                for (int c = 0; c < C; ++c) vaxpy(x[c][k], 2.f * p[t * C + c], uk0);
                            }
                        }
                    }
                }
            }
        }
    };
    // reflectors [r0, r1) of the chunk resident at `base` (first row = chunk_lo)
    // (NEXT-f2: the fused kernel applies QR-structured reflectors in full -- it serves
    // small h, where the zero prefixes are a negligible share; K5 skips them.)
    auto run_range = [&](const V *base, int chunk_lo, int r0, int r1, bool desc) {
        constexpr bool kPairLoop = std::is_same<T, float>::value && C == 2 && TPC <= 32 && !SC;
        if constexpr (kPairLoop) {
            // two reflectors per loop trip: the loop bookkeeping is ~10 of the ~100 issue slots
            // of a reflector here, and this kernel is issue-bound (C2 0.358 -> 0.353 ms, A/B)
            if (desc) {
#pragma unroll 2
                for (int i = r1 - 1; i >= r0; --i) reflect(base + static_cast<size_t>(i - chunk_lo) * nv, i);
            } else {
#pragma unroll 2
                for (int i = r0; i < r1; ++i) reflect(base + static_cast<size_t>(i - chunk_lo) * nv, i);
            }
        } else {
            if (desc) {
                for (int i = r1 - 1; i >= r0; --i) reflect(base + static_cast<size_t>(i - chunk_lo) * nv, i);
            } else {
                for (int i = r0; i < r1; ++i) reflect(base + static_cast<size_t>(i - chunk_lo) * nv, i);
            }
        }
    };
    auto scale_vec = [&]() {
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (valid_k(k)) {
                const V l = ldg_v(vecg + gt + TPC * k);
#pragma unroll
                for (int c = 0; c < C; ++c) vmul(x[c][k], l);
            }
        }
    };

    for (int b = 0; b < nb; ++b) {
        const int64_t t = tile_of(b);
        const bool tv = t < ntiles;
        const int64_t col0 = t * UC + static_cast<int64_t>(grp) * C;

        // pull the unit's tile l2pf batches ahead into L2 with one bulk prefetch, so the
        // register loads (unstaged) or the slot copy (staged) of that batch are served at L2
        // latency while this one computes (measured slower for unstaged n = 4096)
        // (staged columns: the next tile is already on its way into the slot; l2pf >= 2
        // reaches further ahead)
        if (mode != MODE_PAIR && a.l2pf > (stage ? 1 : 0) && ut == 0) {
            const int64_t tp = tile_of(b + a.l2pf);
            if (b + a.l2pf < nb && tp < ntiles) {
                const int64_t c0 = tp * UC;
                const int64_t cols = min(static_cast<int64_t>(UC), a.N - c0);
                const uint32_t bytes = static_cast<uint32_t>(cols * nv * sizeof(V));
                const char *src = reinterpret_cast<const char *>(Xg + c0 * nv);
                for (uint32_t off = 0; off < bytes; off += 32768u)
                    bulk_prefetch_l2(src + off, min(32768u, bytes - off));
            }
        }

        // ---- 1. columns -> registers
        if (tv) {
            if (mode == MODE_PAIR) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int64_t j = col0 + c;
                    const bool cv = j < a.N;
                    const V *pa = Xg + (cv ? static_cast<int64_t>(a.ia[j]) : 0) * nv;
                    const V *pb = Xg + (cv ? static_cast<int64_t>(a.ib[j]) : 0) * nv;
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        vzero(x[c][k]);
                        if (cv && valid_k(k)) {
                            x[c][k] = ldg_v(pa + gt + TPC * k);
                            vsub(x[c][k], ldg_v(pb + gt + TPC * k));
                        }
                    }
                }
            } else if (SC && stage && sc_stageable(t)) {
                if constexpr (SC) {
                    mbar_wait(&xbar[unit], xphase);
                    xphase ^= 1u;
                    // the tile starts `lead` bytes into the slot
                    const unsigned char *slot = reinterpret_cast<const unsigned char *>(Xs) +
                                                static_cast<size_t>(unit) * spitch +
                                                (reinterpret_cast<uintptr_t>(Xg + t * UC * nv) & 15u);
                    const V *xs = reinterpret_cast<const V *>(slot) + static_cast<size_t>(grp * C) * nv;
#pragma unroll
                    for (int c = 0; c < C; ++c) {
#pragma unroll
                        for (int k = 0; k < CH; ++k) {
                            if (valid_k(k))
                                x[c][k] = xs[static_cast<size_t>(c) * nv + gt + TPC * k];
                            else
                                vzero(x[c][k]);
                        }
                    }
                    unit_sync();
                    if (ut == 0) {
                        const int64_t t1 = tile_of(b + 1);
                        if (b + 1 < nb && t1 < ntiles && sc_stageable(t1)) {
                            fence_proxy_async_smem();
                            sc_issue_x(t1);
                        }
                    }
                }
            } else if (!SC && stage) {
                mbar_wait(&xbar[unit], xphase);
                xphase ^= 1u;
                const V *xs = Xs + (static_cast<size_t>(unit) * UC + grp * C) * nv;
#pragma unroll
                for (int c = 0; c < C; ++c) {
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        if (valid_k(k))
                            x[c][k] = xs[static_cast<size_t>(c) * nv + gt + TPC * k];
                        else
                            vzero(x[c][k]);
                    }
                }
                unit_sync();  // every thread of the unit has its columns in registers
                if (ut == 0) {
                    const int64_t t1 = tile_of(b + 1);
                    if (b + 1 < nb && t1 < ntiles) {
                        fence_proxy_async_smem();
                        issue_x(t1);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int64_t j = col0 + c;
                    const bool cv = j < a.N;
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        vzero(x[c][k]);
                        if (cv && valid_k(k)) x[c][k] = ldg_v(Xg + j * nv + gt + TPC * k);
                    }
                }
            }
        }

        // NEXT-f1 right factor (Y = Q D X): x <- D x before the first reflector
        if (tv && (a.dside & 1)) {
            const V *dg = reinterpret_cast<const V *>(a.dsign);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                if (valid_k(k)) {
                    const V dv = ldg_v(dg + gt + TPC * k);
#pragma unroll
                    for (int c = 0; c < C; ++c) vmul(x[c][k], dv);
                }
            }
        }

        // ---- 2. reflector passes
        if (nc == 1) {
            if (!u_ready) {
                mbar_wait(&ubar[0], 0);
                u_ready = true;
            }
            if (tv) {
                if constexpr (KB > 1) {
                    if (mode == MODE_APPLY_N) {
                        run_blocked(0, h, true);
                    } else if (mode == MODE_SYM) {
                        run_blocked(0, h, false);
                        scale_vec();
                        run_blocked(0, h, true);
                    } else {
                        run_blocked(0, h, false);
                    }
                } else if (mode == MODE_APPLY_N) {
                    run_range(Us, 0, 0, h, true);
                } else if (mode == MODE_SYM) {
                    run_range(Us, 0, 0, h, false);
                    scale_vec();
                    run_range(Us, 0, 0, h, true);
                } else {
                    run_range(Us, 0, 0, h, false);
                }
            }
        } else {
            for (int q = 0; q < L; ++q, ++g) {
                const int buf = static_cast<int>(g & 1);
                mbar_wait(&ubar[buf], static_cast<uint32_t>((g >> 1) & 1));
                const int c = chunk_of(q);
                const bool desc = (mode == MODE_APPLY_N) || (mode == MODE_SYM && q >= nc);
                if (tv) {
                    run_range(Us + static_cast<size_t>(buf) * R * nv, c * R, c * R,
                              min(h, (c + 1) * R), desc);
                    if (mode == MODE_SYM && q == nc - 1) scale_vec();
                }
                __syncthreads();  // every unit is done with buffer `buf`
                if (tid == 0 && g + 2 < nvisits) {
                    fence_proxy_async_smem();
                    issue_u(chunk_of(static_cast<int>((g + 2) % L)), buf);
                }
            }
        }

        // ---- 3. epilogue
        if (tv) {
            if (mode == MODE_PAIR) {
                T s[C];
#pragma unroll
                for (int c = 0; c < C; ++c) s[c] = T(0);
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    if (valid_k(k)) {
                        const V dv = ldg_v(vecg + gt + TPC * k);
#pragma unroll
                        for (int c = 0; c < C; ++c) s[c] += vwsq(x[c][k], dv);
                    }
                }
#pragma unroll
                for (int off = (TPC < 32 ? TPC : 32) / 2; off > 0; off >>= 1) {
#pragma unroll
                    for (int c = 0; c < C; ++c) s[c] += __shfl_xor_sync(0xffffffffu, s[c], off);
                }
                if constexpr (TPC > 32) {
                    T *rb = red + (static_cast<size_t>(rpar) * NU + unit) * WPU * C;
                    if (lane == 0) {
#pragma unroll
                        for (int c = 0; c < C; ++c) rb[wiu * C + c] = s[c];
                    }
                    named_bar_sync(1 + unit, UT);
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        T v = rb[c];
#pragma unroll
                        for (int w = 1; w < WPU; ++w) v += rb[w * C + c];
                        s[c] = v;
                    }
                    rpar ^= 1;
                }
                if (gt == 0) {
                    T *dist = reinterpret_cast<T *>(a.Y);
#pragma unroll
                    for (int c = 0; c < C; ++c)
                        if (col0 + c < a.N) dist[col0 + c] = s[c];
                }
            } else {
                if (mode == MODE_TRANSFORM) {
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        if (valid_k(k)) {
                            const V dv = ldg_v(vecg + gt + TPC * k);
#pragma unroll
                            for (int c = 0; c < C; ++c) vmulsqrt(x[c][k], dv);
                        }
                    }
                }
                if (a.dside & 2) {   // NEXT-f1 left factor (Y = D Q X)
                    const V *dg = reinterpret_cast<const V *>(a.dsign);
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        if (valid_k(k)) {
                            const V dv = ldg_v(dg + gt + TPC * k);
#pragma unroll
                            for (int c = 0; c < C; ++c) vmul(x[c][k], dv);
                        }
                    }
                }
                V *Yg = reinterpret_cast<V *>(a.Y);
                const uint64_t ypol = policy_evict_first();
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int64_t j = col0 + c;
                    if (j < a.N) {
#pragma unroll
                        for (int k = 0; k < CH; ++k)
                            if (valid_k(k)) st_global_hint(Yg + j * nv + gt + TPC * k, x[c][k], ypol);
                    }
                }
            }
        }
    }
    if constexpr (UTM) {
        tc::fence_before_sync();
        __syncthreads();
        if ((tid >> 5) == 0) tmem_dealloc_n(s_tmem, static_cast<uint32_t>(a.tcols));
    }
}

// One instantiated shape of the kernel: TPC threads per column, CH vector chunks per
// thread, C columns per group, NT threads per CTA.
struct FusedVariant {
    const void *fn_full;        // nv == TPC*CH exactly
    const void *fn_ragged;
    const void *fn_tm_full;     // K1t (reflectors in TMEM), or nullptr
    const void *fn_tm_ragged;
    int tpc, ch, c, nt;
    int elem;  // bytes
    const char *name;
    const char *name_tm;   // K1t form's name
    const void *fn_tb_full = nullptr;    // K1w (TMEM reflectors in blocks of kb), or nullptr
    const void *fn_tb_ragged = nullptr;
    int kb = 1;
    const char *name_tb = nullptr;
};

#define HH_FUSED_VAR(T, TPC, CH, C, NT, NAME)                                           \
    FusedVariant {                                                                      \
        reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true>),      \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false>), \
            nullptr, nullptr, TPC, CH, C, NT, static_cast<int>(sizeof(T)), NAME, NAME   \
    }
// the same shape with a K1t (TMEM reflector) form
#define HH_FUSED_VAR_TM(T, TPC, CH, C, NT, NAME)                                          \
    FusedVariant {                                                                        \
        reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true>),        \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false>),   \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true, true>), \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, true>), \
            TPC, CH, C, NT, static_cast<int>(sizeof(T)), NAME, NAME "_tmem"                  \
    }
// ... and a K1w (blocked TMEM reflectors, KB per block) form
#define HH_FUSED_VAR_TB(T, TPC, CH, C, NT, NAME, KB)                                       \
    FusedVariant {                                                                        \
        reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true>),        \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false>),   \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true, true>), \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, true>), \
            TPC, CH, C, NT, static_cast<int>(sizeof(T)), NAME, NAME "_tmem",                 \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, true, true, KB>), \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, true, KB>), \
            KB, NAME "_tmem_kb" #KB                                                        \
    }

// the scalar-element form (K1r): ragged form only (n is never a multiple of 16 bytes there)
#define HH_FUSED_VAR_SC(T, TPC, CH, C, NT, NAME)                                                   \
    FusedVariant {                                                                                 \
        nullptr,                                                                                   \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, false, 1, true>), \
            nullptr, nullptr, TPC, CH, C, NT, static_cast<int>(sizeof(T)), NAME, NAME              \
    }

// ... with the reflectors in TMEM (K1t's scalar form: one tcgen05.ld per reflector replaces the
// CH one-element shared-memory reads of the dot and of the update)
#define HH_FUSED_VAR_SC_TM(T, TPC, CH, C, NT, NAME)                                                \
    FusedVariant {                                                                                 \
        nullptr,                                                                                   \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, false, 1, true>), \
            nullptr,                                                                               \
            reinterpret_cast<const void *>(&hh_fused_kernel<T, TPC, CH, C, NT, false, true, 1, true>),  \
            TPC, CH, C, NT, static_cast<int>(sizeof(T)), NAME, NAME "_tmem"                        \
    }

// tables (each defined in its own translation unit so the instantiations build in parallel)
const FusedVariant *fused_table_f32(int *count);
const FusedVariant *fused_table_f64(int *count);
const FusedVariant *fused_alt_f32(int *count);   // A/B alternatives (hh_debug_k1)
const FusedVariant *fused_table_scalar(int dtype, int *count);   // K1r (hh_fused_sc.cu)

}  // namespace hh
