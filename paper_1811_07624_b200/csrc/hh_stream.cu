// hh_stream.cu -- K1s: the fused small-h apply as a NON-persistent streaming kernel for
// n <= 1024 (fp32): a column group of TPC lanes keeps C columns in registers, loaded straight
// from HBM with 128-bit loads that bypass L1; u_i is read through L1 (every CTA of an SM reads
// the same h*n*4 bytes, which stay L1-resident across the CTAs of the launch); the result is
// written once with streaming 128-bit stores.  One CTA handles NT/TPC*C columns and exits.
//
// Why: a persistent CTA that keeps one tile in flight per unit for its whole life streams
// ~12 % below the copy rate (profiles/r1/k1_grid_ab_r1.txt); CTAs that load, compute, store
// and retire stream at the copy rate (tools/micro/k1_stream.cu, profiles/r2).  The staged
// copy of U that made churning CTAs expensive is replaced by L1 hits.  Arithmetic and order
// are those of K1 (hh_fused_kernel.cuh): x <- x - 2 (u^T x) u per reflector,
// applied u_h first for Q X and u_1 first for Q^T X (reading R1).
#include <algorithm>

#include "hh_internal.h"
#include "hh_ptx.cuh"

namespace hh {
namespace {

// X through the non-coherent path, bypassing L1: every element is read exactly once, by the
// thread that later writes the same element of Y -- so an exact alias Y == X (allowed by the
// ABI) never lets a load observe a store of another thread
__device__ __forceinline__ float4 ld_na4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_l14(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs4(float4 *p, const float4 &v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
// two IEEE fp32 FMAs in one instruction (FFMA2), as in K1
__device__ __forceinline__ void ffma2s(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B, D;\n\t"
        "mov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 D, {%0, %1};\n\t"
        "fma.rn.f32x2 D, A, B, D;\n\tmov.b64 {%0, %1}, D;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// d0 += b0, d1 += b1 in one FADD2
__device__ __forceinline__ void fadd2s(float &d0, float &d1, float b0, float b1) {
    asm("{\n\t.reg .b64 A, B;\n\t"
        "mov.b64 A, {%0, %1};\n\tmov.b64 B, {%2, %3};\n\t"
        "add.rn.f32x2 A, A, B;\n\tmov.b64 {%0, %1}, A;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(b0), "f"(b1));
}

template <int TPC, int CH, int C, int NT>
__global__ void __launch_bounds__(NT) hh_stream_kernel(const FusedArgs a) {
    constexpr int GPC = NT / TPC;   // column groups per CTA
    const int tid = threadIdx.x;
    const int grp = tid / TPC, gt = tid % TPC;
    const int nv = static_cast<int>(a.n / 4);
    const int h = static_cast<int>(a.h);
    const int mode = a.mode;
    const float4 *Ug = reinterpret_cast<const float4 *>(a.U);
    const float4 *Xg = reinterpret_cast<const float4 *>(a.X);
    float4 *Yg = reinterpret_cast<float4 *>(a.Y);
    const float4 *vecg = reinterpret_cast<const float4 *>(a.vec);
    const float4 *dg = reinterpret_cast<const float4 *>(a.dsign);
    const int64_t col0 = (static_cast<int64_t>(blockIdx.x) * GPC + grp) * C;
    auto valid = [&](int k) { return gt + TPC * k < nv; };

    float4 x[C][CH];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < CH; ++k)
            x[c][k] = (col0 + c < a.N && valid(k)) ? ld_na4(Xg + (col0 + c) * nv + gt + TPC * k)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.dside & 1) {   // NEXT-f1 right factor: x <- D x first
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (!valid(k)) continue;
            const float4 dv = __ldg(dg + gt + TPC * k);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                x[c][k].x *= dv.x;
                x[c][k].y *= dv.y;
                x[c][k].z *= dv.z;
                x[c][k].w *= dv.w;
            }
        }
    }
    // one reflector (Eq. 2): alpha = u^T x (FFMA2 partial sums, xor butterfly over the group),
    // x <- x - 2 alpha u.  (Loading u_{i+1} during reflector i was measured 1.5x slower at
    // n = 1024: the extra registers cost a quarter of the resident warps.)
    auto reflect = [&](int i) {
        const float4 *u = Ug + static_cast<int64_t>(i) * nv + gt;
        float4 uk[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) uk[k] = valid(k) ? ld_l14(u + TPC * k) : make_float4(0.f, 0.f, 0.f, 0.f);
        float p[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                ffma2s(s0, s1, uk[k].x, uk[k].y, x[c][k].x, x[c][k].y);
                ffma2s(s2, s3, uk[k].z, uk[k].w, x[c][k].z, x[c][k].w);
            }
            fadd2s(s0, s1, s2, s3);   // (s0 + s2, s1 + s3)
            p[c] = s0 + s1;
        }
        // column pairs share packed FADD2s in the butterfly (two IEEE adds per instruction)
#pragma unroll
        for (int off = TPC / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int c = 0; c + 1 < C; c += 2) {
                const float t0 = __shfl_xor_sync(0xffffffffu, p[c], off);
                const float t1 = __shfl_xor_sync(0xffffffffu, p[c + 1], off);
                fadd2s(p[c], p[c + 1], t0, t1);
            }
            if constexpr (C % 2) p[C - 1] += __shfl_xor_sync(0xffffffffu, p[C - 1], off);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const float s = -(p[c] + p[c]);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                ffma2s(x[c][k].x, x[c][k].y, s, s, uk[k].x, uk[k].y);
                ffma2s(x[c][k].z, x[c][k].w, s, s, uk[k].z, uk[k].w);
            }
        }
    };
    auto run_desc = [&]() {
#pragma unroll 2
        for (int i = h - 1; i >= 0; --i) reflect(i);
    };
    auto run_asc = [&]() {
#pragma unroll 2
        for (int i = 0; i < h; ++i) reflect(i);
    };
    if (mode == MODE_APPLY_N)
        run_desc();
    else
        run_asc();   // Q^T X, the Q^T pass of SYM, TRANSFORM
    if (mode == MODE_SYM) {   // x <- lambda (.) x, then the Q pass (eq:thesbar)
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (!valid(k)) continue;
            const float4 l = __ldg(vecg + gt + TPC * k);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                x[c][k].x *= l.x;
                x[c][k].y *= l.y;
                x[c][k].z *= l.z;
                x[c][k].w *= l.w;
            }
        }
        run_desc();
    }
    if (mode == MODE_TRANSFORM) {   // Z = diag(sqrt d) Q^T P
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (!valid(k)) continue;
            const float4 dv = __ldg(vecg + gt + TPC * k);
            float4 sq;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.x) : "f"(dv.x));
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.y) : "f"(dv.y));
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.z) : "f"(dv.z));
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sq.w) : "f"(dv.w));
#pragma unroll
            for (int c = 0; c < C; ++c) {
                x[c][k].x *= sq.x;
                x[c][k].y *= sq.y;
                x[c][k].z *= sq.z;
                x[c][k].w *= sq.w;
            }
        }
    }
    if (a.dside & 2) {   // NEXT-f1 left factor: y <- D y last
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (!valid(k)) continue;
            const float4 dv = __ldg(dg + gt + TPC * k);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                x[c][k].x *= dv.x;
                x[c][k].y *= dv.y;
                x[c][k].z *= dv.z;
                x[c][k].w *= dv.w;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c)
        if (col0 + c < a.N)
#pragma unroll
            for (int k = 0; k < CH; ++k)
                if (valid(k)) st_cs4(Yg + (col0 + c) * nv + gt + TPC * k, x[c][k]);
}

struct StreamVariant {
    const void *fn;
    int tpc, ch, c, nt;
    const char *name;
};
#define HH_STREAM_VAR(TPC, CH, C, NT, NAME) \
    StreamVariant { reinterpret_cast<const void *>(&hh_stream_kernel<TPC, CH, C, NT>), TPC, CH, C, NT, NAME }
const StreamVariant kStream[] = {
    HH_STREAM_VAR(4, 1, 4, 128, "f32s_tpc4_ch1_c4"),     // n <= 16
    HH_STREAM_VAR(4, 2, 4, 128, "f32s_tpc4_ch2_c4"),     // n <= 32
    HH_STREAM_VAR(8, 2, 4, 128, "f32s_tpc8_ch2_c4"),     // n <= 64
    HH_STREAM_VAR(8, 4, 2, 128, "f32s_tpc8_ch4_c2"),     // n <= 128
    HH_STREAM_VAR(16, 4, 2, 128, "f32s_tpc16_ch4_c2"),   // n <= 256
    HH_STREAM_VAR(32, 4, 2, 128, "f32s_tpc32_ch4_c2"),   // n <= 512
    HH_STREAM_VAR(32, 8, 2, 128, "f32s_tpc32_ch8_c2"),   // n <= 1024
};

}  // namespace

// fp32 only, modes APPLY_N / APPLY_T / SYM / TRANSFORM, n <= 1024; the caller decides when
cudaError_t launch_stream(const FusedArgs &a, cudaStream_t stream, LaunchInfo *info) {
    const int64_t nv = a.n / 4;
    const StreamVariant *v = nullptr;
    for (const auto &sv : kStream)
        if (static_cast<int64_t>(sv.tpc) * sv.ch >= nv) {
            v = &sv;
            break;
        }
    if (!v) return cudaErrorNotSupported;
    const int64_t cols = static_cast<int64_t>(v->nt / v->tpc) * v->c;
    const int64_t grid = (a.N + cols - 1) / cols;
    if (grid > 0x7fffffff) return cudaErrorNotSupported;
    FusedArgs b = a;
    void *args[] = {&b};
    const cudaError_t e = cudaLaunchKernel(v->fn, dim3(static_cast<unsigned>(grid)), dim3(v->nt), args, 0, stream);
    if (info) {
        info->variant = v->name;
        info->grid = static_cast<int>(grid);
        info->block = v->nt;
        info->smem = 0;
        info->nchunks = 1;
        info->launches = 1;
    }
    return e;
}

bool stream_supported(const FusedArgs &a, int dtype) {
    return dtype == 0 && a.n <= 1024 && a.n % 4 == 0 &&
           (a.mode == MODE_APPLY_N || a.mode == MODE_APPLY_T || a.mode == MODE_SYM ||
            a.mode == MODE_TRANSFORM);
}

// When K1s replaces K1 (same-box grid n x h at 1 GiB, profiles/r2/k1s_grid_r2.txt): K1s is
// 5-39 % faster for n <= 512 at every h measured (2..32) and for n in (512, 1024] outside
// h = 9..11, where the persistent staged K1 is 1-2 % faster (C2: n = 1024, h = 10); U must stay
// L1-resident next to nothing else (h n 4 <= 128 KB).  (Multi-warp column groups for
// n in (1024, 4096], partial dots summed through shared memory, were measured 8-38 % slower than
// the persistent K1 for h >= 8 at n = 2048 / 4096 and were removed.)
bool stream_preferred(const FusedArgs &a) {
    const int64_t ub = a.h * a.n * 4;
    if (ub > (int64_t(128) << 10)) return false;
    if (a.n > 512 && a.h >= 9 && a.h <= 11) return false;
    // n in (512, 1024], h in [12, 16]: K1 with the reflectors in TMEM (K1t) is ahead -- same box
    // (tools/k1t_ab.py, profiles/r2/k1t_vs_k1s_r2.txt): n = 1024, h = 12 / 14 / 16: 341 / 402 /
    // 435 us vs 455 / 533 / 566; n = 768, h = 16: 660 vs 689-709; symmetric n = 1024, h = 12:
    // 620 vs 793
    if (a.n > 512 && a.h >= 12 && a.h <= 16) return false;
    return true;
}

}  // namespace hh
