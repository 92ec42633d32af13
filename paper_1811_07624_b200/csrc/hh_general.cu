// hh_general.cu -- K1g: the fused reflector kernel for the shapes the vector kernels refuse.
//
// K1 / K1s / K1t move columns with 128-bit accesses and keep a column in the registers of at
// most 256 threads, so they need n*s to be a multiple of 16 bytes, 16-byte aligned pointers and
// n <= 8192 (fp32) / 4096 (fp64).  The paper's operator has no such restriction (Eq. 1-2,
// any n, any h), so every other shape runs here: element-wise accesses (pointers
// aligned to the element only), the CG columns of a CTA in shared memory, the reflectors read
// from global memory (L2-resident) once per CG columns.  Same arithmetic as K1 -- per reflector
// alpha = u^T x, x <- x - 2 alpha u ("4nh operations"), in the order of reading R1 -- and
// the same modes (apply N / T, symmetric, Mahalanobis transform and per-pair distance, the
// diagonal D of Eq. 1 on either side).
//
// A thread owns the elements r = tid + k*blockDim of every column of its CTA for the whole
// kernel, so only the dot products cross threads: xor-shuffle butterfly in the warp, one
// shared-memory slot per warp and column (two buffers: one CTA barrier per reflector), summed
// in warp order by every thread (deterministic; every thread holds the same alpha).
// Not a tuned path: it reads U from L2 once per CG columns (h n s bytes against 2 CG n s of
// HBM traffic), which bounds it at roughly 2 CG / h of the L2 rate; it exists so that the
// boundary takes every shape.
#include <algorithm>
#include <type_traits>

#include "hh_internal.h"

namespace hh {
namespace {

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

template <typename T, int CG>
__global__ void __launch_bounds__(256) hh_general_kernel(const FusedArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t n = a.n;
    const int h = static_cast<int>(a.h);
    const int nt = blockDim.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    T *xs = reinterpret_cast<T *>(smem_raw);   // [CG][n]
    T *red = xs + static_cast<size_t>(CG) * n; // [2][nw][CG]
    const T *U = static_cast<const T *>(a.U);
    const T *X = static_cast<const T *>(a.X);
    const T *vec = static_cast<const T *>(a.vec);
    const T *dsg = static_cast<const T *>(a.dsign);
    const int mode = a.mode;
    int par = 0;

    // sum the CG per-thread partials over the CTA; every thread returns with the same totals
    auto block_sum = [&](T (&p)[CG]) {
#pragma unroll
        for (int c = 0; c < CG; ++c) p[c] = warp_sum(p[c]);
        T *rb = red + static_cast<size_t>(par) * nw * CG;
        if (lane == 0) {
#pragma unroll
            for (int c = 0; c < CG; ++c) rb[warp * CG + c] = p[c];
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < CG; ++c) {
            T s = rb[c];
            for (int w = 1; w < nw; ++w) s += rb[w * CG + c];
            p[c] = s;
        }
        par ^= 1;
    };
    // x <- (I - 2 u u^T) x for the CTA's columns (Eq. 2)
    auto reflect = [&](int i) {
        const T *u = U + static_cast<int64_t>(i) * n;
        T p[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) p[c] = T(0);
        for (int64_t r = tid; r < n; r += nt) {
            const T ur = __ldg(u + r);
#pragma unroll
            for (int c = 0; c < CG; ++c) p[c] = fma(ur, xs[c * n + r], p[c]);
        }
        block_sum(p);
#pragma unroll
        for (int c = 0; c < CG; ++c) p[c] = T(-2) * p[c];
        for (int64_t r = tid; r < n; r += nt) {
            const T ur = __ldg(u + r);
#pragma unroll
            for (int c = 0; c < CG; ++c) xs[c * n + r] = fma(p[c], ur, xs[c * n + r]);
        }
    };
    auto pass_T = [&]() {   // Q^T: u_1 first (R1)
        for (int i = 0; i < h; ++i) reflect(i);
    };
    auto pass_N = [&]() {   // Q: u_h first
        for (int i = h - 1; i >= 0; --i) reflect(i);
    };
    auto scale = [&](const T *v, bool root) {
        for (int64_t r = tid; r < n; r += nt) {
            T f = __ldg(v + r);
            if (root) f = sqrt(f);
#pragma unroll
            for (int c = 0; c < CG; ++c) xs[c * n + r] *= f;
        }
    };

    const int64_t ngroups = (a.N + CG - 1) / CG;
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t j0 = g * CG;
        // columns (or pair differences) -> shared memory; columns past N are zero
#pragma unroll
        for (int c = 0; c < CG; ++c) {
            const int64_t j = j0 + c;
            const bool cv = j < a.N;
            if (mode == MODE_PAIR) {
                const T *pa = X + (cv ? static_cast<int64_t>(a.ia[j]) : 0) * n;
                const T *pb = X + (cv ? static_cast<int64_t>(a.ib[j]) : 0) * n;
                for (int64_t r = tid; r < n; r += nt) xs[c * n + r] = cv ? __ldg(pa + r) - __ldg(pb + r) : T(0);
            } else {
                const T *px = X + (cv ? j : 0) * n;
                for (int64_t r = tid; r < n; r += nt) xs[c * n + r] = cv ? __ldg(px + r) : T(0);
            }
        }
        if (a.dside & 1) scale(dsg, false);   // right factor: D first
        if (mode == MODE_APPLY_N) {
            pass_N();
        } else if (mode == MODE_SYM) {
            pass_T();
            scale(vec, false);
            pass_N();
        } else {
            pass_T();
        }
        if (mode == MODE_PAIR) {
            T s[CG];
#pragma unroll
            for (int c = 0; c < CG; ++c) s[c] = T(0);
            for (int64_t r = tid; r < n; r += nt) {
                const T dv = __ldg(vec + r);
#pragma unroll
                for (int c = 0; c < CG; ++c) s[c] = fma(dv, xs[c * n + r] * xs[c * n + r], s[c]);
            }
            block_sum(s);
            if (tid == 0) {
                T *dist = static_cast<T *>(a.Y);
#pragma unroll
                for (int c = 0; c < CG; ++c)
                    if (j0 + c < a.N) dist[j0 + c] = s[c];
            }
        } else {
            if (mode == MODE_TRANSFORM) scale(vec, true);
            if (a.dside & 2) scale(dsg, false);   // left factor: D last
            T *Y = static_cast<T *>(a.Y);
#pragma unroll
            for (int c = 0; c < CG; ++c) {
                const int64_t j = j0 + c;
                if (j < a.N)
                    for (int64_t r = tid; r < n; r += nt) Y[j * n + r] = xs[c * n + r];
            }
        }
        // (no barrier: a thread only ever touches its own elements of xs, and the reduction
        // buffers alternate)
    }
}

template <typename T, int CG>
cudaError_t launch_cg(const FusedArgs &a, int nt, size_t smem, int sm_count, int max_smem,
                      cudaStream_t stream, LaunchInfo *info, const char *name) {
    const void *fn = reinterpret_cast<const void *>(&hh_general_kernel<T, CG>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorNotSupported;
    const int64_t ngroups = (a.N + CG - 1) / CG;
    const int grid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ngroups, static_cast<int64_t>(occ) * sm_count)));
    FusedArgs b = a;
    void *args[] = {&b};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(nt), args, smem, stream);
    if (info) {
        info->variant = name;
        info->grid = grid;
        info->block = nt;
        info->smem = static_cast<int>(smem);
        info->nchunks = 1;
        info->launches = 1;
    }
    return e;
}

// Row re-pitch: dst[r][e] = e < ncopy ? src[r][e] : fill for e < nwrite (rows of ld_src / ld_dst
// elements).  Pads the columns of an unaligned problem to a 16-byte pitch (and back), so that
// the fast kernels can run on the padded copy.  A warp per row, lanes on consecutive elements
// (coalesced on both sides).
template <typename T>
__global__ void __launch_bounds__(256) repitch_rows_kernel(const T *__restrict__ src, int64_t ld_src,
                                                           T *__restrict__ dst, int64_t ld_dst,
                                                           int64_t rows, int ncopy, int nwrite, T fill) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = w0; r < rows; r += nw) {
        const T *s = src + r * ld_src;
        T *d = dst + r * ld_dst;
        int e = lane;
#pragma unroll 4
        for (; e < ncopy; e += 32) d[e] = __ldg(s + e);
        for (; e < nwrite; e += 32) d[e] = fill;
    }
}

size_t general_smem(int64_t n, int s, int cg, int nt) {
    return static_cast<size_t>(cg) * n * s + static_cast<size_t>(2) * (nt / 32) * cg * s;
}

int general_threads(int64_t n) { return n <= 64 ? 32 : n <= 256 ? 64 : n <= 1024 ? 128 : 256; }

}  // namespace

cudaError_t launch_repitch(const void *src, int64_t ld_src, void *dst, int64_t ld_dst, int64_t rows,
                           int64_t ncopy, int64_t nwrite, double fill, int dtype, cudaStream_t stream) {
    if (rows <= 0) return cudaSuccess;
    const int64_t want = (rows + 7) / 8;   // 8 warps per CTA
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(want, static_cast<int64_t>(device_attr().sm_count) * 16)));
    if (dtype == 0)
        repitch_rows_kernel<float><<<grid, 256, 0, stream>>>(
            static_cast<const float *>(src), ld_src, static_cast<float *>(dst), ld_dst, rows,
            static_cast<int>(ncopy), static_cast<int>(nwrite), static_cast<float>(fill));
    else
        repitch_rows_kernel<double><<<grid, 256, 0, stream>>>(
            static_cast<const double *>(src), ld_src, static_cast<double *>(dst), ld_dst, rows,
            static_cast<int>(ncopy), static_cast<int>(nwrite), fill);
    return cudaGetLastError();
}

bool general_supported(int64_t n, int dtype) {
    const int s = dtype == 0 ? 4 : 8;
    return n >= 1 && general_smem(n, s, 1, general_threads(n)) <=
                         static_cast<size_t>(device_attr().max_smem_optin);
}

namespace {
thread_local int t_scalar = 1;
}
int general_set_scalar(int on) {
    const int prev = t_scalar;
    t_scalar = on;
    return prev;
}

cudaError_t launch_general(const FusedArgs &a, int dtype, cudaStream_t stream, LaunchInfo *info) {
    // K1r first: the register-resident persistent kernel with one-element accesses
    if (t_scalar) {
        const cudaError_t e = launch_fused_scalar(a, dtype, stream, info);
        if (e != cudaErrorNotSupported) return e;
    }
    const DevAttr &da = device_attr();
    const int s = dtype == 0 ? 4 : 8;
    const int nt = general_threads(a.n);
    // four columns per CTA (a quarter of the reflector reads) while two such CTAs fit an SM
    const size_t s4 = general_smem(a.n, s, 4, nt);
    const bool four = 2 * s4 + 2048 <= static_cast<size_t>(da.max_smem_optin) && a.N >= 4;
    const size_t smem = four ? s4 : general_smem(a.n, s, 1, nt);
    if (smem > static_cast<size_t>(da.max_smem_optin)) return cudaErrorNotSupported;
    if (dtype == 0)
        return four ? launch_cg<float, 4>(a, nt, smem, da.sm_count, da.max_smem_optin, stream, info, "f32_general_c4")
                    : launch_cg<float, 1>(a, nt, smem, da.sm_count, da.max_smem_optin, stream, info, "f32_general_c1");
    return four ? launch_cg<double, 4>(a, nt, smem, da.sm_count, da.max_smem_optin, stream, info, "f64_general_c4")
                : launch_cg<double, 1>(a, nt, smem, da.sm_count, da.max_smem_optin, stream, info, "f64_general_c1");
}

}  // namespace hh
