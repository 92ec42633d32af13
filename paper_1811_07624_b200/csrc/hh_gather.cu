// hh_gather.cu -- K3b: gather-fused pair distances on the transform-once points.
//
//   dist[j] = || Z[:, ia[j]] - Z[:, ib[j]] ||^2,   Z = diag(sqrt d) Q^T P   (K3a)
//
// which equals d_S(x_a, x_b) = ||L (x_a - x_b)||^2 with L = sqrt(Lambda) Q^T
// ("perform the transformation x <- L x before running the k-NN").
// The pairs are first counting-sorted by their first point a on the device (a
// histogram, a single-CTA scan and an atomic scatter into a permutation); a group of
// TPC threads then owns one bucket: z_a is loaded once into registers and PP pairs of
// the bucket are gathered at a time (128-bit loads of z_b), so only one endpoint per
// pair crosses L2 -- half the bytes of a per-pair gather.
#include <algorithm>

#include "hh_internal.h"

namespace hh {

namespace {

template <typename T>
struct GV;
template <>
struct GV<float> {
    using V = float4;
    static constexpr int E = 4;
    __device__ static float sqd(const float4 &a, const float4 &b) {
        const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
        return (dx * dx + dy * dy) + (dz * dz + dw * dw);
    }
};
template <>
struct GV<double> {
    using V = double2;
    static constexpr int E = 2;
    __device__ static double sqd(const double2 &a, const double2 &b) {
        const double dx = a.x - b.x, dy = a.y - b.y;
        return dx * dx + dy * dy;
    }
};

struct GVariant {
    const void *full;
    const void *ragged;
    int tpc, ch, pp, nt;
    const char *name;
};


// ---------------------------------------------------------------------------------
// Bucketed gather: pairs grouped by their first point a (a counting sort on device),
// so z_a is read once per bucket (~P/M pairs share it) and only z_b is gathered per
// pair -- half the gathered bytes of the per-pair kernel.
// ---------------------------------------------------------------------------------
__global__ void bucket_hist_kernel(const int32_t *__restrict__ ia, int64_t npairs,
                                   int32_t *__restrict__ cnt) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < npairs;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(cnt + ia[j], 1);
}

// exclusive scan of cnt[0..M) into off[0..M] and cur[0..M), two levels: each CTA scans
// 4096 counts (4 per thread, int4 loads) and writes its total; then every CTA adds the sum
// of the totals before it (a few dozen values, summed in fixed order: deterministic).
// (One CTA scanning all of M had taken ~30 us at M = 65536.)
constexpr int kScanPer = 4096;
__global__ void __launch_bounds__(1024) bucket_scan_local_kernel(const int32_t *__restrict__ cnt,
                                                                 int64_t M,
                                                                 int32_t *__restrict__ off,
                                                                 int32_t *__restrict__ tot) {
    __shared__ int32_t wsum[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kScanPer + 4 * t;
    int4 v = make_int4(0, 0, 0, 0);
    if (i0 + 3 < M) {
        v = *reinterpret_cast<const int4 *>(cnt + i0);
    } else {
        if (i0 < M) v.x = cnt[i0];
        if (i0 + 1 < M) v.y = cnt[i0 + 1];
        if (i0 + 2 < M) v.z = cnt[i0 + 2];
    }
    const int32_t sthr = v.x + v.y + v.z + v.w;
    int32_t x = sthr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int32_t z = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        wsum[lane] = z;
    }
    __syncthreads();
    const int32_t run = (w ? wsum[w - 1] : 0) + x - sthr;
    int4 o;
    o.x = run;
    o.y = run + v.x;
    o.z = o.y + v.y;
    o.w = o.z + v.z;
    if (i0 + 3 < M) {
        *reinterpret_cast<int4 *>(off + i0) = o;
    } else {
        if (i0 < M) off[i0] = o.x;
        if (i0 + 1 < M) off[i0 + 1] = o.y;
        if (i0 + 2 < M) off[i0 + 2] = o.z;
    }
    if (t == 0) tot[blockIdx.x] = wsum[31];
}

__global__ void __launch_bounds__(1024) bucket_scan_add_kernel(const int32_t *__restrict__ tot,
                                                               int64_t M, int32_t *__restrict__ off,
                                                               int32_t *__restrict__ cur) {
    __shared__ int32_t base;
    if (threadIdx.x == 0) {
        int32_t b = 0;
        for (int c = 0; c < static_cast<int>(blockIdx.x); ++c) b += tot[c];
        base = b;
        if (blockIdx.x == gridDim.x - 1) off[M] = b + tot[blockIdx.x];
    }
    __syncthreads();
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kScanPer + 4 * threadIdx.x;
    for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        if (i < M) {
            const int32_t vv = off[i] + base;
            off[i] = vv;
            cur[i] = vv;
        }
    }
}

__global__ void bucket_scatter_kernel(const int32_t *__restrict__ ia, int64_t npairs,
                                      int32_t *__restrict__ cur, int32_t *__restrict__ perm) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < npairs;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        perm[atomicAdd(cur + ia[j], 1)] = static_cast<int32_t>(j);
}

// a group of TPC threads per bucket a: z_a in registers, PP pairs of the bucket in flight
template <typename T, int TPC, int CH, int PP, int NT, bool FULL>
__global__ void __launch_bounds__(NT)
    hh_gather_bucket_kernel(const T *__restrict__ Z, int64_t n, int64_t M,
                            const int32_t *__restrict__ off, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ ib, T *__restrict__ dist) {
    using V = typename GV<T>::V;
    constexpr int E = GV<T>::E;
    const int nv = static_cast<int>(n / E);
    const int gt = threadIdx.x % TPC;
    const int64_t groups = static_cast<int64_t>(gridDim.x) * (NT / TPC);
    const V *Zv = reinterpret_cast<const V *>(Z);
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * (NT / TPC) + threadIdx.x / TPC; a < M;
         a += groups) {
        const int32_t p0 = __ldg(off + a), p1 = __ldg(off + a + 1);
        if (p0 == p1) continue;
        V za[CH];
        const V *pa = Zv + a * nv;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int v = gt + TPC * k;
            za[k] = (FULL || v < nv) ? __ldg(pa + v) : V{};
        }
        for (int32_t q = p0; q < p1; q += PP) {
            int32_t jj[PP];
            const V *pb[PP];
#pragma unroll
            for (int p = 0; p < PP; ++p) {
                const bool ok = q + p < p1;
                jj[p] = ok ? __ldg(perm + q + p) : -1;
                pb[p] = Zv + (ok ? static_cast<int64_t>(__ldg(ib + jj[p])) : a) * nv;
            }
            T s[PP];
#pragma unroll
            for (int p = 0; p < PP; ++p) {
                s[p] = T(0);
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int v = gt + TPC * k;
                    if (FULL || v < nv) s[p] += GV<T>::sqd(za[k], __ldg(pb[p] + v));
                }
            }
#pragma unroll
            for (int o = TPC / 2; o > 0; o >>= 1) {
#pragma unroll
                for (int p = 0; p < PP; ++p) s[p] += __shfl_xor_sync(0xffffffffu, s[p], o);
            }
            if (gt == 0) {
#pragma unroll
                for (int p = 0; p < PP; ++p)
                    if (jj[p] >= 0) dist[jj[p]] = s[p];
            }
        }
    }
}

#define HH_GVAR_B(T, TPC, CH, PP, NT, NAME)                                                   \
    GVariant {                                                                                  \
        reinterpret_cast<const void *>(&hh_gather_bucket_kernel<T, TPC, CH, PP, NT, true>),     \
            reinterpret_cast<const void *>(&hh_gather_bucket_kernel<T, TPC, CH, PP, NT, false>), \
            TPC, CH, PP, NT, NAME                                                               \
    }

const GVariant kB32[] = {
    HH_GVAR_B(float, 8, 2, 4, 256, "bucket_f32_tpc8_ch2"),
    HH_GVAR_B(float, 8, 4, 4, 256, "bucket_f32_tpc8_ch4"),
    HH_GVAR_B(float, 16, 4, 4, 256, "bucket_f32_tpc16_ch4"),
    HH_GVAR_B(float, 32, 4, 8, 256, "bucket_f32_tpc32_ch4"),
    HH_GVAR_B(float, 32, 8, 2, 256, "bucket_f32_tpc32_ch8"),
    HH_GVAR_B(float, 32, 16, 2, 256, "bucket_f32_tpc32_ch16"),
    HH_GVAR_B(float, 32, 32, 1, 256, "bucket_f32_tpc32_ch32"),
    HH_GVAR_B(float, 32, 64, 1, 128, "bucket_f32_tpc32_ch64"),
};
const GVariant kB64[] = {
    HH_GVAR_B(double, 8, 4, 4, 256, "bucket_f64_tpc8_ch4"),
    HH_GVAR_B(double, 16, 4, 4, 256, "bucket_f64_tpc16_ch4"),
    HH_GVAR_B(double, 32, 4, 4, 256, "bucket_f64_tpc32_ch4"),
    HH_GVAR_B(double, 32, 8, 2, 256, "bucket_f64_tpc32_ch8"),
    HH_GVAR_B(double, 32, 16, 2, 256, "bucket_f64_tpc32_ch16"),
    HH_GVAR_B(double, 32, 32, 1, 256, "bucket_f64_tpc32_ch32"),
    HH_GVAR_B(double, 32, 64, 1, 128, "bucket_f64_tpc32_ch64"),
};
#undef HH_GVAR_B

}  // namespace

size_t bucket_ws_bytes(int64_t M, int64_t npairs) {
    auto r = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    return r(static_cast<size_t>(M) * 4) * 2 + r(static_cast<size_t>(M + 1) * 4) +
           r(static_cast<size_t>(npairs) * 4) + r(static_cast<size_t>((M + kScanPer - 1) / kScanPer) * 4);
}

namespace {
struct BucketWs {
    int32_t *cnt, *cur, *off, *perm, *tot;
};
BucketWs bucket_ws(void *ws, int64_t M, int64_t npairs) {
    auto r = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    char *w = static_cast<char *>(ws);
    BucketWs b;
    b.cnt = reinterpret_cast<int32_t *>(w);
    b.cur = reinterpret_cast<int32_t *>(w + r(static_cast<size_t>(M) * 4));
    b.off = reinterpret_cast<int32_t *>(w + 2 * r(static_cast<size_t>(M) * 4));
    b.perm = reinterpret_cast<int32_t *>(w + 2 * r(static_cast<size_t>(M) * 4) +
                                         r(static_cast<size_t>(M + 1) * 4));
    b.tot = b.perm + r(static_cast<size_t>(npairs) * 4) / 4;   // per-CTA scan totals
    return b;
}
}  // namespace

cudaError_t launch_bucket_sort(int64_t M, const int32_t *ia, int64_t npairs, void *ws,
                               cudaStream_t stream) {
    const BucketWs b = bucket_ws(ws, M, npairs);
    const int sms = device_attr().sm_count;
    cudaError_t e = cudaMemsetAsync(b.cnt, 0, static_cast<size_t>(M) * 4, stream);
    if (e != cudaSuccess) return e;
    const int g = static_cast<int>(std::min<int64_t>((npairs + 255) / 256, sms * 8));
    bucket_hist_kernel<<<g, 256, 0, stream>>>(ia, npairs, b.cnt);
    const int nsb = static_cast<int>((M + kScanPer - 1) / kScanPer);
    bucket_scan_local_kernel<<<nsb, 1024, 0, stream>>>(b.cnt, M, b.off, b.tot);
    bucket_scan_add_kernel<<<nsb, 1024, 0, stream>>>(b.tot, M, b.off, b.cur);
    bucket_scatter_kernel<<<g, 256, 0, stream>>>(ia, npairs, b.cur, b.perm);
    return cudaGetLastError();
}

cudaError_t launch_gather_bucketed(const void *Z, int64_t n, int64_t M, const int32_t *ia,
                                   const int32_t *ib, int64_t npairs, void *dist, void *ws,
                                   int dtype, cudaStream_t stream, LaunchInfo *info) {
    cudaError_t e = launch_bucket_sort(M, ia, npairs, ws, stream);
    if (e != cudaSuccess) return e;
    return launch_bucket_gather(Z, n, M, ib, npairs, dist, ws, dtype, stream, info);
}

cudaError_t launch_bucket_gather(const void *Z, int64_t n, int64_t M, const int32_t *ib,
                                 int64_t npairs, void *dist, void *ws, int dtype,
                                 cudaStream_t stream, LaunchInfo *info) {
    const BucketWs b = bucket_ws(ws, M, npairs);
    int32_t *off = b.off, *perm = b.perm;
    const int sms = device_attr().sm_count;
    cudaError_t e = cudaSuccess;

    const int E = dtype == 0 ? 4 : 2;
    const int64_t nv = n / E;
    const GVariant *tab = dtype == 0 ? kB32 : kB64;
    const int cntv = dtype == 0 ? static_cast<int>(sizeof(kB32) / sizeof(kB32[0]))
                                : static_cast<int>(sizeof(kB64) / sizeof(kB64[0]));
    const GVariant *v = nullptr;
    for (int i = 0; i < cntv; ++i)
        if (static_cast<int64_t>(tab[i].tpc) * tab[i].ch >= nv) {
            v = &tab[i];
            break;
        }
    if (!v) return cudaErrorNotSupported;
    const bool full = static_cast<int64_t>(v->tpc) * v->ch == nv;
    const void *fn = full ? v->full : v->ragged;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v->nt, 0);
    if (e != cudaSuccess) return e;
    const int64_t per_block = v->nt / v->tpc;
    const int64_t need = (M + per_block - 1) / per_block;
    const int64_t cap = static_cast<int64_t>(std::max(occ, 1)) * sms;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(need, cap)));
    void *args[] = {const_cast<void **>(&Z), &n, &M, &off, &perm, const_cast<int32_t **>(&ib),
                    &dist};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(v->nt), args, 0, stream);
    if (info) {
        info->variant = v->name;
        info->grid = grid;
        info->block = v->nt;
        info->smem = 0;
        info->nchunks = 0;
        info->launches = 5;   // histogram, scan (2), scatter, gather (+ one memset)
    }
    return e;
}

}  // namespace hh
