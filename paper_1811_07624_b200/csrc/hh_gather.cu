// hh_gather.cu -- K3b: gather-fused pair distances on the transform-once points.
//
//   dist[j] = || Z[:, ia[j]] - Z[:, ib[j]] ||^2,   Z = diag(sqrt d) Q^T P   (K3a)
//
// which equals d_S(x_a, x_b) = ||L (x_a - x_b)||^2 with L = sqrt(Lambda) Q^T
// ("perform the transformation x <- L x before running the k-NN").
// A group of TPC threads owns PP pairs at a time; each thread issues 2*PP*CH
// independent 128-bit loads (both endpoints of every pair) before any arithmetic,
// so the gather keeps enough bytes in flight to stream from L2/HBM.
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

template <typename T, int TPC, int CH, int PP, int NT, bool FULL>
__global__ void __launch_bounds__(NT)
    hh_gather_dist_kernel(const T *__restrict__ Z, int64_t n, const int32_t *__restrict__ ia,
                          const int32_t *__restrict__ ib, int64_t npairs, T *__restrict__ dist) {
    using V = typename GV<T>::V;
    constexpr int E = GV<T>::E;
    const int nv = static_cast<int>(n / E);
    const int gt = threadIdx.x % TPC;
    const int64_t groups = static_cast<int64_t>(gridDim.x) * (NT / TPC);
    const int64_t g0 = static_cast<int64_t>(blockIdx.x) * (NT / TPC) + threadIdx.x / TPC;
    const V *Zv = reinterpret_cast<const V *>(Z);

    constexpr int KB = CH < 4 ? CH : 4;  // chunks loaded per step (register bound)
    for (int64_t base = g0 * PP; base < npairs; base += groups * PP) {
        const V *pa[PP], *pb[PP];
        bool pv[PP];
#pragma unroll
        for (int p = 0; p < PP; ++p) {
            const int64_t j = base + p;
            pv[p] = j < npairs;
            pa[p] = Zv + (pv[p] ? static_cast<int64_t>(__ldg(ia + j)) : 0) * nv;
            pb[p] = Zv + (pv[p] ? static_cast<int64_t>(__ldg(ib + j)) : 0) * nv;
        }
        T s[PP];
#pragma unroll
        for (int p = 0; p < PP; ++p) s[p] = T(0);
#pragma unroll
        for (int k0 = 0; k0 < CH; k0 += KB) {
            V za[PP][KB], zb[PP][KB];
#pragma unroll
            for (int p = 0; p < PP; ++p) {
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    const int v = gt + TPC * (k0 + k);
                    if (pv[p] && (FULL || v < nv)) {
                        za[p][k] = __ldg(pa[p] + v);
                        zb[p][k] = __ldg(pb[p] + v);
                    } else {
                        za[p][k] = V{};
                        zb[p][k] = V{};
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < PP; ++p) {
#pragma unroll
                for (int k = 0; k < KB; ++k) s[p] += GV<T>::sqd(za[p][k], zb[p][k]);
            }
        }
#pragma unroll
        for (int off = TPC / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int p = 0; p < PP; ++p) s[p] += __shfl_xor_sync(0xffffffffu, s[p], off);
        }
        if (gt == 0) {
#pragma unroll
            for (int p = 0; p < PP; ++p)
                if (base + p < npairs) dist[base + p] = s[p];
        }
    }
}

struct GVariant {
    const void *full;
    const void *ragged;
    int tpc, ch, pp, nt;
    const char *name;
};

#define HH_GVAR(T, TPC, CH, PP, NT, NAME)                                                     \
    GVariant {                                                                                \
        reinterpret_cast<const void *>(&hh_gather_dist_kernel<T, TPC, CH, PP, NT, true>),     \
            reinterpret_cast<const void *>(&hh_gather_dist_kernel<T, TPC, CH, PP, NT, false>), \
            TPC, CH, PP, NT, NAME                                                             \
    }

const GVariant kG32[] = {
    HH_GVAR(float, 8, 2, 4, 256, "gather_f32_tpc8_ch2"),    // n <= 64
    HH_GVAR(float, 8, 4, 4, 256, "gather_f32_tpc8_ch4"),    // n <= 128
    HH_GVAR(float, 16, 4, 2, 256, "gather_f32_tpc16_ch4"),  // n <= 256
    HH_GVAR(float, 32, 4, 2, 256, "gather_f32_tpc32_ch4"),  // n <= 512
    HH_GVAR(float, 32, 8, 1, 256, "gather_f32_tpc32_ch8"),  // n <= 1024
    HH_GVAR(float, 32, 16, 1, 256, "gather_f32_tpc32_ch16"),  // n <= 2048
    HH_GVAR(float, 32, 32, 1, 256, "gather_f32_tpc32_ch32"),  // n <= 4096
    HH_GVAR(float, 32, 64, 1, 128, "gather_f32_tpc32_ch64"),  // n <= 8192
};
const GVariant kG64[] = {
    HH_GVAR(double, 8, 4, 4, 256, "gather_f64_tpc8_ch4"),    // n <= 64
    HH_GVAR(double, 16, 4, 2, 256, "gather_f64_tpc16_ch4"),  // n <= 128
    HH_GVAR(double, 32, 4, 2, 256, "gather_f64_tpc32_ch4"),  // n <= 256
    HH_GVAR(double, 32, 8, 1, 256, "gather_f64_tpc32_ch8"),  // n <= 512
    HH_GVAR(double, 32, 16, 1, 256, "gather_f64_tpc32_ch16"),  // n <= 1024
    HH_GVAR(double, 32, 32, 1, 256, "gather_f64_tpc32_ch32"),  // n <= 2048
    HH_GVAR(double, 32, 64, 1, 128, "gather_f64_tpc32_ch64"),  // n <= 4096
};
#undef HH_GVAR

}  // namespace

cudaError_t launch_gather_dist(const void *Z, int64_t n, const int32_t *ia, const int32_t *ib,
                               int64_t npairs, void *dist, int dtype, cudaStream_t stream,
                               LaunchInfo *info) {
    const int E = dtype == 0 ? 4 : 2;
    const int64_t nv = n / E;
    const GVariant *tab = dtype == 0 ? kG32 : kG64;
    const int cnt = dtype == 0 ? static_cast<int>(sizeof(kG32) / sizeof(kG32[0]))
                               : static_cast<int>(sizeof(kG64) / sizeof(kG64[0]));
    const GVariant *v = nullptr;
    for (int i = 0; i < cnt; ++i)
        if (static_cast<int64_t>(tab[i].tpc) * tab[i].ch >= nv) {
            v = &tab[i];
            break;
        }
    if (!v) return cudaErrorNotSupported;
    const bool full = static_cast<int64_t>(v->tpc) * v->ch == nv;
    const void *fn = full ? v->full : v->ragged;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v->nt, 0);
    if (e != cudaSuccess) return e;
    const int64_t per_block = static_cast<int64_t>(v->nt / v->tpc) * v->pp;
    const int64_t need = (npairs + per_block - 1) / per_block;
    const int64_t cap = static_cast<int64_t>(std::max(occ, 1)) * device_attr().sm_count;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(need, cap)));
    void *args[] = {const_cast<void **>(&Z), &n, const_cast<int32_t **>(&ia),
                    const_cast<int32_t **>(&ib), &npairs, &dist};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(v->nt), args, 0, stream);
    if (info) {
        info->variant = v->name;
        info->grid = grid;
        info->block = v->nt;
        info->smem = 0;
        info->nchunks = 0;
        info->launches = 1;
    }
    return e;
}

}  // namespace hh
