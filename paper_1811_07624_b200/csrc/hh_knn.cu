// hh_knn.cu -- NEXT-f3: test-time k-nearest neighbours under the learned metric.
//
// The paper's deployment of the path: with S = Q diag(d) Q^T
// (reading R4) and L = diag(sqrt d) Q^T, "perform the transformation x <- L x before
// running the k-NN"; each point is transformed once (4nh operations instead of 2n^2)
// and neighbours are found by Euclidean distance between transformed points:
//
//   d_S(q, r) = || z_q - z_r ||^2 = ||z_q||^2 + ||z_r||^2 - 2 z_q . z_r,   z = L x.
//
// Steps (all on the GPU):
//   1. K3a (hh_fused.cu, MODE_TRANSFORM): Z = diag(sqrt d) Q^T P for queries and
//      references (one HBM read + write per point).
//   2. knn_pack_kernel: bf16 hi/lo split of Z (K padded to a multiple of 32) and the
//      fp32 squared norms.
//   3. knn_topk_kernel (tcgen05): a CTA owns 128 queries (resident in SMEM, MMA M) and
//      streams a range of reference tiles (128 refs, MMA N) through a TMA ring; the
//      dot products z_q . z_r accumulate in TMEM (bf16x3, fp32 accumulation); the
//      epilogue turns them into distances and keeps a per-query sorted top-k list in
//      registers (ties: smaller reference index first).
//   4. knn_merge_kernel: merges the per-split lists (k-way, same tie rule).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <mutex>

#include "hh_internal.h"
#include "hh_tc.cuh"

namespace hh {

namespace {

constexpr int kQ = 128;           // queries per CTA (MMA M)
constexpr int kRT = 256;          // references per tile (MMA N)
constexpr int kRStage = kRT * 64 * 2;   // one K slab of a tile, hi + lo (32 KB)
constexpr int kKS = 12;           // reference slab ring depth: maximum (runtime nks)
constexpr int kNAcc = 2;          // TMEM accumulators (2 x 256 columns)
constexpr int kKnnMaxK = 16;      // largest k
constexpr int kKnnMaxN = 256;     // largest n (K = n + 1 augmented, padded to 32)
constexpr int kKnnMaxNpad = 288;  // resident query tile: n_pad x 128 x 4 B <= 144 KB

size_t al(size_t x) { return (x + 1023) & ~static_cast<size_t>(1023); }

__device__ __forceinline__ uint16_t f2bf(float x) {
    uint16_t b;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(b) : "f"(x));
    return b;
}
__device__ __forceinline__ float bf2f(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// one warp per point: Zb[hi: row][0..n_pad), Zb[lo: M + row][..] and nrm[row] = ||z||^2.
// Column n is the augmentation that folds the reference norm into the tensor-core dot:
// queries carry 1, references -||z_r||^2 / 2, so the accumulator holds
// D = z_q . z_r - ||z_r||^2 / 2 and d_S(q, r) = ||z_q||^2 - 2 D.
__global__ void knn_pack_kernel(const float *__restrict__ Z, int64_t M, int n, int n_pad,
                                int is_query, uint16_t *__restrict__ Zb, float *__restrict__ nrm) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t row = w0; row < M; row += nw) {
        float ss = 0.f;
        for (int c = lane; c < n; c += 32) {
            const float v = Z[row * n + c];
            ss = fmaf(v, v, ss);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        const float aug = is_query ? 1.f : -0.5f * ss;
        for (int c = lane; c < n_pad; c += 32) {
            const float v = c < n ? Z[row * n + c] : (c == n ? aug : 0.f);
            const uint16_t h = f2bf(v);
            Zb[row * n_pad + c] = h;
            Zb[(M + row) * n_pad + c] = f2bf(v - bf2f(h));
        }
        if (lane == 0) nrm[row] = ss;
    }
}

struct BarsK {
    uint64_t qfull;
    uint64_t full[kKS], empty[kKS];
    uint64_t acc_full[kNAcc], acc_empty[kNAcc];
    uint32_t tmem;
    float thr[4 * kQ];   // per (column group, query): that group's k-th best distance
};

// grid (query tiles, splits).  18 warps: w0 TMA producer, w1 MMA issuer (+TMEM
// owner), w2-17 epilogue (TMEM lane quarter x column group; thread = query).  KM: the
// register top-k capacity (k <= KM).
template <int KM>
__global__ void __launch_bounds__(576, 1)
    knn_topk_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmR,
                    const float *__restrict__ qn, const float *__restrict__ rn, int64_t Mq,
                    int64_t Mr, int n_pad, int k, int tiles_per_split, float *__restrict__ pd,
                    int32_t *__restrict__ pi, int nks, int nk16) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int nslab = n_pad / 32;
    unsigned char *Qhi = smem;                        // nslab x 8 KB
    unsigned char *Qlo = smem + nslab * 8192;
    unsigned char *stg = smem + 2 * nslab * 8192;
    BarsK *bars = reinterpret_cast<BarsK *>(stg + nks * kRStage);
    auto Rhi = [&](int s) { return stg + s * kRStage; };
    auto Rlo = [&](int s) { return stg + s * kRStage + kRStage / 2; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qt = blockIdx.x, split = blockIdx.y;
    const int64_t rtiles = (Mr + kRT - 1) / kRT;
    const int64_t t0 = static_cast<int64_t>(split) * tiles_per_split;
    const int64_t t1 = rtiles < t0 + tiles_per_split ? rtiles : t0 + tiles_per_split;
    if (threadIdx.x == 0) {
        mbar_init(&bars->qfull, 1);
        for (int s = 0; s < nks; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int i = 0; i < 4 * kQ; ++i) bars->thr[i] = FLT_MAX;
        for (int a = 0; a < kNAcc; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 512);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<kNAcc * kRT>(&bars->tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = bars->tmem;

    if (warp == 0) {
        if (lane == 0) {
            tc::prefetch_tmap(&tmQ);
            tc::prefetch_tmap(&tmR);
            mbar_arrive_expect_tx(&bars->qfull, static_cast<uint32_t>(nslab) * 16384u);
            for (int c = 0; c < nslab; ++c) {
                tc::tma_load_2d(Qhi + c * 8192, &tmQ, c * 32, qt * kQ, &bars->qfull);
                tc::tma_load_2d(Qlo + c * 8192, &tmQ, c * 32, static_cast<int>(Mq) + qt * kQ,
                                &bars->qfull);
            }
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = t0; t < t1; ++t) {
                for (int c = 0; c < nslab; ++c) {
                    mbar_wait(&bars->empty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&bars->full[s], static_cast<uint32_t>(kRStage));
                    tc::tma_load_2d(Rhi(s), &tmR, c * 32, static_cast<int>(t * kRT), &bars->full[s]);
                    tc::tma_load_2d(Rlo(s), &tmR, c * 32, static_cast<int>(Mr + t * kRT),
                                    &bars->full[s]);
                    if (++s == nks) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // the whole warp runs the issue loop (uniform descriptors); one lane issues
        const uint32_t idesc = tc::idesc_bf16(kQ, kRT);
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0;
        mbar_wait(&bars->qfull, 0);
        tc::fence_after_sync();
        const uint32_t qh = smem_u32(Qhi), ql = smem_u32(Qlo);
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&bars->acc_empty[a], aph ^ 1u);
            tc::fence_after_sync();
            const uint32_t d = tbase + static_cast<uint32_t>(a * kRT);
            for (int c = 0; c < nslab; ++c) {
                mbar_wait(&bars->full[s], ph);
                tc::fence_after_sync();
                const uint32_t rh = smem_u32(Rhi(s)), rl = smem_u32(Rlo(s));
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    if (2 * c + kk >= nk16) break;   // all-zero K16 step of the padding
                    const uint64_t ah = tc::sdesc_sw64(qh + c * 8192 + kk * 32);
                    const uint64_t alo = tc::sdesc_sw64(ql + c * 8192 + kk * 32);
                    const uint64_t bh = tc::sdesc_sw64(rh + kk * 32), blo = tc::sdesc_sw64(rl + kk * 32);
                    tc::mma_bf16_w(d, ah, bh, idesc, (c | kk) != 0);
                    tc::mma_bf16_w(d, ah, blo, idesc, 1u);
                    tc::mma_bf16_w(d, alo, bh, idesc, 1u);
                }
                tc::mma_commit_w(&bars->empty[s]);
                if (++s == nks) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            tc::mma_commit_w(&bars->acc_full[a]);
            if (++a == kNAcc) {
                a = 0;
                aph ^= 1u;
            }
        }
        __syncwarp();
    } else {
        // 16 epilogue warps: lane quarter q (thread = query), column group grp (32 of
        // the 128 references of a tile).  The accumulator already holds
        // D = z_q.z_r - ||z_r||^2/2 (augmented K column), so per reference the streaming
        // loop is one compare into a hit mask: d_S < worst  <=>  D > (||z_q||^2 - worst)/2.
        // The rare insertions run off the mask, outside the streaming loop.
        const int q = warp & 3, grp = (warp - 2) >> 2;
        const int qi = q * 32 + lane;
        const int64_t row = static_cast<int64_t>(qt) * kQ + qi;
        const float qnorm = row < Mq ? qn[row] : 0.f;
        volatile float *thr_s = bars->thr;   // read racy on purpose: values only decrease
        float bd[KM];
        int32_t bi[KM];
#pragma unroll
        for (int e = 0; e < KM; ++e) {
            bd[e] = FLT_MAX;
            bi[e] = -1;
        }
        float worst = FLT_MAX;   // bd[k-1], kept in a register (no dynamic indexing)
        int a = 0;
        uint32_t aph = 0;
        // one 32-reference chunk of this group's columns (ascending j)
        auto chunk = [&](float (&v)[32], int64_t j0, bool first) {
            const int jvalid = Mr - j0 >= 32 ? 32 : static_cast<int>(Mr - j0);   // may be <= 0
            // the first tile fills the empty list branch-free (every entry would be a hit)
            if (first) {
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    float cd = fmaf(-2.f, v[e], qnorm);
                    int32_t ci = static_cast<int32_t>(j0 + e);
                    if (e >= jvalid) cd = FLT_MAX;
#pragma unroll
                    for (int u = 0; u < KM; ++u) {
                        const bool sw = u < k && cd < bd[u];
                        const float td = bd[u];
                        const int32_t ti = bi[u];
                        bd[u] = sw ? cd : td;
                        bi[u] = sw ? ci : ti;
                        cd = sw ? td : cd;
                        ci = sw ? ti : ci;
                    }
                }
#pragma unroll
                for (int u = 0; u < KM; ++u)
                    if (u == k - 1) worst = bd[u];
                thr_s[grp * kQ + qi] = worst;
                return;
            }
            // prune with the best k-th distance of the query's four column groups (a
            // candidate worse than any group's k-th best cannot be in the top k; <= keeps
            // exact ties for the index rule of the final merge)
            float gw = worst;
#pragma unroll
            for (int g = 0; g < 4; ++g) gw = fminf(gw, thr_s[g * kQ + qi]);
            // (a relative margin keeps every candidate whose rounded distance can reach gw;
            // the exact decision is the insertion's cd < worst)
            const float c = 0.5f * (qnorm - gw) - 1e-6f * (fabsf(qnorm) + fabsf(gw));
            uint32_t hit = 0;
#pragma unroll
            for (int e = 0; e < 32; ++e) hit |= (v[e] >= c ? 1u : 0u) << e;
            if (jvalid < 32) hit &= jvalid > 0 ? (0xffffffffu >> (32 - jvalid)) : 0u;
            const float worst0 = worst;
            while (hit) {   // ascending j: an equal distance keeps the earlier reference
                const int e = __ffs(hit) - 1;
                hit &= hit - 1;
                // v[e] by a 5-level select tree (no dynamic register indexing)
                float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
                for (int u = 0; u < 16; ++u) t16[u] = (e & 16) ? v[u + 16] : v[u];
#pragma unroll
                for (int u = 0; u < 8; ++u) t8[u] = (e & 8) ? t16[u + 8] : t16[u];
#pragma unroll
                for (int u = 0; u < 4; ++u) t4[u] = (e & 4) ? t8[u + 4] : t8[u];
#pragma unroll
                for (int u = 0; u < 2; ++u) t2[u] = (e & 2) ? t4[u + 2] : t4[u];
                float cd = fmaf(-2.f, (e & 1) ? t2[1] : t2[0], qnorm);
                if (!(cd < worst)) continue;
                int32_t ci = static_cast<int32_t>(j0 + e);
#pragma unroll
                for (int u = 0; u < KM; ++u) {
                    if (u < k) {
                        const bool sw = cd < bd[u];
                        const float td = bd[u];
                        const int32_t ti = bi[u];
                        bd[u] = sw ? cd : td;
                        bi[u] = sw ? ci : ti;
                        cd = sw ? td : cd;
                        ci = sw ? ti : ci;
                    }
                }
#pragma unroll
                for (int u = 0; u < KM; ++u)
                    if (u == k - 1) worst = bd[u];
            }
            if (worst != worst0) thr_s[grp * kQ + qi] = worst;
        };
        for (int64_t t = t0; t < t1; ++t) {
            // group grp owns columns [64 grp, 64 grp + 64) of the 256-reference tile
            const int64_t jg = t * kRT + grp * 64;
            mbar_wait(&bars->acc_full[a], aph);
            tc::fence_after_sync();
            const uint32_t tcol = tbase + (static_cast<uint32_t>(q * 32) << 16) +
                                  static_cast<uint32_t>(a * kRT + grp * 64);
            float v[32];
            tc::tmem_ld32(tcol, v);
            chunk(v, jg, t == t0);
            tc::tmem_ld32(tcol + 32, v);
            tc::fence_before_sync();
            tc::mbar_arrive(&bars->acc_empty[a]);   // both chunks are in registers / done
            if (++a == kNAcc) {
                a = 0;
                aph ^= 1u;
            }
            chunk(v, jg + 32, false);
        }
        // merge the four column groups' lists of each query through shared memory (the
        // reference ring is free: every MMA has completed)
        float *md = reinterpret_cast<float *>(stg);
        int32_t *mi = reinterpret_cast<int32_t *>(stg + 4 * kQ * kKnnMaxK * 4);
        fence_proxy_async_smem();
#pragma unroll
        for (int u = 0; u < KM; ++u) {
            if (u < k) {
                md[(grp * kQ + qi) * kKnnMaxK + u] = bd[u];
                mi[(grp * kQ + qi) * kKnnMaxK + u] = bi[u];
            }
        }
        named_bar_sync(1, 512);
        if (grp == 0 && row < Mq) {
            int pos[4] = {0, 0, 0, 0};
            const int64_t o = (static_cast<int64_t>(split) * Mq + row) * k;
            for (int u = 0; u < k; ++u) {
                int best = -1;
                float bdv = 0.f;
                int32_t biv = 0;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (pos[g] >= k) continue;
                    const int32_t idx = mi[(g * kQ + qi) * kKnnMaxK + pos[g]];
                    if (idx < 0) continue;
                    const float dv = md[(g * kQ + qi) * kKnnMaxK + pos[g]];
                    if (best < 0 || dv < bdv || (dv == bdv && idx < biv)) {
                        best = g;
                        bdv = dv;
                        biv = idx;
                    }
                }
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    if (g == best) ++pos[g];
                pd[o + u] = best >= 0 ? bdv : FLT_MAX;
                pi[o + u] = best >= 0 ? biv : -1;
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_free<kNAcc * kRT>(tbase);
}

// thread per query: k-way merge of the sorted per-split lists, ties by smaller index
__global__ void knn_merge_kernel(const float *__restrict__ pd, const int32_t *__restrict__ pi,
                                 int64_t Mq, int k, int splits, float *__restrict__ od,
                                 int32_t *__restrict__ oi) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= Mq) return;
    int pos[64];
    for (int s = 0; s < splits; ++s) pos[s] = 0;
    for (int u = 0; u < k; ++u) {
        int best = -1;
        float bdv = 0.f;
        int32_t biv = 0;
        for (int s = 0; s < splits; ++s) {
            if (pos[s] >= k) continue;
            const int64_t o = (static_cast<int64_t>(s) * Mq + q) * k + pos[s];
            const int32_t idx = pi[o];
            if (idx < 0) continue;
            const float dv = pd[o];
            if (best < 0 || dv < bdv || (dv == bdv && idx < biv)) {
                best = s;
                bdv = dv;
                biv = idx;
            }
        }
        if (best >= 0) ++pos[best];
        od[q * k + u] = best >= 0 ? bdv : FLT_MAX;
        oi[q * k + u] = best >= 0 ? biv : -1;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
std::once_flag g_enc_once;
// the large dynamic shared-memory opt-in belongs to each device's context: once per device
constexpr int kKnnMaxDev = 64;
std::once_flag g_knn_attr_once[kKnnMaxDev];
cudaError_t g_knn_attr_err[kKnnMaxDev];

bool make_map_bf16(CUtensorMap *m, const void *base, uint64_t inner, uint64_t outer, uint32_t rows) {
    std::call_once(g_enc_once, []() {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!g_enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {32, rows};
    cuuint32_t es[2] = {1, 1};
    return g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

constexpr size_t kKnnSmemMax = 232448;
int knn_nks(int n_pad) {   // reference ring stages that fit next to the resident queries
    const long r = (static_cast<long>(kKnnSmemMax) - 2 * (n_pad / 32) * 8192 -
                    static_cast<long>(sizeof(BarsK)) - 1024) / kRStage;
    return static_cast<int>(std::max(2L, std::min(static_cast<long>(kKS), r)));
}
size_t knn_smem(int n_pad) {
    return static_cast<size_t>(2 * (n_pad / 32) * 8192) + knn_nks(n_pad) * kRStage + sizeof(BarsK) +
           1024;
}

}  // namespace

KnnPlan knn_plan(int64_t n, int64_t Mr, int64_t Mq, int k, int sm_count) {
    KnnPlan p{};
    p.n = n;
    p.Mr = Mr;
    p.Mq = Mq;
    p.k = k;
    p.n_pad = static_cast<int>((n + 1 + 31) / 32 * 32);   // + the augmentation column
    const int64_t qtiles = (Mq + kQ - 1) / kQ;
    const int64_t rtiles = (Mr + kRT - 1) / kRT;
    // one CTA per SM (registers): pick the split count whose CTA total fills the last
    // wave best (ties: fewer splits), keeping >= 8 reference tiles per CTA
    int64_t splits = 1;
    double best_eff = -1.0;
    for (int64_t sp = 1; sp <= 64 && sp <= rtiles; ++sp) {
        if (sp > 1 && (rtiles + sp - 1) / sp < 8) break;
        const int64_t ctas = qtiles * sp;
        const int64_t waves = (ctas + sm_count - 1) / sm_count;
        const double eff = static_cast<double>(ctas) / static_cast<double>(waves * sm_count);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            splits = sp;
        }
    }
    p.tiles_per_split = static_cast<int>((rtiles + splits - 1) / splits);
    p.splits = static_cast<int>((rtiles + p.tiles_per_split - 1) / p.tiles_per_split);
    size_t off = 0;
    auto take = [&](size_t b) {
        const size_t o = off;
        off += al(b);
        return o;
    };
    p.off_zr = take(static_cast<size_t>(Mr) * n * 4);
    p.off_zq = take(static_cast<size_t>(Mq) * n * 4);
    p.off_zrb = take(static_cast<size_t>(Mr) * p.n_pad * 2 * 2);
    p.off_zqb = take(static_cast<size_t>(Mq) * p.n_pad * 2 * 2);
    p.off_rn = take(static_cast<size_t>(Mr) * 4);
    p.off_qn = take(static_cast<size_t>(Mq) * 4);
    p.off_pd = take(static_cast<size_t>(p.splits) * Mq * k * 4);
    p.off_pi = take(static_cast<size_t>(p.splits) * Mq * k * 4);
    p.bytes = off;
    return p;
}

bool knn_supported(int64_t n, int64_t Mr, int64_t Mq, int k) {
    return n >= 1 && n <= kKnnMaxN && k >= 1 &&
           k <= kKnnMaxK && Mr >= k && Mq >= 1 && 2 * Mr < (int64_t(1) << 31) &&
           2 * Mq < (int64_t(1) << 31);
}

cudaError_t launch_knn(const KnnPlan &p, const float *U, int64_t h, const float *d,
                       const float *Pr, const float *Pq, int32_t *nn_idx, float *nn_dist, void *ws,
                       cudaStream_t stream, LaunchInfo *info, bool general) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kKnnMaxDev) return cudaErrorInvalidDevice;
    std::call_once(g_knn_attr_once[dev], [dev]() {
        const int sm = static_cast<int>(kKnnSmemMax);
        cudaError_t &err = g_knn_attr_err[dev];
        err = cudaFuncSetAttribute(knn_topk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(knn_topk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(knn_topk_kernel<kKnnMaxK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    });
    if (g_knn_attr_err[dev] != cudaSuccess) return g_knn_attr_err[dev];
    char *w = static_cast<char *>(ws);
    float *Zr = reinterpret_cast<float *>(w + p.off_zr);
    float *Zq = reinterpret_cast<float *>(w + p.off_zq);
    uint16_t *Zrb = reinterpret_cast<uint16_t *>(w + p.off_zrb);
    uint16_t *Zqb = reinterpret_cast<uint16_t *>(w + p.off_zqb);
    float *rn = reinterpret_cast<float *>(w + p.off_rn);
    float *qn = reinterpret_cast<float *>(w + p.off_qn);
    float *pd = reinterpret_cast<float *>(w + p.off_pd);
    int32_t *pi = reinterpret_cast<int32_t *>(w + p.off_pi);

    // 1. transform once: Z = diag(sqrt d) Q^T P
    for (int which = 0; which < 2; ++which) {
        FusedArgs a{};
        a.U = U;
        a.X = which ? Pq : Pr;
        a.Y = which ? Zq : Zr;
        a.vec = d;
        a.n = p.n;
        a.h = h;
        a.N = which ? p.Mq : p.Mr;
        a.mode = MODE_TRANSFORM;
        // (K1g when n * 4 is not a multiple of 16 bytes or an operand is only element-aligned)
        cudaError_t e = general ? launch_general(a, 0, stream, nullptr)
                                : launch_fused(a, 0, stream, nullptr);
        if (e != cudaSuccess) return e;
    }
    // 2. bf16 hi/lo split + squared norms
    const int sms = device_attr().sm_count;
    knn_pack_kernel<<<sms * 4, 256, 0, stream>>>(Zr, p.Mr, static_cast<int>(p.n), p.n_pad, 0, Zrb, rn);
    knn_pack_kernel<<<sms * 4, 256, 0, stream>>>(Zq, p.Mq, static_cast<int>(p.n), p.n_pad, 1, Zqb, qn);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // 3. distances on the tensor cores + per-query top-k
    CUtensorMap mQ, mR;
    if (!make_map_bf16(&mQ, Zqb, p.n_pad, 2 * p.Mq, kQ) ||
        !make_map_bf16(&mR, Zrb, p.n_pad, 2 * p.Mr, kRT))
        return cudaErrorNotSupported;
    const dim3 grid(static_cast<unsigned>((p.Mq + kQ - 1) / kQ), static_cast<unsigned>(p.splits));
    const size_t sm = knn_smem(p.n_pad);
    if (p.k <= 4)
        knn_topk_kernel<4><<<grid, 576, sm, stream>>>(mQ, mR, qn, rn, p.Mq, p.Mr, p.n_pad, p.k,
                                                      p.tiles_per_split, pd, pi, knn_nks(p.n_pad),
            static_cast<int>((p.n + 1 + 15) / 16));
    else if (p.k <= 8)
        knn_topk_kernel<8><<<grid, 576, sm, stream>>>(mQ, mR, qn, rn, p.Mq, p.Mr, p.n_pad, p.k,
                                                      p.tiles_per_split, pd, pi, knn_nks(p.n_pad),
            static_cast<int>((p.n + 1 + 15) / 16));
    else
        knn_topk_kernel<kKnnMaxK><<<grid, 576, sm, stream>>>(mQ, mR, qn, rn, p.Mq, p.Mr, p.n_pad,
                                                             p.k, p.tiles_per_split, pd, pi, knn_nks(p.n_pad),
            static_cast<int>((p.n + 1 + 15) / 16));
    // 4. merge the per-split lists
    knn_merge_kernel<<<static_cast<int>((p.Mq + 127) / 128), 128, 0, stream>>>(
        pd, pi, p.Mq, p.k, p.splits, nn_dist, nn_idx);
    if (info) {
        info->variant = "knn_bf16x3_tcgen05_topk";
        info->grid = static_cast<int>(grid.x * grid.y);
        info->block = 576;
        info->smem = static_cast<int>(knn_smem(p.n_pad));
        info->nchunks = p.splits;
        info->launches = 6;   // 2 transforms, 2 packs, distance/top-k, merge
    }
    return cudaGetLastError();
}

}  // namespace hh
