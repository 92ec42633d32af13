// hh_internal.h -- declarations shared by the libhh.so translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hh {

enum Mode : int {
    MODE_APPLY_N = 0,    // Y = Q X        (u_h first)
    MODE_APPLY_T = 1,    // Y = Q^T X      (u_1 first)
    MODE_SYM = 2,        // Y = Q diag(vec) Q^T X
    MODE_TRANSFORM = 3,  // Y = diag(sqrt(vec)) Q^T X       (Mahalanobis transform-once)
    MODE_PAIR = 4        // dist[j] = sum_r vec_r (Q^T (X[:,ia_j] - X[:,ib_j]))_r^2
};

struct FusedArgs {
    const void *U;      // (h, n) row-major reflectors
    const void *X;      // (N, n) columns (or points for MODE_PAIR)
    void *Y;            // (N, n) output columns (or dist[npairs] for MODE_PAIR)
    const void *vec;    // lambda (SYM) or d (TRANSFORM / PAIR), n values
    const int32_t *ia;  // MODE_PAIR
    const int32_t *ib;  // MODE_PAIR
    int64_t n, h, N;    // N = #columns, or #pairs in MODE_PAIR
    int mode;
    int R;              // reflectors per shared-memory U chunk
    int nchunks;        // ceil(h / R); 1 = U resident for the whole kernel
    int stage_x;        // 1 = stage column tiles through shared memory (bulk copy)
    int nbatches;       // batches per unit (uniform over the grid)
    const void *dsign;  // NEXT-f1: the diagonal D of Eq. 1 (n values) or NULL
    int dside;          // bit 0: x <- D x before the reflectors, bit 1: y <- D y after
    int qr;             // NEXT-f2: u_i[r] = 0 for r < i (partial-QR reflectors)
    int l2pf;           // unstaged columns: prefetch the tile this many batches ahead into L2
    int tcols;          // K1t: TMEM columns allocated per CTA (power of 2 >= 32)
};

struct LaunchInfo {
    const char *variant = nullptr;
    int grid = 0, block = 0, smem = 0, nchunks = 0;
    int launches = 0;   // kernels this call enqueued
};

// Launch the fused reflector kernel (K1 / K2 / K3a / K3c).  dtype: 0 f32, 1 f64.
// Returns cudaSuccess or the launch error; cudaErrorNotSupported if n is too big.
cudaError_t launch_fused(FusedArgs a, int dtype, cudaStream_t stream, LaunchInfo *info);

// K3b, bucketed: pairs counting-sorted by their first point on device (histogram, scan,
// scatter), then one z_a load per bucket; needs bucket_ws_bytes(M, npairs) of scratch.
size_t bucket_ws_bytes(int64_t M, int64_t npairs);
cudaError_t launch_gather_bucketed(const void *Z, int64_t n, int64_t M, const int32_t *ia,
                                   const int32_t *ib, int64_t npairs, void *dist, void *ws,
                                   int dtype, cudaStream_t stream, LaunchInfo *info);
// ... the same in two halves: the counting sort of the pairs by ia (memset, histogram, scan,
// scatter: needs only ia) and the gather (needs the sort and Z), so that the sort can run on a
// second stream beside the transform K3a
cudaError_t launch_bucket_sort(int64_t M, const int32_t *ia, int64_t npairs, void *ws,
                               cudaStream_t stream);
cudaError_t launch_bucket_gather(const void *Z, int64_t n, int64_t M, const int32_t *ib,
                                 int64_t npairs, void *dist, void *ws, int dtype,
                                 cudaStream_t stream, LaunchInfo *info);

// A/B hook (hh_debug_k1): force an alternative fused variant (-1: none), grid multiplier.
void k1_set_debug(int alt, int gridx);
// K1s (hh_stream.cu): the non-persistent streaming form of K1 for fp32 n <= 1024
bool stream_supported(const FusedArgs &a, int dtype);
bool stream_preferred(const FusedArgs &a);   // the measured K1 / K1s policy
cudaError_t launch_stream(const FusedArgs &a, cudaStream_t stream, LaunchInfo *info);
int k1_set_prefetch(int dist);
int k1_set_tmem(int on);      // A/B hook (hh_debug_k1_tmem): -1 policy, 0 never, 1 when eligible; previous
int k7_set_rows(int rw);      // A/B hook (hh_debug_k7_rows): K7 rows per warp pass; previous
int k1_set_blocked(int on);   // A/B hook (hh_debug_k1_blocked): K1w -1 policy, 0 never, 1 when K1t runs; previous
int k1_set_stream(int on);   // A/B hook (hh_debug_k1_stream): -1 auto, 0 K1, 1 K1s; previous

// K8 (hh_shf.cu): the SHF objective C(u) and its gradient for K candidates (NEXT-f4)
size_t shf_ws_bytes(int64_t n, int64_t K, int dtype);
cudaError_t launch_shf(int64_t n, const void *A, const void *B, const void *Uc, int64_t K, void *cost,
                       void *grad, int dtype, void *ws, cudaStream_t stream, LaunchInfo *info);

// Largest n the vector kernels support for this dtype.
int64_t max_n(int dtype);

// K1g (hh_general.cu): the same modes for any n whose column fits in shared memory and
// operands aligned to the element only (scalar accesses; the shapes K1 refuses).
bool general_supported(int64_t n, int dtype);
cudaError_t launch_general(const FusedArgs &a, int dtype, cudaStream_t stream, LaunchInfo *info);
// K1r (hh_fused_sc.cu): the persistent fused kernel with one-element accesses, for the same
// shapes while n is within the K1 tables and U fits in shared memory; cudaErrorNotSupported
// otherwise (launch_general tries it first)
cudaError_t launch_fused_scalar(FusedArgs a, int dtype, cudaStream_t stream, LaunchInfo *info);
// rows of ld_src elements -> rows of ld_dst elements: the first ncopy copied, then `fill` up to
// nwrite (pads an unaligned problem to a 16-byte pitch, and strips the pad again)
cudaError_t launch_repitch(const void *src, int64_t ld_src, void *dst, int64_t ld_dst, int64_t rows,
                           int64_t ncopy, int64_t nwrite, double fill, int dtype, cudaStream_t stream);
int k1r_set_stage(int on);  // A/B / test hook (hh_debug_k1r_stage): K1r staged column tiles (default 1) or direct loads (0); previous
int k1r_set_tmem(int on);   // A/B / test hook (hh_debug_k1r_tmem): K1r with U in TMEM (default 1) or shared memory (0); previous
int general_set_scalar(int on);   // A/B / test hook (hh_debug_general_scalar): 1 K1r first (default), 0 K1g only

// Device attributes (cached per device, thread-safe).
struct DevAttr {
    int sm_count = 0;
    int max_smem_optin = 0;
    int l2_bytes = 0;
};
const DevAttr &device_attr();

}  // namespace hh

namespace hh {

// ---- K4/K5 compact-WY tensor-core path (hh_wy.cu) ----
enum WyKind : int { WY_APPLY_N = 0, WY_APPLY_T = 1, WY_SYM = 2 };
struct WyPlan {
    int kind = 0;
    int64_t n = 0, h = 0, N = 0;
    int b = 0, nblk = 0, h_pad = 0, extra = 0, nsplit = 0, gram_rows = 0;
    int qr = 0;   // NEXT-f2: block k's W rows (and V rows) are zero above row k*b
    int64_t n_pad = 0;
    size_t off_wf = 0, off_wb = 0, off_sp = 0, off_s = 0, off_t = 0, off_v = 0, off_v2 = 0,
           off_asym = 0, off_vf = 0, off_vpf = 0, off_pp = 0, off_p = 0, off_m = 0, off_gt = 0,
           off_ld = 0, off_part = 0, off_flag = 0;
    // K5f (single dataflow launch): G ring, partial slots, per-(pass, tile) counters
    int np = 0, ntiles = 0, fD = 0, fnkc = 0, fkw = 0, fG = 1;
    size_t off_ring = 0, off_fpart = 0, off_cnt = 0;
    size_t bytes = 0;
};
WyPlan wy_plan(int kind, int64_t n, int64_t h, int64_t N);
void wy_set_timeline(unsigned long long *buf);   // debug: per-role barrier wait cycles
int wy_set_ts_min(int kw);                       // test: TS-mode update threshold (prev.)
// test / A-B hook: K5f dataflow launch on (1, default) or off (0); project-CTA count
// (0 = default); returns the previous on/off
int wy_set_flow(int on, int project_ctas);
void wy_set_flow_knobs(const int *k, int cnt);   // [on, P, nkc, rseg, D, G, pol]
int wy_set_pdl(int on);   // A/B hook: bit 0 PDL launches, bit 1 prep beside the first projection
int wy_set_tsa(int on);       // A/B hook: K5a converts X into TMEM (b <= 128); previous
int wy_set_symfuse(int on);   // A/B hook: the symmetric folded block's operands in one launch
bool wy_supported(int kind, int64_t n, int64_t h, int64_t N);   // incl. the pass cap
// Y = Q X / Q^T X / Q diag(lam) Q^T X by the compact-WY block program (fp32 in/out).
// debug_stop_blocks >= 0: run the preparation and only the first projection (test hook).
// dsign/dside: optional diagonal D (bit 0: right factor, D applied first; bit 1: left
// factor, D applied last), fused into the first project/update and the last update.
cudaError_t launch_wy(const WyPlan &p, const float *U, const float *lam, const float *X, float *Y,
                      void *ws, cudaStream_t stream, LaunchInfo *info, int debug_stop_blocks = -1,
                      const float *dsign = nullptr, int dside = 0);

}  // namespace hh

namespace hh {

// ---- NEXT-f3: test-time k-NN under the learned metric (hh_knn.cu) ----
struct KnnPlan {
    int64_t n = 0, Mr = 0, Mq = 0;
    int k = 0, n_pad = 0, splits = 0, tiles_per_split = 0;
    size_t off_zr = 0, off_zq = 0, off_zrb = 0, off_zqb = 0, off_rn = 0, off_qn = 0, off_pd = 0,
           off_pi = 0;
    size_t bytes = 0;
};
KnnPlan knn_plan(int64_t n, int64_t Mr, int64_t Mq, int k, int sm_count);
bool knn_supported(int64_t n, int64_t Mr, int64_t Mq, int k);
cudaError_t launch_knn(const KnnPlan &p, const float *U, int64_t h, const float *d,
                       const float *Pr, const float *Pq, int32_t *nn_idx, float *nn_dist, void *ws,
                       cudaStream_t stream, LaunchInfo *info, bool general = false);

}  // namespace hh

namespace hh {
// NEXT-f4 (hh_cong.cu): B_b = A_b^T for `count` column-major n x n matrices.
cudaError_t launch_transpose(const void *A, void *B, int64_t n, int64_t count, int dtype,
                             cudaStream_t stream);
// K7: out_b = A_b op(Q)^T (every row through op(Q)) for fp32 n <= 1024
bool row_apply_supported(int64_t n, int64_t h, int dtype);
cudaError_t launch_row_apply(const void *A, void *B, const void *U, int64_t n, int64_t h,
                             int64_t count, int op, cudaStream_t stream);
}  // namespace hh
