// hh_api.cu -- the extern "C" boundary of libhh.so (declared in include/hh.h).
//
// Validation happens before any launch (nothing is written on error); the
// library allocates nothing for the caller's data and keeps only a cached
// device-attribute table.  Every computational step runs in this library's own
// kernels (hh_fused.cu, hh_gather.cu); there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "hh.h"
#include "hh_internal.h"

namespace hh {

namespace {
constexpr int kMaxDev = 64;
DevAttr g_attr[kMaxDev];
std::once_flag g_once[kMaxDev];
thread_local LaunchInfo t_last;
thread_local bool t_has_last = false;
thread_local int t_algo = HH_ALGO_AUTO;

// K1 (fused SIMT; K1s for fp32 n <= 512, hh_stream.cu) vs K5 (compact-WY on tcgen05) crossover
// in h, fp32 only, by n and by the problem size E = n*N elements.  K1 is one HBM pass but its
// FMA work grows with h; K5 moves ~1.5 passes and its cost is flat in h up to one block
// (b <= 32), plus a fixed cost of its kernel chain that only large problems amortise.
// Thresholds are the first h where K5 won in same-box sweeps: n <= 512 against K1s
// (profiles/r2/crossover_r2.txt, round 2: K1s moved them up by 2-10), n > 512 against K1
// (profiles/r1/crossover_r1.txt); E = 2^28 for the large band, 2^25 for the middle one.
int64_t wy_min_h(int64_t n, int64_t N) {
    if (n < 128) return int64_t(1) << 30;
    if (n > 8192) {
        // beyond the K1 tables the alternative is K1g (U from L2 per column: ~0.45 ms per
        // reflector at E = 2^28, against ~0.6 ms flat for one block of K5 --
        // n = 16384, N = 16384: h = 4 1.78 ms on K1g, h = 8 / 64 0.60 / 0.63 ms on K5)
        const int64_t E = n * N;
        return E >= (int64_t(1) << 27) ? 2 : E >= (int64_t(1) << 25) ? 3 : 12;
    }
    // bands follow K1's variant table (measured at the top n of each band)
    const int i = n <= 128 ? 0 : n <= 256 ? 1 : n <= 512 ? 2 : n <= 1024 ? 3 : n <= 2048 ? 4
                : n <= 4096 ? 5 : 6;
    // (n in (1024, 4096]: re-swept after K1t / K1w and the TMEM-A K5a, profiles/r2/xover_r2b.txt --
    // K1w stays ahead through h = 16, the most its TMEM holds: n = 4096 13 -> 17, n = 2048 mid
    // band 22 -> 19)
    // (n in (512, 1024] likewise after K1t took h = 12..16 from K1s, profiles/r2/xover_r2c.txt:
    // 19 -> 17, middle band 26 -> 20)
    static const int big[7] = {24, 20, 18, 17, 17, 17, 7};    // E >= 2^27
    static const int mid[7] = {28, 25, 23, 20, 19, 17, 16};   // 2^25 <= E < 2^27
    const int64_t E = n * N;
    if (E >= (int64_t(1) << 27)) return big[i];
    if (E >= (int64_t(1) << 25)) return mid[i];
    return 32;   // small problems: K5's fixed cost dominates below h = 32
}

// the block program is measured and tested up to this n (its own limit is 2^20)
constexpr int64_t kWyMaxN = 65536;

bool use_wy(hh_dtype dtype, int64_t n, int64_t h, int64_t N, int algo) {
    if (dtype != HH_F32 || n > kWyMaxN || !wy_supported(WY_APPLY_N, n, h, N)) return false;
    if (algo == HH_ALGO_WY) return true;
    if (algo == HH_ALGO_FUSED) return false;
    return h >= wy_min_h(n, N);
}

// Symmetric apply: K2 does 2h reflectors per column and is FMA-bound from h ~ 5; the
// tensor-core block program moves ~1.5 passes of X plus a fixed cost for its kernel chain.
// Same-box sweeps: n <= 512 against the streaming K2 (profiles/r2/crossover_r2.txt, E = 2^28;
// the middle band raised by the same margin), n > 512 against K2 (profiles/r1/crossover_r1.txt).
int64_t wy_min_h_sym(int64_t n, int64_t N) {
    if (n < 128) return int64_t(1) << 30;
    if (n > 8192) {   // K1g runs 2h reflectors per column there (see wy_min_h)
        const int64_t E = n * N;
        return E >= (int64_t(1) << 27) ? 1 : E >= (int64_t(1) << 25) ? 2 : 6;
    }
    const int i = n <= 128 ? 0 : n <= 256 ? 1 : n <= 512 ? 2 : n <= 1024 ? 3 : n <= 2048 ? 4 : 5;
    // (n in (1024, 4096] re-swept in round 2, profiles/r2/xover_r2b.txt: 10 -> 12 and 8 -> 10 for
    // E >= 2^27, 15 -> 12 for n = 4096 in the middle band)
    static const int big[6] = {16, 13, 10, 11, 12, 10};      // E >= 2^27
    static const int mid[6] = {24, 19, 18, 15, 18, 12};      // 2^25 <= E < 2^27 (n <= 1024: 19 -> 15)
    const int64_t E = n * N;
    if (E >= (int64_t(1) << 27)) return big[i];
    if (E >= (int64_t(1) << 25)) return mid[i];
    return 32;
}

bool use_wy_sym(hh_dtype dtype, int64_t n, int64_t h, int64_t N, int algo) {
    if (dtype != HH_F32 || n > kWyMaxN || !wy_supported(WY_SYM, n, h, N)) return false;
    if (algo == HH_ALGO_WY) return true;
    if (algo == HH_ALGO_FUSED) return false;
    return h >= wy_min_h_sym(n, N);
}

// HH_ALGO_WY forces the tensor-core program: a shape it cannot run (fp64, n < 32, more than
// kMaxPasses block passes, ...) is an error, never a silent switch to the SIMT kernel
bool wy_forced_unsupported(int kind, hh_dtype dtype, int64_t n, int64_t h, int64_t N) {
    return t_algo == HH_ALGO_WY && h > 0 && N > 0 &&
           (dtype != HH_F32 || n > kWyMaxN || !wy_supported(kind, n, h, N));
}

// the bucketed Mahalanobis path indexes pairs and points with int32
constexpr int64_t kMaxPairs = (int64_t(1) << 31) - 1;

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t elem(hh_dtype dt) { return dt == HH_F32 ? 4 : 8; }
bool dtype_ok(int dt) { return dt == HH_F32 || dt == HH_F64; }
size_t round256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

hh_status map_err(cudaError_t e) {
    if (e == cudaSuccess) return HH_OK;
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return HH_ERR_UNSUPPORTED;
    }
    return HH_ERR_CUDA;
}

// The vector kernels (K1 / K1s / K1t, K5) move columns with 128-bit accesses: column stride a
// multiple of 16 bytes and n within their variant tables.  Every other shape runs K1g
// (hh_general.cu), which needs element alignment only.
bool vector_shape(int64_t n, hh_dtype dtype) {
    return (static_cast<size_t>(n) * elem(dtype)) % 16 == 0 && n <= max_n(dtype);
}
bool aligned_elem(const void *p, hh_dtype dtype) {
    return reinterpret_cast<uintptr_t>(p) % elem(dtype) == 0;
}

// ---- the padded detour for column strides that are not a multiple of 16 bytes
// With a workspace, the columns (and U, lambda, D) are copied to a 16-byte pitch n4 (pads zero,
// so every dot product and update is unchanged: Eq. 2 on the zero-extended vectors), the call
// runs on the copy with the fast kernels (K1 family or the block program K5), and the result is
// copied back: two extra passes over X against K1r's / K1g's cost per reflector (policy and
// measurements in use_padded below).
thread_local int t_pad = -1;   // test hook (hh_debug_general_pad): -1 policy, 0 never, 1 whenever possible
bool stride_unaligned(int64_t n, hh_dtype dtype) {
    return (static_cast<size_t>(n) * elem(dtype)) % 16 != 0;
}
int64_t padded_n(int64_t n, hh_dtype dtype) {
    const int64_t q = 16 / static_cast<int64_t>(elem(dtype));
    return (n + q - 1) / q * q;
}
bool k1r_capable(int64_t n, int64_t h, hh_dtype dtype) {
    if (n > max_n(dtype) / 2) return false;   // K1r's tables: n <= 4096 (fp32) / 2048 (fp64)
    if (dtype == HH_F32 && n > 512 && h <= 16) return true;   // U in TMEM
    int64_t pitch = 64;                       // U in shared memory at its variant's row pitch
    while (pitch < n) pitch *= 2;
    return static_cast<size_t>(h) * pitch * elem(dtype) + 1024 <=
           static_cast<size_t>(device_attr().max_smem_optin);
}
bool use_padded(int64_t n, int64_t h, hh_dtype dtype, bool sym) {
    if (!stride_unaligned(n, dtype) || h < 1 || t_pad == 0) return false;
    const int64_t n4 = padded_n(n, dtype);
    if (n4 > max_n(dtype) && !(dtype == HH_F32 && n4 <= kWyMaxN)) return false;
    if (t_pad == 1 || t_algo == HH_ALGO_WY) return true;   // (a forced K5 runs on the padded copy)
    // same-box sweep at 1 GiB (tools/pad_time.py, profiles/r2/pad_time_r2.jsonl): the detour costs
    // ~0.87 ms of copies + the aligned call; K1r (no per-element predicates) grows by 0.02-0.03 ms
    // per reflector -- n = 1023: h = 16 0.48 (U in TMEM) vs 1.36, h = 40 1.26 (U in shared
    // memory) vs 1.53, h = 56 K1g 12.2 vs 1.52; sym h = 16 0.94 vs 1.53; n = 101: h = 40 1.01 vs
    // 1.02, h = 56 1.36 vs 1.24, sym h = 16 0.85 vs 0.91; n = 4095: h = 16 0.67 vs 1.51, then
    // only K1g: h = 20 4.8 vs 1.55; n = 9001 (K1g): h = 4 1.56 vs 1.42, sym h = 2 1.69 vs 1.50
    if (!k1r_capable(n, h, dtype)) return h >= (sym ? 2 : 4);
    if (n <= 256) return h >= (sym ? 19 : 44);
    if (n <= 1024) return h >= (sym ? 22 : 50);
    return h >= (sym ? 17 : 40);
}
// scratch of the detour itself (U, X and up to two n-vectors at the padded pitch)
struct PadPlan {
    int64_t n4 = 0;
    size_t off_u = 0, off_x = 0, off_v0 = 0, off_v1 = 0, off_inner = 0;
};
PadPlan pad_plan(int64_t n, int64_t h, int64_t N, hh_dtype dtype) {
    PadPlan p;
    p.n4 = padded_n(n, dtype);
    const size_t s = elem(dtype);
    p.off_u = 0;
    p.off_x = round256(static_cast<size_t>(h) * p.n4 * s);
    p.off_v0 = p.off_x + round256(static_cast<size_t>(N) * p.n4 * s);
    p.off_v1 = p.off_v0 + round256(static_cast<size_t>(p.n4) * s);
    p.off_inner = p.off_v1 + round256(static_cast<size_t>(p.n4) * s);
    return p;
}

// shape checks shared by the column calls; returns HH_OK or the error.  general_ok: the call
// has the K1g path, so shapes / alignments outside the vector kernels' are accepted when K1g
// takes them (the call itself then checks element alignment of its operands).
hh_status check_common(int64_t n, int64_t h, const void *U, int64_t N, hh_dtype dtype,
                       bool device_u = true, bool general_ok = false) {
    if (!dtype_ok(dtype) || n < 1 || h < 0 || N < 0) return HH_ERR_INVALID_VALUE;
    if (h > 0 && !U) return HH_ERR_INVALID_VALUE;
    if (h > (int64_t(1) << 30)) return HH_ERR_UNSUPPORTED;
    if (general_ok) {
        // (n past K1g's shared memory: only the block program can serve it -- fp32, 16-byte
        // strides, past the crossover and with a workspace; otherwise the launch is refused)
        if (!vector_shape(n, dtype) && !general_supported(n, dtype == HH_F32 ? 0 : 1) &&
            !(dtype == HH_F32 && n % 4 == 0 && n <= kWyMaxN))
            return HH_ERR_UNSUPPORTED;
        if (device_u && h > 0 && !aligned_elem(U, dtype)) return HH_ERR_UNSUPPORTED;
        return HH_OK;
    }
    if (!vector_shape(n, dtype)) return HH_ERR_UNSUPPORTED;
    if (device_u && h > 0 && !aligned16(U)) return HH_ERR_UNSUPPORTED;
    return HH_OK;
}

hh_status run_fused(FusedArgs a, hh_dtype dtype, cudaStream_t stream, bool general = false) {
    LaunchInfo info;
    cudaError_t e = general ? launch_general(a, dtype == HH_F32 ? 0 : 1, stream, &info)
                            : launch_fused(a, dtype == HH_F32 ? 0 : 1, stream, &info);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (info.variant) {
        t_last = info;
        t_has_last = true;
    }
    return map_err(e);
}

// columns per ring slot of hh_apply_host
int64_t host_chunk_cols(int64_t n, int64_t N, hh_dtype dtype) {
    const int64_t colB = n * static_cast<int64_t>(elem(dtype));
    const int64_t cols = std::max<int64_t>(1, (int64_t(64) << 20) / colB);
    return std::max<int64_t>(1, std::min(cols, N));
}
constexpr int kRing = 3;

}  // namespace

// hh_mahalanobis's second stream (the pair sort beside the transform): created once per
// calling thread and device, with its fork / join events; the hook hh_debug_mahal_fork turns
// the overlap off for A/B (the sort then runs on the caller's stream)
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    bool tried = false;
    ~SideStream() {
        // (at thread exit; errors ignored -- the context may already be gone)
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (s) cudaStreamDestroy(s);
    }
};
thread_local SideStream t_side[kMaxDev];
thread_local int t_mahal_fork = 1;

SideStream *side_stream() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    SideStream &ss = t_side[dev];
    if (!ss.tried) {
        ss.tried = true;
        if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            ss.s = nullptr;
        }
    }
    return ss.s ? &ss : nullptr;
}

void drop_side_stream() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return;
    t_side[dev] = SideStream{};   // (the old handles are abandoned, not destroyed: they are stale)
    t_side[dev].tried = true;     // and not re-created in this thread
}

const DevAttr &device_attr() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    std::call_once(g_once[dev], [dev]() {
        DevAttr a;
        cudaDeviceGetAttribute(&a.sm_count, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&a.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaDeviceGetAttribute(&a.l2_bytes, cudaDevAttrL2CacheSize, dev);
        if (a.sm_count <= 0) a.sm_count = 148;
        if (a.max_smem_optin <= 0) a.max_smem_optin = 227 * 1024;
        g_attr[dev] = a;
    });
    return g_attr[dev];
}

}  // namespace hh

using namespace hh;

extern "C" {

const char *hh_status_string(hh_status s) {
    switch (s) {
        case HH_OK: return "HH_OK";
        case HH_ERR_INVALID_VALUE: return "HH_ERR_INVALID_VALUE";
        case HH_ERR_UNSUPPORTED: return "HH_ERR_UNSUPPORTED";
        case HH_ERR_WORKSPACE: return "HH_ERR_WORKSPACE";
        case HH_ERR_CUDA: return "HH_ERR_CUDA";
    }
    return "HH_ERR_UNKNOWN";
}

const char *hh_version(void) { return "0.2.0"; }

// Debug hook (not part of hh.h): a device buffer of >= 16 uint64 that CTA 0 of every
// subsequent K5b launch fills with per-role barrier wait cycles (NULL switches it off).
hh_status hh_debug_wy_timeline(void *device_buf) {
    wy_set_timeline(static_cast<unsigned long long *>(device_buf));
    return HH_OK;
}

// Test hook (not part of hh.h): block width from which the update runs in TS mode (G in
// TMEM, wy_update_ts_kernel); default 256.  Lets the GPU tests cover the TS kernel at every
// block width.  Returns the previous value.
int hh_debug_wy_ts_min(int kw) { return wy_set_ts_min(kw); }

// Test / A-B hook (not part of hh.h): the single-launch dataflow form of the block program
// (K5f) on (default) or off for the calling thread, and its project-CTA count (0: default).
// Returns the previous on/off.
int hh_debug_wy_flow(int on, int project_ctas) { return wy_set_flow(on, project_ctas); }
void hh_debug_wy_flow_knobs(const int *k, int cnt) { wy_set_flow_knobs(k, cnt); }
void hh_debug_k1(int alt, int gridx) { k1_set_debug(alt, gridx); }
int hh_debug_k1_stream(int on) { return k1_set_stream(on); }
int hh_debug_k1_prefetch(int dist) { return k1_set_prefetch(dist); }
int hh_debug_k1_tmem(int on) { return k1_set_tmem(on); }
int hh_debug_k1_blocked(int on) { return k1_set_blocked(on); }
int hh_debug_k7_rows(int rw) { return k7_set_rows(rw); }
int hh_debug_general_scalar(int on) { return general_set_scalar(on); }
int hh_debug_k1r_tmem(int on) { return k1r_set_tmem(on); }
int hh_debug_k1r_stage(int on) { return k1r_set_stage(on); }
int hh_debug_general_pad(int on) {
    const int prev = t_pad;
    t_pad = on;
    return prev;
}
int hh_debug_mahal_fork(int on) {
    const int prev = t_mahal_fork;
    t_mahal_fork = on;
    return prev;
}
int hh_debug_wy_pdl(int on) { return wy_set_pdl(on); }
int hh_debug_wy_symfuse(int on) { return wy_set_symfuse(on); }
int hh_debug_wy_tsa(int on) { return wy_set_tsa(on); }

// Test hook (not part of hh.h): runs the compact-WY preparation and the first
// projection only, leaving G (bf16 hi/lo rows) and V in the workspace at the
// offsets written to off[0..1] (G, V) and the block size b / count nblk to off[2..3].
hh_status hh_debug_wy_project(int op, int64_t n, int64_t h, const void *U, const void *X,
                              int64_t N, void *workspace, size_t workspace_bytes, int64_t *off,
                              hh_stream_t stream) {
    if (!wy_supported(op ? WY_APPLY_T : WY_APPLY_N, n, h, N) || !workspace || !off)
        return HH_ERR_INVALID_VALUE;
    const WyPlan p = wy_plan(op ? WY_APPLY_T : WY_APPLY_N, n, h, N);
    if (workspace_bytes < p.bytes) return HH_ERR_WORKSPACE;
    off[0] = static_cast<int64_t>(p.off_gt);
    off[1] = static_cast<int64_t>(p.off_v);
    off[2] = p.b;
    off[3] = p.nblk;
    off[4] = p.n_pad;
    off[5] = static_cast<int64_t>(p.off_t);
    return map_err(launch_wy(p, static_cast<const float *>(U), nullptr,
                             static_cast<const float *>(X), nullptr, workspace, stream, nullptr, 1));
}

hh_status hh_last_launch_count(int *kernels) {
    if (!t_has_last || !kernels) return HH_ERR_INVALID_VALUE;
    *kernels = t_last.launches;
    return HH_OK;
}

hh_status hh_last_launch_info(const char **variant, int *grid, int *block, int *smem_bytes,
                              int *nchunks) {
    if (!t_has_last) return HH_ERR_INVALID_VALUE;
    if (variant) *variant = t_last.variant;
    if (grid) *grid = t_last.grid;
    if (block) *block = t_last.block;
    if (smem_bytes) *smem_bytes = t_last.smem;
    if (nchunks) *nchunks = t_last.nchunks;
    return HH_OK;
}

hh_status hh_workspace_bytes(hh_call call, int64_t n, int64_t h, int64_t N_or_M, int64_t npairs,
                             hh_dtype dtype, size_t *bytes) {
    if (!bytes || !dtype_ok(dtype) || n < 1 || h < 0 || N_or_M < 0 || npairs < 0)
        return HH_ERR_INVALID_VALUE;
    switch (call) {
        case HH_CALL_APPLY:
        case HH_CALL_SYM: {
            const bool sym = call == HH_CALL_SYM;
            if (use_padded(n, h, dtype, sym)) {
                // unaligned column stride: the padded copy + what the call needs on it
                const PadPlan pp = pad_plan(n, h, N_or_M, dtype);
                size_t inner = 0;
                hh_workspace_bytes(call, pp.n4, h, N_or_M, 0, dtype, &inner);
                *bytes = pp.off_inner + inner;
                return HH_OK;
            }
            if (stride_unaligned(n, dtype)) {   // K1r / K1g: no scratch
                *bytes = 0;
                return HH_OK;
            }
            if (sym)
                *bytes = use_wy_sym(dtype, n, h, N_or_M, t_algo) ? wy_plan(WY_SYM, n, h, N_or_M).bytes : 0;
            else
                *bytes = use_wy(dtype, n, h, N_or_M, t_algo) ? wy_plan(WY_APPLY_N, n, h, N_or_M).bytes : 0;
            return HH_OK;
        }
        case HH_CALL_MAHALANOBIS:
            if (npairs >= kMaxPairs || N_or_M >= kMaxPairs) return HH_ERR_UNSUPPORTED;
            if (stride_unaligned(n, dtype) && t_pad != 0 && padded_n(n, dtype) <= max_n(dtype)) {
                // the padded copies of U, P, d, then the aligned call's scratch
                const PadPlan pp = pad_plan(n, h, N_or_M, dtype);
                *bytes = pp.off_inner +
                         round256(static_cast<size_t>(pp.n4) * static_cast<size_t>(N_or_M) * elem(dtype)) +
                         bucket_ws_bytes(N_or_M, npairs);
                return HH_OK;
            }
            *bytes = round256(static_cast<size_t>(n) * static_cast<size_t>(N_or_M) * elem(dtype)) +
                     bucket_ws_bytes(N_or_M, npairs);
            return HH_OK;
        case HH_CALL_CONGRUENCE: {   /* N_or_M = count */
            const size_t mb =
                round256(static_cast<size_t>(n) * n * N_or_M * elem(dtype));
            const size_t aw = use_wy(dtype, n, h, n * N_or_M, t_algo)
                                  ? wy_plan(WY_APPLY_N, n, h, n * N_or_M).bytes
                                  : 0;
            *bytes = 2 * mb + aw;
            return HH_OK;
        }
        case HH_CALL_SHF:   /* N_or_M = K candidates */
            *bytes = shf_ws_bytes(n, N_or_M, dtype == HH_F32 ? 0 : 1);
            return HH_OK;
        case HH_CALL_KNN:   /* N_or_M = M_ref, npairs = M_query; k = h is not needed: max */
            *bytes = knn_plan(n, N_or_M, npairs, 16, device_attr().sm_count).bytes;
            return HH_OK;
        case HH_CALL_APPLY_HOST: {
            const size_t ub = round256(static_cast<size_t>(n) * static_cast<size_t>(h) * elem(dtype));
            const int64_t cols = host_chunk_cols(n, std::max<int64_t>(N_or_M, 1), dtype);
            const size_t slot = round256(static_cast<size_t>(cols) * n * elem(dtype));
            // past the crossover each chunk runs the compact-WY program (its own scratch)
            const size_t wyb = (h > 0 && use_wy(dtype, n, h, cols, t_algo))
                                   ? round256(wy_plan(WY_APPLY_N, n, h, cols).bytes) : 0;
            *bytes = ub + kRing * slot + wyb;
            return HH_OK;
        }
    }
    return HH_ERR_INVALID_VALUE;
}

hh_status hh_set_algo(hh_algo algo) {
    if (algo != HH_ALGO_AUTO && algo != HH_ALGO_FUSED && algo != HH_ALGO_WY)
        return HH_ERR_INVALID_VALUE;
    t_algo = algo;
    return HH_OK;
}

hh_algo hh_get_algo(void) { return static_cast<hh_algo>(t_algo); }

static hh_status apply_impl(hh_op op, int64_t n, int64_t h, const void *U, const void *X,
                            void *Y, int64_t N, hh_dtype dtype, void *workspace,
                            size_t workspace_bytes, hh_stream_t stream, const void *dsign,
                            int dside, int qr = 0) {
    if (op != HH_OP_N && op != HH_OP_T) return HH_ERR_INVALID_VALUE;
    hh_status st = check_common(n, h, U, N, dtype, true, true);
    if (st != HH_OK) return st;
    if (N == 0) return HH_OK;
    if (!X || !Y) return HH_ERR_INVALID_VALUE;
    if (dside && !dsign) return HH_ERR_INVALID_VALUE;
    if (!aligned_elem(X, dtype) || !aligned_elem(Y, dtype) || (dside && !aligned_elem(dsign, dtype)))
        return HH_ERR_UNSUPPORTED;
    // K1g for the shapes and alignments the vector kernels do not take
    const bool al16 = (static_cast<size_t>(n) * elem(dtype)) % 16 == 0 && aligned16(X) &&
                      aligned16(Y) && (h == 0 || aligned16(U)) && (!dside || aligned16(dsign));
    const bool general = !al16 || n > max_n(dtype);   // (the fused path then runs K1r / K1g)
    if (workspace && use_padded(n, h, dtype, false)) {
        if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        const PadPlan pp = pad_plan(n, h, N, dtype);
        size_t inner = 0;
        hh_workspace_bytes(HH_CALL_APPLY, pp.n4, h, N, 0, dtype, &inner);
        if (workspace_bytes < pp.off_inner + inner) return HH_ERR_WORKSPACE;
        char *w = static_cast<char *>(workspace);
        const int dt = dtype == HH_F32 ? 0 : 1;
        cudaError_t e = launch_repitch(U, n, w + pp.off_u, pp.n4, h, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess) e = launch_repitch(X, n, w + pp.off_x, pp.n4, N, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess && dside)
            e = launch_repitch(dsign, n, w + pp.off_v0, pp.n4, 1, n, pp.n4, 1.0, dt, stream);
        if (e != cudaSuccess) return map_err(e);
        st = apply_impl(op, pp.n4, h, w + pp.off_u, w + pp.off_x, w + pp.off_x, N, dtype,
                        inner ? w + pp.off_inner : nullptr, inner, stream,
                        dside ? w + pp.off_v0 : nullptr, dside, qr);
        if (st != HH_OK) return st;
        e = launch_repitch(w + pp.off_x, pp.n4, Y, n, N, n, n, 0.0, dt, stream);
        if (t_has_last) t_last.launches += 3 + (dside ? 1 : 0);
        return map_err(e);
    }
    if (wy_forced_unsupported(WY_APPLY_N, dtype, n, h, N)) return HH_ERR_UNSUPPORTED;
    if (!al16 && t_algo == HH_ALGO_WY && h > 0) return HH_ERR_UNSUPPORTED;
    if (al16 && h > 0 && use_wy(dtype, n, h, N, t_algo)) {
        WyPlan p = wy_plan(op == HH_OP_T ? WY_APPLY_T : WY_APPLY_N, n, h, N);
        p.qr = qr;
        if (workspace && workspace_bytes < p.bytes) return HH_ERR_WORKSPACE;
        if (workspace && !aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        if (!workspace && t_algo == HH_ALGO_WY) return HH_ERR_WORKSPACE;
        if (workspace) {
            LaunchInfo info;
            cudaError_t e = launch_wy(p, static_cast<const float *>(U), nullptr,
                                      static_cast<const float *>(X), static_cast<float *>(Y),
                                      workspace, stream, &info, -1,
                                      static_cast<const float *>(dsign), dside);
            if (info.variant) {
                t_last = info;
                t_has_last = true;
            }
            return map_err(e);
        }
        // no workspace in AUTO mode: the fused kernel (K1) runs instead
    }
    FusedArgs a{};
    a.U = U;
    a.X = X;
    a.Y = Y;
    a.n = n;
    a.h = h;
    a.N = N;
    a.mode = op == HH_OP_N ? MODE_APPLY_N : MODE_APPLY_T;
    a.dsign = dsign;
    a.dside = dside;
    a.qr = qr;
    return run_fused(a, dtype, stream, general);
}

hh_status hh_apply_qr(hh_op op, int64_t n, int64_t h, const void *U, const void *X, void *Y,
                      int64_t N, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                      hh_stream_t stream) {
    return apply_impl(op, n, h, U, X, Y, N, dtype, workspace, workspace_bytes, stream, nullptr, 0,
                      1);
}

hh_status hh_apply(hh_op op, int64_t n, int64_t h, const void *U, const void *X, void *Y,
                   int64_t N, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                   hh_stream_t stream) {
    return apply_impl(op, n, h, U, X, Y, N, dtype, workspace, workspace_bytes, stream, nullptr, 0);
}

hh_status hh_apply_signed(hh_op op, hh_side side, int64_t n, int64_t h, const void *U,
                          const void *d, const void *X, void *Y, int64_t N, hh_dtype dtype,
                          void *workspace, size_t workspace_bytes, hh_stream_t stream) {
    if (side != HH_SIDE_LEFT && side != HH_SIDE_RIGHT) return HH_ERR_INVALID_VALUE;
    if (N > 0 && !d) return HH_ERR_INVALID_VALUE;
    return apply_impl(op, n, h, U, X, Y, N, dtype, workspace, workspace_bytes, stream, d,
                      side == HH_SIDE_RIGHT ? 1 : 2);
}


static hh_status sym_impl(int64_t n, int64_t h, const void *U, const void *lambda, const void *X,
                          void *Y, int64_t N, hh_dtype dtype, void *workspace,
                          size_t workspace_bytes, hh_stream_t stream, const void *dsign) {
    hh_status st = check_common(n, h, U, N, dtype, true, true);
    if (st != HH_OK) return st;
    if (N == 0) return HH_OK;
    if (!X || !Y || !lambda) return HH_ERR_INVALID_VALUE;
    if (!aligned_elem(X, dtype) || !aligned_elem(Y, dtype) || !aligned_elem(lambda, dtype) ||
        (dsign && !aligned_elem(dsign, dtype)))
        return HH_ERR_UNSUPPORTED;
    const bool al16 = (static_cast<size_t>(n) * elem(dtype)) % 16 == 0 && aligned16(X) &&
                      aligned16(Y) && aligned16(lambda) && (h == 0 || aligned16(U)) &&
                      (!dsign || aligned16(dsign));
    const bool general = !al16 || n > max_n(dtype);
    if (workspace && use_padded(n, h, dtype, true)) {
        if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        const PadPlan pp = pad_plan(n, h, N, dtype);
        size_t inner = 0;
        hh_workspace_bytes(HH_CALL_SYM, pp.n4, h, N, 0, dtype, &inner);
        if (workspace_bytes < pp.off_inner + inner) return HH_ERR_WORKSPACE;
        char *w = static_cast<char *>(workspace);
        const int dt = dtype == HH_F32 ? 0 : 1;
        cudaError_t e = launch_repitch(U, n, w + pp.off_u, pp.n4, h, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess) e = launch_repitch(X, n, w + pp.off_x, pp.n4, N, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess)
            e = launch_repitch(lambda, n, w + pp.off_v0, pp.n4, 1, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess && dsign)
            e = launch_repitch(dsign, n, w + pp.off_v1, pp.n4, 1, n, pp.n4, 1.0, dt, stream);
        if (e != cudaSuccess) return map_err(e);
        st = sym_impl(pp.n4, h, w + pp.off_u, w + pp.off_v0, w + pp.off_x, w + pp.off_x, N, dtype,
                      inner ? w + pp.off_inner : nullptr, inner, stream,
                      dsign ? w + pp.off_v1 : nullptr);
        if (st != HH_OK) return st;
        e = launch_repitch(w + pp.off_x, pp.n4, Y, n, N, n, n, 0.0, dt, stream);
        if (t_has_last) t_last.launches += 4 + (dsign ? 1 : 0);
        return map_err(e);
    }
    if (wy_forced_unsupported(WY_SYM, dtype, n, h, N)) return HH_ERR_UNSUPPORTED;
    if (!al16 && t_algo == HH_ALGO_WY && h > 0) return HH_ERR_UNSUPPORTED;
    if (al16 && h > 0 && use_wy_sym(dtype, n, h, N, t_algo)) {
        const WyPlan p = wy_plan(WY_SYM, n, h, N);
        if (workspace && workspace_bytes < p.bytes) return HH_ERR_WORKSPACE;
        if (workspace && !aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        if (!workspace && t_algo == HH_ALGO_WY) return HH_ERR_WORKSPACE;
        if (workspace) {
            LaunchInfo info;
            cudaError_t e = launch_wy(p, static_cast<const float *>(U),
                                      static_cast<const float *>(lambda),
                                      static_cast<const float *>(X), static_cast<float *>(Y),
                                      workspace, stream, &info, -1,
                                      static_cast<const float *>(dsign), dsign ? 3 : 0);
            if (info.variant) {
                t_last = info;
                t_has_last = true;
            }
            return map_err(e);
        }
    }
    FusedArgs a{};
    a.U = U;
    a.X = X;
    a.Y = Y;
    a.vec = lambda;
    a.n = n;
    a.h = h;
    a.N = N;
    a.mode = MODE_SYM;
    a.dsign = dsign;
    a.dside = dsign ? 3 : 0;
    return run_fused(a, dtype, stream, general);
}

hh_status hh_sym_apply(int64_t n, int64_t h, const void *U, const void *lambda, const void *X,
                       void *Y, int64_t N, hh_dtype dtype, void *workspace,
                       size_t workspace_bytes, hh_stream_t stream) {
    return sym_impl(n, h, U, lambda, X, Y, N, dtype, workspace, workspace_bytes, stream, nullptr);
}

hh_status hh_sym_apply_signed(int64_t n, int64_t h, const void *U, const void *d,
                              const void *lambda, const void *X, void *Y, int64_t N,
                              hh_dtype dtype, void *workspace, size_t workspace_bytes,
                              hh_stream_t stream) {
    if (N > 0 && !d) return HH_ERR_INVALID_VALUE;
    return sym_impl(n, h, U, lambda, X, Y, N, dtype, workspace, workspace_bytes, stream, d);
}


hh_status hh_mahalanobis(int64_t n, int64_t h, const void *U, const void *d, const void *P,
                         int64_t M, const int32_t *ia, const int32_t *ib, int64_t npairs,
                         void *dist, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                         hh_stream_t stream) {
    if (npairs < 0 || M < 0) return HH_ERR_INVALID_VALUE;
    if (npairs > 0 && M < 1) return HH_ERR_INVALID_VALUE;
    if (npairs >= kMaxPairs || M >= kMaxPairs) return HH_ERR_UNSUPPORTED;
    hh_status st = check_common(n, h, U, M, dtype, true, true);
    if (st != HH_OK) return st;
    if (npairs == 0) return HH_OK;
    if (!d || !P || !ia || !ib || !dist) return HH_ERR_INVALID_VALUE;
    if (!aligned_elem(d, dtype) || !aligned_elem(P, dtype) || !aligned_elem(dist, dtype))
        return HH_ERR_UNSUPPORTED;
    // shapes / alignments outside the vector kernels': the per-pair form on K1g (no scratch)
    const bool general = !vector_shape(n, dtype) || !aligned16(d) || !aligned16(P) ||
                         (h > 0 && !aligned16(U));
    size_t need = 0;
    hh_workspace_bytes(HH_CALL_MAHALANOBIS, n, h, M, npairs, dtype, &need);
    if (workspace && stride_unaligned(n, dtype) && t_pad != 0 && padded_n(n, dtype) <= max_n(dtype)) {
        // unaligned stride: transform-once on a copy of the points at a 16-byte pitch (pads
        // zero: they stay zero through Q^T and add nothing to the distance)
        if (workspace_bytes < need) return HH_ERR_WORKSPACE;
        if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        const PadPlan pp = pad_plan(n, h, M, dtype);
        char *w = static_cast<char *>(workspace);
        const int dt = dtype == HH_F32 ? 0 : 1;
        cudaError_t e = cudaSuccess;
        if (h > 0) e = launch_repitch(U, n, w + pp.off_u, pp.n4, h, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess) e = launch_repitch(P, n, w + pp.off_x, pp.n4, M, n, pp.n4, 0.0, dt, stream);
        if (e == cudaSuccess) e = launch_repitch(d, n, w + pp.off_v0, pp.n4, 1, n, pp.n4, 0.0, dt, stream);
        if (e != cudaSuccess) return map_err(e);
        st = hh_mahalanobis(pp.n4, h, h > 0 ? w + pp.off_u : nullptr, w + pp.off_v0, w + pp.off_x, M,
                            ia, ib, npairs, dist, dtype, w + pp.off_inner, need - pp.off_inner, stream);
        if (st == HH_OK && t_has_last) t_last.launches += 2 + (h > 0 ? 1 : 0);
        return st;
    }
    if (workspace && !general) {
        if (workspace_bytes < need) return HH_ERR_WORKSPACE;
        if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
        // The counting sort of the pairs needs only ia: it runs on a second stream beside
        // K3a (fork / join through events, so the call stays stream-ordered and graph-
        // capturable), and the gather waits for both.
        const size_t zb = round256(static_cast<size_t>(n) * static_cast<size_t>(M) * elem(dtype));
        void *bws = static_cast<char *>(workspace) + zb;
        SideStream *side = t_mahal_fork ? side_stream() : nullptr;
        cudaError_t e = cudaSuccess;
        if (side) {
            e = cudaEventRecord(side->fork, stream);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(side->s, side->fork, 0);
            if (e == cudaSuccess) e = launch_bucket_sort(M, ia, npairs, bws, side->s);
            if (e == cudaSuccess) e = cudaEventRecord(side->join, side->s);
            if (e != cudaSuccess && e != cudaErrorStreamCaptureUnsupported &&
                e != cudaErrorStreamCaptureInvalidated) {
                // a stale cached stream (e.g. after a device reset): forget it and sort on the
                // caller's stream instead
                cudaGetLastError();
                drop_side_stream();
                side = nullptr;
                e = launch_bucket_sort(M, ia, npairs, bws, stream);
            }
            if (e != cudaSuccess) return map_err(e);
        } else {
            e = launch_bucket_sort(M, ia, npairs, bws, stream);
            if (e != cudaSuccess) return map_err(e);
        }
        // K3a: Z = diag(sqrt d) Q^T P  (transform each point once)
        FusedArgs a{};
        a.U = U;
        a.X = P;
        a.Y = workspace;
        a.vec = d;
        a.n = n;
        a.h = h;
        a.N = M;
        a.mode = MODE_TRANSFORM;
        st = run_fused(a, dtype, stream);
        if (side) {   // join (also when K3a failed: the side stream's work stays ordered)
            e = cudaStreamWaitEvent(stream, side->join, 0);
            if (e != cudaSuccess) return map_err(e);
        }
        if (st != HH_OK) return st;
        // K3b: dist[j] = ||Z[:,ia[j]] - Z[:,ib[j]]||^2, pairs bucketed by ia on device
        LaunchInfo info;
        e = launch_bucket_gather(workspace, n, M, ib, npairs, dist, bws, dtype == HH_F32 ? 0 : 1,
                                 stream, &info);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (info.variant) {
            info.launches += 1;   // + K3a
            t_last = info;
            t_has_last = true;
        }
        return map_err(e);
    }
    // K3c: per-pair fused, no scratch
    FusedArgs a{};
    a.U = U;
    a.X = P;
    a.Y = dist;
    a.vec = d;
    a.ia = ia;
    a.ib = ib;
    a.n = n;
    a.h = h;
    a.N = npairs;
    a.mode = MODE_PAIR;
    return run_fused(a, dtype, stream, general);
}

hh_status hh_shf_cost(int64_t n, const void *A, const void *B, const void *Uc, int64_t K,
                      void *cost, void *grad, hh_dtype dtype, void *workspace,
                      size_t workspace_bytes, hh_stream_t stream) {
    if (n < 1 || K < 0 || !dtype_ok(dtype)) return HH_ERR_INVALID_VALUE;
    if (K == 0) return HH_OK;
    if (!A || !B || !Uc || !cost || !workspace) return HH_ERR_INVALID_VALUE;
    const size_t s = elem(dtype);
    for (const void *q : {A, B, Uc, static_cast<const void *>(cost), static_cast<const void *>(grad),
                          static_cast<const void *>(workspace)})
        if (reinterpret_cast<uintptr_t>(q) % s != 0) return HH_ERR_UNSUPPORTED;
    if (workspace_bytes < shf_ws_bytes(n, K, dtype == HH_F32 ? 0 : 1)) return HH_ERR_WORKSPACE;
    LaunchInfo info;
    cudaError_t e = launch_shf(n, A, B, Uc, K, cost, grad, dtype == HH_F32 ? 0 : 1, workspace,
                               static_cast<cudaStream_t>(stream), &info);
    if (e == cudaSuccess) {
        t_last = info;
        t_has_last = true;
    }
    return map_err(e);
}

hh_status hh_congruence(hh_op op, int64_t n, int64_t h, const void *U, const void *M, void *Mout,
                        int64_t count, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                        hh_stream_t stream) {
    if (op != HH_OP_N && op != HH_OP_T) return HH_ERR_INVALID_VALUE;
    if (count < 0) return HH_ERR_INVALID_VALUE;
    hh_status st = check_common(n, h, U, n * count, dtype, true, true);
    if (st != HH_OK) return st;
    if (count == 0) return HH_OK;
    if (!M || !Mout) return HH_ERR_INVALID_VALUE;
    // (shapes / alignments outside the vector kernels': the applies run on K1g around the
    // transposes, which take any n)
    if (!aligned_elem(M, dtype) || !aligned_elem(Mout, dtype)) return HH_ERR_UNSUPPORTED;
    const bool general = !vector_shape(n, dtype) || !aligned16(M) || !aligned16(Mout) ||
                         (h > 0 && !aligned16(U));
    size_t need = 0;
    hh_workspace_bytes(HH_CALL_CONGRUENCE, n, h, count, 0, dtype, &need);
    if (!workspace || workspace_bytes < need) return HH_ERR_WORKSPACE;
    if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
    const size_t mb = round256(static_cast<size_t>(n) * n * count * elem(dtype));
    char *w = static_cast<char *>(workspace);
    void *T1 = w, *T2 = w + mb;
    void *aws = w + 2 * mb;
    const size_t awsb = need - 2 * mb;
    const int64_t NC = n * count;
    const int dt = dtype == HH_F32 ? 0 : 1;
    if (!general && h > 0 && row_apply_supported(n, h, dt)) {
        // two passes: T1 = op(Q) M (columns), M_out = T1 op(Q)^T (rows, K7)
        st = apply_impl(op, n, h, U, M, T1, NC, dtype, awsb ? aws : nullptr, awsb, stream, nullptr, 0);
        if (st != HH_OK) return st;
        if (map_err(launch_row_apply(T1, Mout, U, n, h, count, op == HH_OP_N ? 0 : 1, stream)) != HH_OK)
            return HH_ERR_CUDA;
        if (t_has_last) t_last.launches += 1;
        return HH_OK;
    }
    // (op(Q) (op(Q) M)^T)^T = op(Q) M op(Q)^T
    st = apply_impl(op, n, h, U, M, T1, NC, dtype, awsb ? aws : nullptr, awsb, stream, nullptr, 0);
    if (st != HH_OK) return st;
    if (map_err(launch_transpose(T1, T2, n, count, dt, stream)) != HH_OK) return HH_ERR_CUDA;
    st = apply_impl(op, n, h, U, T2, T1, NC, dtype, awsb ? aws : nullptr, awsb, stream, nullptr, 0);
    if (st != HH_OK) return st;
    if (map_err(launch_transpose(T1, Mout, n, count, dt, stream)) != HH_OK) return HH_ERR_CUDA;
    if (t_has_last) {
        t_last.launches = 2 * t_last.launches + 2;
    }
    return HH_OK;
}

hh_status hh_knn(int64_t n, int64_t h, const void *U, const void *d, const void *P_ref,
                 int64_t M_ref, const void *P_query, int64_t M_query, int k, int32_t *nn_idx,
                 void *nn_dist, hh_dtype dtype, void *workspace, size_t workspace_bytes,
                 hh_stream_t stream) {
    if (dtype != HH_F32 && dtype != HH_F64) return HH_ERR_INVALID_VALUE;
    if (n < 1 || h < 0 || M_ref < 0 || M_query < 0 || k < 1) return HH_ERR_INVALID_VALUE;
    if (M_query == 0) return HH_OK;
    if (M_ref < k) return HH_ERR_INVALID_VALUE;
    if ((h > 0 && !U) || !d || !P_ref || !P_query || !nn_idx || !nn_dist)
        return HH_ERR_INVALID_VALUE;
    if (dtype != HH_F32 || !knn_supported(n, M_ref, M_query, k)) return HH_ERR_UNSUPPORTED;
    if (!aligned_elem(d, dtype) || !aligned_elem(P_ref, dtype) || !aligned_elem(P_query, dtype) ||
        (h > 0 && !aligned_elem(U, dtype)) || !aligned_elem(nn_dist, dtype))
        return HH_ERR_UNSUPPORTED;
    // the transform runs on K1g when the points are not 16-byte strided / aligned
    const bool general = !vector_shape(n, dtype) || !aligned16(d) || !aligned16(P_ref) ||
                         !aligned16(P_query) || (h > 0 && !aligned16(U));
    const KnnPlan p = knn_plan(n, M_ref, M_query, k, device_attr().sm_count);
    if (!workspace || workspace_bytes < p.bytes) return HH_ERR_WORKSPACE;
    if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;
    LaunchInfo info;
    cudaError_t e = launch_knn(p, static_cast<const float *>(U), h, static_cast<const float *>(d),
                               static_cast<const float *>(P_ref),
                               static_cast<const float *>(P_query), nn_idx,
                               static_cast<float *>(nn_dist), workspace, stream, &info, general);
    if (info.variant) {
        t_last = info;
        t_has_last = true;
    }
    return map_err(e);
}

hh_status hh_apply_host(hh_op op, int64_t n, int64_t h, const void *U_host, const void *X_host,
                        void *Y_host, int64_t N, hh_dtype dtype, void *workspace,
                        size_t workspace_bytes, hh_stream_t stream) {
    if (op != HH_OP_N && op != HH_OP_T) return HH_ERR_INVALID_VALUE;
    hh_status st = check_common(n, h, U_host, N, dtype, /*device_u=*/false, /*general_ok=*/true);
    if (st != HH_OK) return st;
    if (N == 0) return HH_OK;
    if (!X_host || !Y_host || !workspace) return HH_ERR_INVALID_VALUE;
    size_t need = 0;
    hh_workspace_bytes(HH_CALL_APPLY_HOST, n, h, N, 0, dtype, &need);
    if (workspace_bytes < need) return HH_ERR_WORKSPACE;
    if (!aligned16(workspace)) return HH_ERR_UNSUPPORTED;

    const size_t s = elem(dtype);
    const size_t colB = static_cast<size_t>(n) * s;
    const size_t ub = round256(static_cast<size_t>(h) * colB);
    const int64_t cols = host_chunk_cols(n, N, dtype);
    const size_t slotB = round256(static_cast<size_t>(cols) * colB);
    char *ws = static_cast<char *>(workspace);
    char *Ud = ws;
    char *slots = ws + ub;
    char *wyws = slots + kRing * slotB;
    const size_t wyb = need - (ub + kRing * slotB);   // compact-WY scratch (0: fused path)

    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    cudaEvent_t start = nullptr, ev_in[kRing] = {}, ev_cp[kRing] = {}, ev_out[kRing] = {};
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t r) {
        if (e == cudaSuccess && r != cudaSuccess) e = r;
        return e == cudaSuccess;
    };
    chk(cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking));
    chk(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    chk(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
    chk(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    for (int i = 0; i < kRing; ++i) {
        chk(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_cp[i], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming));
    }
    hh_status kst = HH_OK;
    if (e == cudaSuccess) {
        // order after everything already queued on the caller's stream
        chk(cudaEventRecord(start, stream));
        chk(cudaStreamWaitEvent(sh, start, 0));
        if (h > 0) chk(cudaMemcpyAsync(Ud, U_host, static_cast<size_t>(h) * colB,
                                       cudaMemcpyHostToDevice, sh));
        const int64_t nchunks = (N + cols - 1) / cols;
        for (int64_t i = 0; i < nchunks && e == cudaSuccess && kst == HH_OK; ++i) {
            const int r = static_cast<int>(i % kRing);
            const int64_t c0 = i * cols;
            const int64_t cc = std::min(cols, N - c0);
            char *slot = slots + static_cast<size_t>(r) * slotB;
            const size_t bytes = static_cast<size_t>(cc) * colB;
            if (i >= kRing) chk(cudaStreamWaitEvent(sh, ev_out[r], 0));
            chk(cudaMemcpyAsync(slot, static_cast<const char *>(X_host) + c0 * colB, bytes,
                                cudaMemcpyHostToDevice, sh));
            chk(cudaEventRecord(ev_in[r], sh));
            chk(cudaStreamWaitEvent(sc, ev_in[r], 0));
            // the same path selection as hh_apply on a device chunk (K1, or the compact-WY
            // program past the crossover, with its scratch after the ring)
            if (e == cudaSuccess)
                kst = apply_impl(op, n, h, Ud, slot, slot, cc, dtype, wyb ? wyws : nullptr, wyb,
                                 sc, nullptr, 0);
            chk(cudaEventRecord(ev_cp[r], sc));
            chk(cudaStreamWaitEvent(sd, ev_cp[r], 0));
            chk(cudaMemcpyAsync(static_cast<char *>(Y_host) + c0 * colB, slot, bytes,
                                cudaMemcpyDeviceToHost, sd));
            chk(cudaEventRecord(ev_out[r], sd));
        }
        chk(cudaStreamSynchronize(sh));
        chk(cudaStreamSynchronize(sc));
        chk(cudaStreamSynchronize(sd));
    }
    for (int i = 0; i < kRing; ++i) {
        if (ev_in[i]) cudaEventDestroy(ev_in[i]);
        if (ev_cp[i]) cudaEventDestroy(ev_cp[i]);
        if (ev_out[i]) cudaEventDestroy(ev_out[i]);
    }
    if (start) cudaEventDestroy(start);
    if (sh) cudaStreamDestroy(sh);
    if (sc) cudaStreamDestroy(sc);
    if (sd) cudaStreamDestroy(sd);
    if (kst != HH_OK) return kst;
    return e == cudaSuccess ? HH_OK : HH_ERR_CUDA;
}

}  // extern "C"
