// hh_fused.cu -- host launcher of the fused SIMT kernel (K1 / K2 / K3a / K3c): variant
// choice by n, the shared-memory plan and the persistent grid.
#include <algorithm>
#include <cstdio>

#include "hh_fused_kernel.cuh"

namespace hh {
namespace {

// A/B knobs (hh_debug_k1, per calling thread): a forced alternative variant (-1: the table)
// and a multiplier of the persistent grid (1: persistent)
thread_local int t_k1_alt = -1;
thread_local int t_k1_gridx = 1;
thread_local int t_k1_stream = -1;
thread_local int t_k1_pf = 0;       // unstaged K1: L2 prefetch distance in batches (0: off;
                                    // measured slower at n = 4096, tools/k1_pf_ab.py)
thread_local int t_k1_tmem = -1;    // K1t (reflectors in TMEM): -1 policy, 0 never, 1 when eligible
thread_local int t_k1_blk = -1;     // K1w (K1t in blocks of kb reflectors): -1 policy, 0 never,
                                    // 1 when the variant has the form and K1t runs

// K1t policy (reflectors in TMEM), from a same-box A/B (tools/k1t_ab.py,
// profiles/r2/k1t_ab_r2.txt; outputs bit-identical): multi-warp groups (n > 1024) always --
// n = 4096, h = 8 / 12 / 16: 404 / 542 / 880 -> 338 / 439 / 535 us, n = 2048, h = 12 / 16:
// 461 / 602 -> 381 / 487 us; one-warp groups (n <= 1024) from h = 12 (n = 1024, h = 16:
// 499 -> 430 us, but h = 10: 350 -> 380 us: the tcgen05.ld wait sits on the reflector's
// serial chain where the shared-memory loads pipelined with the FMAs); never for the two-CTA
// (256-thread) variants (n = 512, h = 10: 448 -> 609 us; K1s serves those shapes)
bool k1t_preferred(const FusedVariant *v, int64_t h) {
    if (v->nt <= 256) return false;
    return v->tpc > 32 || h >= 12;
}

const FusedVariant *pick(int dtype, int64_t nv) {
    int cnt = 0;
    if (dtype == 0 && t_k1_alt >= 0) {
        const FusedVariant *alt = fused_alt_f32(&cnt);
        if (t_k1_alt < cnt && static_cast<int64_t>(alt[t_k1_alt].tpc) * alt[t_k1_alt].ch >= nv)
            return &alt[t_k1_alt];
        cnt = 0;
    }
    const FusedVariant *tab = dtype == 0 ? fused_table_f32(&cnt) : fused_table_f64(&cnt);
    for (int i = 0; i < cnt; ++i)
        if (static_cast<int64_t>(tab[i].tpc) * tab[i].ch >= nv) return &tab[i];
    return nullptr;
}

}  // namespace

int64_t max_n(int dtype) { return dtype == 0 ? 8192 : 4096; }

int k1_set_prefetch(int dist) {
    const int prev = t_k1_pf;
    t_k1_pf = dist < 0 ? 0 : dist;
    return prev;
}

int k1_set_tmem(int on) {
    const int prev = t_k1_tmem;
    t_k1_tmem = on;
    return prev;
}

int k1_set_blocked(int on) {
    const int prev = t_k1_blk;
    t_k1_blk = on;
    return prev;
}

// K1w policy, from a same-box A/B (tools/k1w_ab.py, profiles/r2/k1w_ab_r2.txt): blocks of 4
// reflectors for multi-warp groups from h = 12 -- n = 4096, h = 12 / 16: 431-441 / 560 ->
// 421-437 / 548-550 us, n = 2048, h = 12 / 16: 392-424 / 530-571 -> 383-415 / 516-552 us;
// at h = 8 / 10 and for one-warp groups (n <= 1024) the second TMEM read of each u costs
// more than the saved per-reflector exchanges; block sizes 2 and 8 measured slower
bool k1w_preferred(const FusedVariant *v, int64_t h) {
    return v->tpc > 32 && h >= 12;
}

int k1_set_stream(int on) {
    const int prev = t_k1_stream;
    t_k1_stream = on;
    return prev;
}

void k1_set_debug(int alt, int gridx) {
    t_k1_alt = alt;
    t_k1_gridx = gridx > 0 ? gridx : 1;
}

cudaError_t launch_fused(FusedArgs a, int dtype, cudaStream_t stream, LaunchInfo *info) {
    if (t_k1_stream != 0 && stream_supported(a, dtype) && (t_k1_stream >= 1 || stream_preferred(a)))
        return launch_stream(a, stream, info);
    const int E = dtype == 0 ? 4 : 2;
    const int s = dtype == 0 ? 4 : 8;
    const int64_t nv = a.n / E;
    const FusedVariant *v = pick(dtype, nv);
    if (!v) return cudaErrorNotSupported;
    const bool full = static_cast<int64_t>(v->tpc) * v->ch == nv;

    const DevAttr &da = device_attr();
    const int UT = v->tpc > 32 ? v->tpc : 32;
    const int UC = (UT / v->tpc) * v->c;
    const int NU = v->nt / UT;
    const int WPU = UT / 32;
    const size_t colB = static_cast<size_t>(a.n) * s;
    const size_t bars0 = 8 * static_cast<size_t>(2 + NU) + 8;   // + the K1t TMEM address slot
    const size_t maxs = static_cast<size_t>(da.max_smem_optin);
    const int64_t h = a.h;

    // K1t: the reflectors in TMEM (4 CH columns each; a CTA per SM may take all 512 columns,
    // two CTAs 256 each) -- fp32 variants built with the TMEM form, U resident, no gathers
    int tcols = 32;
    while (tcols < h * 4 * v->ch) tcols *= 2;
    const bool tm_ok = v->fn_tm_full != nullptr && a.mode != MODE_PAIR && h > 0 &&
                       tcols <= (v->nt <= 256 ? 256 : 512);
    const bool utm = tm_ok && (t_k1_tmem == 1 || (t_k1_tmem < 0 && k1t_preferred(v, h)));
    // K1w: the blocked form of K1t (its h x h Gram and per-pair partials follow the barriers)
    const bool ublk = utm && v->fn_tb_full != nullptr &&
                      (t_k1_blk == 1 || (t_k1_blk < 0 && k1w_preferred(v, h)));
    const int kv = ublk ? v->kb * v->c : v->c;
    const size_t red = v->tpc > 32 ? static_cast<size_t>(2) * NU * WPU * kv * s : 0;
    const size_t bars = bars0 + (ublk ? 4 * static_cast<size_t>(h * h + (h * (h + 1) / 2) * (v->tpc / 32)) : 0);

    // Shared-memory plan, in order of preference: (1) staged column tiles + resident U,
    // (2) resident U with columns loaded straight into registers (a chunked U would be
    // re-streamed from L2 for every tile: h*n*s bytes per tile), (3) staged tiles + U
    // chunks through two buffers, (4) unstaged + U chunks.
    const size_t xs_st = static_cast<size_t>(NU) * UC * colB;
    const bool pair = a.mode == MODE_PAIR;
    const size_t ub = static_cast<size_t>(h) * colB;
    int stage = 0, R = 0, nc = 1;
    size_t smem = 0;
    if (h == 0 || utm) {   // (K1t: no U in shared memory, R = 0)
        stage = pair ? 0 : 1;
        smem = (stage ? xs_st : 0) + red + bars;
    } else if (!pair && ub + xs_st + red + bars <= maxs) {
        stage = 1;
        R = static_cast<int>(h);
        smem = ub + xs_st + red + bars;
    } else if (ub + red + bars <= maxs) {
        stage = 0;
        R = static_cast<int>(h);
        smem = ub + red + bars;
    } else {
        bool ok = false;
        for (int st = pair ? 0 : 1; st >= 0 && !ok; --st) {
            const size_t fixed = (st ? xs_st : 0) + red + bars;
            const int64_t r = fixed < maxs ? static_cast<int64_t>((maxs - fixed) / (2 * colB)) : 0;
            if (r >= 1) {
                stage = st;
                R = static_cast<int>(std::min<int64_t>(r, h));
                nc = static_cast<int>((h + R - 1) / R);
                smem = 2 * static_cast<size_t>(R) * colB + fixed;
                ok = true;
            }
        }
        if (!ok) return cudaErrorNotSupported;
    }
    a.R = R;
    a.nchunks = nc;
    a.stage_x = stage;
    a.l2pf = t_k1_pf;
    a.tcols = utm ? tcols : 0;
    const void *fn = ublk ? (full ? v->fn_tb_full : v->fn_tb_ragged)
                     : utm ? (full ? v->fn_tm_full : v->fn_tm_ragged) : (full ? v->fn_full : v->fn_ragged);

    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(maxs));
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v->nt, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorNotSupported;
    const int64_t ntiles = (a.N + UC - 1) / UC;
    const int64_t need = (ntiles + NU - 1) / NU;
    const int64_t cap = static_cast<int64_t>(occ) * da.sm_count * t_k1_gridx;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(need, cap)));
    a.nbatches = static_cast<int>((ntiles + static_cast<int64_t>(grid) * NU - 1) /
                                  (static_cast<int64_t>(grid) * NU));

    void *args[] = {&a};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(v->nt), args, smem, stream);
    if (info) {
        info->variant = ublk ? v->name_tb : utm ? v->name_tm : v->name;
        info->grid = grid;
        info->block = v->nt;
        info->smem = static_cast<int>(smem);
        info->nchunks = nc;
        info->launches = 1;
    }
    return e;
}

}  // namespace hh
