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
thread_local int t_k1_stream = -1;   // K1s (hh_stream.cu): -1 measured policy, 0 never, 1 always

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
    const size_t red = v->tpc > 32 ? static_cast<size_t>(2) * NU * WPU * v->c * s : 0;
    const size_t bars = 8 * static_cast<size_t>(2 + NU);
    const size_t maxs = static_cast<size_t>(da.max_smem_optin);
    const int64_t h = a.h;

    // Shared-memory plan, in order of preference: (1) staged column tiles + resident U,
    // (2) resident U with columns loaded straight into registers (a chunked U would be
    // re-streamed from L2 for every tile: h*n*s bytes per tile), (3) staged tiles + U
    // chunks through two buffers, (4) unstaged + U chunks.
    const size_t xs_st = static_cast<size_t>(NU) * UC * colB;
    const bool pair = a.mode == MODE_PAIR;
    const size_t ub = static_cast<size_t>(h) * colB;
    int stage = 0, R = 0, nc = 1;
    size_t smem = 0;
    if (h == 0) {
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
    const void *fn = full ? v->fn_full : v->fn_ragged;

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
        info->variant = v->name;
        info->grid = grid;
        info->block = v->nt;
        info->smem = static_cast<int>(smem);
        info->nchunks = nc;
        info->launches = 1;
    }
    return e;
}

}  // namespace hh
