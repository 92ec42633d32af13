// hh_fused_sc.cu -- K1r: the scalar-element instantiations of the fused kernel and their
// launcher.  Same persistent kernel as K1 (hh_fused_kernel.cuh, SC = true): a group of TPC
// threads owns a column, thread gt the elements gt + TPC k, the column stays in registers for
// all h reflectors; but every access is one element wide (lanes on consecutive elements:
// coalesced 128-byte rows per warp access), so the column stride and the pointers need
// element alignment only.  Serves the shapes K1 refuses (n * size not a multiple of 16 bytes,
// or merely element-aligned operands) for n up to the K1 tables when U fits in shared memory;
// K1g (hh_general.cu) takes what is left.
#include <algorithm>

#include "hh_fused_kernel.cuh"

namespace hh {
namespace {

const FusedVariant kF32S[] = {
    HH_FUSED_VAR_SC(float, 8, 8, 1, 256, "f32r_tpc8_ch8_c1"),        // n <= 64
    HH_FUSED_VAR_SC(float, 8, 16, 1, 256, "f32r_tpc8_ch16_c1"),      // n <= 128
    HH_FUSED_VAR_SC(float, 16, 16, 1, 256, "f32r_tpc16_ch16_c1"),    // n <= 256
    HH_FUSED_VAR_SC(float, 32, 16, 2, 256, "f32r_tpc32_ch16_c2"),    // n <= 512
    HH_FUSED_VAR_SC_TM(float, 32, 32, 2, 512, "f32r_tpc32_ch32_c2"),    // n <= 1024
    HH_FUSED_VAR_SC_TM(float, 64, 32, 2, 512, "f32r_tpc64_ch32_c2"),    // n <= 2048
    HH_FUSED_VAR_SC_TM(float, 128, 32, 2, 512, "f32r_tpc128_ch32_c2"),  // n <= 4096
    // (a 256-thread one-column form for n <= 8192 measured slower than K1g -- n = 4097, h = 12:
    // 4.0 vs 3.4 ms -- and was dropped: K1g or the padded detour serve n > 4096)
};
const FusedVariant kF64S[] = {
    HH_FUSED_VAR_SC(double, 8, 8, 1, 256, "f64r_tpc8_ch8_c1"),        // n <= 64
    HH_FUSED_VAR_SC(double, 16, 8, 1, 256, "f64r_tpc16_ch8_c1"),      // n <= 128
    HH_FUSED_VAR_SC(double, 32, 8, 1, 256, "f64r_tpc32_ch8_c1"),      // n <= 256
    HH_FUSED_VAR_SC(double, 32, 16, 1, 256, "f64r_tpc32_ch16_c1"),    // n <= 512
    HH_FUSED_VAR_SC(double, 64, 16, 1, 512, "f64r_tpc64_ch16_c1"),    // n <= 1024
    HH_FUSED_VAR_SC(double, 128, 16, 1, 512, "f64r_tpc128_ch16_c1"),  // n <= 2048
};

}  // namespace

const FusedVariant *fused_table_scalar(int dtype, int *count) {
    if (dtype == 0) {
        *count = static_cast<int>(sizeof(kF32S) / sizeof(kF32S[0]));
        return kF32S;
    }
    *count = static_cast<int>(sizeof(kF64S) / sizeof(kF64S[0]));
    return kF64S;
}

namespace {
thread_local int t_sc_tmem = 1;   // A/B / test hook (hh_debug_k1r_tmem): 0 = shared-memory U only
}
namespace {
thread_local int t_sc_stage = 1;   // A/B / test hook (hh_debug_k1r_stage): 0 = columns straight into registers
}
int k1r_set_stage(int on) {
    const int prev = t_sc_stage;
    t_sc_stage = on;
    return prev;
}
int k1r_set_tmem(int on) {
    const int prev = t_sc_tmem;
    t_sc_tmem = on;
    return prev;
}

// cudaErrorNotSupported when no variant holds n or U does not fit in shared memory (the
// caller then runs K1g)
cudaError_t launch_fused_scalar(FusedArgs a, int dtype, cudaStream_t stream, LaunchInfo *info) {
    int cnt = 0;
    const FusedVariant *tab = fused_table_scalar(dtype, &cnt);
    const FusedVariant *v = nullptr;
    for (int i = 0; i < cnt && !v; ++i)
        if (static_cast<int64_t>(tab[i].tpc) * tab[i].ch >= a.n) v = &tab[i];
    if (!v) return cudaErrorNotSupported;
    const DevAttr &da = device_attr();
    const int s = dtype == 0 ? 4 : 8;
    const int UT = v->tpc > 32 ? v->tpc : 32;
    const int UC = (UT / v->tpc) * v->c;
    const int NU = v->nt / UT;
    const int WPU = UT / 32;
    // the reflectors in TMEM (CH columns each, 512 per CTA) when the variant has the form:
    // one tcgen05.ld per reflector instead of 2 CH one-element shared-memory reads
    int tcols = 32;
    while (tcols < a.h * v->ch) tcols *= 2;
    // Same-box A/B (tools/k1g_time.py, profiles/r2/k1r_time_r2.jsonl), with staged tiles:
    // n = 1023, h = 10 / 16: 0.75 / 1.11 -> 0.56 / 0.80 ms; n = 2047, h = 12: 1.00 -> 0.78;
    // n = 4095, h = 12: 1.16 -> 1.04 (U in TMEM also leaves the shared memory to the slots)
    const bool utm = t_sc_tmem != 0 && v->fn_tm_ragged != nullptr && a.mode != MODE_PAIR && a.h > 0 &&
                     tcols <= 512;
    // (shared-memory U: rows at pitch TPC CH, zero padded -- see the kernel; the kernel places
    // what follows U at R n elements, so R covers the padded rows)
    const int64_t Rpad = utm ? 0 : (a.h * v->tpc * v->ch + a.n - 1) / a.n;
    const size_t ub = static_cast<size_t>(Rpad) * a.n * s;
    const size_t red = v->tpc > 32 ? static_cast<size_t>(2) * NU * WPU * v->c * s : 0;
    const size_t bars = 8 * static_cast<size_t>(2 + NU) + 8;
    // staged column tiles (bulk copies of each tile's 16-byte superset, the next tile in flight
    // while this one computes, as in K1) when X is 16-byte aligned and the slots fit
    const size_t spitch = (static_cast<size_t>(UC) * a.n * s + 31) & ~static_cast<size_t>(15);
    const size_t base = ub + 16 + red + bars + 16;
    const bool stage = t_sc_stage != 0 && a.mode != MODE_PAIR && a.N > UC &&
                       (reinterpret_cast<uintptr_t>(a.X) & 15u) == 0 &&
                       base + NU * spitch <= static_cast<size_t>(da.max_smem_optin);
    const size_t smem = base + (stage ? NU * spitch : 0);
    if (smem > static_cast<size_t>(da.max_smem_optin)) return cudaErrorNotSupported;
    a.nchunks = 1;
    a.stage_x = stage ? 1 : 0;
    a.l2pf = 0;
    a.tcols = utm ? tcols : 0;
    a.R = static_cast<int>(Rpad);   // (TMEM form: no U in shared memory)
    const void *fn = utm ? v->fn_tm_ragged : v->fn_ragged;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         da.max_smem_optin);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, v->nt, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorNotSupported;
    const int64_t ntiles = (a.N + UC - 1) / UC;
    const int64_t need = (ntiles + NU - 1) / NU;
    const int64_t cap = static_cast<int64_t>(occ) * da.sm_count;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(need, cap)));
    a.nbatches = static_cast<int>((ntiles + static_cast<int64_t>(grid) * NU - 1) /
                                  (static_cast<int64_t>(grid) * NU));
    void *args[] = {&a};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(v->nt), args, smem, stream);
    if (info) {
        info->variant = utm ? v->name_tm : v->name;
        info->grid = grid;
        info->block = v->nt;
        info->smem = static_cast<int>(smem);
        info->nchunks = 1;
        info->launches = 1;
    }
    return e;
}

}  // namespace hh
