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
    HH_FUSED_VAR_SC(float, 256, 32, 1, 512, "f32r_tpc256_ch32_c1"),  // n <= 8192
};
const FusedVariant kF64S[] = {
    HH_FUSED_VAR_SC(double, 8, 8, 1, 256, "f64r_tpc8_ch8_c1"),        // n <= 64
    HH_FUSED_VAR_SC(double, 16, 8, 1, 256, "f64r_tpc16_ch8_c1"),      // n <= 128
    HH_FUSED_VAR_SC(double, 32, 8, 1, 256, "f64r_tpc32_ch8_c1"),      // n <= 256
    HH_FUSED_VAR_SC(double, 32, 16, 1, 256, "f64r_tpc32_ch16_c1"),    // n <= 512
    HH_FUSED_VAR_SC(double, 64, 16, 1, 512, "f64r_tpc64_ch16_c1"),    // n <= 1024
    HH_FUSED_VAR_SC(double, 128, 16, 1, 512, "f64r_tpc128_ch16_c1"),  // n <= 2048
    HH_FUSED_VAR_SC(double, 256, 16, 1, 512, "f64r_tpc256_ch16_c1"),  // n <= 4096
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
thread_local int t_sc_tmem = 1;   // A/B / test hook (hh_debug_k1r_tmem): 0 shared-memory U only, 1 policy, 2 TMEM whenever possible
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
    // Policy (same-box A/B, tools/k1g_time.py, profiles/r2/k1r_time_r2.jsonl): one-warp groups
    // (n in (512, 1024]) -- n = 1023, h = 10 / 16: 0.827 / 1.192 -> 0.648 / 0.878 ms; multi-warp
    // groups gain nothing (n = 2047 / 4095, h = 12: 1.024 / 1.073 vs 1.047 / 1.063 ms) and keep
    // the shared-memory form unless the hook forces it (2)
    const bool utm = t_sc_tmem != 0 && v->fn_tm_ragged != nullptr && a.mode != MODE_PAIR && a.h > 0 &&
                     tcols <= 512 && (v->tpc == 32 || t_sc_tmem == 2);
    const size_t ub = utm ? 0 : static_cast<size_t>(a.h) * a.n * s;
    const size_t red = v->tpc > 32 ? static_cast<size_t>(2) * NU * WPU * v->c * s : 0;
    const size_t bars = 8 * static_cast<size_t>(2 + NU) + 8;
    const size_t smem = ub + 16 + red + bars + 16;
    if (smem > static_cast<size_t>(da.max_smem_optin)) return cudaErrorNotSupported;
    a.nchunks = 1;
    a.stage_x = 0;
    a.l2pf = 0;
    a.tcols = utm ? tcols : 0;
    a.R = utm ? 0 : static_cast<int>(a.h);   // (TMEM form: no U in shared memory)
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
