// hh_fused_f32.cu -- fp32 instantiations of the fused kernel.
#include "hh_fused_kernel.cuh"

namespace hh {

namespace {
// n in (512, 4096]: one 512-thread CTA per SM (16 warps, U staged once per SM) rather than two
// 256-thread CTAs that each hold a copy of U -- the copy halved the occupancy from h = 11
// (n = 1024) / h = 7 (n = 2048); same-box sweep: n = 2048, h = 12 0.634 -> 0.469 ms, C5 h=12
// 0.553 -> 0.534 ms, C2 unchanged (profiles/r1/crossover_r1.txt); n in (4096, 8192] likewise
// (two 256-thread units): h = 4 / 8 / 12 0.529 / 1.093 / 1.510 -> 0.384 / 0.815 / 1.133 ms
const FusedVariant kF32[] = {
    HH_FUSED_VAR(float, 8, 2, 1, 256, "f32_tpc8_ch2_c1"),      // n <= 64
    HH_FUSED_VAR(float, 8, 4, 1, 256, "f32_tpc8_ch4_c1"),      // n <= 128
    HH_FUSED_VAR(float, 16, 4, 1, 256, "f32_tpc16_ch4_c1"),    // n <= 256
    HH_FUSED_VAR_TM(float, 32, 4, 2, 256, "f32_tpc32_ch4_c2"),    // n <= 512
    HH_FUSED_VAR_TB(float, 32, 8, 2, 512, "f32_tpc32_ch8_c2", 4),    // n <= 1024
    HH_FUSED_VAR_TB(float, 64, 8, 2, 512, "f32_tpc64_ch8_c2", 4),    // n <= 2048
    HH_FUSED_VAR_TB(float, 128, 8, 2, 512, "f32_tpc128_ch8_c2", 4),  // n <= 4096
    HH_FUSED_VAR(float, 256, 8, 1, 512, "f32_tpc256_ch8_c1"),  // n <= 8192
};
// alternatives for same-box A/B only (hh_debug_k1 forces one): two-warp column groups with
// four columns each (half the u reads per column), 256-thread CTAs
const FusedVariant kF32Alt[] = {
    HH_FUSED_VAR(float, 64, 4, 4, 512, "f32_tpc64_ch4_c4_nt512"),
    HH_FUSED_VAR(float, 64, 4, 2, 512, "f32_tpc64_ch4_c2_nt512"),
    HH_FUSED_VAR(float, 32, 8, 2, 256, "f32_tpc32_ch8_c2_nt256"),
    HH_FUSED_VAR(float, 128, 2, 4, 512, "f32_tpc128_ch2_c4_nt512"),
    HH_FUSED_VAR_TB(float, 128, 8, 2, 512, "f32_tpc128_ch8_c2", 2),   // K1w block sizes
    HH_FUSED_VAR_TB(float, 128, 8, 2, 512, "f32_tpc128_ch8_c2", 8),
    HH_FUSED_VAR_TB(float, 64, 8, 2, 512, "f32_tpc64_ch8_c2", 2),
    HH_FUSED_VAR_TB(float, 64, 8, 2, 512, "f32_tpc64_ch8_c2", 8),
};
}  // namespace

const FusedVariant *fused_alt_f32(int *count) {
    *count = static_cast<int>(sizeof(kF32Alt) / sizeof(kF32Alt[0]));
    return kF32Alt;
}

const FusedVariant *fused_table_f32(int *count) {
    *count = static_cast<int>(sizeof(kF32) / sizeof(kF32[0]));
    return kF32;
}

}  // namespace hh
