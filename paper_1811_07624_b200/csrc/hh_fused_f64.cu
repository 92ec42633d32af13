// hh_fused_f64.cu -- fp64 instantiations of the fused kernel.
#include "hh_fused_kernel.cuh"

namespace hh {

namespace {
// n in (512, 4096]: one 512-thread CTA per SM sharing one staged U (as for fp32); same-box A/B
// (2^26 elements): n = 2048, h = 8 414 -> 308 us; n = 4096, h = 6 / 12 359 / 820 -> 299 / 607 us;
// n = 1024 equal; n = 512 2.5 % slower at 512 threads, so it keeps 256
const FusedVariant kF64[] = {
    HH_FUSED_VAR(double, 8, 4, 1, 256, "f64_tpc8_ch4_c1"),      // n <= 64
    HH_FUSED_VAR(double, 16, 4, 1, 256, "f64_tpc16_ch4_c1"),    // n <= 128
    HH_FUSED_VAR(double, 32, 4, 1, 256, "f64_tpc32_ch4_c1"),    // n <= 256
    HH_FUSED_VAR(double, 32, 8, 1, 256, "f64_tpc32_ch8_c1"),    // n <= 512
    HH_FUSED_VAR(double, 64, 8, 1, 512, "f64_tpc64_ch8_c1"),    // n <= 1024
    HH_FUSED_VAR(double, 128, 8, 1, 512, "f64_tpc128_ch8_c1"),  // n <= 2048
    HH_FUSED_VAR(double, 256, 8, 1, 512, "f64_tpc256_ch8_c1"),  // n <= 4096
};
}  // namespace

const FusedVariant *fused_table_f64(int *count) {
    *count = static_cast<int>(sizeof(kF64) / sizeof(kF64[0]));
    return kF64;
}

}  // namespace hh
