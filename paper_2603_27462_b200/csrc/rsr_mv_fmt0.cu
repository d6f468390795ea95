// Instantiations: u16 chunk stream (flag bit 15), tiles <= 32768 columns;
// shared-memory buckets up to 2187 keys, register flush above.
#include "rsr_mv_impl.cuh"

namespace rsr {
#define RSR_F0(M, B) [&](int k) -> KernelFn { RSR_K_SWITCH(RSR_F0K_##M##_##B) }(k)
#define RSR_F0K_0_1(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_U16, true>)
#define RSR_F0K_1_1(KK) (rsr_mv_kernel<KK, MODE_INT, FMT_U16, true>)
#define RSR_F0K_2_1(KK) (rsr_mv_kernel<KK, MODE_FUSED, FMT_U16, true>)
#define RSR_F0K_0_0(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_U16, false>)
#define RSR_F0K_1_0(KK) (rsr_mv_kernel<KK, MODE_INT, FMT_U16, false>)
#define RSR_F0K_2_0(KK) (rsr_mv_kernel<KK, MODE_FUSED, FMT_U16, false>)
KernelFn pick_fmt0(int mode, int k, bool bucket) {
    if (bucket) {
        if (k > 11) return nullptr;
        if (mode == MODE_FLOAT) return RSR_F0(0, 1);
        if (mode == MODE_INT) return RSR_F0(1, 1);
        return RSR_F0(2, 1);
    }
    if (k < 8) return nullptr;  // every pattern space below 3^8 / 2^12 uses buckets
    if (mode == MODE_FLOAT) return RSR_F0(0, 0);
    if (mode == MODE_INT) return RSR_F0(1, 0);
    return RSR_F0(2, 0);
}
}  // namespace rsr
