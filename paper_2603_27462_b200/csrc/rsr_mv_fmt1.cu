// Instantiations: scaled u16 chunk stream with shared-memory pattern buckets
// (tiles <= 16384 columns, <= 2187 pattern keys) -- the hot configuration.
#include "rsr_mv_impl.cuh"

namespace rsr {
#define RSR_F1(M) [&](int k) -> KernelFn { RSR_K_SWITCH(RSR_F1K_##M) }(k)
#define RSR_F1K_0(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_U16_SCALED, true>)
#define RSR_F1K_1(KK) (rsr_mv_kernel<KK, MODE_INT, FMT_U16_SCALED, true>)
#define RSR_F1K_2(KK) (rsr_mv_kernel<KK, MODE_FUSED, FMT_U16_SCALED, true>)
KernelFn pick_fmt1(int mode, int k) {
    if (k > 11) return nullptr;
    if (mode == MODE_FLOAT) return RSR_F1(0);
    if (mode == MODE_INT) return RSR_F1(1);
    return RSR_F1(2);
}
}  // namespace rsr
