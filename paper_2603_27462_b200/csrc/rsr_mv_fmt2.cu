// Instantiations: u32 chunk stream (tiles wider than 32768 columns or pattern
// spaces above 2^15), register flush, v gathered from global scratch.
#include "rsr_mv_impl.cuh"

namespace rsr {
#define RSR_F2(M) [&](int k) -> KernelFn { RSR_K_SWITCH(RSR_F2K_##M) }(k)
#define RSR_F2K_0(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_U32, false>)
#define RSR_F2K_1(KK) (rsr_mv_kernel<KK, MODE_INT, FMT_U32, false>)
#define RSR_F2K_2(KK) (rsr_mv_kernel<KK, MODE_FUSED, FMT_U32, false>)
KernelFn pick_fmt2(int mode, int k) {
    if (mode == MODE_FLOAT) return RSR_F2(0);
    if (mode == MODE_INT) return RSR_F2(1);
    return RSR_F2(2);
}
}  // namespace rsr
