// Instantiations: halfword chunk stream (format 3, rsr_stream_h.cu) with
// shared-memory pattern buckets -- the hot configuration (tiles <= 16384
// columns, <= 2187 pattern keys).  Float vectors: bf16 staged as halfwords
// (f32 += bf16 adds), f32/f16 staged as f32; int8 and fused: int16.
#include "rsr_mv_impl.cuh"

namespace rsr {
#define RSR_F3(M, V) [&](int k) -> KernelFn { RSR_K_SWITCH(RSR_F3K_##M##_##V) }(k)
#define RSR_F3K_0_1(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_H, true, VK_BF16>)
#define RSR_F3K_0_2(KK) (rsr_mv_kernel<KK, MODE_FLOAT, FMT_H, true, VK_F32X2>)
#define RSR_F3K_1_3(KK) (rsr_mv_kernel<KK, MODE_INT, FMT_H, true, VK_I16>)
#define RSR_F3K_2_3(KK) (rsr_mv_kernel<KK, MODE_FUSED, FMT_H, true, VK_I16>)
KernelFn pick_fmt3(int mode, int vk, int k) {
    if (k > 11) return nullptr;
    if (mode == MODE_FLOAT) return vk == VK_BF16 ? RSR_F3(0, 1) : RSR_F3(0, 2);
    if (mode == MODE_INT) return RSR_F3(1, 3);
    return RSR_F3(2, 3);
}
}  // namespace rsr
