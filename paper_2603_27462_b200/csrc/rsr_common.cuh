// rsr_common.cuh -- shared device helpers for the sm_100a RSR kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "../../include/rsr_b200.h"

#define RSR_FULL_MASK 0xffffffffu

namespace rsr {

// Records the last CUDA error string for rsr_last_cuda_error().
void set_cuda_error(cudaError_t e);

inline rsr_status launch_status() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return RSR_ERR_CUDA;
    }
    return RSR_OK;
}

// SM count of the current device (cached per device ordinal).
inline int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cache[dev] > 0) return cache[dev];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    if (dev >= 0 && dev < 64) cache[dev] = n;
    return n;
}

// Makes `device` current for the scope of a launch and restores the previous
// device (a view's arrays may live on a device other than the current one).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device) {
        if (device < 0) return;
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != device) {
            cudaSetDevice(device);
            prev = cur;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---- mbarrier / bulk-copy helpers (sm_90+ async proxy) -------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tTC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC_WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// Inclusive warp scan (Kogge-Stone over shuffles).
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(RSR_FULL_MASK, x, d);
        if (lane >= (uint32_t)d) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(RSR_FULL_MASK, x, d);
    return x;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint32_t bits16) {
    return __uint_as_float(bits16 << 16);
}

// Number of pattern buckets for a block of height h: 2^h binary, 3^h ternary
// (ternary keys are base-3; the order they induce equals the reference's
// 4^h code-key order because every digit is < 3 in both bases).
__host__ __device__ __forceinline__ int64_t bucket_count(int bitwidth, int h) {
    if (bitwidth == RSR_BINARY) return (int64_t)1 << h;
    int64_t b = 1;
    for (int i = 0; i < h; ++i) b *= 3;
    return b;
}

}  // namespace rsr
