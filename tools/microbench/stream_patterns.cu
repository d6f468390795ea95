// Micro-benchmark: DRAM read bandwidth of the access patterns the multiply
// kernel could use (B200).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// pattern 0: each warp streams its own contiguous region in 1 KB rounds,
// PD rounds in flight (register ring), like the multiply.
template <int PD>
__global__ void per_warp_regions(const uint4 *__restrict__ src, int64_t region_rounds,
                                 int64_t nwarps_total, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= nwarps_total) return;
    const uint4 *base = src + gw * region_rounds * 64;
    uint4 ring[PD][2];
    uint32_t acc = 0;
#pragma unroll
    for (int u = 0; u < PD; ++u) {
        ring[u][0] = __ldg(base + u * 64 + lane);
        ring[u][1] = __ldg(base + u * 64 + 32 + lane);
    }
    for (int64_t r = 0; r < region_rounds; r += PD) {
#pragma unroll
        for (int u = 0; u < PD; ++u) {
            if (r + u < region_rounds) {
                uint4 a = ring[u][0], b = ring[u][1];
                if (r + u + PD < region_rounds) {
                    ring[u][0] = __ldg(base + (r + u + PD) * 64 + lane);
                    ring[u][1] = __ldg(base + (r + u + PD) * 64 + 32 + lane);
                }
                acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// pattern 1: interleaved -- round r of warp w at (r * nwarps + w) KB.
template <int PD>
__global__ void interleaved(const uint4 *__restrict__ src, int64_t region_rounds,
                            int64_t nwarps_total, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= nwarps_total) return;
    uint4 ring[PD][2];
    uint32_t acc = 0;
    auto addr = [&](int64_t r) { return src + (r * nwarps_total + gw) * 64; };
#pragma unroll
    for (int u = 0; u < PD; ++u) {
        ring[u][0] = __ldg(addr(u) + lane);
        ring[u][1] = __ldg(addr(u) + 32 + lane);
    }
    for (int64_t r = 0; r < region_rounds; r += PD) {
#pragma unroll
        for (int u = 0; u < PD; ++u) {
            if (r + u < region_rounds) {
                uint4 a = ring[u][0], b = ring[u][1];
                if (r + u + PD < region_rounds) {
                    ring[u][0] = __ldg(addr(r + u + PD) + lane);
                    ring[u][1] = __ldg(addr(r + u + PD) + 32 + lane);
                }
                acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void linear(const uint4 *__restrict__ src, int64_t n16, uint32_t *out) {
    uint32_t acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint4 a = __ldg(src + i);
        acc ^= a.x ^ a.y ^ a.z ^ a.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
float time_it(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main1() {
    const int64_t warps_per_cta = 19, ctas = 144, nw = warps_per_cta * ctas;
    const int64_t rounds = 36;  // 36 KB per warp (like a C2 cell)
    const int64_t bytes = nw * rounds * 1024;
    // 4 copies to defeat L2 (rotate)
    uint4 *buf[4];
    for (auto &b : buf) cudaMalloc(&b, bytes), cudaMemset(b, 1, bytes);
    uint32_t *out;
    cudaMalloc(&out, 4);
    int it = 0;
    auto report = [&](const char *name, float ms) {
        printf("%-40s %8.2f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    report("per-warp regions PD=4 (19w x 144)", time_it([&] {
        per_warp_regions<4><<<ctas, warps_per_cta * 32>>>(buf[it++ & 3], rounds, nw, out); }));
    report("per-warp regions PD=8", time_it([&] {
        per_warp_regions<8><<<ctas, warps_per_cta * 32>>>(buf[it++ & 3], rounds, nw, out); }));
    report("per-warp regions PD=2", time_it([&] {
        per_warp_regions<2><<<ctas, warps_per_cta * 32>>>(buf[it++ & 3], rounds, nw, out); }));
    report("interleaved PD=4", time_it([&] {
        interleaved<4><<<ctas, warps_per_cta * 32>>>(buf[it++ & 3], rounds, nw, out); }));
    report("interleaved PD=8", time_it([&] {
        interleaved<8><<<ctas, warps_per_cta * 32>>>(buf[it++ & 3], rounds, nw, out); }));
    // same total bytes with 2x the warps (half regions)
    report("per-warp regions PD=4, 38w x 144", time_it([&] {
        per_warp_regions<4><<<ctas * 2, warps_per_cta * 32>>>(buf[it++ & 3], rounds / 2, nw * 2, out); }));
    report("linear grid-stride 148x1024", time_it([&] {
        linear<<<148 * 2, 1024>>>(buf[it++ & 3], bytes / 16, out); }));
    report("linear grid-stride 148x8x256", time_it([&] {
        linear<<<148 * 8, 256>>>(buf[it++ & 3], bytes / 16, out); }));
    return 0;
}

// ---- pattern 2: TMA 1-D bulk copies into a per-warp shared ring -----------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile("{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra LAB_WAIT;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase) : "memory");
}

template <int S, int STAGE_BYTES>
__global__ void tma_ring(const char *__restrict__ src, int64_t region_bytes, int64_t nwarps_total,
                         uint32_t *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    unsigned char *ring = sm + (size_t)warp * S * STAGE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)(blockDim.x >> 5) * S * STAGE_BYTES) + warp * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    if (gw >= nwarps_total) return;
    const char *base = src + gw * region_bytes;
    const int64_t nst = region_bytes / STAGE_BYTES;
    if (lane == 0)
        for (int s = 0; s < S && s < nst; ++s) {
            mbar_expect_tx(bars + s, STAGE_BYTES);
            bulk_g2s(ring + s * STAGE_BYTES, base + s * STAGE_BYTES, STAGE_BYTES, bars + s);
        }
    uint32_t acc = 0;
    for (int64_t i = 0; i < nst; ++i) {
        const int s = (int)(i % S);
        mbar_wait(bars + s, (uint32_t)((i / S) & 1));
        const uint4 *st = reinterpret_cast<const uint4 *>(ring + s * STAGE_BYTES);
#pragma unroll
        for (int q = 0; q < STAGE_BYTES / 512; ++q) {
            uint4 a = st[q * 32 + lane];
            acc ^= a.x ^ a.y ^ a.z ^ a.w;
        }
        __syncwarp();
        if (lane == 0 && i + S < nst) {
            mbar_expect_tx(bars + s, STAGE_BYTES);
            bulk_g2s(ring + s * STAGE_BYTES, base + (i + S) * STAGE_BYTES, STAGE_BYTES, bars + s);
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main2() {
    const int64_t warps_per_cta = 19, ctas = 144, nw = warps_per_cta * ctas;
    const int64_t region = 36 * 1024;
    const int64_t bytes = nw * region;
    char *buf[4];
    for (auto &b : buf) cudaMalloc(&b, bytes), cudaMemset(b, 1, bytes);
    uint32_t *out;
    cudaMalloc(&out, 4);
    int it = 0;
    auto report = [&](const char *name, float ms) {
        printf("%-40s %8.2f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
#define TMA_CASE(S, SB)                                                                          \
    {                                                                                            \
        size_t smem = warps_per_cta * (S) * (SB) + warps_per_cta * (S) * 8;                     \
        cudaFuncSetAttribute(tma_ring<S, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        char name[64];                                                                           \
        snprintf(name, 64, "tma ring S=%d stage=%dB (19w)", S, SB);                             \
        report(name, time_it([&] { tma_ring<S, SB><<<ctas, warps_per_cta * 32, smem>>>(buf[it++ & 3], region, nw, out); })); \
        printf("   err=%s\n", cudaGetErrorString(cudaGetLastError()));                          \
    }
    TMA_CASE(2, 1024)
    TMA_CASE(4, 1024)
    TMA_CASE(8, 1024)
    TMA_CASE(4, 2048)
    TMA_CASE(2, 4096)
    return 0;
}
int main() { main1(); main2(); return 0; }
