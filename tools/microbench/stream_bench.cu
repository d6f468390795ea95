// stream_bench.cu -- how fast can 2731 warps each stream their own ~36 KB
// region (the C2 cell pattern: rounds of 2 KiB per warp) on a B200?
// Variants: grid-stride read (reference), per-warp rounds through registers
// with D rounds in flight, and per-warp rounds through a cp.async.bulk ring of
// S stages.  No compute: the XOR of the data is written once per warp.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/stream_bench tools/microbench/stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <string>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_na(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__global__ void grid_read(const uint4 *p, int64_t n4, uint32_t *out) {
    uint32_t x = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = ldg_na(p + i);
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678u) out[0] = x;
}

// each warp: `rounds` rounds of 2 KiB starting at warp * rounds * 2 KiB
template <int D>
__global__ void warp_reg(const uint4 *p, int64_t ncells, int rounds, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= ncells) return;
    const uint4 *base = p + w * (int64_t)rounds * 128;
    uint4 q[D][4];
    uint32_t x = 0;
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < rounds)
#pragma unroll
            for (int j = 0; j < 4; ++j) q[d][j] = ldg_na(base + d * 128 + j * 32 + lane);
    for (int r = 0; r < rounds; r += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if (r + d < rounds) {
#pragma unroll
                for (int j = 0; j < 4; ++j) x ^= q[d][j].x ^ q[d][j].y ^ q[d][j].z ^ q[d][j].w;
                if (r + d + D < rounds)
#pragma unroll
                    for (int j = 0; j < 4; ++j) q[d][j] = ldg_na(base + (r + d + D) * 128 + j * 32 + lane);
            }
        }
    }
    if (x == 0x12345678u) out[0] = x;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

__global__ void warp_tma(const uint4 *p, int64_t ncells, int rounds, int S, uint32_t *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t w = (int64_t)blockIdx.x * nw + warp;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sm) + warp * S * 2048;
    const uint32_t bars = (uint32_t)__cvta_generic_to_shared(sm) + nw * S * 2048 + warp * S * 8;
    if (w >= ncells) return;
    const char *base = reinterpret_cast<const char *>(p + w * (int64_t)rounds * 128);
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bars + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    int is = 0;
    for (int r = 0; r < S - 1 && r < rounds; ++r, ++is)
        if (lane == 0) { mbar_expect(bars + 8 * r, 2048); bulk(ring + 2048 * r, base + 2048 * r, 2048, bars + 8 * r); }
    uint32_t x = 0;
    for (int r = 0; r < rounds; ++r) {
        __syncwarp();
        if (is < rounds) {
            const int st = is % S;
            if (lane == 0) { mbar_expect(bars + 8 * st, 2048); bulk(ring + 2048 * st, base + 2048 * (int64_t)is, 2048, bars + 8 * st); }
            ++is;
        }
        const int st = r % S;
        mbar_wait(bars + 8 * st, (r / S) & 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ring + 2048 * st + (j * 32 + lane) * 16));
            x ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (x == 0x12345678u) out[0] = x;
}

int main() {
    const int64_t ncells = 2731, rounds = 18;
    const int64_t bytes = ncells * rounds * 2048;  // 100.7 MB
    const int ncopies = 4;
    uint4 *buf[ncopies];
    for (int i = 0; i < ncopies; ++i) { CK(cudaMalloc(&buf[i], bytes)); CK(cudaMemset(buf[i], i, bytes)); }
    uint32_t *out; CK(cudaMalloc(&out, 64));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 40;
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 8; ++i) launch(buf[i % ncopies]);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) launch(buf[i % ncopies]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("%-40s %7.2f us  %6.2f TB/s  (%s)\n", name, us, bytes / us / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int g : {148 * 2, 148 * 4, 148 * 8})
        run((std::string("grid-stride read, grid ") + std::to_string(g)).c_str(), [&](uint4 *p) { grid_read<<<g, 1024>>>(p, bytes / 16, out); });
    for (int wpc : {19, 16, 32}) {
        const int grid = (ncells + wpc - 1) / wpc;
        char nm[64];
        snprintf(nm, 64, "warp regs D=1 w/cta %d", wpc); run(nm, [&](uint4 *p) { warp_reg<1><<<grid, wpc * 32>>>(p, ncells, rounds, out); });
        snprintf(nm, 64, "warp regs D=2 w/cta %d", wpc); run(nm, [&](uint4 *p) { warp_reg<2><<<grid, wpc * 32>>>(p, ncells, rounds, out); });
        snprintf(nm, 64, "warp regs D=3 w/cta %d", wpc); run(nm, [&](uint4 *p) { warp_reg<3><<<grid, wpc * 32>>>(p, ncells, rounds, out); });
        snprintf(nm, 64, "warp regs D=4 w/cta %d", wpc); run(nm, [&](uint4 *p) { warp_reg<4><<<grid, wpc * 32>>>(p, ncells, rounds, out); });
        for (int S : {2, 3, 4, 6}) {
            const size_t smem = (size_t)wpc * S * (2048 + 8);
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(warp_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            snprintf(nm, 64, "warp TMA ring S=%d w/cta %d", S, wpc);
            run(nm, [&](uint4 *p) { warp_tma<<<grid, wpc * 32, smem>>>(p, ncells, rounds, S, out); });
        }
    }
    return 0;
}
