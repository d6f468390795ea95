// umma_bench.cu -- tcgen05.mma throughput per SM vs N (M = 128):
// kind::f16 (bf16 x bf16 -> f32, K = 16 per instruction) and kind::i8
// (s8 x s8 -> s32, K = 32), A from shared memory (SS) or tensor memory
// (TS).  One CTA per SM; one thread issues R back-to-back MMAs (8 per loop
// iteration, descriptors precomputed) into one accumulator, commits, waits.
// Operand contents are zero (timing only).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench/umma_bench.bin tools/microbench/umma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <bool TS, bool I8>
__device__ __forceinline__ void mma(uint32_t td, uint32_t ta, uint64_t da, uint64_t db,
                                    uint32_t idesc) {
    if (TS && I8)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(td), "r"(ta),
                     "l"(db), "r"(idesc));
    else if (I8)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(td), "l"(da),
                     "l"(db), "r"(idesc));
    else if (TS)
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(td),
                     "r"(ta), "l"(db), "r"(idesc));
    else
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(td), "l"(da),
                     "l"(db), "r"(idesc));
}

// ST: warps 4.. keep storing 32 columns per thread into TMEM (columns 288+
// of their lane quarter) while the MMAs run, as the expanders do
// CM: one tcgen05.commit (to a barrier nobody waits on) after every 8 MMAs,
// as the multiply's MMA thread commits once per step
template <bool TS, bool I8, bool ST = false, bool CM = false>
__global__ void __launch_bounds__(512) umma_kernel(int N, int R, unsigned long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2;
    __shared__ volatile int stop;
    const int tid = threadIdx.x;
    if (tid == 0) stop = 0;
    for (int i = tid; i < (64 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t td = tbase;
    if (tid == 0) {
        const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
        const uint32_t idesc = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) |
                               (TS || I8 ? 0u : (1u << 15)) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        const uint64_t da = I8 ? smem_desc(s0, 128, 1024) : smem_desc(s0, 16 * 128, 128);
        const uint64_t db = smem_desc(s0 + 32768, 128, 8 * 128);
        // first MMA initializes the accumulator (enable-input-d = 0)
        if (TS && I8)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 0;" ::"r"(td),
                         "r"(td + 256u), "l"(db), "r"(idesc));
        else if (I8)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;" ::"r"(td),
                         "l"(da), "l"(db), "r"(idesc));
        else if (TS)
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;" ::"r"(td),
                         "r"(td + 256u), "l"(db), "r"(idesc));
        else
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(td),
                         "l"(da), "l"(db), "r"(idesc));
        const long long t0 = clock64();
        for (int i = 0; i < R; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) mma<TS, I8>(td, td + 256u + 8u * j, da, db, idesc);
            if (CM)
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        (uint32_t)__cvta_generic_to_shared(&bar2))
                    : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(b) : "memory");
        const long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
        stop = 1;
    } else if (ST && tid >= 128) {
        const int q = (tid >> 5) & 3;
        uint32_t w[32];
        for (int j = 0; j < 32; ++j) w[j] = 0x3F80BF80u ^ (j * 7);
        int k = 0;
        while (!stop) {
            const uint32_t ta = td + ((uint32_t)(32 * q) << 16) + 288u + 32u * (k++ % 7);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
                "%28, %29, %30, %31, %32};" ::"r"(ta),
                "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
                "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]),
                "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]),
                "r"(w[29]), "r"(w[30]), "r"(w[31]) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(td), "r"(512));
}

template <bool TS, bool I8, bool ST = false, bool CM = false>
int run(int sms, unsigned long long *cyc) {
    const int smem = 64 * 1024, R = 4096;
    CK(cudaFuncSetAttribute(umma_kernel<TS, I8, ST, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            smem));
    for (int N : {16, 64, 128, 256}) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            umma_kernel<TS, I8, ST, CM><<<sms, ST ? 512 : 128, smem>>>(N, R, cyc);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            cudaEventElapsedTime(&ms, e0, e1);
        }
        unsigned long long h[1024];
        CK(cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += (double)h[i];
        avg /= sms;
        const double flops = 2.0 * 128 * N * (I8 ? 32 : 16) * R * sms;
        printf("%-10s %s%s N=%3d: %6.1f cycles per MMA (M128 x K%d), %7.1f T(FL)OP/s over %d SMs (%.3f ms)\n",
               I8 ? "kind::i8" : "kind::f16", TS ? "TS (A in TMEM)" : "SS (A in smem)",
               ST ? " + 12 warps of tcgen05.st" : CM ? " + commit / 8 MMAs" : "", N,
               avg / R, I8 ? 32 : 16, flops / (ms * 1e-3) / 1e12, sms, ms);
    }
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long *cyc;
    CK(cudaMalloc(&cyc, sizeof(unsigned long long) * 1024));
    if (run<false, false>(sms, cyc) || run<true, false>(sms, cyc) || run<false, true>(sms, cyc) ||
        run<true, true>(sms, cyc) || run<true, false, true>(sms, cyc) ||
        run<true, true, true>(sms, cyc) || run<true, false, false, true>(sms, cyc))
        return 1;
    return 0;
}
