// rsr_mv_impl.cuh -- the sm_100a RSR multiply kernel (templates).
//
// Replaces the reference's matvec cores (pkg/src/rsrmv/_native.py:167-285)
// and its fused quantize/multiply/dequantize path (_native.py:313-353).
//
// Input: the chunk stream (include/rsr_b200.h): per cell, 32-byte chunks of
// entries; an entry is a column to gather or the pattern key of the group
// whose columns follow.  u16 formats use the quad layout (keys at slots = 0
// mod 4, column 0 = zero padding, the tile's real column 0 added from
// col0_key in the epilogue); u32 the even layout (place_group* in
// rsr_preprocess.cu).
//
// Work decomposition:
//   * grid.y = column tile.  Each CTA stages its tile of v in shared memory
//     once (the fused path quantizes while staging, after a CTA-local absmax
//     over the whole vector -- no separate quantization launch);
//   * one warp (or a team of warps) owns one (block, tile) cell at a time; a
//     round is up to 32 chunk pairs (lane runs: lane L owns a contiguous run
//     of pairs and takes one pair per round, four 16-byte loads straight into
//     registers, one round ahead), gathers v from shared memory per column
//     slot and keeps a running partial group sum;
//   * at a key slot the partial sum is flushed into the warp's PATTERN BUCKET
//     for that key (3^k ternary / 2^k binary buckets in shared memory) --
//     branch-free, predicated;
//   * when the cell is done, the pattern-table reduction y_i = sum_key
//     sgn_i(key) * bucket[key] (sign table in shared memory) produces the k
//     rows, warp-reduced and written once.
// For pattern spaces too large for shared-memory buckets the register
// variant flushes straight into k row accumulators instead.
// Integer accumulation is exact, so the int8 and fused paths are
// bit-identical to the reference.  The float path accumulates in fp32.
#pragma once

#include "rsr_common.cuh"

namespace rsr {

enum MvMode { MODE_FLOAT = 0, MODE_INT = 1, MODE_FUSED = 2 };

// chunk-stream entry formats (rsr_stream_view.format)
enum StreamFormat {
    FMT_U16 = 0,         // u16: column | key<<..., flag bit 15, tiles <= 32768
    FMT_U16_SCALED = 1,  // u16: column*4, or key*4|1; tiles <= 16384, <= 16384 keys
    FMT_U32 = 2,         // u32: column, or key | 1<<31
    FMT_H = 3            // u16: column*2 (2-byte elements), key*4|1, or a zero word
                         // h_zero_b(tn) + 4*bank; tiles <= 32704, <= 2187 keys
                         // (rsr_stream_h.cu)
};

// How format-3 kernels stage v in shared memory (template parameter VK):
enum VKind {
    VK_DEFAULT = 0,  // formats 0-2: f32 (float) / int32 or int8 (integer paths)
    VK_BF16 = 1,     // bf16 halfwords; gathers add them with add.f32.bf16
    VK_F32X2 = 2,    // f32 words, even / odd columns in two images (float32 / float16 vectors)
    VK_I16 = 3       // int16 halfwords (int8 and quantized vectors)
};
// Format 3: the 32 zero words the padding entries name sit right after the
// tile's image, at byte h_zero_b(tn) of the 2-byte image (twice that for f32
// staging); tiles up to H_MAX_TN columns keep every entry below 65536.
constexpr int64_t H_MAX_TN = 32704;
__host__ __device__ constexpr uint32_t h_zero_b(int64_t tn) {
    return (uint32_t)(((tn + 63) / 64) * 64 * 2);
}

constexpr int MV_MAX_WARPS = 20;  // 640 threads: up to 102 registers per thread
constexpr int64_t BUCKET_MAX_KEYS = 2187;  // 3^7: buckets live in smem up to here

struct MvParams {
    const void *entries;
    const int64_t *e_off;
    const uint32_t *col0_key;  // u16 formats: per-cell key of the tile's column 0
    int64_t m_rows;      // rows of the full matrix
    int64_t n;           // columns
    int64_t tw, tc;      // tile width / count
    int64_t blk0;        // first global block of this view
    int64_t nblk;        // blocks in this view
    int k;
    int bitwidth;
    int nkeys;           // pattern buckets: 3^k or 2^k
    const void *v;
    int vdtype;
    const void *vstaged; // FMT_U32: v converted/quantized in global memory
    void *y;             // output slice (view rows)
    int accumulate;
    void *part;          // tc > 1: [tc][nblk*k] partials (float or int32)
    double beta;         // fused
    double *scale_dev;   // fused: device scale slot (may be null when tc == 1)
    int dbg;             // experiment knobs (RSR_MV_DEBUG); 0 in production
    int team;            // warps per cell (bucket path): 1, 2, 4 or 8
    int pf;              // L2 prefetch distance in rounds (0 = off)
    int pdl;             // launched with programmatic stream serialization
    const double *row_beta;  // fused: per-row beta (sibling stacks), or null
    int out_bf16;        // fused: write bf16 instead of f32
    unsigned long long *probe;  // debug timeline (rsr_debug_set_probe), null in production
    const uint16_t *norm_w;  // fused: RMSNorm weight (bf16, n) applied before quantizing, or null
    float norm_eps;
    // all-gather over peer memory (rsr_matvec_peers): every output row is
    // stored to each of npeers buffers (this view's row 0 inside each
    // rank's full output; peers mapped into this device's address space)
    void *const *y_peers;
    int npeers;
};

// The output store: this view's row r into y, or into every peer's buffer.
template <class T>
__device__ __forceinline__ void put_row(const MvParams &p, int64_t r, T x) {
    if (p.npeers) {
        for (int j = 0; j < p.npeers; ++j) reinterpret_cast<T *>(p.y_peers[j])[r] = x;
    } else {
        reinterpret_cast<T *>(p.y)[r] = x;
    }
}

// CTA-wide sum of one float per thread, fixed order (identical in every CTA
// of the same shape); the result is broadcast to every thread.
__device__ __forceinline__ float cta_reduce_sum_f32(float a) {
    __shared__ float red_s[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a += __shfl_xor_sync(RSR_FULL_MASK, a, d);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red_s[warp] = a;
    __syncthreads();
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red_s[w];
    __syncthreads();
    return t;
}

// HF BitNetRMSNorm on eight bf16 values packed in a uint4 (in place):
// bf16(w * bf16(x * rs)), each product in fp32 as torch computes it.
__device__ __forceinline__ void rmsnorm8(uint4 &r, const uint4 &w8, float rs) {
    uint32_t *x = reinterpret_cast<uint32_t *>(&r);
    const uint32_t *w = reinterpret_cast<const uint32_t *>(&w8);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float lo = __uint_as_float(x[q] << 16), hi = __uint_as_float(x[q] & 0xFFFF0000u);
        const float wl = __uint_as_float(w[q] << 16), wh = __uint_as_float(w[q] & 0xFFFF0000u);
        const float nl = __bfloat162float(__float2bfloat16_rn(lo * rs));
        const float nh = __bfloat162float(__float2bfloat16_rn(hi * rs));
        const uint32_t ol = __bfloat16_as_ushort(__float2bfloat16_rn(wl * nl));
        const uint32_t oh = __bfloat16_as_ushort(__float2bfloat16_rn(wh * nh));
        x[q] = ol | (oh << 16);
    }
}

__device__ __forceinline__ float load_as_f32(const void *v, int dtype, int64_t i) {
    switch (dtype) {
        case RSR_F32: return __ldg((const float *)v + i);
        case RSR_BF16: return bf16_bits_to_f32(__ldg((const uint16_t *)v + i));
        case RSR_F16: return __half2float(__ldg((const __half *)v + i));
        default: return 0.f;
    }
}

// Reference absmax quantization of one element (_native.py:326-335).
__device__ __forceinline__ int8_t quantize_one(float x, double scale) {
    const double xs = (double)x * scale;
    double r = xs >= 0.0 ? floor(xs + 0.5) : -floor(-xs + 0.5);
    r = r > 127.0 ? 127.0 : (r < -127.0 ? -127.0 : r);
    return (int8_t)(int)r;
}

// CTA-wide max of |v| over the whole vector in float64 (order-independent,
// hence exact and identical in every CTA).
__device__ __forceinline__ double cta_absmax(const void *v, int dtype, int64_t n) {
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = fabs((double)load_as_f32(v, dtype, i));
        a = x > a ? x : a;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
        a = o > a ? o : a;
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[warp] = a;
    __syncthreads();
    if (warp == 0) {
        a = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
            a = o > a ? o : a;
        }
        if (threadIdx.x == 0) red[0] = a;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

// Sign of row i in the pattern with dense key `key`.
__device__ __forceinline__ int key_sign(uint32_t key, int i, int bitwidth) {
    if (bitwidth == RSR_BINARY) return (int)((key >> i) & 1u);
    for (int j = 0; j < i; ++j) key /= 3u;
    const uint32_t d = key % 3u;
    return d == 1u ? 1 : (d == 2u ? -1 : 0);
}

template <int K>
struct KPad {
    static constexpr int value = (K + 3) & ~3;
};

// ---- shared-memory primitives on 32-bit shared addresses -----------------
// Gathers are plain (non-volatile) asm: v is read-only while they run, so the
// compiler may schedule them freely.  Bucket updates are volatile asm and keep
// their program order with respect to each other.
template <typename Acc, int VSZ>
__device__ __forceinline__ Acc lds_v(uint32_t addr) {
    if constexpr (VSZ == 4) {
        if constexpr (std::is_same<Acc, float>::value) {
            float r;
            asm("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(addr));
            return r;
        } else {
            int r;
            asm("ld.shared.s32 %0, [%1];" : "=r"(r) : "r"(addr));
            return r;
        }
    } else {
        int r;
        asm("ld.shared.s8 %0, [%1];" : "=r"(r) : "r"(addr));
        return (Acc)r;
    }
}

// v[addr] unless `skip` (then 0): the load is predicated off for key slots.
template <typename Acc, int VSZ>
__device__ __forceinline__ Acc lds_v_unless(uint32_t skip, uint32_t addr) {
    if constexpr (VSZ == 4 && std::is_same<Acc, float>::value) {
        float r;
        asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\tmov.f32 %0, 0f00000000;\n\t"
            "@p ld.shared.f32 %0, [%2];\n\t}"
            : "=f"(r) : "r"(skip), "r"(addr));
        return r;
    } else if constexpr (VSZ == 4) {
        int r;
        asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\tmov.u32 %0, 0;\n\t"
            "@p ld.shared.s32 %0, [%2];\n\t}"
            : "=r"(r) : "r"(skip), "r"(addr));
        return r;
    } else {
        int r;
        asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\tmov.u32 %0, 0;\n\t"
            "@p ld.shared.s8 %0, [%2];\n\t}"
            : "=r"(r) : "r"(skip), "r"(addr));
        return (Acc)r;
    }
}

// if (pred) bucket += s.  In-loop flushes of one warp instruction never share
// a key (a group's in-chunk segment ends at exactly one slot), so the float
// path can use a plain read-modify-write.
__device__ __forceinline__ void bucket_flush_pred(uint32_t pred, uint32_t addr, float s) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .f32 t;\n\tsetp.ne.u32 p, %0, 0;\n\t"
        "@p ld.shared.f32 t, [%1];\n\t@p add.f32 t, t, %2;\n\t@p st.shared.f32 [%1], t;\n\t}" ::"r"(pred),
        "r"(addr), "f"(s));
}
__device__ __forceinline__ void bucket_flush_pred(uint32_t pred, uint32_t addr, int32_t s) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p red.shared.add.s32 [%1], %2;\n\t}" ::"r"(pred),
        "r"(addr), "r"(s));
}
// Batched float flush halves (volatile: ordered against every other bucket op).
__device__ __forceinline__ float lds_bucket(uint32_t addr) {
    float r;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(addr));
    return r;
}
// Eight bucket loads issued back to back (one latency for the whole batch).
__device__ __forceinline__ void lds_bucket8(const uint32_t (&a)[8], float (&r)[8]) {
    asm volatile(
        "ld.shared.f32 %0, [%8];\n\tld.shared.f32 %1, [%9];\n\tld.shared.f32 %2, [%10];\n\t"
        "ld.shared.f32 %3, [%11];\n\tld.shared.f32 %4, [%12];\n\tld.shared.f32 %5, [%13];\n\t"
        "ld.shared.f32 %6, [%14];\n\tld.shared.f32 %7, [%15];"
        : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
          "=f"(r[7])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
}
__device__ __forceinline__ void sts_bucket(uint32_t addr, float x) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(x));
}
// A chunk's last segment may continue in the next lane's chunk: atomic.
__device__ __forceinline__ void bucket_flush_final(uint32_t addr, float s) {
    asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(addr), "f"(s));
}
__device__ __forceinline__ void bucket_flush_final(uint32_t addr, int32_t s) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(s));
}

template <int K, typename Acc>
__device__ __forceinline__ void reg_flush(Acc (&acc)[K], uint32_t key, Acc s, int bitwidth) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] += (Acc)key_sign(key, i, bitwidth) * s;
}

template <int MODE, int FMT, int VK = VK_DEFAULT>
struct MvTypes {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    // staged element of v: format 3 by VK; 4 bytes for the scaled format
    // (column*4 addressing); else f32 (float) / int8 (integer paths)
    static constexpr int VSZ = FMT == FMT_H ? (VK == VK_F32X2 ? 4 : 2)
                               : ((FMT == FMT_U16_SCALED || MODE == MODE_FLOAT) ? 4 : 1);
    static constexpr bool SMEM_V = FMT != FMT_U32;
};

// Bytes of the format-3 v image in shared memory: the staged tile plus the
// 32 zero words the padding entries name.
__host__ __device__ constexpr size_t h_image_bytes(int vk, int64_t tn) {
    return vk == VK_F32X2 ? (size_t)2 * h_zero_b(tn) + 256 : (size_t)h_zero_b(tn) + 128;
}

// f32 += bf16 in one instruction (FHADD.BF16 on sm_100a).
__device__ __forceinline__ float add_bf16(float acc, uint16_t h) {
    asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(h));
    return acc;
}
__device__ __forceinline__ uint16_t lds_u16(uint32_t addr) {
    uint16_t r;
    asm("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(addr));
    return r;
}
__device__ __forceinline__ int lds_s16(uint32_t addr) {
    int r;
    asm("ld.shared.s16 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}
// u16 load unless `skip` (then +0.0 as bf16 bits)
__device__ __forceinline__ uint16_t lds_u16_unless(uint32_t skip, uint32_t addr) {
    uint16_t r;
    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\tmov.u16 %0, 0;\n\t"
        "@p ld.shared.u16 %0, [%2];\n\t}"
        : "=h"(r) : "r"(skip), "r"(addr));
    return r;
}
__device__ __forceinline__ int lds_s16_unless(uint32_t skip, uint32_t addr) {
    int r;
    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\tmov.u32 %0, 0;\n\t"
        "@p ld.shared.s16 %0, [%2];\n\t}"
        : "=r"(r) : "r"(skip), "r"(addr));
    return r;
}

// Element loader for the staging loops, templated on the input dtype.
template <int DT>
__device__ __forceinline__ float ld_elem(const void *v, int64_t i) {
    if constexpr (DT == RSR_F32) return __ldg((const float *)v + i);
    else if constexpr (DT == RSR_BF16) return bf16_bits_to_f32(__ldg((const uint16_t *)v + i));
    else if constexpr (DT == RSR_F16) return __half2float(__ldg((const __half *)v + i));
    else return (float)__ldg((const int8_t *)v + i);
}

// fn(i, x) for i in [0, cnt) with x = v[c0 + i]; 16 independent coalesced
// loads in flight per thread (a plain strided loop is a chain of L2 latencies).
template <int DT, typename Fn>
__device__ __forceinline__ void for_each_v_t(const void *v, int64_t c0, int64_t cnt, Fn fn) {
    constexpr int U = 8;
    const int64_t nt = blockDim.x;
    for (int64_t i0 = threadIdx.x; i0 < cnt; i0 += U * nt) {
        float x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * nt;
            x[u] = i < cnt ? ld_elem<DT>(v, c0 + i) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * nt;
            if (i < cnt) fn(i, x[u]);
        }
    }
}
// Real vectors only (float / fused paths): three instantiations, not four --
// the multiply kernels are i-cache sensitive when launched between other work.
template <typename Fn>
__device__ __forceinline__ void for_each_v_real(const void *v, int dtype, int64_t c0,
                                                int64_t cnt, Fn fn) {
    switch (dtype) {
        case RSR_F32: for_each_v_t<RSR_F32>(v, c0, cnt, fn); break;
        case RSR_BF16: for_each_v_t<RSR_BF16>(v, c0, cnt, fn); break;
        default: for_each_v_t<RSR_F16>(v, c0, cnt, fn); break;
    }
}
template <typename Fn>
__device__ __forceinline__ void for_each_v(const void *v, int dtype, int64_t c0, int64_t cnt,
                                           Fn fn) {
    switch (dtype) {
        case RSR_F32: for_each_v_t<RSR_F32>(v, c0, cnt, fn); break;
        case RSR_BF16: for_each_v_t<RSR_BF16>(v, c0, cnt, fn); break;
        case RSR_F16: for_each_v_t<RSR_F16>(v, c0, cnt, fn); break;
        default: for_each_v_t<RSR_I8>(v, c0, cnt, fn); break;
    }
}

// CTA-wide max |v| (float64, exact), with the batched loader.
__device__ __forceinline__ double cta_absmax_fast(const void *v, int dtype, int64_t n) {
    __shared__ double red[32];
    double a = 0.0;
    for_each_v_real(v, dtype, 0, n, [&](int64_t, float x) {
        const double ax = fabs((double)x);
        a = ax > a ? ax : a;
    });
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
        a = o > a ? o : a;
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[warp] = a;
    __syncthreads();
    if (warp == 0) {
        a = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
            a = o > a ? o : a;
        }
        if (threadIdx.x == 0) red[0] = a;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

}  // namespace rsr
#include "rsr_mv_kernel.cuh"
namespace rsr {
using KernelFn = void (*)(MvParams);

// Kernel lookup, defined per format in rsr_mv_fmt*.cu (parallel compilation).
KernelFn pick_fmt1(int mode, int k);             // FMT_U16_SCALED, buckets
KernelFn pick_fmt0(int mode, int k, bool bucket);  // FMT_U16
KernelFn pick_fmt2(int mode, int k);             // FMT_U32, register flush
KernelFn pick_fmt3(int mode, int vk, int k);     // FMT_H, buckets

#define RSR_K_SWITCH(EXPR)                                                                   \
    switch (k) {                                                                             \
        case 1: return EXPR(1); case 2: return EXPR(2); case 3: return EXPR(3);              \
        case 4: return EXPR(4); case 5: return EXPR(5); case 6: return EXPR(6);              \
        case 7: return EXPR(7); case 8: return EXPR(8); case 9: return EXPR(9);              \
        case 10: return EXPR(10); case 11: return EXPR(11); case 12: return EXPR(12);        \
        case 13: return EXPR(13); case 14: return EXPR(14); case 15: return EXPR(15);        \
        case 16: return EXPR(16);                                                            \
        default: return nullptr;                                                             \
    }

}  // namespace rsr
