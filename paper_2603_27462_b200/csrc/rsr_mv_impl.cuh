// rsr_mv_impl.cuh -- the sm_100a RSR multiply kernel (templates).
//
// Replaces the reference's matvec cores (pkg/src/rsrmv/_native.py:167-285)
// and its fused quantize/multiply/dequantize path (_native.py:313-353).
//
// Input: the chunk stream (include/rsr_b200.h): per cell, 32-byte chunks of
// entries; an entry is a column to gather or the pattern key of the group
// whose columns follow; every chunk starts with a key and keys only sit at
// even slots (place_group in rsr_preprocess.cu).
//
// Work decomposition:
//   * grid.y = column tile.  Each CTA stages its tile of v in shared memory
//     once (the fused path quantizes while staging, after a CTA-local absmax
//     over the whole vector -- no separate quantization launch);
//   * one warp owns one (block, tile) cell at a time; in each round lane L
//     owns chunk L (two coalesced 16-byte loads per lane, the next round
//     prefetched), gathers v from shared memory per column slot and keeps a
//     running partial group sum;
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
    FMT_U32 = 2          // u32: column, or key | 1<<31
};

constexpr int MV_MAX_WARPS = 20;  // 640 threads: up to 102 registers per thread
constexpr int64_t BUCKET_MAX_KEYS = 2187;  // 3^7: buckets live in smem up to here

struct MvParams {
    const void *entries;
    const int64_t *e_off;
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
    int pf;              // L2 prefetch distance in rounds (0 = off)
    int team;            // warps per cell (ring path): 1, 2, 4 or 8
    const double *row_beta;  // fused: per-row beta (sibling stacks), or null
    int out_bf16;        // fused: write bf16 instead of f32
    int stages;          // TMA ring depth per warp (bucket path)
    unsigned long long *probe;  // debug timeline (rsr_debug_set_probe), null in production
};

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

template <int MODE, int FMT>
struct MvTypes {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    // staged element of v: 4 bytes for the scaled format (column*4 addressing),
    // else f32 (float) / int8 (integer paths)
    static constexpr int VSZ = (FMT == FMT_U16_SCALED || MODE == MODE_FLOAT) ? 4 : 1;
    static constexpr bool SMEM_V = FMT != FMT_U32;
};

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
    constexpr int U = 16;
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
    for_each_v(v, dtype, 0, n, [&](int64_t, float x) {
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
#if 0  // superseded register-ring kernel (kept out of the build)
template <int K, int MODE, int FMT, bool BUCKET>
__global__ void __launch_bounds__(MV_MAX_WARPS * 32)
rsr_mv_kernel_old(MvParams p) {
    using T = MvTypes<MODE, FMT>;
    using Acc = typename T::Acc;
    constexpr int VSZ = T::VSZ;
    constexpr bool SMEM_V = T::SMEM_V;
    constexpr int CH = FMT == FMT_U32 ? 8 : 16;  // entries per 32-byte chunk
    constexpr int KP = KPad<K>::value;
    constexpr int PD = 4;                        // rounds in flight (bucket path)

    extern __shared__ __align__(16) unsigned char mv_smem[];
    const int nwarps = blockDim.x >> 5;
    const int64_t t = blockIdx.y;
    const int64_t c0 = t * p.tw;
    const int64_t tn = min(p.tw, p.n - c0);
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const uint4 *__restrict__ ent4 = reinterpret_cast<const uint4 *>(p.entries);
    const int64_t bstride = (int64_t)gridDim.x * nwarps;

    // smem carve-up: [v tile][sign table NB x KP][buckets nwarps x NB]
    size_t off = 0;
    unsigned char *vsm = mv_smem;
    if constexpr (SMEM_V) off += ((size_t)tn * VSZ + 15) & ~(size_t)15;
    Acc *__restrict__ stab = reinterpret_cast<Acc *>(mv_smem + off);
    if constexpr (BUCKET) off += (size_t)p.nkeys * KP * sizeof(Acc);
    Acc *__restrict__ buckets = reinterpret_cast<Acc *>(mv_smem + off);
    Acc *__restrict__ bk = buckets + (size_t)warp * p.nkeys;
    const uint32_t vbase = (uint32_t)__cvta_generic_to_shared(vsm);
    const uint32_t bkbase = (uint32_t)__cvta_generic_to_shared(bk);

    // ---- bucket-path stream helpers (see the round loop below) -------------
    constexpr bool SC = FMT == FMT_U16_SCALED;
    auto load_round = [&](int64_t gb, int64_t cend, uint4 &q0, uint4 &q1) {
        const int64_t nr = min((int64_t)32, cend - gb);
        q0 = make_uint4(0, 0, 0, 0);
        q1 = q0;
        if ((int64_t)lane < nr) {
            q0 = __ldg(ent4 + 2 * gb + lane);
            q1 = __ldg(ent4 + 2 * gb + nr + lane);
        }
    };
    uint4 ring[PD][2];
    int64_t b = (int64_t)blockIdx.x * nwarps + warp;
    int64_t ch0 = 0, ch1 = 0;
    if constexpr (FMT != FMT_U32 && BUCKET) {
        // start the first cell's stream before the prologue so its DRAM
        // latency overlaps the staging of v
        if (b < p.nblk && !(p.dbg & 512)) {
            const int64_t dc = b * p.tc + t;
            ch0 = p.e_off[dc] / CH;
            ch1 = p.e_off[dc + 1] / CH;
#pragma unroll
            for (int u = 0; u < PD; ++u) load_round(ch0 + 32 * u, ch1, ring[u][0], ring[u][1]);
        }
    }

    // ---- prologue -------------------------------------------------------
    double scale = 1.0;
    if constexpr (MODE == MODE_FUSED) {
        if constexpr (SMEM_V) {
            const double amax = cta_absmax_fast(p.v, p.vdtype, p.n);
            scale = amax == 0.0 ? 1.0 : 127.0 / amax;
            if (p.scale_dev && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
                *p.scale_dev = scale;
        } else {
            scale = *p.scale_dev;  // written by the staging kernel
        }
    }
    if (!(p.dbg & 128)) if constexpr (SMEM_V) {
        if constexpr (MODE == MODE_FLOAT) {
            for_each_v(p.v, p.vdtype, c0, tn,
                       [&](int64_t i, float x) { reinterpret_cast<float *>(vsm)[i] = x; });
        } else {
            const int dt = MODE == MODE_INT ? (int)RSR_I8 : p.vdtype;
            for_each_v(p.v, dt, c0, tn, [&](int64_t i, float x) {
                const int8_t q = MODE == MODE_INT ? (int8_t)x : quantize_one(x, scale);
                if constexpr (VSZ == 4) reinterpret_cast<int32_t *>(vsm)[i] = q;
                else reinterpret_cast<int8_t *>(vsm)[i] = q;
            });
        }
    }
    if (!(p.dbg & 256)) if constexpr (BUCKET) {
        for (int key = threadIdx.x; key < p.nkeys; key += blockDim.x) {
            uint32_t kk = (uint32_t)key;
#pragma unroll
            for (int i = 0; i < KP; ++i) {
                int sg = 0;
                if (p.bitwidth == RSR_BINARY) {
                    sg = (int)((kk >> i) & 1u);
                } else {
                    const uint32_t q3 = kk / 3u, d = kk - 3u * q3;
                    kk = q3;
                    sg = d == 1u ? 1 : (d == 2u ? -1 : 0);
                }
                stab[key * KP + i] = (Acc)(i < K ? sg : 0);
            }
        }
        for (int i = threadIdx.x; i < nwarps * p.nkeys; i += blockDim.x) buckets[i] = (Acc)0;
    }
    __syncthreads();
    if (p.dbg & 64) return;  // prologue only (experiment)

    using VG = typename std::conditional<MODE == MODE_FLOAT, float, int8_t>::type;
    const VG *__restrict__ vglob = reinterpret_cast<const VG *>(p.vstaged) + c0;

    // ---- per-cell epilogue: pattern-table reduction + warp reduce + store ----
    auto finish_cell = [&](int64_t bb, Acc (&acc)[K]) {
        // y_i = sum_key sgn_i(key) * bucket[key]  (bucket 0 collects padding)
        if constexpr (BUCKET) {
            for (int key = lane; key < ((p.dbg & 4) ? 0 : p.nkeys); key += 32) {
                const Acc bv = key ? bk[key] : (Acc)0;
                bk[key] = (Acc)0;
                const Acc *row = stab + key * KP;
#pragma unroll
                for (int i = 0; i < K; ++i) acc[i] += row[i] * bv;
            }
            __syncwarp();
        }
        const int64_t row0 = bb * p.k;  // row within the view
        const int64_t grow0 = (p.blk0 + bb) * p.k;
        Acc mine = (Acc)0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const Acc r = warp_sum(acc[i]);
            if (lane == (uint32_t)i) mine = r;
        }
        if (lane < (uint32_t)K && grow0 + lane < p.m_rows) {
            const int64_t r = row0 + lane;
            if (p.tc > 1) {
                const int64_t rows_view = p.nblk * p.k;
                reinterpret_cast<Acc *>(p.part)[t * rows_view + r] = mine;
            } else if constexpr (MODE == MODE_FLOAT) {
                float *y = reinterpret_cast<float *>(p.y);
                y[r] = p.accumulate ? y[r] + (float)mine : (float)mine;
            } else if constexpr (MODE == MODE_INT) {
                int32_t *y = reinterpret_cast<int32_t *>(p.y);
                y[r] = p.accumulate ? y[r] + (int32_t)mine : (int32_t)mine;
            } else {
                reinterpret_cast<float *>(p.y)[r] =
                    (float)((double)(int32_t)mine * (p.beta / scale));
            }
        }
    };

    if constexpr (FMT != FMT_U32 && BUCKET) {
        // ===== bucket path =====================================================
        // A round is 32 chunks; lane L owns chunk L.  Each round is stored as
        // [first 16B halves][second 16B halves], so both loads are coalesced
        // 512B accesses.  Rounds are fetched PD ahead into a register ring and
        // the next cell's first rounds are fetched before this cell's epilogue.
        // Chunks past the cell end read as zeros, which decode to column-0
        // gathers flushed into bucket 0 (never reduced): no divergence.
        auto is_key = [](uint32_t x) -> uint32_t { return SC ? (x & 1u) : (x & 0x8000u); };
        auto key_off = [](uint32_t x) -> uint32_t { return SC ? (x & 0xFFFCu) : (x & 0x7FFFu) * 4u; };
        auto lo_off = [](uint32_t x) -> uint32_t { return SC ? (x & 0xFFFCu) : (x & 0x7FFFu) * VSZ; };
        auto hi_off = [](uint32_t x) -> uint32_t { return SC ? (x >> 16) : (x >> 16) * VSZ; };
        while (b < p.nblk) {
            Acc acc[K];
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] = (Acc)0;
            auto do_round = [&](const uint4 &a0, const uint4 &a1) {
                if (p.dbg & 32) {  // stream only (bandwidth experiment)
                    acc[0] += (Acc)(a0.x ^ a0.y ^ a0.z ^ a0.w ^ a1.x ^ a1.y ^ a1.z ^ a1.w);
                    return;
                }
                const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                uint32_t cur = key_off(w[0]);
                Acc s = lds_v<Acc, VSZ>(vbase + hi_off(w[0]));
                uint32_t fk[7];
                float fs[7];
#pragma unroll
                for (int i = 1; i < 8; ++i) {
                    const uint32_t x = w[i];
                    const uint32_t isk = is_key(x);
                    const uint32_t ko = key_off(x);
                    const uint32_t ga = (p.dbg & 8) ? lane * 4u : lo_off(x);
                    const uint32_t ha = (p.dbg & 8) ? lane * 4u + 128u : hi_off(x);
                    const Acc g = lds_v_unless<Acc, VSZ>(isk, vbase + ga);
                    const Acc h = lds_v<Acc, VSZ>(vbase + ha);
                    if constexpr (MODE == MODE_FLOAT) {
                        // record completed segments; flushed below as one batch
                        const bool newseg = isk && ko != cur;
                        fk[i - 1] = newseg ? cur : 0u;
                        fs[i - 1] = s;
                        cur = newseg ? ko : cur;
                        s = (newseg ? (Acc)0 : s) + g + h;
                    } else {
                        if (!(p.dbg & 1)) bucket_flush_pred(isk, bkbase + cur, s);  // native red
                        cur = isk ? ko : cur;
                        s = (isk ? (Acc)0 : s) + g + h;
                    }
                }
                if constexpr (MODE == MODE_FLOAT) {
                    // all bucket loads, then all adds/stores: one latency per
                    // round.  Keys of completed segments are distinct across the
                    // round (a group completes inside a chunk at most once; a
                    // repeated equal key continues the segment), bucket 0 aside.
                    if (!(p.dbg & 1)) {
                        float tb[7];
#pragma unroll
                        for (int i = 0; i < 7; ++i) tb[i] = lds_bucket(bkbase + fk[i]);
#pragma unroll
                        for (int i = 0; i < 7; ++i) sts_bucket(bkbase + fk[i], tb[i] + fs[i]);
                    }
                }
                // A chunk's last segment may continue in the next lane's chunk.
                // Integer: native shared red handles same-key lanes.  Float:
                // lanes with equal final keys form contiguous runs; a segmented
                // suffix sum over the run lets the run's first lane flush alone
                // (no CAS loop, fixed summation order).
                if (!(p.dbg & 2)) {
                    if constexpr (MODE == MODE_FLOAT) {
                        float sj = s;
                        const uint32_t kj = cur;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const float os = __shfl_down_sync(RSR_FULL_MASK, sj, d);
                            const uint32_t ok = __shfl_down_sync(RSR_FULL_MASK, kj, d);
                            if (lane + d < 32 && ok == kj) sj += os;
                        }
                        const uint32_t pk = __shfl_up_sync(RSR_FULL_MASK, kj, 1);
                        const bool head = lane == 0 || pk != kj;
                        if (head) sts_bucket(bkbase + kj, lds_bucket(bkbase + kj) + sj);
                    } else {
                        bucket_flush_final(bkbase + cur, s);
                    }
                } else {
                    acc[0] += s;
                }
                __syncwarp();
            };
            for (int64_t base = ch0; base < ch1; base += 32 * PD) {
#pragma unroll
                for (int u = 0; u < PD; ++u) {
                    const int64_t rb = base + 32 * u;
                    if (rb < ch1) {
                        const uint4 a0 = ring[u][0], a1 = ring[u][1];
                        load_round(rb + 32 * PD, ch1, ring[u][0], ring[u][1]);
                        do_round(a0, a1);
                    }
                }
            }
            // prefetch the next cell before this cell's epilogue
            const int64_t nb = b + bstride;
            const int64_t cb = b;
            if (nb < p.nblk) {
                const int64_t dc = nb * p.tc + t;
                ch0 = p.e_off[dc] / CH;
                ch1 = p.e_off[dc + 1] / CH;
#pragma unroll
                for (int u = 0; u < PD; ++u) load_round(ch0 + 32 * u, ch1, ring[u][0], ring[u][1]);
            }
            asm volatile("" ::: "memory");
            finish_cell(cb, acc);
            b = nb;
        }
    } else {
        // ===== generic path (register flush and/or u32 entries) ================
        for (; b < p.nblk; b += bstride) {
            const int64_t dc = b * p.tc + t;
            const int64_t cch0 = p.e_off[dc] / CH, cch1 = p.e_off[dc + 1] / CH;
            Acc acc[K];
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] = (Acc)0;
            int64_t nr = min((int64_t)32, cch1 - cch0);
            uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
            if ((int64_t)lane < nr) {
                q0 = __ldg(ent4 + 2 * cch0 + lane);
                q1 = __ldg(ent4 + 2 * cch0 + nr + lane);
            }
            for (int64_t base = cch0; base < cch1; base += 32) {
                const bool valid = (int64_t)lane < nr;
                const uint4 a0 = q0, a1 = q1;
                const int64_t nbase = base + 32;
                const int64_t nnr = min((int64_t)32, cch1 - nbase);
                if ((int64_t)lane < nnr) {  // prefetch the next round
                    q0 = __ldg(ent4 + 2 * nbase + lane);
                    q1 = __ldg(ent4 + 2 * nbase + nnr + lane);
                }
                if (valid) {
                    const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    if constexpr (FMT == FMT_U16) {
                        uint32_t cur = w[0] & 0x7FFFu;
                        Acc s = lds_v<Acc, VSZ>(vbase + (w[0] >> 16) * VSZ);
#pragma unroll
                        for (int i = 1; i < 8; ++i) {
                            const uint32_t lo = w[i] & 0xFFFFu;
                            const uint32_t isk = lo & 0x8000u;
                            const Acc g = lds_v_unless<Acc, VSZ>(isk, vbase + (lo & 0x7FFFu) * VSZ);
                            const Acc h = lds_v<Acc, VSZ>(vbase + (w[i] >> 16) * VSZ);
                            if (isk) reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                            cur = isk ? (lo & 0x7FFFu) : cur;
                            s = (isk ? (Acc)0 : s) + g + h;
                        }
                        reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                    } else {  // FMT_U32, register flush, v gathered from global scratch
                        constexpr uint32_t KF = 1u << 31;
                        uint32_t cur = w[0] & ~KF;
                        Acc s = (Acc)__ldg(vglob + w[1]);
#pragma unroll
                        for (int i = 2; i < 8; i += 2) {
                            const Acc h = (Acc)__ldg(vglob + w[i + 1]);
                            if (w[i] & KF) {
                                reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                                cur = w[i] & ~KF;
                                s = (Acc)0;
                            } else {
                                s += (Acc)__ldg(vglob + w[i]);
                            }
                            s += h;
                        }
                        reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                    }
                }
                nr = nnr;
            }
            finish_cell(b, acc);
        }
    }
}

#endif

using KernelFn = void (*)(MvParams);

// Kernel lookup, defined per format in rsr_mv_fmt*.cu (parallel compilation).
KernelFn pick_fmt1(int mode, int k);             // FMT_U16_SCALED, buckets
KernelFn pick_fmt0(int mode, int k, bool bucket);  // FMT_U16
KernelFn pick_fmt2(int mode, int k);             // FMT_U32, register flush

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
