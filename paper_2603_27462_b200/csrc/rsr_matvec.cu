// rsr_matvec.cu -- online RSR multiply for sm_100a.
//
// Replaces the reference's matvec cores (pkg/src/rsrmv/_native.py:167-285)
// and its fused quantize/multiply/dequantize path (_native.py:313-353).
//
// Input: the chunk stream (include/rsr_b200.h): per cell, 32-byte chunks of
// entries; an entry is a column to gather or (top bit set) the pattern key of
// the group whose columns follow; every chunk starts with a key.
//
// Work decomposition:
//   * grid.y = column tile.  Each CTA stages its tile of v in shared memory
//     once (fp32 for the float path, int8 for the integer/fused paths; the
//     fused path quantizes while staging, after a CTA-local absmax over the
//     whole vector -- no separate quantization launch);
//   * one warp owns one (block, tile) cell at a time; lane L of a round owns
//     chunk L: one 32-byte load, then a gather from shared memory per column
//     entry and a running partial group sum;
//   * at every key entry the partial sum is flushed into the warp's PATTERN
//     BUCKET for that key (3^k ternary / 2^k binary buckets in shared memory);
//   * when the cell is done, the pattern-table reduction y_i = sum_key
//     sgn_i(key) * bucket[key] (sign table in shared memory) produces the k
//     rows, warp-reduced and written once.
// For pattern spaces too large for shared-memory buckets the "register"
// variant flushes straight into k row accumulators instead.
// Integer accumulation is exact, so the int8 and fused paths are
// bit-identical to the reference.  The float path accumulates in fp32.

#include "rsr_common.cuh"

namespace rsr {

enum MvMode { MODE_FLOAT = 0, MODE_INT = 1, MODE_FUSED = 2 };

constexpr int MV_MAX_WARPS = 32;
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
    const void *vstaged; // u32-entry variant: v converted/quantized in global memory
    void *y;             // output slice (view rows)
    int accumulate;
    void *part;          // tc > 1: [tc][nblk*k] partials (float or int32)
    double beta;         // fused
    double *scale_dev;   // fused: device scale slot (may be null when tc == 1)
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
__device__ double cta_absmax(const void *v, int dtype, int64_t n) {
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

template <typename Acc>
__device__ __forceinline__ void bucket_add_atomic(Acc *b, Acc s) {
    atomicAdd(b, s);
}

template <int K, int MODE, typename E, bool BUCKET>
__global__ void __launch_bounds__(MV_MAX_WARPS * 32)
rsr_mv_kernel(MvParams p) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    using VS = typename std::conditional<MODE == MODE_FLOAT, float, int8_t>::type;
    constexpr bool SMEM_V = sizeof(E) == 2;
    constexpr int CH = 32 / (int)sizeof(E);           // entries per chunk (32 bytes)
    constexpr E KEYFLAG = (E)1 << (8 * sizeof(E) - 1);
    constexpr int KP = KPad<K>::value;

    extern __shared__ __align__(16) unsigned char mv_smem[];
    const int nwarps = blockDim.x >> 5;
    const int64_t t = blockIdx.y;
    const int64_t c0 = t * p.tw;
    const int64_t tn = min(p.tw, p.n - c0);

    // smem carve-up: [v tile][sign table NB x KP][buckets nwarps x NB]
    size_t off = 0;
    VS *vs = reinterpret_cast<VS *>(mv_smem);
    if (SMEM_V) off += ((size_t)tn * sizeof(VS) + 15) & ~(size_t)15;
    Acc *stab = reinterpret_cast<Acc *>(mv_smem + off);
    if (BUCKET) off += (size_t)p.nkeys * KP * sizeof(Acc);
    Acc *buckets = reinterpret_cast<Acc *>(mv_smem + off);

    // ---- prologue -------------------------------------------------------
    double scale = 1.0;
    if (MODE == MODE_FUSED) {
        if (SMEM_V) {
            const double amax = cta_absmax(p.v, p.vdtype, p.n);
            scale = amax == 0.0 ? 1.0 : 127.0 / amax;
            if (p.scale_dev && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
                *p.scale_dev = scale;
        } else {
            scale = *p.scale_dev;  // written by the staging kernel
        }
    }
    if (SMEM_V) {
        for (int64_t i = threadIdx.x; i < tn; i += blockDim.x) {
            if (MODE == MODE_FLOAT)
                vs[i] = (VS)load_as_f32(p.v, p.vdtype, c0 + i);
            else if (MODE == MODE_INT)
                vs[i] = __ldg((const int8_t *)p.v + c0 + i);
            else
                vs[i] = quantize_one(load_as_f32(p.v, p.vdtype, c0 + i), scale);
        }
    }
    if (BUCKET) {
        for (int key = threadIdx.x; key < p.nkeys; key += blockDim.x) {
#pragma unroll
            for (int i = 0; i < KP; ++i)
                stab[key * KP + i] = (Acc)(i < K ? key_sign((uint32_t)key, i, p.bitwidth) : 0);
        }
        for (int i = threadIdx.x; i < nwarps * p.nkeys; i += blockDim.x) buckets[i] = (Acc)0;
    }
    __syncthreads();

    const VS *vg = SMEM_V ? vs : reinterpret_cast<const VS *>(p.vstaged) + c0;
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    Acc *bk = buckets + (size_t)warp * p.nkeys;
    const uint4 *ent4 = reinterpret_cast<const uint4 *>(p.entries);

    for (int64_t b = (int64_t)blockIdx.x * nwarps + warp; b < p.nblk;
         b += (int64_t)gridDim.x * nwarps) {
        const int64_t dc = b * p.tc + t;
        const int64_t ch0 = p.e_off[dc] / CH, ch1 = p.e_off[dc + 1] / CH;  // chunk range
        Acc acc[K];
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = (Acc)0;

        int64_t ch = ch0 + lane;
        uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
        if (ch < ch1) {
            q0 = __ldg(ent4 + 2 * ch);
            q1 = __ldg(ent4 + 2 * ch + 1);
        }
        for (int64_t base = ch0; base < ch1; base += 32) {
            const bool valid = ch < ch1;
            const uint4 a0 = q0, a1 = q1;
            const int64_t nch = ch + 32;
            if (nch < ch1) {  // prefetch the next round
                q0 = __ldg(ent4 + 2 * nch);
                q1 = __ldg(ent4 + 2 * nch + 1);
            }
            if (valid) {
                const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                uint32_t cur = 0;
                Acc s = (Acc)0;
#pragma unroll
                for (int e = 0; e < CH; ++e) {
                    uint32_t x;
                    if (sizeof(E) == 2)
                        x = (e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xFFFFu);
                    else
                        x = w[e];
                    if (x & (uint32_t)KEYFLAG) {
                        if (e > 0) {
                            if (BUCKET) {
                                if (MODE == MODE_FLOAT) bk[cur] += s;  // distinct keys per instruction
                                else atomicAdd(bk + cur, s);
                            } else {
#pragma unroll
                                for (int i = 0; i < K; ++i)
                                    acc[i] += (Acc)key_sign(cur, i, p.bitwidth) * s;
                            }
                        }
                        cur = x & ~(uint32_t)KEYFLAG;
                        s = (Acc)0;
                    } else {
                        s += (Acc)vg[x];
                    }
                }
                if (BUCKET) {
                    bucket_add_atomic(bk + cur, s);  // tails of one group may coincide
                } else {
#pragma unroll
                    for (int i = 0; i < K; ++i) acc[i] += (Acc)key_sign(cur, i, p.bitwidth) * s;
                }
            }
            __syncwarp();
            ch = nch;
        }

        // ---- pattern-table reduction: y_i = sum_key sgn_i(key) * bucket[key] ----
        if (BUCKET) {
            for (int key = lane; key < p.nkeys; key += 32) {
                const Acc bv = bk[key];
                bk[key] = (Acc)0;
                const Acc *row = stab + key * KP;
#pragma unroll
                for (int i = 0; i < K; ++i) acc[i] += row[i] * bv;
            }
            __syncwarp();
        }
        const int64_t row0 = b * p.k;  // row within the view
        const int64_t grow0 = (p.blk0 + b) * p.k;
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
            } else if (MODE == MODE_FLOAT) {
                float *y = reinterpret_cast<float *>(p.y);
                y[r] = p.accumulate ? y[r] + (float)mine : (float)mine;
            } else if (MODE == MODE_INT) {
                int32_t *y = reinterpret_cast<int32_t *>(p.y);
                y[r] = p.accumulate ? y[r] + (int32_t)mine : (int32_t)mine;
            } else {
                reinterpret_cast<float *>(p.y)[r] =
                    (float)((double)(int32_t)mine * (p.beta / scale));
            }
        }
    }
}

// tc > 1: sum the tile partials in ascending tile order (the reference order).
template <int MODE>
__global__ void tile_finalize_kernel(MvParams p, int64_t rows_view) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    const Acc *part = reinterpret_cast<const Acc *>(p.part);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows_view;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (p.blk0 * p.k + r >= p.m_rows) continue;
        Acc s = (Acc)0;
        for (int64_t t = 0; t < p.tc; ++t) s += part[t * rows_view + r];
        if (MODE == MODE_FLOAT) {
            float *y = reinterpret_cast<float *>(p.y);
            y[r] = p.accumulate ? y[r] + s : s;
        } else if (MODE == MODE_INT) {
            int32_t *y = reinterpret_cast<int32_t *>(p.y);
            y[r] = p.accumulate ? y[r] + s : s;
        } else {
            reinterpret_cast<float *>(p.y)[r] = (float)((double)s * (p.beta / *p.scale_dev));
        }
    }
}

// u32-entry variant (tiles wider than 32768 columns): v converted/quantized
// once into global scratch; the multiply gathers it through L1/L2.
__global__ void stage_global_kernel(const void *v, int dtype, int64_t n, int mode, void *out,
                                    double *scale_dev) {
    double scale = 1.0;
    if (mode == MODE_FUSED) {
        const double amax = cta_absmax(v, dtype, n);
        scale = amax == 0.0 ? 1.0 : 127.0 / amax;
        if (blockIdx.x == 0 && threadIdx.x == 0) *scale_dev = scale;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (mode == MODE_FLOAT) ((float *)out)[i] = load_as_f32(v, dtype, i);
        else if (mode == MODE_INT) ((int8_t *)out)[i] = ((const int8_t *)v)[i];
        else ((int8_t *)out)[i] = quantize_one(load_as_f32(v, dtype, i), scale);
    }
}

__global__ void absmax_quantize_kernel(const void *v, int dtype, int64_t n, int8_t *q,
                                       double *scale_out) {
    const double amax = cta_absmax(v, dtype, n);
    const double scale = amax == 0.0 ? 1.0 : 127.0 / amax;
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        q[i] = quantize_one(load_as_f32(v, dtype, i), scale);
}

// ---------------------------------------------------------------------------
// host-side dispatch

using KernelFn = void (*)(MvParams);

template <int MODE, typename E, bool BUCKET>
static KernelFn pick_k(int k) {
    switch (k) {
#define RSR_K_CASE(KK) \
    case KK: return rsr_mv_kernel<KK, MODE, E, BUCKET>;
        RSR_K_CASE(1) RSR_K_CASE(2) RSR_K_CASE(3) RSR_K_CASE(4) RSR_K_CASE(5) RSR_K_CASE(6)
        RSR_K_CASE(7) RSR_K_CASE(8) RSR_K_CASE(9) RSR_K_CASE(10) RSR_K_CASE(11) RSR_K_CASE(12)
        RSR_K_CASE(13) RSR_K_CASE(14) RSR_K_CASE(15) RSR_K_CASE(16)
#undef RSR_K_CASE
        default: return nullptr;
    }
}

template <int MODE>
static KernelFn pick_kernel(int k, int entry_bytes, bool bucket) {
    if (entry_bytes == 4) return pick_k<MODE, uint32_t, false>(k);
    return bucket ? pick_k<MODE, uint16_t, true>(k) : pick_k<MODE, uint16_t, false>(k);
}

static rsr_status check_view(const rsr_stream_view *vw) {
    if (!vw || !vw->entries || !vw->e_off) return RSR_ERR_INVALID;
    if (vw->k < 1 || vw->k > 16 || vw->m < 1 || vw->n < 1 || vw->tile_count < 1 ||
        vw->n_blocks < 0 || vw->tile_width < 1)
        return RSR_ERR_INVALID;
    if (vw->bitwidth != RSR_BINARY && vw->bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    if (vw->entry_bytes != 2 && vw->entry_bytes != 4) return RSR_ERR_INVALID;
    if (vw->chunk != 32 / vw->entry_bytes) return RSR_ERR_INVALID;
    if (vw->entry_bytes == 2 &&
        (vw->tile_width > 32768 || bucket_count(vw->bitwidth, vw->k) > 32768))
        return RSR_ERR_INVALID;
    return RSR_OK;
}

// workspace: [tile partials][16B: fused scale][staged v (u32 entries)]
static size_t part_bytes(const rsr_stream_view *vw) {
    return vw->tile_count <= 1 ? 0
                               : (((size_t)vw->tile_count * vw->n_blocks * vw->k * 4 + 15) & ~15);
}
static size_t ws_bytes_for(const rsr_stream_view *vw) {
    size_t b = part_bytes(vw) + 16;
    if (vw->entry_bytes == 4) b += (size_t)vw->n * 4;
    return b;
}

template <int MODE>
static rsr_status launch_mv(const rsr_stream_view *vw, const void *v, int vdtype, void *y,
                            int accumulate, double beta, double *scale_out, void *ws,
                            size_t ws_bytes, cudaStream_t s) {
    rsr_status st = check_view(vw);
    if (st != RSR_OK) return st;
    if (!v || !y) return RSR_ERR_INVALID;
    if (vw->n_blocks == 0) return RSR_OK;
    const bool need_ws = vw->tile_count > 1 || vw->entry_bytes == 4 ||
                         (MODE == MODE_FUSED && !scale_out && vw->tile_count > 1);
    if (need_ws && (ws_bytes < ws_bytes_for(vw) || !ws)) return RSR_ERR_WORKSPACE;
    MvParams p;
    p.entries = vw->entries;
    p.e_off = vw->e_off;
    p.m_rows = vw->m;
    p.n = vw->n;
    p.tw = vw->tile_width;
    p.tc = vw->tile_count;
    p.blk0 = vw->row_begin_block;
    p.nblk = vw->n_blocks;
    p.k = vw->k;
    p.bitwidth = vw->bitwidth;
    p.nkeys = (int)bucket_count(vw->bitwidth, vw->k);
    p.v = v;
    p.vdtype = vdtype;
    p.y = y;
    p.accumulate = accumulate;
    p.part = ws;
    p.beta = beta;
    p.scale_dev = scale_out;
    if (MODE == MODE_FUSED && !p.scale_dev && need_ws)
        p.scale_dev = (double *)((char *)ws + part_bytes(vw));
    p.vstaged = nullptr;
    if (vw->entry_bytes == 4) {
        void *stg = (char *)ws + part_bytes(vw) + 16;
        p.vstaged = stg;
        stage_global_kernel<<<MODE == MODE_FUSED ? 1 : 256, 1024, 0, s>>>(v, vdtype, vw->n, MODE,
                                                                          stg, p.scale_dev);
        if (MODE == MODE_FUSED) {
            // one CTA computed the scale; re-stage in parallel is unnecessary (n small)
        }
    }
    const bool bucket = vw->entry_bytes == 2 && p.nkeys <= BUCKET_MAX_KEYS;
    KernelFn fn = pick_kernel<MODE>(vw->k, vw->entry_bytes, bucket);
    if (!fn) return RSR_ERR_INVALID;

    // size: one persistent CTA per SM, as many warps as fit (<= 32) and needed
    const int sms = sm_count();
    const size_t vsz = MODE == MODE_FLOAT ? 4 : 1;
    const int64_t tn = std::min(vw->tile_width, vw->n);
    const size_t kp = (size_t)((vw->k + 3) & ~3);
    size_t fixed = 0;
    if (vw->entry_bytes == 2) fixed += ((size_t)tn * vsz + 15) & ~(size_t)15;
    if (bucket) fixed += (size_t)p.nkeys * kp * 4;
    const size_t per_warp = bucket ? (size_t)p.nkeys * 4 : 0;
    const size_t smem_cap = 227 * 1024;
    int64_t cells_per_tile = vw->n_blocks;
    int64_t ctas_per_tile = std::max<int64_t>(1, sms / vw->tile_count);
    int64_t warps = (cells_per_tile + ctas_per_tile - 1) / ctas_per_tile;
    warps = std::max<int64_t>(1, std::min<int64_t>(warps, MV_MAX_WARPS));
    while (warps > 1 && fixed + warps * per_warp > smem_cap) --warps;
    if (fixed + warps * per_warp > smem_cap) return RSR_ERR_INVALID;
    const size_t smem = fixed + warps * per_warp;
    ctas_per_tile = std::min<int64_t>(ctas_per_tile, (cells_per_tile + warps - 1) / warps);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)ctas_per_tile, (unsigned)vw->tile_count);
    fn<<<grid, (unsigned)(warps * 32), smem, s>>>(p);
    if (vw->tile_count > 1) {
        const int64_t rows_view = vw->n_blocks * vw->k;
        const int g2 = (int)std::min<int64_t>((rows_view + 255) / 256, 4096);
        tile_finalize_kernel<MODE><<<g2, 256, 0, s>>>(p, rows_view);
    }
    return launch_status();
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_matvec_workspace_bytes(const rsr_stream_view *view) {
    if (!view) return 0;
    if (view->tile_count <= 1 && view->entry_bytes != 4) return 0;
    return ws_bytes_for(view);
}

rsr_status rsr_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype, void *y,
                      int32_t accumulate, void *workspace, size_t workspace_bytes,
                      rsr_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (v_dtype == RSR_I8)
        return launch_mv<MODE_INT>(view, v, v_dtype, y, accumulate, 1.0, nullptr, workspace,
                                   workspace_bytes, s);
    if (v_dtype == RSR_F32 || v_dtype == RSR_BF16 || v_dtype == RSR_F16)
        return launch_mv<MODE_FLOAT>(view, v, v_dtype, y, accumulate, 1.0, nullptr, workspace,
                                     workspace_bytes, s);
    return RSR_ERR_INVALID;
}

rsr_status rsr_fused_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                            double beta, float *out, double *scale_out, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream) {
    if (v_dtype != RSR_F32 && v_dtype != RSR_BF16 && v_dtype != RSR_F16) return RSR_ERR_INVALID;
    if (view && view->bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    return launch_mv<MODE_FUSED>(view, v, v_dtype, out, 0, beta, scale_out, workspace,
                                 workspace_bytes, (cudaStream_t)stream);
}

rsr_status rsr_absmax_quantize(const void *v, int32_t v_dtype, int64_t n, int8_t *q,
                               double *scale_out, rsr_stream_t stream) {
    if (!v || !q || n < 0) return RSR_ERR_INVALID;
    if (v_dtype != RSR_F32 && v_dtype != RSR_BF16 && v_dtype != RSR_F16) return RSR_ERR_INVALID;
    if (n == 0) return RSR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (int)std::min<int64_t>((n + 1023) / 1024, 64);
    absmax_quantize_kernel<<<grid, 1024, 0, s>>>(v, v_dtype, n, q, scale_out);
    return launch_status();
}

}  // extern "C"
