// rsr_matvec.cu -- online RSR multiply for sm_100a.
//
// Replaces the reference's matvec cores (pkg/src/rsrmv/_native.py:167-285)
// and the fused quantize/multiply/dequantize path (_native.py:313-353).
//
// Work decomposition:
//   * grid.y = column tile; each CTA stages its tile of v in shared memory
//     once (fp32 for the float path, int8 for the integer/fused paths; the
//     fused path quantizes while staging after a CTA-local absmax over the
//     whole vector, so no separate quantization pass exists);
//   * one warp owns one (block, tile) cell at a time and streams the cell's
//     entries (u16 column | head<<15) with 2 x 16-byte loads per lane per
//     round (1 KiB per warp-round), prefetching the next round;
//   * each lane owns 16 consecutive entries: it gathers v from shared memory,
//     keeps a running partial group sum, and at every group head flushes the
//     partial sum into its k row accumulators with the group's signs
//     (linearity: y_i = sum_g sgn_i(g) * S_g = sum over partial segments);
//     the group index of a lane's first entry comes from a warp scan of the
//     head counts;
//   * at the end of the cell the k accumulators are warp-reduced and written.
// Integer accumulation is exact, so the int8 and fused paths are
// bit-identical to the reference.  The float path accumulates in fp32.

#include "rsr_common.cuh"

namespace rsr {

constexpr int MV_WARPS = 8;
constexpr int MV_EPL = 16;  // u16 entries per lane per round (32 bytes)

enum MvMode { MODE_FLOAT = 0, MODE_INT = 1, MODE_FUSED = 2 };

struct MvParams {
    const uint16_t *entries;
    const uint32_t *gsigns;
    const int64_t *e_off;
    const int64_t *g_off;
    int64_t m_rows;      // rows of the full matrix
    int64_t n;           // columns
    int64_t tw, tc;      // tile width / count
    int64_t blk0;        // first global block of this view
    int64_t nblk;        // blocks in this view
    int k;
    const void *v;
    int vdtype;
    void *y;             // output slice (view rows)
    int accumulate;
    void *part;          // tc > 1: [tc][nblk*k] partials (float or int32)
    double beta;         // fused
    double *scale_out;   // fused (may be null)
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

// CTA-wide max of |v| over the whole vector, in float64 (exact: max is
// order-independent).  Result broadcast to every thread.
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

template <typename Acc>
__device__ __forceinline__ Acc sign_of(uint32_t m, int i) {
    return (Acc)((int)((m >> i) & 1u) - (int)((m >> (16 + i)) & 1u));
}

// Flush a partial group sum into the k row accumulators (FMA with the
// group's sign, so a non-finite partial poisons every row of the block
// exactly as the reference's `y += sgn * s` does).
template <int K, typename Acc>
__device__ __forceinline__ void flush(Acc (&acc)[K], Acc s, uint32_t m) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] += sign_of<Acc>(m, i) * s;
}

template <int K, int MODE>
__global__ void __launch_bounds__(MV_WARPS * 32)
rsr_mv_kernel(MvParams p) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    using VS = typename std::conditional<MODE == MODE_FLOAT, float, int8_t>::type;
    extern __shared__ __align__(16) unsigned char mv_smem[];
    VS *vs = reinterpret_cast<VS *>(mv_smem);

    const int64_t t = blockIdx.y;
    const int64_t c0 = t * p.tw;
    const int64_t tn = min(p.tw, p.n - c0);

    // ---- prologue: stage this tile of v (quantizing on the fused path) ----
    double scale = 1.0;
    if (MODE == MODE_FUSED) {
        const double amax = cta_absmax(p.v, p.vdtype, p.n);
        scale = amax == 0.0 ? 1.0 : 127.0 / amax;
        if (p.scale_out && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
            *p.scale_out = scale;
    }
    for (int64_t i = threadIdx.x; i < tn; i += blockDim.x) {
        if (MODE == MODE_FLOAT) {
            vs[i] = (VS)load_as_f32(p.v, p.vdtype, c0 + i);
        } else if (MODE == MODE_INT) {
            vs[i] = __ldg((const int8_t *)p.v + c0 + i);
        } else {
            vs[i] = quantize_one(load_as_f32(p.v, p.vdtype, c0 + i), scale);
        }
    }
    __syncthreads();

    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const uint4 *ent4 = reinterpret_cast<const uint4 *>(p.entries);

    for (int64_t b = (int64_t)blockIdx.x * MV_WARPS + warp; b < p.nblk;
         b += (int64_t)gridDim.x * MV_WARPS) {
        const int64_t dc = b * p.tc + t;
        const int64_t e0 = p.e_off[dc], e1 = p.e_off[dc + 1];
        int64_t g = p.g_off[dc] - 1;  // index of the group before the cell's first entry
        Acc acc[K];
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = (Acc)0;

        // 16 entries (two uint4) per lane per round; prefetch one round ahead.
        int64_t idx = e0 + (int64_t)lane * MV_EPL;
        uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
        if (idx < e1) {
            q0 = __ldg(ent4 + (idx >> 3));
            q1 = __ldg(ent4 + (idx >> 3) + 1);
        }
        for (int64_t base = e0; base < e1; base += 32 * MV_EPL) {
            const bool valid = idx < e1;
            const uint4 c0q = q0, c1q = q1;
            const int64_t nidx = idx + 32 * MV_EPL;
            if (nidx < e1) {
                q0 = __ldg(ent4 + (nidx >> 3));
                q1 = __ldg(ent4 + (nidx >> 3) + 1);
            }
            const uint32_t w[8] = {c0q.x, c0q.y, c0q.z, c0q.w, c1q.x, c1q.y, c1q.z, c1q.w};
            // head bits of the 16 entries, packed: bit e = head of entry e
            uint32_t hm = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                hm |= ((w[j] >> 15) & 1u) << (2 * j) | ((w[j] >> 31) & 1u) << (2 * j + 1);
            const uint32_t cnt = valid ? __popc(hm) : 0u;
            const uint32_t incl = warp_inclusive_scan(cnt, lane);
            const uint32_t total = __shfl_sync(RSR_FULL_MASK, incl, 31);
            if (valid) {
                int64_t gg = g + (int64_t)(incl - cnt);
                uint32_t msk = gg >= 0 ? __ldg(p.gsigns + gg) : 0u;
                Acc s = (Acc)0;
#pragma unroll
                for (int e = 0; e < MV_EPL; ++e) {
                    const uint32_t x = (e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xFFFFu);
                    if ((hm >> e) & 1u) {
                        if (e > 0) flush<K, Acc>(acc, s, msk);
                        s = (Acc)0;
                        ++gg;
                        msk = __ldg(p.gsigns + gg);
                    }
                    s += (Acc)vs[x & 0x7FFFu];
                }
                flush<K, Acc>(acc, s, msk);
            }
            g += total;
            idx = nidx;
        }

        // ---- epilogue: warp-reduce the k rows, write ----
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

// tc > 1: sum tile partials in ascending tile order (the reference's order).
template <int MODE>
__global__ void tile_finalize_kernel(MvParams p, int64_t rows_view, const double *scale_dev) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    const Acc *part = reinterpret_cast<const Acc *>(p.part);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows_view;
         r += (int64_t)gridDim.x * blockDim.x) {
        if ((p.blk0 * p.k) + r >= p.m_rows) continue;
        Acc s = (Acc)0;
        for (int64_t t = 0; t < p.tc; ++t) s += part[t * rows_view + r];
        if (MODE == MODE_FLOAT) {
            float *y = reinterpret_cast<float *>(p.y);
            y[r] = p.accumulate ? y[r] + s : s;
        } else if (MODE == MODE_INT) {
            int32_t *y = reinterpret_cast<int32_t *>(p.y);
            y[r] = p.accumulate ? y[r] + s : s;
        } else {
            reinterpret_cast<float *>(p.y)[r] = (float)((double)s * (p.beta / *scale_dev));
        }
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

template <int MODE>
static KernelFn pick_kernel(int k) {
    switch (k) {
#define RSR_K_CASE(KK) \
    case KK: return rsr_mv_kernel<KK, MODE>;
        RSR_K_CASE(1) RSR_K_CASE(2) RSR_K_CASE(3) RSR_K_CASE(4) RSR_K_CASE(5) RSR_K_CASE(6)
        RSR_K_CASE(7) RSR_K_CASE(8) RSR_K_CASE(9) RSR_K_CASE(10) RSR_K_CASE(11) RSR_K_CASE(12)
        RSR_K_CASE(13) RSR_K_CASE(14) RSR_K_CASE(15) RSR_K_CASE(16)
#undef RSR_K_CASE
        default: return nullptr;
    }
}

static rsr_status check_view(const rsr_stream_view *vw) {
    if (!vw || !vw->entries || !vw->gsigns || !vw->e_off || !vw->g_off) return RSR_ERR_INVALID;
    if (vw->k < 1 || vw->k > 16 || vw->m < 1 || vw->n < 1 || vw->tile_count < 1 ||
        vw->n_blocks < 0)
        return RSR_ERR_INVALID;
    if (vw->entry_bytes != 2) return RSR_ERR_INVALID;  // u32 entries: see DESIGN.md
    if (vw->tile_width > 32768) return RSR_ERR_INVALID;
    return RSR_OK;
}

static size_t part_bytes(const rsr_stream_view *vw) {
    if (vw->tile_count <= 1) return 0;
    return (size_t)vw->tile_count * (size_t)vw->n_blocks * (size_t)vw->k * 4 + 16;
}

template <int MODE>
static rsr_status launch_mv(const rsr_stream_view *vw, const void *v, int vdtype, void *y,
                            int accumulate, double beta, double *scale_out, void *ws,
                            size_t ws_bytes, cudaStream_t s) {
    rsr_status st = check_view(vw);
    if (st != RSR_OK) return st;
    if (!v || !y) return RSR_ERR_INVALID;
    if (vw->n_blocks == 0) return RSR_OK;
    const size_t need = part_bytes(vw);
    if (need && (ws_bytes < need || !ws)) return RSR_ERR_WORKSPACE;
    MvParams p;
    p.entries = (const uint16_t *)vw->entries;
    p.gsigns = vw->gsigns;
    p.e_off = vw->e_off;
    p.g_off = vw->g_off;
    p.m_rows = vw->m;
    p.n = vw->n;
    p.tw = vw->tile_width;
    p.tc = vw->tile_count;
    p.blk0 = vw->row_begin_block;
    p.nblk = vw->n_blocks;
    p.k = vw->k;
    p.v = v;
    p.vdtype = vdtype;
    p.y = y;
    p.accumulate = accumulate;
    p.part = ws;
    p.beta = beta;
    double *scale_dev = nullptr;
    if (MODE == MODE_FUSED) {
        // with tiles, the finalize pass needs the scale: keep it in the workspace tail
        scale_dev = scale_out;
        if (!scale_dev && need) scale_dev = (double *)((char *)ws + need - 16);
    }
    p.scale_out = scale_dev;
    KernelFn fn = pick_kernel<MODE>(vw->k);
    if (!fn) return RSR_ERR_INVALID;
    const size_t vsz = MODE == MODE_FLOAT ? 4 : 1;
    const size_t smem = (size_t)std::min(vw->tile_width, vw->n) * vsz;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, MV_WARPS * 32, smem);
    if (occ < 1) occ = 1;
    const int64_t want = (vw->n_blocks + MV_WARPS - 1) / MV_WARPS;
    const int64_t cap = std::max<int64_t>(1, ((int64_t)sm_count() * occ) / vw->tile_count);
    dim3 grid((unsigned)std::min(want, cap), (unsigned)vw->tile_count);
    fn<<<grid, MV_WARPS * 32, smem, s>>>(p);
    if (vw->tile_count > 1) {
        const int64_t rows_view = vw->n_blocks * vw->k;
        const int g2 = (int)std::min<int64_t>((rows_view + 255) / 256, 4096);
        tile_finalize_kernel<MODE><<<g2, 256, 0, s>>>(p, rows_view, scale_dev);
    }
    return launch_status();
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_matvec_workspace_bytes(const rsr_stream_view *view) {
    return view ? part_bytes(view) : 0;
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
