// rsr_mm.cu -- batched multi-vector RSR multiply Y[b] = M . V[b] (SURVEY.md
// section 8a K9, config C4).  Not in the reference (its kernels.py:196 takes a
// 1-D vector); the oracle is the single-vector path column by column.
//
// Same chunk stream as the single-vector kernel (quad layout, lane runs; see
// rsr_mv_kernel.cuh).  Each CTA stages a chunk of BV vectors as a [tn][BV]
// shared-memory tile, so one column gather is one 16-byte load feeding BV
// running group sums, and a pattern bucket is a BV-wide row.  grid.z walks
// the vector chunks: every chunk re-reads the stream, but the chunks run
// concurrently and the stream (29 MB at C4) stays resident in L2, so HBM sees
// it about once.  The pattern-table step runs once per cell per chunk.
#include <cstdio>

#include "rsr_mv_impl.cuh"

namespace rsr {

constexpr int MM_MAX_WARPS = 16;
constexpr int MM_BV = 4;  // vectors per pass

struct MmParams {
    const void *entries;
    const int64_t *e_off;
    const uint32_t *col0_key;
    int64_t m_rows, n, tw, tc, blk0, nblk;
    int k, bitwidth, nkeys;
    const void *V;   // V[b * ldv + col]
    int vdtype;
    int64_t ldv;
    int B;
    void *Y;         // Y[b * ldy + row] (rows of the view)
    int64_t ldy;
    void *part;      // tc > 1: [tc][B][rows_view] partials
};

template <int K, int MODE, int FMT>
__global__ void __launch_bounds__(MM_MAX_WARPS * 32) rsr_mm_kernel(MmParams p) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    using Vec = typename std::conditional<MODE == MODE_FLOAT, float4, int4>::type;
    constexpr int BV = MM_BV;
    constexpr bool FH = FMT == FMT_H;  // halfword format: every column in the stream
    constexpr bool SC = FMT == FMT_U16_SCALED;
    extern __shared__ __align__(16) unsigned char mm_sbuf[];
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int64_t t = blockIdx.y;
    const int64_t c0 = t * p.tw;
    const int64_t tn = min(p.tw, p.n - c0);
    const int b0 = blockIdx.z * BV;
    const int nb = min(BV, p.B - b0);

    // smem: [v tile tn x BV][sign table K x NB][buckets W x NB x BV]
    Acc *vt = reinterpret_cast<Acc *>(mm_sbuf);
    size_t off = (size_t)(FH ? h_zero_b(tn) / 2 + 64 : tn) * BV * sizeof(Acc);
    Acc *stab = reinterpret_cast<Acc *>(mm_sbuf + off);
    off += ((size_t)p.nkeys * K * sizeof(Acc) + 15) & ~(size_t)15;
    Acc *bk = reinterpret_cast<Acc *>(mm_sbuf + off) + (size_t)warp * p.nkeys * BV;
    const uint32_t vbase = (uint32_t)__cvta_generic_to_shared(vt);
    const uint32_t bkbase = (uint32_t)__cvta_generic_to_shared(bk);

    // ---- prologue: stage the vector chunk, sign table, zero buckets ---------
    // vector j of the chunk -> column j of the [tn][BV] tile (16-deep batched
    // loads per thread; unused columns of a short last chunk are zero)
#pragma unroll
    for (int j = 0; j < BV; ++j) {
        if (j < nb) {
            const int64_t base = (int64_t)(b0 + j) * p.ldv;
            const char *vj = reinterpret_cast<const char *>(p.V) +
                             base * (p.vdtype == RSR_F32 ? 4 : (p.vdtype == RSR_I8 ? 1 : 2));
            for_each_v(vj, MODE == MODE_FLOAT ? p.vdtype : (int)RSR_I8, c0, tn,
                       [&](int64_t i, float x) { vt[i * BV + j] = (Acc)x; });
        } else {
            for (int64_t i = threadIdx.x; i < tn; i += blockDim.x) vt[i * BV + j] = (Acc)0;
        }
    }
    if constexpr (FH) {
        // padding names the zero columns [Z, Z + 64) after the tile
        const int64_t z = h_zero_b(tn) / 2;
        for (int64_t i = threadIdx.x; i < 64 * BV; i += blockDim.x) vt[z * BV + i] = (Acc)0;
    } else if (threadIdx.x == 0) {  // column 0 is the zero padding entry (see col0_key);
#pragma unroll                      // thread 0 staged element 0 of every column
        for (int j = 0; j < BV; ++j) vt[j] = (Acc)0;
    }
    for (int key = threadIdx.x; key < p.nkeys; key += blockDim.x) {
        uint32_t kk = (uint32_t)key;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            int sg;
            if (p.bitwidth == RSR_BINARY) {
                sg = (int)((kk >> i) & 1u);
            } else {
                const uint32_t q3 = kk / 3u, d = kk - 3u * q3;
                kk = q3;
                sg = d == 1u ? 1 : (d == 2u ? -1 : 0);
            }
            stab[i * p.nkeys + key] = (Acc)sg;
        }
    }
    {
        Acc *ball = reinterpret_cast<Acc *>(mm_sbuf + off);
        for (int64_t i = threadIdx.x; i < (int64_t)nwarps * p.nkeys * BV; i += blockDim.x)
            ball[i] = (Acc)0;
    }
    Acc v0[BV];  // the tile's column-0 values (added via col0_key)
#pragma unroll
    for (int j = 0; j < BV; ++j) {
        v0[j] = (Acc)0;
        if (j < nb) {
            const int64_t src = (int64_t)(b0 + j) * p.ldv + c0;
            if constexpr (MODE == MODE_FLOAT) v0[j] = load_as_f32(p.V, p.vdtype, src);
            else v0[j] = (Acc)reinterpret_cast<const int8_t *>(p.V)[src];
        }
    }
    __syncthreads();

    // byte offsets of a column / key entry into the v tile / bucket rows
    // (format 3: a column entry is 2*column, a key entry key*4|1)
    auto col_off = [](uint32_t e) -> uint32_t {
        return FH ? (e & 0xFFFEu) * (2u * BV) : (SC ? (e & 0xFFFCu) * BV : (e & 0x7FFFu) * (4u * BV));
    };
    auto key_off = [](uint32_t e) -> uint32_t {
        return FH ? (e & 0xFFFCu) * BV : (SC ? (e & 0xFFFCu) * BV : (e & 0x7FFFu) * (4u * BV));
    };
    auto hi_off = [](uint32_t x) -> uint32_t {
        return FH ? (x >> 16) * (2u * BV) : (SC ? (x >> 16) * BV : (x >> 16) * (4u * BV));
    };
    auto is_key = [](uint32_t x) -> bool { return (SC || FH) ? (x & 1u) != 0u : (x & 0x8000u) != 0u; };
    auto gat = [&](uint32_t o) -> Vec {
        Vec r;
        if constexpr (MODE == MODE_FLOAT) {
            asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(vbase + o));
        } else {
            asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(vbase + o));
        }
        return r;
    };
    auto add4 = [](Vec &a, const Vec &b) {
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
    };
    // bucket[key] += s when `on`; otherwise a harmless update of the sink
    // bucket 0 (never reduced).  One round's closing keys are distinct.
    auto flush = [&](bool on, uint32_t key_o, const Vec &s) {
        const uint32_t a = bkbase + (on ? key_o : 0u);
        Vec b;
        if constexpr (MODE == MODE_FLOAT) {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "r"(a));
            b.x += s.x; b.y += s.y; b.z += s.z; b.w += s.w;
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};"
                         ::"r"(a), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w));
        } else {
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "r"(a));
            b.x += s.x; b.y += s.y; b.z += s.z; b.w += s.w;
            asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};"
                         ::"r"(a), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w));
        }
    };
    const uint4 *__restrict__ ent4 = reinterpret_cast<const uint4 *>(p.entries);

    for (int64_t b = (int64_t)blockIdx.x * nwarps + warp; b < p.nblk;
         b += (int64_t)gridDim.x * nwarps) {
        const int64_t dc = b * p.tc + t;
        const uint32_t ch0 = (uint32_t)(p.e_off[dc] >> 4);
        const uint32_t N = ((uint32_t)(p.e_off[dc + 1] >> 4) - ch0) >> 1;
        const uint32_t P = (N + 31u) >> 5;
        const uint32_t Lf = P ? N / P : 0u, rem = N - Lf * P;
        uint32_t cur = 0;
        Vec s = Vec{0, 0, 0, 0};
        auto load = [&](uint32_t r, uint4 (&q)[4]) {
            // lanes past the round: the sink key, then padding
            const uint32_t zb = FH ? h_zero_b(tn) : 0u;
            const uint32_t PW = zb | (zb << 16);
            q[0] = make_uint4(FH ? (1u | (zb << 16)) : 0u, PW, PW, PW);
#pragma unroll
            for (int j = 1; j < 4; ++j) q[j] = make_uint4(PW, PW, PW, PW);
            if (r >= P) return;
            const uint32_t np = Lf + (r < rem ? 1u : 0u);
            const uint32_t R = r * Lf + min(r, rem);
            if (lane < np) {
                const uint4 *src = ent4 + 2 * ((size_t)ch0 + 2 * (size_t)R) + lane;
#pragma unroll
                for (int j = 0; j < 4; ++j) q[j] = ld_stream(src + j * np);
            }
        };
        uint4 nq[4];
        load(0, nq);
        for (uint32_t r = 0; r < P; ++r) {
            const uint4 a0 = nq[0], a1 = nq[1], a2 = nq[2], a3 = nq[3];
            load(r + 1, nq);
            const uint32_t w[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                                    a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
            {   // slot 0: a key; a new one closes the open group
                const uint32_t k0 = key_off(w[0]);
                const bool ns = k0 != cur;
                flush(ns, cur, s);
                cur = k0;
                if (ns) s = Vec{0, 0, 0, 0};
                Vec g = gat(hi_off(w[0]));
                add4(g, gat(col_off(w[1])));
                add4(g, gat(hi_off(w[1])));
                add4(s, g);
            }
#pragma unroll
            for (int qd = 1; qd < 8; ++qd) {
                const uint32_t x = w[2 * qd], y = w[2 * qd + 1];
                const bool isk = is_key(x);
                const uint32_t xo = col_off(x);
                flush(isk, cur, s);
                cur = isk ? key_off(x) : cur;
                Vec g = gat(hi_off(x));
                add4(g, gat(col_off(y)));
                add4(g, gat(hi_off(y)));
                if (isk) {
                    s = g;
                } else {
                    add4(s, gat(xo));  // slot 4q is a column here
                    add4(s, g);
                }
            }
        }
        // close every lane's open group (equal open keys are contiguous lanes)
        if constexpr (MODE == MODE_FLOAT) {
            Vec sj = s;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t ok = __shfl_down_sync(RSR_FULL_MASK, cur, d);
                const float ox = __shfl_down_sync(RSR_FULL_MASK, sj.x, d);
                const float oy = __shfl_down_sync(RSR_FULL_MASK, sj.y, d);
                const float oz = __shfl_down_sync(RSR_FULL_MASK, sj.z, d);
                const float ow = __shfl_down_sync(RSR_FULL_MASK, sj.w, d);
                if (lane + d < 32 && ok == cur) {
                    sj.x += ox; sj.y += oy; sj.z += oz; sj.w += ow;
                }
            }
            const uint32_t pk = __shfl_up_sync(RSR_FULL_MASK, cur, 1);
            if (lane == 0 || pk != cur) flush(true, cur, sj);
        } else {
            const uint32_t a = bkbase + cur;
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(s.x));
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a + 4), "r"(s.y));
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a + 8), "r"(s.z));
            asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a + 12), "r"(s.w));
        }
        __syncwarp();
        // epilogue: column 0, then y[i][j] = sum_key sgn_i(key) * bucket[key][j]
        const uint32_t key0 = FH ? 0u : p.col0_key[dc];
        if (lane == 0 && key0) {
            Acc *row = bk + (size_t)key0 * BV;
#pragma unroll
            for (int j = 0; j < BV; ++j) row[j] += v0[j];
        }
        __syncwarp();
        Acc acc[K][BV];
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < BV; ++j) acc[i][j] = (Acc)0;
        for (int key = (int)lane; key < p.nkeys; key += 32) {
            Vec bv = reinterpret_cast<Vec *>(bk)[key];
            reinterpret_cast<Vec *>(bk)[key] = Vec{0, 0, 0, 0};
            if (key == 0) bv = Vec{0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const Acc sg = stab[i * p.nkeys + key];
                acc[i][0] += sg * bv.x;
                acc[i][1] += sg * bv.y;
                acc[i][2] += sg * bv.z;
                acc[i][3] += sg * bv.w;
            }
        }
        __syncwarp();
        const int64_t row0 = b * p.k, grow0 = (p.blk0 + b) * p.k;
#pragma unroll
        for (int i = 0; i < K; ++i) {
#pragma unroll
            for (int j = 0; j < BV; ++j) {
                const Acc r = warp_sum(acc[i][j]);
                if (lane == 0 && j < nb && grow0 + i < p.m_rows) {
                    if (p.tc > 1) {
                        const int64_t rows_view = p.nblk * p.k;
                        reinterpret_cast<Acc *>(p.part)[(t * p.B + b0 + j) * rows_view + row0 + i] = r;
                    } else {
                        reinterpret_cast<Acc *>(p.Y)[(int64_t)(b0 + j) * p.ldy + row0 + i] = r;
                    }
                }
            }
        }
    }
}

template <int MODE>
__global__ void mm_finalize_kernel(MmParams p, int64_t rows_view) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    const Acc *part = reinterpret_cast<const Acc *>(p.part);
    const int64_t total = rows_view * p.B;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bi = e / rows_view, r = e - bi * rows_view;
        if (p.blk0 * p.k + r >= p.m_rows) continue;
        Acc s = (Acc)0;
        for (int64_t t = 0; t < p.tc; ++t) s += part[(t * p.B + bi) * rows_view + r];
        reinterpret_cast<Acc *>(p.Y)[bi * p.ldy + r] = s;
    }
}

using MmFn = void (*)(MmParams);
#define RSR_MM_K(M, F) [&](int k) -> MmFn { RSR_K_SWITCH(RSR_MMK_##M##_##F) }
#define RSR_MMK_0_0(KK) (rsr_mm_kernel<KK, MODE_FLOAT, FMT_U16>)
#define RSR_MMK_0_1(KK) (rsr_mm_kernel<KK, MODE_FLOAT, FMT_U16_SCALED>)
#define RSR_MMK_1_0(KK) (rsr_mm_kernel<KK, MODE_INT, FMT_U16>)
#define RSR_MMK_1_1(KK) (rsr_mm_kernel<KK, MODE_INT, FMT_U16_SCALED>)
#define RSR_MMK_0_3(KK) (rsr_mm_kernel<KK, MODE_FLOAT, FMT_H>)
#define RSR_MMK_1_3(KK) (rsr_mm_kernel<KK, MODE_INT, FMT_H>)
static MmFn pick_mm(int mode, int fmt, int k) {
    if (k > 11) return nullptr;
    if (mode == MODE_FLOAT)
        return fmt == FMT_U16 ? RSR_MM_K(0, 0)(k)
               : (fmt == FMT_H ? RSR_MM_K(0, 3)(k) : RSR_MM_K(0, 1)(k));
    return fmt == FMT_U16 ? RSR_MM_K(1, 0)(k)
           : (fmt == FMT_H ? RSR_MM_K(1, 3)(k) : RSR_MM_K(1, 1)(k));
}

static size_t mm_part_bytes(const rsr_stream_view *vw, int B) {
    return vw->tile_count <= 1 ? 0
                               : (size_t)vw->tile_count * B * vw->n_blocks * vw->k * 4;
}

// smem need of the batched kernel for `warps` warps (0 when unsupported)
static size_t mm_smem(const rsr_stream_view *vw, int warps) {
    const int64_t tn = std::min(vw->tile_width, vw->n);
    const size_t nkeys = (size_t)bucket_count(vw->bitwidth, vw->k);
    // format 3: the tile plus the 64 zero columns the padding names
    const size_t cols = vw->format == FMT_H ? (size_t)h_zero_b(tn) / 2 + 64 : (size_t)tn;
    return cols * MM_BV * 4 + ((nkeys * vw->k * 4 + 15) & ~(size_t)15) +
           (size_t)warps * nkeys * MM_BV * 4;
}

template <int MODE>
static rsr_status launch_mm(const rsr_stream_view *vw, const void *V, int vdtype, int64_t ldv,
                            int B, void *Y, int64_t ldy, void *ws, size_t ws_bytes,
                            cudaStream_t s) {
    if (!vw || !vw->entries || !vw->e_off || !V || !Y || B < 1) return RSR_ERR_INVALID;
    if (vw->format == FMT_U32 || !vw->col0_key) return RSR_ERR_INVALID;
    const int64_t rows = std::min(vw->n_blocks * vw->k, vw->m - vw->row_begin_block * vw->k);
    if (ldv < vw->n || ldy < rows) return RSR_ERR_INVALID;
    if (vw->n_blocks == 0) return RSR_OK;
    DeviceGuard guard(vw->device);
    const size_t pb = mm_part_bytes(vw, B);
    if (pb && (!ws || ws_bytes < pb)) return RSR_ERR_WORKSPACE;
    const int64_t nkeys = bucket_count(vw->bitwidth, vw->k);
    if (nkeys > BUCKET_MAX_KEYS) return RSR_ERR_INVALID;
    MmFn fn = pick_mm(MODE, vw->format, vw->k);
    if (!fn) return RSR_ERR_INVALID;
    const size_t cap = 227 * 1024;
    int warps = MM_MAX_WARPS;
    while (warps > 1 && mm_smem(vw, warps) > cap) --warps;
    if (mm_smem(vw, warps) > cap) return RSR_ERR_INVALID;
    const size_t smem = mm_smem(vw, warps);
    MmParams p;
    p.entries = vw->entries;
    p.e_off = vw->e_off;
    p.col0_key = vw->col0_key;
    p.m_rows = vw->m;
    p.n = vw->n;
    p.tw = vw->tile_width;
    p.tc = vw->tile_count;
    p.blk0 = vw->row_begin_block;
    p.nblk = vw->n_blocks;
    p.k = vw->k;
    p.bitwidth = vw->bitwidth;
    p.nkeys = (int)nkeys;
    p.V = V;
    p.vdtype = vdtype;
    p.ldv = ldv;
    p.B = B;
    p.Y = Y;
    p.ldy = ldy;
    p.part = ws;
    const int sms = sm_count();
    const int64_t chunks = (B + MM_BV - 1) / MM_BV;
    // one wave: the vector chunks and tiles share the SMs
    int64_t ctas = std::max<int64_t>(1, sms / (chunks * vw->tile_count));
    ctas = std::min<int64_t>(ctas, (vw->n_blocks + warps - 1) / warps);
    if (smem > 46 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return launch_status();
    }
    dim3 grid((unsigned)ctas, (unsigned)vw->tile_count, (unsigned)chunks);
    fn<<<grid, warps * 32, smem, s>>>(p);
    if (vw->tile_count > 1) {
        const int64_t rows_view = vw->n_blocks * vw->k;
        const int g2 = (int)std::min<int64_t>((rows_view * B + 255) / 256, 4096);
        mm_finalize_kernel<MODE><<<g2, 256, 0, s>>>(p, rows_view);
    }
    return launch_status();
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_matmul_workspace_bytes(const rsr_stream_view *view, int32_t B) {
    if (!view || B < 1) return 0;
    return mm_part_bytes(view, B);
}

rsr_status rsr_matmul(const rsr_stream_view *view, const void *V, int32_t v_dtype, int64_t ldv,
                      int32_t B, void *Y, int64_t ldy, void *workspace, size_t workspace_bytes,
                      rsr_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (v_dtype == RSR_I8)
        return launch_mm<MODE_INT>(view, V, v_dtype, ldv, B, Y, ldy, workspace, workspace_bytes, s);
    if (v_dtype == RSR_F32 || v_dtype == RSR_BF16 || v_dtype == RSR_F16)
        return launch_mm<MODE_FLOAT>(view, V, v_dtype, ldv, B, Y, ldy, workspace,
                                     workspace_bytes, s);
    return RSR_ERR_INVALID;
}

}  // extern "C"
