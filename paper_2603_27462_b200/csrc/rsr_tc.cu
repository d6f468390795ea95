// rsr_tc.cu -- batched multi-vector multiply on the 5th-generation tensor
// cores: Y[b] = M . V[b] for bf16 V.
//
// RSR's pattern-table step y_blk = T . S_blk (T in {0,+-1}^{k x P}) is a
// dense contraction; with B vectors it is cheaper to apply T before the
// segment sums: every column's pattern key, expanded through T, is one
// column of the block's k rows.  So this path keeps every column's pattern
// key in the reference's 2-bit code form (pattern_key, preproc.py:183-197:
// row i's code at bits 2i, 2i+1), concatenated down the rows and cut into
// 8-row groups (one u16 per (row group, column); 16.8 MB at C4 -- 2 bits
// per matrix entry), expands it straight into the A operand of tcgen05.mma
// and accumulates in TMEM:
//
//   D[row][b] += A[row][col] * B[b][col],  A = T[:, key(blk, col)] (bf16 +-1/0),
//                                          B = V chunk (bf16, K-major)
//
// Tile: M = 128 rows (16 row groups), K = 64 columns per step, N = vectors
// (16..256).  Warp-specialized, TC_STAGES-deep ring per CTA:
//   warp 8  (producer)  bulk-copies (cp.async.bulk, mbarrier complete_tx) the
//                       step's code chunk and its pre-packed B tile;
//   warps 0-7 (expand)  build the MN-major A tile: per (row group, column)
//                       one u16 of codes -> 4 PRMTs (a register byte table)
//                       -> one 16-byte store (conflict-free: a quarter warp
//                       covers 128 B);
//   warp 9  (MMA)       one thread issues tcgen05.mma (fp32 in TMEM) and
//                       commits to the stage's "empty" barrier.
// Code matrix layout [step = col / 64][row group][col % 64], so a tile's
// step is one contiguous chunk; a row-block view starting mid-group takes
// the enclosing groups and skips the outside rows in the epilogue.  V is
// repacked once per call into the K-major no-swizzle core-matrix image of
// each step (tc_pack_v_kernel), so its B tile is one bulk copy too.  Products
// with +-1 are exact and accumulate in fp32: the float-path tolerance holds.
// Split-K over grid.y fills the SMs; partials are summed in a fixed order
// by tc_finalize_kernel (deterministic).
#include <cstdio>
#include <cstdlib>

#include "rsr_mv_impl.cuh"

namespace rsr {

constexpr int TC_M = 128;           // tile rows = TMEM lanes
constexpr int TC_MAXBPT = 128;      // row blocks per tile: floor(128 / k)
constexpr int TC_K = 64;            // columns per pipeline step
constexpr int TC_STAGES = 4;       // ring depth (at most; fewer when shared memory is short)
#ifndef RSR_TC_EXP_WARPS
#define RSR_TC_EXP_WARPS 8
#endif
constexpr int TC_EXP_WARPS = RSR_TC_EXP_WARPS;
constexpr int TC_THREADS = TC_EXP_WARPS * 32 + 64;  // expanders, producer, MMA
constexpr int TC_UNITS = 16 * TC_K / (TC_EXP_WARPS * 32);  // (row group, column) units per thread


__host__ __device__ inline int64_t tc_steps(int64_t n) { return (n + TC_K - 1) / TC_K; }

// ---- key matrix: KM[step][g][col % 64] = the 2-bit row codes of rows
// 8g .. 8g + 7 at column col (each block's pattern key, in code form, lands at
// bit 2 (row % 8) of its row group; a block straddling two groups is split)
__global__ void keymat_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                              const uint16_t *__restrict__ perm, const int64_t *__restrict__ po,
                              int64_t bc, int64_t tc, int64_t tw, int k, int64_t ng,
                              uint32_t *__restrict__ km32) {
    const uint32_t lane = lane_id();
    const int64_t cells = bc * tc;
    for (int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; cell < cells;
         cell += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = cell / bc, b = cell - t * bc;  // reference cells are tile-major
        const int64_t c0 = t * tw;
        const int64_t r0 = b * k, g0 = r0 >> 3;
        const int sh = 2 * (int)(r0 & 7);
        for (int64_t g = go[cell]; g < go[cell + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu), L = (int64_t)((w >> 16) & 0xFFFFu);
            const uint32_t pos = (uint32_t)((w >> 32) & 0xFFu), neg = (uint32_t)((w >> 48) & 0xFFu);
            uint32_t code = 0;  // +1 -> 01, -1 -> 10 (binary keys have no neg bits)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                code |= (((pos >> i) & 1u) | (((neg >> i) & 1u) << 1)) << (2 * i);
            const uint32_t lo = (code << sh) & 0xFFFFu, hi = (code << sh) >> 16;
            const uint16_t *cols = perm + po[cell] + ps;
            for (int64_t j = lane; j < L; j += 32) {
                const int64_t col = c0 + cols[j];
                const int64_t e = ((col / TC_K) * ng + g0) * TC_K + (col % TC_K);
                atomicOr(km32 + (e >> 1), lo << (16 * (e & 1)));
                if (hi) {
                    const int64_t e2 = e + TC_K;  // next row group, same column
                    atomicOr(km32 + (e2 >> 1), hi << (16 * (e2 & 1)));
                }
            }
        }
    }
}

// ---- V repack: vp[step][N/8][kg 8][8 vectors][8 columns] bf16 (the B tile image) ----
__global__ void tc_pack_v_kernel(const uint16_t *__restrict__ V, int64_t ldv, int64_t n, int B,
                                 int N, int64_t steps, uint4 *__restrict__ vp) {
    const int64_t pieces = steps * N * 8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pieces;
         e += (int64_t)gridDim.x * blockDim.x) {
        // e = ((st * N/8 + vg) * 8 + kg) * 8 + vi
        const int vi = (int)(e & 7), kg = (int)((e >> 3) & 7);
        const int64_t r = e >> 6;
        const int64_t st = r / (N >> 3);
        const int vb = (int)(r - st * (N >> 3)) * 8 + vi;
        const int64_t c = st * TC_K + kg * 8;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (vb < B) {
            const uint16_t *src = V + (int64_t)vb * ldv + c;
            if (c + 8 <= n && ((ldv & 7) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0)) {
                val = *reinterpret_cast<const uint4 *>(src);
            } else {
                uint32_t h[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) h[q] = c + q < n ? src[q] : 0u;
                val = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                                 h[6] | (h[7] << 16));
            }
        }
        vp[e] = val;
    }
}

// ---- tcgen05 / mbarrier / bulk-copy helpers -------------------------------------
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // no-swizzle canonical layout; fields in 16-byte units; version 1 (sm_100)
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     mbar)
                 : "memory");
}

#ifdef RSR_TC_DBG
__device__ unsigned long long tc_dbg[64 * 4 + 4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TC_MARK(cond, idx) \
    if ((cond) && blockIdx.x == 0 && blockIdx.y == 0 && (idx) < 64 * 4 + 4) tc_dbg[idx] = gtime();
#else
#define TC_MARK(cond, idx)
#endif

struct TcParams {
    const uint16_t *km;  // key matrix [steps][bc][64] (2-bit row codes)
    const uint4 *vp;     // packed V [steps][N/8][8][8][8] bf16
    float *Y;            // [B][ldy] rows of the view
    int64_t ldy;
    float *part;         // split-K partials [ksplit][B][rows]
    int64_t m_rows, n, nblk, blk0, bc;
    int64_t ng;           // row groups of 8 in the whole matrix
    int k, B, N, ksplit, stages;
    uint32_t tab0, tab1;  // PRMT byte table {00 3F BF 00 | 00 80 80 00} (kept in registers)
};

// 8 row codes (2 bits each, +1 -> 01, -1 -> 10) of two units at once
// (x = unit0 | unit1 << 16) -> the 8 bf16 signs of each as 4 words of two:
// PRMT picks each byte from a register table {00 3F BF 00 | 00 80 80 00}
// with selector nibbles (4 + c0, c0, 4 + c1, c1) =
// 0x0404 + 0x11 * (c0 + (c1 << 8)), built per 16-bit half with two IMADs
__device__ __forceinline__ void expand_codes2(uint32_t x, uint4 &lo, uint4 &hi, uint32_t tab0,
                                              uint32_t tab1, uint32_t c0404) {
    uint32_t w0[4], w1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t t = x >> (4 * q);
        const uint32_t tm = t & 0x000F000Fu, th = t & 0x000C000Cu;
        // 0x11 * (c0 + 4 c1) + 0x42F * 4 c1 = 0x11 * (c0 + (c1 << 8)), + 0x0404;
        // explicit mads (one immediate each: no constant rematerialization)
        uint32_t u, sel;
        asm("mad.lo.u32 %0, %1, 0x11, %2;" : "=r"(u) : "r"(tm), "r"(c0404));
        asm("mad.lo.u32 %0, %1, 0x42F, %2;" : "=r"(sel) : "r"(th), "r"(u));
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(w0[q]) : "r"(tab0), "r"(tab1), "r"(sel));
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(w1[q]) : "r"(tab0), "r"(tab1), "r"(sel >> 16));
    }
    lo = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    hi = make_uint4(w1[0], w1[1], w1[2], w1[3]);
}

// N = 16 * NP: MMA N (vectors padded up, <= 256)
template <int NP>
__global__ void __launch_bounds__(TC_THREADS) rsr_tc_kernel(TcParams p) {
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t bars[3 * TC_STAGES + 1];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    constexpr int N = 16 * NP;
    const int S = p.stages;
    // PDL: the finalize may launch now (it waits for this grid to finish)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // this tile: row groups [g_first, g_first + 16) of the matrix, covering
    // the view's rows [row0, row0 + rows_view) (rows outside are skipped)
    const int64_t row0 = p.blk0 * p.k;
    const int64_t rows_view = min(p.nblk * p.k, p.m_rows - row0);
    const int64_t g_first = (row0 >> 3) + (int64_t)blockIdx.x * 16;
    const int ng_here = (int)min((int64_t)16, p.ng - g_first);
    const int64_t nsteps_all = tc_steps(p.n);
    const int64_t s0 = nsteps_all * blockIdx.y / p.ksplit;
    const int64_t s1 = nsteps_all * (blockIdx.y + 1) / p.ksplit;
    const int64_t nst = s1 - s0;

    // smem: per stage [A 16 KB][B N x 128 B][codes 16 x 64 x u16]
    constexpr uint32_t A_BYTES = TC_M * TC_K * 2;
    constexpr uint32_t B_BYTES = (uint32_t)N * TC_K * 2;
    constexpr uint32_t C_BYTES = 16 * TC_K * 2;
    constexpr uint32_t st_bytes = (A_BYTES + B_BYTES + C_BYTES + 1023) / 1024 * 1024;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tc_smem);
    const uint32_t bar_full = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    const uint32_t bar_aready = bar_full + 8 * TC_STAGES;
    const uint32_t bar_empty = bar_aready + 8 * TC_STAGES;
    const uint32_t bar_done = bar_empty + 8 * TC_STAGES;

    // code rows past the matrix (never written by the producer) read as 0
    for (int s = 0; s < S; ++s) {
        uint32_t *kz = reinterpret_cast<uint32_t *>(tc_smem + s * st_bytes + A_BYTES + B_BYTES +
                                                    (size_t)ng_here * TC_K * 2);
        for (int i = tid; i < (16 - ng_here) * TC_K / 2; i += TC_THREADS) kz[i] = 0u;
    }
    if (warp == TC_EXP_WARPS + 1) {  // TMEM: N fp32 columns x 128 lanes
        uint32_t cols = 32;
        while (cols < (uint32_t)N) cols <<= 1;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base_sh)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_aready + 8 * s, TC_EXP_WARPS * 32);
            mbar_init(bar_empty + 8 * s, 1);
        }
        mbar_init(bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;
    TC_MARK(tid == 0, 256)

    if (warp == TC_EXP_WARPS) {
        // ---- producer ----
        if (lane == 0) {
            const uint32_t kbytes = (uint32_t)ng_here * TC_K * 2;
            // PDL: the packed V comes from the previous kernel; everything
            // before this point overlapped its tail
            asm volatile("griddepcontrol.wait;" ::: "memory");
            for (int64_t it = 0; it < nst; ++it) {
                const int s = (int)(it % S);
                if (it >= S) mbar_wait_parity(bar_empty + 8 * s, (uint32_t)((it / S - 1) & 1));
                const int64_t st = s0 + it;
                TC_MARK(it < 64, it * 4 + 2)
                const uint32_t sa = sbase + s * st_bytes;
                mbar_expect_tx(bar_full + 8 * s, kbytes + B_BYTES);
                bulk_g2s(sa + A_BYTES + B_BYTES, p.km + (st * p.ng + g_first) * TC_K, kbytes,
                         bar_full + 8 * s);
                bulk_g2s(sa + A_BYTES, p.vp + (size_t)st * (B_BYTES / 16), B_BYTES,
                         bar_full + 8 * s);
            }
        }
    } else if (warp == TC_EXP_WARPS + 1) {
        // ---- MMA issuer ----
        if (lane == 0) {
            // instruction descriptor: kind::f16, A = B = BF16, D = F32, A MN-major,
            // B K-major, N >> 3 at [17,23), M >> 4 at [24,29)
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                                   ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            int s = 0;
            uint32_t par = 0;
            for (int64_t it = 0; it < nst; ++it) {
                mbar_wait_parity(bar_full + 8 * s, par);
                mbar_wait_parity(bar_aready + 8 * s, par);
                TC_MARK(it < 64, it * 4 + 3)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a0 = sbase + s * st_bytes, b0 = a0 + A_BYTES;
#pragma unroll
                for (int kk = 0; kk < TC_K / 16; ++kk) {
                    // A MN-major: LBO = K-group stride (16 row groups x 128 B), SBO = M-group stride
                    const uint64_t da = smem_desc(a0 + kk * 2 * (16 * 128), 16 * 128, 128);
                    // B K-major: LBO = K-group stride (128 B), SBO = N-group stride (8 x 128 B)
                    const uint64_t db = smem_desc(b0 + kk * 2 * 128, 128, 8 * 128);
                    mma_bf16(tmem_d, da, db, idesc, (it > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(bar_empty + 8 * s);
                if (++s == S) {
                    s = 0;
                    par ^= 1u;
                }
            }
            mma_commit(bar_done);
        }
    } else {
        // ---- expanders: thread owns column c_t of row groups mg_t .. mg_t +
        // TC_UNITS - 1 (tile rows 8 mg .. 8 mg + 7); a quarter warp's 16-byte
        // A stores are 128 contiguous bytes ----
        const int c_t = tid & 63, mg_t = (tid >> 6) * TC_UNITS;
        // table words and the selector bias in plain registers, set once
        // (shuffled: per-thread values ptxas keeps in vector registers
        // instead of re-copying uniform ones at every use)
        const uint32_t tab0 = __shfl_sync(RSR_FULL_MASK, p.tab0, 0);
        const uint32_t tab1 = __shfl_sync(RSR_FULL_MASK, p.tab1, 0);
        const uint32_t c0404 = __shfl_sync(RSR_FULL_MASK, 0x04040404u, 0);
        int s = 0;
        uint32_t par = 0;
        for (int64_t it = 0; it < nst; ++it) {
            mbar_wait_parity(bar_full + 8 * s, par);
            TC_MARK(tid == 0 && it < 64, it * 4 + 0)
            unsigned char *stg = tc_smem + s * st_bytes;
            const uint16_t *sk =
                reinterpret_cast<const uint16_t *>(stg + A_BYTES + B_BYTES) + mg_t * TC_K + c_t;
            // A (MN-major core layout [kg 8][row group 16][8 columns][16 B = 8 rows])
            unsigned char *dA = stg + (size_t)(c_t & 7) * 16 + (size_t)(c_t >> 3) * 16 * 128;
#pragma unroll
            for (int j = 0; j < TC_UNITS; j += 2) {
                // the row codes of two row groups, one per 16-bit half
                uint32_t x;
                asm("prmt.b32 %0, %1, %2, 0x5410;"
                    : "=r"(x)
                    : "r"((uint32_t)sk[j * TC_K]), "r"((uint32_t)sk[(j + 1) * TC_K]));
                uint4 lo, hi;
                expand_codes2(x, lo, hi, tab0, tab1, c0404);
                *reinterpret_cast<uint4 *>(dA + (size_t)(mg_t + j) * 128) = lo;
                *reinterpret_cast<uint4 *>(dA + (size_t)(mg_t + j + 1) * 128) = hi;
            }
            // generic-proxy writes -> visible to the tensor core (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(bar_aready + 8 * s);
            TC_MARK(tid == 0 && it < 64, it * 4 + 1)
            if (++s == S) {
                s = 0;
                par ^= 1u;
            }
        }
    }
    __syncwarp();
    mbar_wait_parity(bar_done, 0);
    TC_MARK(tid == 0, 257)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    if (warp < 4) {
        // --- epilogue: warp w reads TMEM lanes 32w..32w+31 (tile rows), 8 columns at a time
        const int row_t = warp * 32 + (int)lane;
        const int64_t vrow = g_first * 8 + row_t - row0;  // row within the view
        const bool valid = vrow >= 0 && vrow < rows_view;
        for (int c = 0; c < N; c += 8) {
            uint32_t r[8];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7])
                : "r"(tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (valid) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int vb = c + j;
                    if (vb < p.B) {
                        const float x = nst > 0 ? __uint_as_float(r[j]) : 0.f;
                        if (p.ksplit == 1) p.Y[(int64_t)vb * p.ldy + vrow] = x;
                        else p.part[((int64_t)blockIdx.y * p.B + vb) * rows_view + vrow] = x;
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    TC_MARK(tid == 0, 258)
    if (warp == TC_EXP_WARPS + 1) {
        uint32_t cols = 32;
        while (cols < (uint32_t)N) cols <<= 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(cols));
    }
}

__global__ void tc_finalize_kernel(TcParams p, int64_t rows_view) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the partials are complete
    const int64_t total = rows_view * p.B;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t vb = e / rows_view, r = e - vb * rows_view;
        float s = 0.f;
        for (int ks = 0; ks < p.ksplit; ++ks) s += p.part[((int64_t)ks * p.B + vb) * rows_view + r];
        p.Y[vb * p.ldy + r] = s;
    }
}

static int tc_np(int B) {
    int np = 1;
    while (16 * np < B) np *= 2;
    return np;
}

static size_t tc_stage_bytes(int N) {
    return ((size_t)TC_M * TC_K * 2 + (size_t)N * TC_K * 2 + 16 * TC_K * 2 + 1023) / 1024 * 1024;
}

static int tc_stages(int N) {
    // deepest ring that still lets two CTAs share an SM (16 expander warps
    // per SM); failing that the deepest ring that fits one CTA
    const size_t sb = tc_stage_bytes(N);
    for (int st = TC_STAGES; st >= 3; --st)
        if (2 * (st * sb + 2048) <= 228 * 1024) return st;
    int st = TC_STAGES;
    while (st > 2 && st * sb > 220 * 1024) --st;
    return st;
}

static size_t tc_smem_bytes(int N) { return tc_stages(N) * tc_stage_bytes(N); }

// row tiles (16 row groups) covering the view's rows
static int64_t tc_tiles(int64_t block_begin, int64_t n_blocks, int32_t k, int64_t m) {
    const int64_t r0 = block_begin * k, r1 = std::min((block_begin + n_blocks) * k, m);
    if (r1 <= r0) return 0;
    const int64_t g0 = r0 >> 3, g1 = (r1 + 7) >> 3;
    return (g1 - g0 + 15) / 16;
}

static int tc_ksplit(int64_t tiles, int64_t n, int B) {
    // split K so that the tiles x splits fill the resident CTA slots in as
    // few waves as possible; a wave costs about its steps plus ~6 steps of
    // prologue / epilogue
    const int64_t steps = tc_steps(n);
    const size_t smem = tc_smem_bytes(16 * tc_np(B)) + 2048;
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (228 * 1024) / (int64_t)smem));
    const int64_t slots = per_sm * sm_count();
    static const int forced = [] {
        const char *e = getenv("RSR_TC_KSPLIT");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) return (int)std::max<int64_t>(1, std::min<int64_t>(forced, steps));
    int best = 1;
    double best_cost = 1e30;
    for (int ks = 1; ks <= 32 && ks <= steps; ++ks) {
        const int64_t waves = (tiles * ks + slots - 1) / slots;
        const double cost = (double)waves * ((double)((steps + ks - 1) / ks) + 6.0) +
                            0.02 * ks;  // partial traffic
        if (cost < best_cost) {
            best_cost = cost;
            best = ks;
        }
    }
    return best;
}

}  // namespace rsr

using namespace rsr;

extern "C" {

#ifdef RSR_TC_DBG
int rsr_tc_debug(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, tc_dbg, sizeof(unsigned long long) * (64 * 4 + 4));
}
#endif

size_t rsr_keymat_bytes(int64_t block_count, int64_t cols, int32_t bitwidth, int32_t k) {
    (void)bitwidth;
    if (k < 1 || k > 8 || block_count < 0 || cols < 0) return 0;
    const int64_t ng = (block_count * k + 7) / 8;
    return (size_t)tc_steps(cols) * ng * TC_K * 2;
}

rsr_status rsr_keymat_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                            void *keymat, rsr_stream_t stream) {
    const size_t bytes = rsr_keymat_bytes(block_count, cols, bitwidth, k);
    if (!bytes || !keymat || !go || !po || (reinterpret_cast<uintptr_t>(keymat) & 3))
        return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(keymat, 0, bytes, s);
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells * 32 + 255) / 256, (int64_t)sm_count() * 16);
    keymat_kernel<<<grid, 256, 0, s>>>(words, go, perm, po, block_count, tile_count, tile_width, k,
                                       (block_count * k + 7) / 8, (uint32_t *)keymat);
    return launch_status();
}

// workspace: [packed V (256-byte aligned)][split-K partials]
static size_t tc_vpack_bytes(int64_t n, int32_t B) {
    return ((size_t)tc_steps(n) * 16 * tc_np(B) * TC_K * 2 + 255) / 256 * 256;
}

size_t rsr_matmul_tc_workspace_bytes(int64_t m, int64_t n, int32_t k, int64_t block_begin,
                                     int64_t n_blocks, int32_t B) {
    if (B < 1 || B > 256 || k < 1 || k > 8 || n_blocks < 0) return 0;
    const int ks = tc_ksplit(tc_tiles(block_begin, n_blocks, k, m), n, B);
    const int64_t rows = std::max<int64_t>(0, std::min(n_blocks * k, m - block_begin * k));
    return tc_vpack_bytes(n, B) + (ks > 1 ? (size_t)ks * B * rows * 4 : 0);
}

rsr_status rsr_matmul_tc(const void *keymat, int64_t m, int64_t n, int32_t bitwidth, int32_t k,
                         int64_t block_begin, int64_t n_blocks, const void *V, int32_t v_dtype,
                         int64_t ldv, int32_t B, float *Y, int64_t ldy, void *workspace,
                         size_t workspace_bytes, rsr_stream_t stream) {
    (void)bitwidth;
    if (!keymat || !V || !Y || B < 1 || B > 256 || v_dtype != RSR_BF16 || k < 1 || k > 8)
        return RSR_ERR_INVALID;
    const int64_t rows = std::min(n_blocks * k, m - block_begin * k);
    if (ldv < n || ldy < rows || n_blocks < 0 || block_begin < 0) return RSR_ERR_INVALID;
    if (n_blocks == 0) return RSR_OK;
    const int64_t tiles = tc_tiles(block_begin, n_blocks, k, m);
    const int ks = tc_ksplit(tiles, n, B);
    const size_t wsb = rsr_matmul_tc_workspace_bytes(m, n, k, block_begin, n_blocks, B);
    if (!workspace || workspace_bytes < wsb || (reinterpret_cast<uintptr_t>(workspace) & 255))
        return RSR_ERR_WORKSPACE;
    const int np = tc_np(B);
    TcParams p;
    p.km = (const uint16_t *)keymat;
    p.vp = (const uint4 *)workspace;
    p.Y = Y;
    p.ldy = ldy;
    p.part = (float *)((char *)workspace + tc_vpack_bytes(n, B));
    p.m_rows = m;
    p.n = n;
    p.nblk = n_blocks;
    p.blk0 = block_begin;
    p.bc = (m + k - 1) / k;
    p.ng = (p.bc * k + 7) / 8;
    p.k = k;
    p.B = B;
    p.N = 16 * np;
    p.ksplit = ks;
    p.stages = tc_stages(p.N);
    p.tab0 = 0x00BF3F00u;
    p.tab1 = 0x00808000u;
    if (block_begin + n_blocks > p.bc) return RSR_ERR_INVALID;
    const size_t smem = tc_smem_bytes(p.N);
    if (smem > 227 * 1024) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    {
        const int64_t pieces = tc_steps(n) * p.N * 8;
        const int g = (int)std::min<int64_t>((pieces + 255) / 256, (int64_t)sm_count() * 8);
        tc_pack_v_kernel<<<g, 256, 0, s>>>((const uint16_t *)V, ldv, n, B, p.N, tc_steps(n),
                                           (uint4 *)workspace);
    }
    dim3 grid((unsigned)tiles, (unsigned)ks);
    // the tcgen05 kernel and the finalize launch as programmatic dependents
    // (PDL): each one's prologue overlaps the previous kernel's tail
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
#define RSR_TC_LAUNCH(NPV)                                                                      \
    {                                                                                          \
        cudaFuncSetAttribute(rsr_tc_kernel<NPV>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)smem);                                                       \
        cudaLaunchKernelEx(&cfg, rsr_tc_kernel<NPV>, p);                                       \
    }
    switch (np) {
        case 1: RSR_TC_LAUNCH(1) break;
        case 2: RSR_TC_LAUNCH(2) break;
        case 4: RSR_TC_LAUNCH(4) break;
        case 8: RSR_TC_LAUNCH(8) break;
        default: RSR_TC_LAUNCH(16) break;
    }
#undef RSR_TC_LAUNCH
    if (ks > 1) {
        cudaLaunchConfig_t fcfg = cfg;
        fcfg.gridDim = dim3((unsigned)std::min<int64_t>((rows * B + 255) / 256, 4096));
        fcfg.blockDim = dim3(256);
        fcfg.dynamicSmemBytes = 0;
        cudaLaunchKernelEx(&fcfg, tc_finalize_kernel, p, rows);
    }
    return launch_status();
}

}  // extern "C"
