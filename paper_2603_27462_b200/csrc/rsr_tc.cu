// rsr_tc.cu -- batched multi-vector multiply on the 5th-generation tensor
// cores: Y[b] = M . V[b] for bf16 V.
//
// RSR's pattern-table step y_blk = T . S_blk (T in {0,+-1}^{k x P}) is a
// dense contraction; with B vectors it is cheaper to apply T before the
// segment sums: every column's pattern key, expanded through T, is one
// column of the block's k rows.  So this path keeps, per row block, the
// pattern key of every column (the RSR keys before the grouping sort, 1 byte
// per column when the pattern space fits in a byte -- 13.4 MB at C4, less
// than the 29 MB artifact), expands keys through a shared-memory copy of T
// straight into the A operand of tcgen05.mma, and accumulates in TMEM:
//
//   D[row][b] += A[row][col] * B[b][col],  A = T[:, key(blk, col)] (bf16 +-1/0),
//                                          B = V chunk (bf16, K-major)
//
// Tile: 16 row blocks x 8 (padded) rows = M 128, K 64 columns per step,
// N = vectors (16..256).  A is MN-major (one 16-byte write per (block,
// column): the block's 8 rows), B is K-major; both in the no-swizzle
// canonical core-matrix layout (8 x 16 B core matrices).  Products with +-1
// are exact and accumulate in fp32: the float-path tolerance holds.
// Split-K over grid.y keeps every SM busy; partials are summed in a fixed
// order by rsr_tc_finalize (deterministic).
#include <cstdio>

#include "rsr_mv_impl.cuh"

namespace rsr {

constexpr int TC_BLOCKS = 16;       // row blocks per tile (8 padded rows each)
constexpr int TC_M = TC_BLOCKS * 8; // 128 rows = TMEM lanes
constexpr int TC_K = 64;            // columns per pipeline step
constexpr int TC_THREADS = 128;

// ---- key matrix: KM[blk][col] = pattern key of column col in block blk ----
template <typename KeyT>
__global__ void keymat_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                              const uint16_t *__restrict__ perm, const int64_t *__restrict__ po,
                              int64_t bc, int64_t tc, int64_t tw, int bitwidth, int64_t n,
                              KeyT *__restrict__ km) {
    const uint32_t lane = lane_id();
    const int64_t cells = bc * tc;
    for (int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; cell < cells;
         cell += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = cell / bc, b = cell - t * bc;  // reference cells are tile-major
        const int64_t c0 = t * tw;
        KeyT *row = km + b * n + c0;
        for (int64_t g = go[cell]; g < go[cell + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu), L = (int64_t)((w >> 16) & 0xFFFFu);
            const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
            uint32_t key = pos;
            if (bitwidth != RSR_BINARY) {
                key = 0;
                uint32_t p3 = 1;
                for (int i = 0; i < 16; ++i) {
                    key += (((pos >> i) & 1u) + 2u * ((neg >> i) & 1u)) * p3;
                    p3 *= 3u;
                }
            }
            const uint16_t *cols = perm + po[cell] + ps;
            for (int64_t j = lane; j < L; j += 32) row[cols[j]] = (KeyT)key;
        }
    }
}

// ---- tcgen05 helpers ---------------------------------------------------------
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

__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tTC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC_WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

struct TcParams {
    const void *km;      // key matrix [bc][n] (u8 or u16)
    const void *V;       // bf16 [B][ldv]
    int64_t ldv;
    float *Y;            // [B][ldy] rows of the view
    int64_t ldy;
    float *part;         // split-K partials [ksplit][B][rows]
    int64_t m_rows, n, nblk, blk0;
    int k, bitwidth, nkeys, B, N, ksplit;
};

// N = 16 * NP: MMA N (vectors padded up, <= 256)
template <typename KeyT, int NP>
__global__ void __launch_bounds__(TC_THREADS) rsr_tc_kernel(TcParams p) {
    extern __shared__ __align__(128) unsigned char tc_smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t bars[2];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    constexpr int N = 16 * NP;
    const int64_t blk_first = (int64_t)blockIdx.x * TC_BLOCKS;
    const int nblk_here = (int)min((int64_t)TC_BLOCKS, p.nblk - blk_first);
    // split-K: columns [kc0, kc1) of this CTA, in TC_K steps
    const int64_t nsteps_all = (p.n + TC_K - 1) / TC_K;
    const int64_t s0 = nsteps_all * blockIdx.y / p.ksplit;
    const int64_t s1 = nsteps_all * (blockIdx.y + 1) / p.ksplit;

    // smem: [A x2: 128 rows x 64 cols bf16 = 16 KB][B x2: N x 64 bf16][sign LUT nkeys x 16 B]
    constexpr uint32_t A_BYTES = TC_M * TC_K * 2;
    constexpr uint32_t B_BYTES = (uint32_t)N * TC_K * 2;
    unsigned char *sA = tc_smem;
    unsigned char *sB = tc_smem + 2 * A_BYTES;
    uint32_t *lut = reinterpret_cast<uint32_t *>(tc_smem + 2 * A_BYTES + 2 * B_BYTES);
    const uint32_t aA = (uint32_t)__cvta_generic_to_shared(sA);
    const uint32_t aB = (uint32_t)__cvta_generic_to_shared(sB);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);

    // pair table: two rows' digits (d0 + 3*d1, digit 0 / +1 / -1 for 0 / 1 / 2)
    // -> the two bf16 signs packed in one 32-bit word
    if (tid < 9) {
        const uint32_t d0 = tid % 3, d1 = tid / 3;
        auto h = [](uint32_t d) -> uint32_t { return d == 0 ? 0u : (d == 1 ? 0x3F80u : 0xBF80u); };
        lut[tid] = h(d0) | (h(d1) << 16);
    }
    if (warp == 0) {  // TMEM: N fp32 columns x 128 lanes
        uint32_t cols = 32;
        while (cols < (uint32_t)N) cols <<= 1;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base_sh)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init1(bar0);
        mbar_init1(bar0 + 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;

    // instruction descriptor: kind::f16, A = B = BF16, D = F32, A MN-major,
    // B K-major, N >> 3 at [17,23), M >> 4 at [24,29)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

    const KeyT *km = reinterpret_cast<const KeyT *>(p.km);
    const uint16_t *V = reinterpret_cast<const uint16_t *>(p.V);
    // Per step each thread owns: column tid % 64 of the 8 blocks (tid / 64)*8
    // + j (so a warp's 16-byte A stores cover all banks), and NP 16-byte
    // pieces of the vector chunk (8 consecutive threads take 8 vectors of one
    // 8-column group: conflict-free B stores).  Both are loaded one step
    // ahead into registers (ping-pong), so global latency overlaps the
    // previous step's expansion and MMAs.
    const int c_t = tid & 63, bg_t = (tid >> 6) * 8;
    struct Step {
        uint32_t keys[8];
        uint4 vp[NP];
    };
    auto load_step = [&](int64_t st, Step &S) {
        const int64_t col = st * TC_K + c_t;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int bi = bg_t + j;
            S.keys[j] = (bi < nblk_here && col < p.n)
                            ? (uint32_t)__ldg(km + (blk_first + bi) * p.n + col) : 0u;
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int piece = tid + j * TC_THREADS;
            const int vb = (piece & 7) + 8 * (piece >> 6), kg = (piece >> 3) & 7;
            const int64_t c = st * TC_K + kg * 8;
            uint4 val = make_uint4(0, 0, 0, 0);
            if (vb < p.B) {
                const uint16_t *src = V + (int64_t)vb * p.ldv + c;
                if (c + 8 <= p.n && ((p.ldv & 7) == 0)) {
                    val = ld_stream(reinterpret_cast<const uint4 *>(src));
                } else {
                    uint32_t h[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) h[q] = c + q < p.n ? src[q] : 0u;
                    val = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                                     h[6] | (h[7] << 16));
                }
            }
            S.vp[j] = val;
        }
    };
    const bool binary = p.bitwidth == RSR_BINARY;
    // the 8 (padded) rows of a key as 4 words of two bf16 signs
    auto expand = [&](uint32_t key) -> uint4 {
        uint32_t w[4];
        if (binary) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t two = (key >> (2 * q)) & 3u;
                w[q] = lut[(two & 1u) + 3u * (two >> 1)];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t nk = key / 9u;  // digits 2q, 2q+1 of the base-3 key
                w[q] = lut[key - 9u * nk];
                key = nk;
            }
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    };
    uint32_t phase[2] = {0u, 0u};
    auto do_step = [&](int64_t st, const Step &S) {
        const int buf = (int)((st - s0) & 1);
        if (st - s0 >= 2) {  // the MMAs that read this buffer two steps ago are done
            mbar_wait_parity(bar0 + 8 * buf, phase[buf]);
            phase[buf] ^= 1u;
        }
        // A (MN-major core layout [kg 8][block 16][8 columns][16 B = 8 rows])
        unsigned char *dA = sA + buf * A_BYTES + (size_t)(c_t & 7) * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4 *>(dA + ((size_t)(c_t >> 3) * TC_BLOCKS + bg_t + j) * 128) =
                expand(S.keys[j]);
        // B (K-major core layout [N/8][kg 8][8 vectors][16 B = 8 columns])
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int piece = tid + j * TC_THREADS;
            const int vb = (piece & 7) + 8 * (piece >> 6), kg = (piece >> 3) & 7;
            *reinterpret_cast<uint4 *>(sB + buf * B_BYTES +
                                       (((size_t)(vb >> 3) * 8 + kg) * 8 + (vb & 7)) * 16) = S.vp[j];
        }
        // generic-proxy writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = aA + buf * A_BYTES, b0 = aB + buf * B_BYTES;
#pragma unroll
            for (int kk = 0; kk < TC_K / 16; ++kk) {
                // A MN-major: LBO = K-group stride (16 blocks x 128 B), SBO = M-group stride
                const uint64_t da = smem_desc(a0 + kk * 2 * (TC_BLOCKS * 128), TC_BLOCKS * 128, 128);
                // B K-major: LBO = K-group stride (128 B), SBO = N-group stride (8 x 128 B)
                const uint64_t db = smem_desc(b0 + kk * 2 * 128, 128, 8 * 128);
                mma_bf16(tmem_d, da, db, idesc, (st > s0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(bar0 + 8 * buf);
        }
        __syncwarp();
    };
    Step SA, SB;
    if (s0 < s1) load_step(s0, SA);
    for (int64_t st = s0; st < s1; st += 2) {
        if (st + 1 < s1) load_step(st + 1, SB);
        do_step(st, SA);
        if (st + 1 >= s1) break;
        if (st + 2 < s1) load_step(st + 2, SA);
        do_step(st + 1, SB);
    }
    // wait for the last MMAs of both buffers
    const int64_t nst = s1 - s0;
    for (int b = 0; b < 2; ++b) {
        // buffer b was committed ceil((nst - b) / 2) times; the waits above
        // consumed max(0, that - 1) of them
        const int64_t commits = (nst - b + 1) / 2;
        if (commits > 0) mbar_wait_parity(bar0 + 8 * b, phase[b]);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // --- epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 8 columns at a time
    const int row_t = warp * 32 + (int)lane;  // tile row = block * 8 + i
    const int bi = row_t >> 3, i = row_t & 7;
    const int64_t blk = blk_first + bi;
    const bool valid = bi < nblk_here && i < p.k && (p.blk0 + blk) * p.k + i < p.m_rows;
    const int64_t vrow = blk * p.k + i;  // row within the view
    const int64_t rows_view = min(p.nblk * p.k, p.m_rows - p.blk0 * p.k);
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7])
            : "r"(tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int vb = c + j;
                if (vb < p.B) {
                    const float x = __uint_as_float(r[j]);
                    if (p.ksplit == 1) p.Y[(int64_t)vb * p.ldy + vrow] = x;
                    else p.part[((int64_t)blockIdx.y * p.B + vb) * rows_view + vrow] = x;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        uint32_t cols = 32;
        while (cols < (uint32_t)N) cols <<= 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(cols));
    }
}

__global__ void tc_finalize_kernel(TcParams p, int64_t rows_view) {
    const int64_t total = rows_view * p.B;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t vb = e / rows_view, r = e - vb * rows_view;
        float s = 0.f;
        for (int ks = 0; ks < p.ksplit; ++ks) s += p.part[((int64_t)ks * p.B + vb) * rows_view + r];
        p.Y[vb * p.ldy + r] = s;
    }
}

static size_t tc_smem_bytes(int N, int) {
    return 2 * (size_t)TC_M * TC_K * 2 + 2 * (size_t)N * TC_K * 2 + 64;
}

static int tc_ksplit(int64_t nblk, int64_t n) {
    // about four CTAs per SM (52-100 KB of shared memory each)
    const int64_t tiles = (nblk + TC_BLOCKS - 1) / TC_BLOCKS;
    const int64_t steps = (n + TC_K - 1) / TC_K;
    int64_t ks = std::max<int64_t>(1, (4 * (int64_t)sm_count() + tiles - 1) / tiles);
    return (int)std::min<int64_t>(std::min<int64_t>(ks, std::max<int64_t>(1, steps / 4)), 32);
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_keymat_bytes(int64_t block_count, int64_t cols, int32_t bitwidth, int32_t k) {
    const int64_t nkeys = bucket_count(bitwidth, k);
    if (k > 8 || nkeys > 65536) return 0;
    return (size_t)block_count * cols * (nkeys <= 256 ? 1 : 2);
}

rsr_status rsr_keymat_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                            void *keymat, rsr_stream_t stream) {
    const size_t bytes = rsr_keymat_bytes(block_count, cols, bitwidth, k);
    if (!bytes || !keymat || !go || !po) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(keymat, 0, bytes, s);
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells * 32 + 255) / 256, (int64_t)sm_count() * 16);
    if (bucket_count(bitwidth, k) <= 256)
        keymat_kernel<uint8_t><<<grid, 256, 0, s>>>(words, go, perm, po, block_count, tile_count,
                                                    tile_width, bitwidth, cols, (uint8_t *)keymat);
    else
        keymat_kernel<uint16_t><<<grid, 256, 0, s>>>(words, go, perm, po, block_count, tile_count,
                                                     tile_width, bitwidth, cols,
                                                     (uint16_t *)keymat);
    return launch_status();
}

size_t rsr_matmul_tc_workspace_bytes(int64_t m, int64_t n, int32_t k, int64_t block_begin,
                                     int64_t n_blocks, int32_t B) {
    const int ks = tc_ksplit(n_blocks, n);
    if (ks <= 1) return 0;
    const int64_t rows = std::min(n_blocks * k, m - block_begin * k);
    return (size_t)ks * B * rows * 4;
}

rsr_status rsr_matmul_tc(const void *keymat, int64_t m, int64_t n, int32_t bitwidth, int32_t k,
                         int64_t block_begin, int64_t n_blocks, const void *V, int32_t v_dtype,
                         int64_t ldv, int32_t B, float *Y, int64_t ldy, void *workspace,
                         size_t workspace_bytes, rsr_stream_t stream) {
    if (!keymat || !V || !Y || B < 1 || B > 256 || v_dtype != RSR_BF16 || k < 1 || k > 8)
        return RSR_ERR_INVALID;
    const int64_t rows = std::min(n_blocks * k, m - block_begin * k);
    if (ldv < n || ldy < rows || n_blocks < 0) return RSR_ERR_INVALID;
    if (n_blocks == 0) return RSR_OK;
    const int nkeys = (int)bucket_count(bitwidth, k);
    const int ks = tc_ksplit(n_blocks, n);
    const size_t wsb = rsr_matmul_tc_workspace_bytes(m, n, k, block_begin, n_blocks, B);
    if (wsb && (!workspace || workspace_bytes < wsb)) return RSR_ERR_WORKSPACE;
    TcParams p;
    p.km = (const char *)keymat + (size_t)block_begin * n * (nkeys <= 256 ? 1 : 2);
    p.V = V;
    p.ldv = ldv;
    p.Y = Y;
    p.ldy = ldy;
    p.part = (float *)workspace;
    p.m_rows = m;
    p.n = n;
    p.nblk = n_blocks;
    p.blk0 = block_begin;
    p.k = k;
    p.bitwidth = bitwidth;
    p.nkeys = nkeys;
    p.B = B;
    int np = 1;
    while (16 * np < B) np *= 2;
    p.N = 16 * np;
    p.ksplit = ks;
    const size_t smem = tc_smem_bytes(p.N, nkeys);
    if (smem > 200 * 1024) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    dim3 grid((unsigned)((n_blocks + TC_BLOCKS - 1) / TC_BLOCKS), (unsigned)ks);
#define RSR_TC_LAUNCH(KT, NPV)                                                                  \
    {                                                                                          \
        cudaFuncSetAttribute(rsr_tc_kernel<KT, NPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                       \
        rsr_tc_kernel<KT, NPV><<<grid, TC_THREADS, smem, s>>>(p);                              \
    }
#define RSR_TC_NP(KT)                          \
    switch (np) {                              \
        case 1: RSR_TC_LAUNCH(KT, 1) break;    \
        case 2: RSR_TC_LAUNCH(KT, 2) break;    \
        case 4: RSR_TC_LAUNCH(KT, 4) break;    \
        case 8: RSR_TC_LAUNCH(KT, 8) break;    \
        default: RSR_TC_LAUNCH(KT, 16) break;  \
    }
    if (nkeys <= 256) {
        RSR_TC_NP(uint8_t)
    } else {
        RSR_TC_NP(uint16_t)
    }
#undef RSR_TC_NP
#undef RSR_TC_LAUNCH
    if (ks > 1) {
        const int g2 = (int)std::min<int64_t>((rows * B + 255) / 256, 4096);
        tc_finalize_kernel<<<g2, 256, 0, s>>>(p, rows);
    }
    return launch_status();
}

}  // extern "C"
