// rsr_tc.cu -- batched multi-vector multiply on the 5th-generation tensor
// cores: Y[b] = M . V[b] for a batch of
// bf16 vectors (kind::f16, fp32 accumulation) or int8 vectors (kind::i8,
// exact int32 -- optionally dequantized in the epilogue for the batched
// fused path).
//
// RSR's pattern-table step y_blk = T . S_blk (T in {0,+-1}^{k x P}) is a
// dense contraction; with B vectors it is cheaper to apply T before the
// segment sums: every column's pattern key, expanded through T, is one
// column of the block's k rows.  So this path keeps every column's pattern
// key in the reference's 2-bit code form (pattern_key, preproc.py:183-197:
// +1 -> 01, -1 -> 10), one row at a time -- the code matrix, 2 bits per
// matrix entry (16.8 MB at C4) -- and expands it straight into the A operand
// of tcgen05.mma, which reads A from TENSOR MEMORY:
//
//   D[row][b] += A[row][col] * B[b][col],  A = T[:, key(blk, col)] (TMEM),
//                                          B = V (TMA box, shared memory)
//
// Tile: M = 128 rows (TMEM lanes), K = 128 columns per step, N = vectors
// padded to 16 .. 256.  One 576-thread CTA per SM (all 512 TMEM columns),
// warp-specialized:
//   warp 16 (producer)  lanes 0-7 each own a step: one cp.async.bulk of the
//                       step's 128 code rows (4 KB) into a codes ring of up
//                       to 16 slots (freed by the expanders once they have
//                       read them), and the step's B tile as 2-d TMA boxes of
//                       V itself (SWIZZLE_128B K-major; vectors >= B and
//                       columns >= n zero-filled) into a B ring paired with
//                       the TMEM A ring (freed by the MMA's one commit);
//   warps 0-15 (expand) 2 step groups x 2 column halves x 4 TMEM lane
//                       quarters; thread = (row, 64 columns): one 16-byte
//                       code load -> 32 bf16-pair words (shift, mask, IMAD,
//                       2 PRMT per pair) or 16 int8-quad words (mask + PRMT)
//                       -> one tcgen05.st into the row's TMEM lane, in an A
//                       ring of TMEM stages (64 / 32 columns per step);
//   warp 17 (MMA)       one thread waits on the A stage and its B tile,
//                       issues 8 x K16 (bf16) / 4 x K32 (int8) MMAs and one
//                       commit that frees both (a commit costs the pipe ~45
//                       cycles, so one per step, not two).
// The A tile never touches shared memory (round 1 staged it there: 32 KB of
// shared traffic per step and ~22 us at C4 for every B).  Split-K runs
// inside thread-block clusters (below); the tensor pipe's A rate -- ~45
// cycles per M128 x K16 / K32 instruction at N <= 64 -- is the bound
// (profiles/r02_umma_microbench.txt).
//
// Code matrix layout [step][row][u32]: bf16 steps of 128 columns (8 words
// per row), int8 steps of 256 (16 words: the int8 expansion and MMAs are
// half as long per column, so the per-step overheads are paid half as
// often); u32 q holds columns 16q .. 16q + 15 of the step, permuted so the
// expansion needs one shift + mask per pair of words (bf16: tc_code_bit;
// int8: tc_code_bit_i8).  A tile's step is one contiguous run of rows.
#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime)

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "rsr_mv_impl.cuh"

namespace rsr {

constexpr int TC_M = 128;           // tile rows = TMEM lanes
constexpr int TC_K = 128;           // columns per pipeline step (bf16; int8 steps are 2 x TC_K)
constexpr int TC_RB = 32;           // code bytes per (step, row): 128 x 2 bits (int8: 2 x)
constexpr int TC_LMAX = 16;         // load-ring depth (at most)
constexpr int TC_AMAX = 16;         // A-ring depth in TMEM (at most)
constexpr int TC_MAXK = 16;         // rows per block (16-bit pos / neg masks)
constexpr int TC_GROUPS = 2;        // expander step groups (8 warps: 2 column halves x 4 lane quarters)
constexpr int TC_EXP_WARPS = 8 * TC_GROUPS;
constexpr int TC_THREADS = TC_EXP_WARPS * 32 + 64;  // expanders, producer, MMA

__host__ __device__ inline int64_t tc_steps(int64_t n, bool i8 = false) {
    const int ks = i8 ? 2 * TC_K : TC_K;
    return (n + ks - 1) / ks;
}
__host__ __device__ inline int64_t tc_rows_pad(int64_t bc, int k) { return (bc * k + 7) / 8 * 8; }

// bit offset of column c (c % 16 within its u32) in the permuted code word
// of the bf16 path: column pair j at bits 2 (j % 4) of bytes 2 (j / 4) and
// 2 (j / 4) + 1
__device__ __forceinline__ uint32_t tc_code_bit(uint32_t c) {
    const uint32_t j = (c >> 1) & 7;
    return 8 * (2 * (j >> 2) + (c & 1)) + 2 * (j & 3);
}

// ... and of the int8 path: column 4w + i (word w of 4 int8) in nibble
// i + 4 (w / 2) at bit offset 2 (w % 2), so (x >> 2j) & 0x33333333 holds the
// PRMT selectors of words j (low half) and j + 2 (high half)
__device__ __forceinline__ uint32_t tc_code_bit_i8(uint32_t c) {
    const uint32_t w = (c >> 2) & 3, i = c & 3;
    return 4 * (i + 4 * (w >> 1)) + 2 * (w & 1);
}

// ---- code matrix: KM[step][row][q] (see the header) from the artifact's
// groups: each column of a cell's group carries the group's pattern key; row
// r0 + i gets code (pos_i, neg_i)
template <bool I8, bool W2 = false>
__global__ void keymat_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                              const uint16_t *__restrict__ perm, const int64_t *__restrict__ po,
                              int64_t bc, int64_t tc, int64_t tw, int k, int64_t rows_pad,
                              uint32_t *__restrict__ km32) {
    const uint32_t lane = lane_id();
    const int64_t cells = bc * tc;
    for (int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; cell < cells;
         cell += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = cell / bc, b = cell - t * bc;  // reference cells are tile-major
        const int64_t c0 = t * tw, r0 = b * k;
        for (int64_t g = go[cell]; g < go[cell + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu), L = (int64_t)((w >> 16) & 0xFFFFu);
            const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
            const uint16_t *cols = perm + po[cell] + ps;
            for (int64_t j = lane; j < L; j += 32) {
                const int64_t col = c0 + cols[j];
                const uint32_t bit =
                    I8 ? tc_code_bit_i8((uint32_t)col & 15) : tc_code_bit((uint32_t)col & 15);
                uint32_t *dst = I8 || W2
                                    ? km32 + ((col >> 8) * rows_pad + r0) * 16 + ((col & 255) >> 4)
                                    : km32 + ((col >> 7) * rows_pad + r0) * 8 + ((col & 127) >> 4);
                for (int i = 0; i < k; ++i) {
                    const uint32_t code = ((pos >> i) & 1u) | (((neg >> i) & 1u) << 1);
                    if (code) atomicOr(dst + (int64_t)i * (I8 || W2 ? 16 : 8), code << bit);
                }
            }
        }
    }
}

// ---- tcgen05 helpers -------------------------------------------------------------
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // no-swizzle canonical layout; fields in 16-byte units; version 1 (sm_100)
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// D (TMEM) += A (TMEM, K-major: row = lane, 2 bf16 per column) * B (smem)
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     mbar)
                 : "memory");
}

// 2-d tensor TMA (global -> shared, mbarrier complete_tx); out-of-bounds
// elements are zero-filled and still counted in the transaction bytes
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *tm, int c0, int c1,
                                       uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

#ifdef RSR_TC_DBG
__device__ unsigned long long tc_dbg[64 * 8 + 4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long tc_cta_t[1024 * 8];
__device__ long long tc_mma_cyc[64 * 3];
#define TC_CTA_MARK(j) \
    if (threadIdx.x == 0 && blockIdx.x < 1024) tc_cta_t[blockIdx.x * 8 + (j)] = gtime();
#define TC_MARK(cond, idx) \
    if ((cond) && blockIdx.x == 0 && blockIdx.y == 0 && (idx) < 64 * 8 + 4) tc_dbg[idx] = gtime();
#else
#define TC_MARK(cond, idx)
#define TC_CTA_MARK(j)
#endif

struct TcParams {
    // V [B][n] (bf16 / int8) as a 2-d TMA view, 128-byte swizzle: a box of
    // 128 bytes of columns x N vectors is one K-half (bf16) / the whole K of
    // a step's B tile in the canonical K-major SWIZZLE_128B image (vectors
    // >= B, columns >= n zero-filled)
    CUtensorMap tm_v;
    const uint32_t *km;  // code matrix [steps][rows_pad][8]
    float *Y;            // [B][ldy] rows of the view (f32; int32 on the int8 path)
    int64_t ldy;
    // int8 path with the fused dequantization (prefill): out[b][i] =
    // f32(f64(y) * (beta_i / scales[b])), beta_i = row_beta[i] or beta; f32
    // or bf16 (RNE of that f32) -- rsr_dequant_rows' arithmetic
    const double *dq_scales, *dq_row_beta;
    double dq_beta;
    int dq_bf16;
    int64_t n, row0, rows_view, rows_pad;
    int64_t S;           // steps per tile (= tc_steps(n))
    int B, N, ks, ls, as;  // ks: CTAs per tile (cluster size)
    uint32_t recv_off;     // N <= 64: byte offset of the cluster-reduction receive buffer
    uint32_t a_col, tmem_cols;  // TMEM column of A stage 0; columns allocated
    uint32_t tab0, tab1;        // PRMT byte table {00 3F BF 00 | 00 80 80 00}
};

// one output element from its raw accumulator bits (fp32 bits; int32 bits
// on the int8 path, optionally dequantized)
template <bool I8>
__device__ __forceinline__ void tc_store(const TcParams &p, int b, int64_t vrow, uint32_t bits) {
    const int64_t o = (int64_t)b * p.ldy + vrow;
    if (I8 && p.dq_scales) {
        const double beta = p.dq_row_beta ? p.dq_row_beta[vrow] : p.dq_beta;
        const float v = (float)((double)(int32_t)bits * (beta / p.dq_scales[b]));
        if (p.dq_bf16) reinterpret_cast<__nv_bfloat16 *>(p.Y)[o] = __float2bfloat16_rn(v);
        else p.Y[o] = v;
    } else {
        reinterpret_cast<uint32_t *>(p.Y)[o] = bits;
    }
}

// 64 columns' codes of one row (x[q]: columns 16q .. 16q + 15, permuted
// layout) -> 32 words of two bf16 each: per pair of words, sel = ((x >> 2i)
// & 0x03030303) * 0x11 + 0x04040404 holds the PRMT selector nibbles
// (4 + c0, c0, 4 + c1, c1) of word i in its low half and of word i + 4 in
// its high half
__device__ __forceinline__ void expand64(const uint4 &x, uint32_t (&w)[32], uint32_t tab0,
                                         uint32_t tab1, uint32_t c0404) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const uint32_t xv = h == 0 ? x.x : h == 1 ? x.y : h == 2 ? x.z : x.w;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t sel;
            asm("mad.lo.u32 %0, %1, 0x11, %2;" : "=r"(sel) : "r"((xv >> (2 * i)) & 0x03030303u),
                "r"(c0404));
            asm("prmt.b32 %0, %1, %2, %3;" : "=r"(w[8 * h + i]) : "r"(tab0), "r"(tab1), "r"(sel));
            asm("prmt.b32 %0, %1, %2, %3;"
                : "=r"(w[8 * h + i + 4])
                : "r"(tab0), "r"(tab1), "r"(sel >> 16));
        }
    }
}

// 64 columns' codes of one row (int8 layout) -> 16 words of four int8 (+1,
// -1, 0): one mask + one PRMT per word from the byte table {00 01 FF 00}
__device__ __forceinline__ void expand64_i8(const uint4 &x, uint32_t (&w)[16], uint32_t tab) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const uint32_t xv = h == 0 ? x.x : h == 1 ? x.y : h == 2 ? x.z : x.w;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint32_t sel = (xv >> (2 * j)) & 0x33333333u;
            asm("prmt.b32 %0, %1, 0, %2;" : "=r"(w[4 * h + j]) : "r"(tab), "r"(sel));
            asm("prmt.b32 %0, %1, 0, %2;" : "=r"(w[4 * h + j + 2]) : "r"(tab), "r"(sel >> 16));
        }
    }
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&w)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
        "r"(w[15])
        : "memory");
}

__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&w)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
        "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]),
        "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]),
        "r"(w[29]), "r"(w[30]), "r"(w[31])
        : "memory");
}

// N = 16 * NP: MMA N (vectors padded up, <= 256).
// Split-K over thread-block clusters: cluster t (ks CTAs) owns row tile t,
// CTA rank r its steps [r S / ks, (r + 1) S / ks).  Each CTA accumulates in
// TMEM; rank r then owns rows [r 128 / ks, (r + 1) 128 / ks) of the tile and
// sums them over all ranks' accumulators in rank order (deterministic):
// N <= 64 pushes every accumulator row into its owner's receive buffer
// (DSMEM stores, one cluster barrier); larger N parks the accumulator in the
// CTA's idle load ring and the owners read it through DSMEM.  No partials
// in global memory, one launch per call.
template <int NP, bool I8, bool W2 = false>
__global__ void __launch_bounds__(TC_THREADS, 1) rsr_tc_kernel(const __grid_constant__ TcParams p) {
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(8) uint64_t bars[2 * TC_LMAX + 3 * TC_AMAX + 1];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = lane_id();
    constexpr int N = 16 * NP;
    const int LS = p.ls, AS = p.as, ks = p.ks;
    TC_CTA_MARK(0)
    const int64_t t0 = blockIdx.x / ks;
    const int rank = (int)(blockIdx.x - t0 * ks);  // = %cluster_ctarank (1-d clusters)
    const int64_t w0 = t0 * p.S + p.S * rank / ks, w1 = t0 * p.S + p.S * (rank + 1) / ks;
    const int64_t nst = w1 - w0;

    // smem: per load stage [B tile: 2 K-halves x N x 128 B][codes 128 rows x 32 B]
    // int8 steps take 256 columns: the same 256-byte B rows and twice the
    // code bytes, so the per-step overheads are paid half as often
    // W2 (bf16, N <= 32): 256-column steps too -- a 128-column TMEM stage,
    // four 64-column B boxes, 16 MMAs per commit
    constexpr int KS = I8 || W2 ? 2 * TC_K : TC_K;   // columns per step
    constexpr int RB = I8 || W2 ? 2 * TC_RB : TC_RB;  // code bytes per (step, row)
    constexpr uint32_t B_BYTES = (uint32_t)N * KS * (I8 ? 1 : 2);
    constexpr int NBOX = (int)(KS * (I8 ? 1 : 2) / 128);  // 128-byte column boxes per B row
    // TMEM columns per A stage (128 bf16 pairs / 256 int8 quads; W2: 256 bf16)
    constexpr uint32_t ASC = W2 ? 128u : 64u;
    constexpr uint32_t C_BYTES = TC_M * RB;
    // shared memory: the codes ring [LS x 4 KB] (freed by the expanders),
    // then the B ring [AS x B tile] that pairs with the TMEM A ring (one MMA
    // commit frees both), then (N <= 64) the reduction's receive buffer
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tc_smem);
    const uint32_t bbase = sbase + (uint32_t)LS * C_BYTES;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    const uint32_t bar_cfull = bar0, bar_cempty = bar0 + 8 * TC_LMAX;
    const uint32_t bar_bfull = bar0 + 16 * TC_LMAX, bar_aready = bar_bfull + 8 * TC_AMAX;
    const uint32_t bar_free = bar_aready + 8 * TC_AMAX;
    const uint32_t bar_done = bar_free + 8 * TC_AMAX;  // accumulator complete

    if (warp == TC_EXP_WARPS + 1) {  // TMEM: accumulators + the A ring
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base_sh)),
                     "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // barriers, one per thread: codes full / B full (the producer's
    // expect_tx), codes empty and A ready (the 256 threads of an expander
    // group), stage free / done (an MMA commit)
    if (tid < 2 * TC_LMAX + 3 * TC_AMAX + 1) {
        const bool grp = (tid >= TC_LMAX && tid < 2 * TC_LMAX) ||
                         (tid >= 2 * TC_LMAX + TC_AMAX && tid < 2 * TC_LMAX + 2 * TC_AMAX);
        mbar_init(bar0 + 8 * tid, grp ? 8u * 32u : 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_sh;
    TC_MARK(tid == 0, 512)
    TC_CTA_MARK(1)

    if (warp == TC_EXP_WARPS) {
        // ---- producer: lanes 0 .. J-1 load J consecutive steps at once (a
        // lane per step, each its own slot): the step's code rows (bulk
        // copy) and its B tile straight from V (two 2-d TMAs, one per 64
        // columns) ----
        const int J = min(min(LS, AS), 8);
        const unsigned char *kb = reinterpret_cast<const unsigned char *>(p.km);
        if (lane == 0)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tm_v))
                         : "memory");
        // PDL: V may come from the previous kernel; everything before this
        // point overlapped its tail
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if ((int)lane < J) {
            int s = (int)lane, a = (int)lane;
            uint32_t par = 0, apar = 0;
            const int64_t w = w0 + lane;
            int64_t t = w / p.S, st = w - t * p.S;
            for (int64_t it = lane; it < nst; it += J) {
                const int64_t r_first = t * TC_M;
                const uint32_t kbytes =
                    (uint32_t)min((int64_t)TC_M, p.rows_view - r_first) * RB;
                TC_MARK(it < 64, it * 8 + 2)
                // codes: the slot's previous step has been read by its expanders
                if (it >= LS) mbar_wait_parity(bar_cempty + 8 * s, par ^ 1u);
                mbar_expect_tx(bar_cfull + 8 * s, kbytes);
                bulk_g2s(sbase + s * C_BYTES, kb + (st * p.rows_pad + p.row0 + r_first) * RB,
                         kbytes, bar_cfull + 8 * s);
                // B tile: the stage's previous MMAs are complete
                if (it >= AS) mbar_wait_parity(bar_free + 8 * a, apar ^ 1u);
                const uint32_t ba = bbase + a * B_BYTES, fb = bar_bfull + 8 * a;
                mbar_expect_tx(fb, B_BYTES);
                // boxes of 128 bytes of columns (64 bf16 / 128 int8)
#pragma unroll
                for (int j = 0; j < NBOX; ++j)
                    tma_2d(ba + j * (B_BYTES / NBOX), &p.tm_v, (int)st * KS + j * (KS / NBOX), 0,
                           fb);
                s += J;
                if (s >= LS) {
                    s -= LS;
                    par ^= 1u;
                }
                a += J;
                if (a >= AS) {
                    a -= AS;
                    apar ^= 1u;
                }
                st += J;
                while (st >= p.S) {
                    st -= p.S;
                    ++t;
                }
            }
        }
    } else if (warp == TC_EXP_WARPS + 1) {
        // ---- MMA issuer ----
        if (lane == 0) {
            // instruction descriptor: kind::f16, A = B = BF16, D = F32, A and B
            // K-major, N >> 3 at [17,23), M >> 4 at [24,29)
            // (kind::i8: D = S32 (2), A = B = S8 (1))
            const uint32_t idesc = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            // B K-major SWIZZLE_128B (layout type 2 at [61,64)): rows of 128 B,
            // SBO = 8 rows (1024 B); a K = 16 slice starts 32 B further into
            // its 64-column half (the swizzle applies to the absolute address)
            const uint64_t db0 = smem_desc(bbase, 16, 1024) | ((uint64_t)2 << 61);
            int a = 0;
            uint32_t apar = 0;
#ifdef RSR_TC_DBG
            long long c_prev = 0;
#endif
            for (int64_t it = 0; it < nst; ++it) {
                const bool first = it == 0;
#ifdef RSR_TC_DBG
                const long long c0 = clock64();
                const long long c1 = c0;
                const long long dstep = it ? c0 - c_prev : 0;
                c_prev = c0;
#endif
                // A stage expanded, B tile landed
                mbar_wait_parity(bar_aready + 8 * a, apar);
                mbar_wait_parity(bar_bfull + 8 * a, apar);
#ifdef RSR_TC_DBG
                const long long c2 = clock64();
#endif
                TC_MARK(it < 64, it * 8 + 3)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t db = db0 + ((a * B_BYTES) >> 4);
                const uint32_t ta = tmem_d + p.a_col + ASC * a;
                const uint32_t td = tmem_d;
                if (I8) {
                    // K = 32 int8 per MMA: 32 B into a half's 128-byte swizzled rows
#pragma unroll
                    for (int kk = 0; kk < KS / 32; ++kk)
                        mma_i8_ts(td, ta + 8u * kk,
                                  db + (uint64_t)(((kk >> 2) * (B_BYTES / 2) + (kk & 3) * 32) >> 4),
                                  idesc, (!first || kk > 0) ? 1u : 0u);
                } else {
#pragma unroll
                    for (int kk = 0; kk < KS / 16; ++kk)
                        mma_bf16_ts(
                            td, ta + 8u * kk,
                            db + (uint64_t)(((kk >> 2) * (B_BYTES / NBOX) + (kk & 3) * 32) >> 4),
                            idesc, (!first || kk > 0) ? 1u : 0u);
                }
                // one commit frees the A stage and its B tile
                mma_commit(bar_free + 8 * a);
                if (it + 1 == nst) mma_commit(bar_done);
#ifdef RSR_TC_DBG
                if (blockIdx.x == 0 && it < 64) {
                    const long long c3 = clock64();
                    tc_mma_cyc[it * 3 + 0] = dstep + (c1 - c0);
                    tc_mma_cyc[it * 3 + 1] = c2 - c1;
                    tc_mma_cyc[it * 3 + 2] = c3 - c2;
                }
#endif
                if (++a == AS) {
                    a = 0;
                    apar ^= 1u;
                }
            }
        }
    } else {
        // ---- expanders: thread = (tile row 32 (warp % 4) + lane, column half
        // (warp / 4) % 2); a warp's TMEM lanes are its quarter, warp % 4.
        // Group h = warp / 8 expands the steps it = h (mod TC_GROUPS) ----
        const int q = warp & 3, hh = (warp >> 2) & 1, h = warp >> 3;
        const int row = 32 * q + (int)lane;
        const uint32_t t_row = tmem_d + ((uint32_t)(32 * q) << 16) + p.a_col + (ASC / 2) * hh;
        // table words and the selector bias in plain registers, set once
        const uint32_t tab0 = __shfl_sync(RSR_FULL_MASK, p.tab0, 0);
        const uint32_t tab1 = __shfl_sync(RSR_FULL_MASK, p.tab1, 0);
        const uint32_t c0404 = __shfl_sync(RSR_FULL_MASK, 0x04040404u, 0);
        const unsigned char *codes0 = tc_smem + row * RB + hh * (RB / 2);
        // this warp's steps it = h, h + TC_GROUPS, ...: load slot it % LS, A stage it % AS
        int s = h % LS, a = h % AS;
        uint32_t par = (uint32_t)(h / LS) & 1u, apar = (uint32_t)(h / AS) & 1u;
        for (int64_t it = h; it < nst; it += TC_GROUPS) {
            mbar_wait_parity(bar_cfull + 8 * s, par);
            TC_MARK(tid == 0 && it < 64, it * 8 + 0)
            const uint4 x = *reinterpret_cast<const uint4 *>(codes0 + s * C_BYTES);
            uint4 x2 = make_uint4(0, 0, 0, 0);
            if (I8 || W2) x2 = *reinterpret_cast<const uint4 *>(codes0 + s * C_BYTES + 16);
            mbar_arrive(bar_cempty + 8 * s);  // (release: the loads are ordered before)
            if (I8) {
                // 128 columns: two code words -> 32 int8-quad words
                uint32_t w[32];
                expand64_i8(x, *reinterpret_cast<uint32_t(*)[16]>(&w[0]), tab0);
                expand64_i8(x2, *reinterpret_cast<uint32_t(*)[16]>(&w[16]), tab0);
                if (it >= AS) mbar_wait_parity(bar_free + 8 * a, apar ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                tmem_st32(t_row + ASC * a, w);
            } else {
                uint32_t w[32];
                expand64(x, w, tab0, tab1, c0404);
                TC_MARK(tid == 0 && it < 64, it * 8 + 4)
                if (it >= AS) mbar_wait_parity(bar_free + 8 * a, apar ^ 1u);
                TC_MARK(tid == 0 && it < 64, it * 8 + 5)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                tmem_st32(t_row + ASC * a, w);
                if (W2) {  // the half's second 64 columns
                    expand64(x2, w, tab0, tab1, c0404);
                    tmem_st32(t_row + ASC * a + 32u, w);
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            TC_MARK(tid == 0 && it < 64, it * 8 + 6)
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(bar_aready + 8 * a);
            TC_MARK(tid == 0 && it < 64, it * 8 + 1)
            // advance TC_GROUPS steps (LS, AS >= TC_GROUPS)
            s += TC_GROUPS;
            if (s >= LS) {
                s -= LS;
                par ^= 1u;
            }
            a += TC_GROUPS;
            if (a >= AS) {
                a -= AS;
                apar ^= 1u;
            }
        }
    }
    __syncwarp();
    TC_MARK(tid == 0, 513)
    TC_CTA_MARK(2)

    // --- epilogue: warps 0-3 read the accumulator (warp w: TMEM lanes
    // 32w .. 32w + 31 = tile rows), 8 columns at a time; alone in its
    // cluster a CTA writes Y, otherwise it parks the accumulator in its own
    // (now idle) load ring as acc[column][row] for the cluster reduction
    const int64_t r_first = t0 * TC_M;
    float *acc_sm = reinterpret_cast<float *>(tc_smem);
    // N <= 64: push mode -- each rank stores its accumulator straight into
    // the owning rank's receive buffer recv[rank][b][row - owner's first row]
    // (DSMEM stores, no round trip), one cluster barrier, local sums
    constexpr bool PUSH = N <= 64;
    const int RM = (TC_M + ks - 1) / ks;  // rows per rank slot
    if (warp < 4) {
        const int row_t = warp * 32 + (int)lane;
        const int64_t vrow = r_first + row_t;
        const bool valid = vrow < p.rows_view;
        const int owner = ((row_t + 1) * ks - 1) / TC_M;
        const int orow = row_t - owner * TC_M / ks;
        uint32_t owin = 0;
        if (PUSH && ks > 1)
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(owin)
                         : "r"((uint32_t)__cvta_generic_to_shared(tc_smem) + p.recv_off),
                           "r"(owner));
        mbar_wait_parity(bar_done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // 16 accumulator columns per TMEM load (one wait each)
        for (int c = 0; c < N; c += 16) {
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
                "%10, %11, %12, %13, %14, %15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                  "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (ks == 1) {
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c + j < p.B)
                            tc_store<I8>(p, c + j, vrow, r[j]);
                }
            } else if (PUSH) {
                const uint32_t dst = owin + (uint32_t)(((rank * p.B + c) * RM + orow) * 4);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c + j < p.B)
                        asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(
                                         dst + (uint32_t)(j * RM * 4)),
                                     "r"(r[j])
                                     : "memory");
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    reinterpret_cast<uint32_t *>(acc_sm)[(c + j) * TC_M + row_t] = r[j];
            }
        }
    }
    TC_CTA_MARK(4)
    if (PUSH && ks > 1) {
        // every rank's pushes are in (release / acquire): sum this rank's rows
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        TC_CTA_MARK(5)
        const int rbase = rank * TC_M / ks, rows = (rank + 1) * TC_M / ks - rbase;
        const uint32_t *recv = reinterpret_cast<const uint32_t *>(tc_smem + p.recv_off);
        // 32-bit outputs with 16-byte aligned rows: a thread takes four
        // consecutive rows (one 16-byte shared load per rank, one 16-byte
        // store); otherwise one row
        const bool vec4 = !(I8 && p.dq_scales) && (rows & 3) == 0 && (rbase & 3) == 0 &&
                          (p.ldy & 3) == 0 && (reinterpret_cast<uintptr_t>(p.Y) & 15) == 0 &&
                          (RM & 3) == 0;
        if (vec4) {
            const int r4 = rows >> 2, bstep = TC_THREADS / r4, rq = tid % r4, b0 = tid / r4;
            const int64_t vrow = r_first + rbase + 4 * rq;
            if (b0 < bstep)
                for (int b = b0; b < p.B; b += bstep) {
                    uint4 acc = *reinterpret_cast<const uint4 *>(recv + b * RM + 4 * rq);
                    for (int q = 1; q < ks; ++q) {
                        const uint4 x =
                            *reinterpret_cast<const uint4 *>(recv + (q * p.B + b) * RM + 4 * rq);
                        if (I8) {
                            acc.x += x.x, acc.y += x.y, acc.z += x.z, acc.w += x.w;
                        } else {
                            acc.x = __float_as_uint(__uint_as_float(acc.x) + __uint_as_float(x.x));
                            acc.y = __float_as_uint(__uint_as_float(acc.y) + __uint_as_float(x.y));
                            acc.z = __float_as_uint(__uint_as_float(acc.z) + __uint_as_float(x.z));
                            acc.w = __float_as_uint(__uint_as_float(acc.w) + __uint_as_float(x.w));
                        }
                    }
                    uint32_t *yo = reinterpret_cast<uint32_t *>(p.Y) + (int64_t)b * p.ldy + vrow;
                    if (vrow + 3 < p.rows_view) {
                        *reinterpret_cast<uint4 *>(yo) = acc;
                    } else {
                        const uint32_t v4[4] = {acc.x, acc.y, acc.z, acc.w};
                        for (int j = 0; j < 4 && vrow + j < p.rows_view; ++j) yo[j] = v4[j];
                    }
                }
        } else {
        // thread = (row rr, vectors b0, b0 + bstep, ...): no divisions in the
        // loop, consecutive threads on consecutive rows (coalesced Y stores)
        const int bstep = TC_THREADS / rows, rr = tid % rows, b0 = tid / rows;
        if (b0 < bstep)
#pragma unroll 4
        for (int b = b0; b < p.B; b += bstep) {
            uint32_t sum;
            if (I8) {
                sum = 0u;
                for (int q = 0; q < ks; ++q) sum += recv[(q * p.B + b) * RM + rr];
            } else {
                float f = __uint_as_float(recv[b * RM + rr]);
                for (int q = 1; q < ks; ++q) f += __uint_as_float(recv[(q * p.B + b) * RM + rr]);
                sum = __float_as_uint(f);
            }
            const int64_t vrow = r_first + rbase + rr;
            if (vrow < p.rows_view) tc_store<I8>(p, b, vrow, sum);
        }
        }
        TC_CTA_MARK(6)
    } else if (ks > 1) {
        // every rank's accumulator is in its shared memory -> each rank sums
        // rows [rank 128 / ks, (rank + 1) 128 / ks) over ranks 0 .. ks-1
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        TC_CTA_MARK(5)
        const int rbase = rank * TC_M / ks, rows = (rank + 1) * TC_M / ks - rbase;
        const uint32_t own = (uint32_t)__cvta_generic_to_shared(acc_sm);
        // the ranks' shared-memory windows (same offsets in every CTA)
        uint32_t win[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(win[q]) : "r"(own),
                         "r"(q < ks ? q : 0));
        for (int e = tid; e < p.B * rows; e += TC_THREADS) {
            const int b = e / rows, rt = rbase + (e - b * rows);
            const uint32_t off = (uint32_t)((b * TC_M + rt) * 4);
            // every rank's value loaded before any is summed (fp32 in rank
            // order; int32 for the int8 path, exact)
            uint32_t x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                x[q] = 0u;
                if (q < ks)
                    asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(x[q]) : "r"(win[q] + off)
                                 : "memory");
            }
            uint32_t sum;
            if (I8) {
                sum = x[0];
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    if (q < ks) sum += x[q];
            } else {
                float f = __uint_as_float(x[0]);
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    if (q < ks) f += __uint_as_float(x[q]);
                sum = __float_as_uint(f);
            }
            const int64_t vrow = r_first + rt;
            if (vrow < p.rows_view) tc_store<I8>(p, b, vrow, sum);
        }
        TC_CTA_MARK(6)
        // no rank leaves (freeing its shared memory) before all have read it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        TC_CTA_MARK(7)
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    TC_MARK(tid == 0, 514)
    TC_CTA_MARK(3)
    if (warp == TC_EXP_WARPS + 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                     "r"(p.tmem_cols));
}

static int tc_np(int B) {
    int np = 1;
    while (16 * np < B) np *= 2;
    return np;
}

// N <= 64: the cluster reduction's receive buffer after the rings, sized
// for any ks <= 8 (ks x B x ceil(128 / ks) words <= N x 135)
static size_t tc_recv_bytes(int N) { return N <= 64 ? (size_t)N * (TC_M + 7) * 4 : 0; }

struct TcRings {
    int ls, as;  // codes-ring depth (4 KB slots), A / B-ring depth (TMEM stage + B tile)
    size_t smem;
};

// Ring depths within 216 KB of shared memory and the TMEM left after the
// accumulator: the A / B ring as deep as both allow (at most TC_AMAX), the
// codes ring with the rest (at most TC_LMAX); both at least TC_GROUPS.
static TcRings tc_rings(int N, bool i8, bool w2 = false) {
    const size_t bbytes = (size_t)N * TC_K * 2 * (w2 ? 2 : 1);
    const size_t cbytes = (size_t)TC_M * TC_RB * (i8 || w2 ? 2 : 1);
    const size_t budget = 216 * 1024 - tc_recv_bytes(N);
    const int a_col = std::max(N, 64), asc = w2 ? 128 : 64;
    TcRings r;
    r.as = std::min<int>(TC_AMAX, (512 - a_col) / asc);
    r.as = std::max<int>(TC_GROUPS,
                         std::min<int>(r.as, (int)((budget - TC_GROUPS * cbytes) / bbytes)));
    r.ls = (int)std::max<size_t>(TC_GROUPS,
                                 std::min<size_t>(TC_LMAX, (budget - r.as * bbytes) / cbytes));
    r.smem = r.ls * cbytes + r.as * bbytes + tc_recv_bytes(N);
    return r;
}

static int64_t tc_view_rows(int64_t block_begin, int64_t n_blocks, int32_t k, int64_t m) {
    return std::max<int64_t>(0, std::min((block_begin + n_blocks) * k, m) - block_begin * k);
}

// cluster-size choice per (device, N, tiles, steps, smem): the occupancy
// query is a host round trip worth skipping on repeated shapes
struct TcKsKey {
    int dev, np;
    int64_t tiles, S;
    size_t smem;
    bool operator<(const TcKsKey &o) const {
        return std::tie(dev, np, tiles, S, smem) < std::tie(o.dev, o.np, o.tiles, o.S, o.smem);
    }
};
static std::mutex tc_ks_mu;
static std::map<TcKsKey, int> tc_ks_map;

static TcKsKey tc_ks_key(int np, int64_t tiles, int64_t S, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    return TcKsKey{dev, np, tiles, S, smem};
}

static int tc_ks_cached(int np, int64_t tiles, int64_t S, size_t smem) {
    const TcKsKey key = tc_ks_key(np, tiles, S, smem);
    std::lock_guard<std::mutex> g(tc_ks_mu);
    auto it = tc_ks_map.find(key);
    return it == tc_ks_map.end() ? 0 : it->second;
}

static void tc_ks_store(int np, int64_t tiles, int64_t S, size_t smem, int ks) {
    const TcKsKey key = tc_ks_key(np, tiles, S, smem);
    std::lock_guard<std::mutex> g(tc_ks_mu);
    tc_ks_map[key] = ks;
}

}  // namespace rsr

using namespace rsr;

extern "C" {

#ifdef RSR_TC_DBG
int rsr_tc_debug_mma(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, tc_mma_cyc, sizeof(long long) * 64 * 3);
}
int rsr_tc_debug_ctas(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, tc_cta_t, sizeof(unsigned long long) * 1024 * 8);
}
int rsr_tc_debug(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, tc_dbg, sizeof(unsigned long long) * (64 * 8 + 4));
}
#endif

size_t rsr_keymat_bytes(int64_t block_count, int64_t cols, int32_t bitwidth, int32_t k) {
    (void)bitwidth;
    if (k < 1 || k > TC_MAXK || block_count < 0 || cols < 0) return 0;
    // sized for the int8 layout (256-column steps), which the bf16 one
    // (128-column steps) never exceeds
    return (size_t)tc_steps(cols, true) * tc_rows_pad(block_count, k) * (2 * TC_RB);
}

}  // extern "C"

template <bool I8, bool W2 = false>
static rsr_status keymat_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                               const int64_t *po, int64_t block_count, int64_t tile_count,
                               int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                               void *keymat, rsr_stream_t stream) {
    const size_t bytes = rsr_keymat_bytes(block_count, cols, bitwidth, k);
    if (!bytes || !keymat || !go || !po || (reinterpret_cast<uintptr_t>(keymat) & 15))
        return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(keymat, 0, bytes, s);
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells * 32 + 255) / 256, (int64_t)sm_count() * 16);
    keymat_kernel<I8, W2><<<grid, 256, 0, s>>>(words, go, perm, po, block_count, tile_count,
                                           tile_width, k, tc_rows_pad(block_count, k),
                                           (uint32_t *)keymat);
    return launch_status();
}

extern "C" {

rsr_status rsr_keymat_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                            void *keymat, rsr_stream_t stream) {
    return keymat_build<false>(words, go, perm, po, block_count, tile_count, tile_width, cols,
                               bitwidth, k, keymat, stream);
}

rsr_status rsr_keymat_build_wide(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                                 const int64_t *po, int64_t block_count, int64_t tile_count,
                                 int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                                 void *keymat, rsr_stream_t stream) {
    return keymat_build<false, true>(words, go, perm, po, block_count, tile_count, tile_width,
                                     cols, bitwidth, k, keymat, stream);
}

rsr_status rsr_keymat_build_i8(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                               const int64_t *po, int64_t block_count, int64_t tile_count,
                               int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                               void *keymat, rsr_stream_t stream) {
    return keymat_build<true>(words, go, perm, po, block_count, tile_count, tile_width, cols,
                              bitwidth, k, keymat, stream);
}

}  // extern "C"

typedef CUresult (*TcEncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// V [B][n] (bf16 or int8) rows of pitch ldv elements -> the 2-d
// SWIZZLE_128B view, box (128 bytes of columns) x N vectors
static bool tc_encode_v(CUtensorMap *tm, const void *V, int64_t n, int B, int64_t ldv, int N,
                        bool i8) {
    static TcEncodeTiled enc = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (TcEncodeTiled)f;
    }();
    const int esize = i8 ? 1 : 2;
    if (!enc || (reinterpret_cast<uintptr_t>(V) & 15) || ((ldv * esize) & 15)) return false;
    const cuuint64_t gdim[2] = {(cuuint64_t)n, (cuuint64_t)B};
    const cuuint64_t gstride[1] = {(cuuint64_t)ldv * esize};
    const cuuint32_t box[2] = {(cuuint32_t)(128 / esize), (cuuint32_t)N};
    const cuuint32_t estr[2] = {1, 1};
    return enc(tm, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
               const_cast<void *>(V), gdim, gstride, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

extern "C" {

// workspace: not used by this path (kept in the signature for ABI
// stability; 256 bytes)
size_t rsr_matmul_tc_workspace_bytes(int64_t m, int64_t n, int32_t k, int64_t block_begin,
                                     int64_t n_blocks, int32_t B) {
    (void)m, (void)n, (void)block_begin;
    if (B < 1 || B > 256 || k < 1 || k > TC_MAXK || n_blocks < 0) return 0;
    return 256;
}

}  // extern "C"

template <bool I8, bool W2 = false>
static rsr_status tc_launch(const void *keymat, int64_t m, int64_t n, int32_t k,
                            int64_t block_begin, int64_t n_blocks, const void *V, int64_t ldv,
                            int32_t B, void *Y, int64_t ldy, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream,
                            const double *dq_scales = nullptr, const double *dq_row_beta = nullptr,
                            double dq_beta = 1.0, int dq_bf16 = 0) {
    if (!keymat || !V || !Y || B < 1 || B > 256 || k < 1 || k > TC_MAXK) return RSR_ERR_INVALID;
    if (n_blocks < 0 || block_begin < 0) return RSR_ERR_INVALID;
    const int64_t bc = (m + k - 1) / k;
    if (block_begin + n_blocks > bc) return RSR_ERR_INVALID;
    const int64_t rows = tc_view_rows(block_begin, n_blocks, k, m);
    if (ldv < n || ldy < rows) return RSR_ERR_INVALID;
    if (rows == 0) return RSR_OK;
    if (reinterpret_cast<uintptr_t>(keymat) & 15) return RSR_ERR_INVALID;
    const int64_t tiles = (rows + TC_M - 1) / TC_M;
    const size_t wsb = rsr_matmul_tc_workspace_bytes(m, n, k, block_begin, n_blocks, B);
    if (!workspace || workspace_bytes < wsb || (reinterpret_cast<uintptr_t>(workspace) & 255))
        return RSR_ERR_WORKSPACE;
    const int np = tc_np(B);
    // the wide steps serve N <= 32 (at N = 64 the 3-deep A ring they leave
    // costs what the halved per-step overheads save)
    if (W2 && np > 2) return RSR_ERR_INVALID;
    TcParams p;
    p.km = (const uint32_t *)keymat;
    if (!tc_encode_v(&p.tm_v, V, n, B, ldv, 16 * np, I8)) return RSR_ERR_INVALID;
    p.Y = (float *)Y;
    p.ldy = ldy;
    p.dq_scales = dq_scales;
    p.dq_row_beta = dq_row_beta;
    p.dq_beta = dq_beta;
    p.dq_bf16 = dq_bf16;
    p.n = n;
    p.row0 = block_begin * k;
    p.rows_view = rows;
    p.rows_pad = tc_rows_pad(bc, k);
    p.B = B;
    p.N = 16 * np;
    p.S = tc_steps(n, I8 || W2);
    // TMEM (all 512 columns): the accumulator [0, N) (64-column aligned),
    // then the A ring: one step's 128 K elements per stage (64 columns of
    // bf16 pairs, 32 of int8 quads)
    const TcRings rings = tc_rings(p.N, I8, W2);
    p.ls = rings.ls;
    p.as = rings.as;
    p.recv_off = (uint32_t)(rings.smem - tc_recv_bytes(p.N));
    p.a_col = (uint32_t)std::max(p.N, 64);
    p.tmem_cols = 512;
    {
        static const int forced_as = [] {
            const char *e = getenv("RSR_TC_ASTAGES");
            return e ? atoi(e) : 0;
        }();
        if (forced_as >= TC_GROUPS) p.as = std::min(forced_as, p.as);
    }
    // PRMT byte tables: bf16 {00 3F BF 00 | 00 80 80 00}; int8 {00 01 FF 00}
    p.tab0 = I8 ? 0x00FF0100u : 0x00BF3F00u;
    p.tab1 = 0x00808000u;
    // exactly one CTA per SM: each allocates all 512 TMEM columns, and a
    // second resident CTA would block in tcgen05.alloc while its cluster
    // partners wait for it at the cluster barrier.  Shared memory above half
    // the SM's 228 KB guarantees it (registers alone would not for small
    // int8 batches).
    const size_t smem = std::max<size_t>(rings.smem, 116 * 1024);
    if (smem > 227 * 1024) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    // programmatic dependent launch (PDL): the prologue overlaps the previous
    // kernel's tail; clusters of ks CTAs split each tile's steps
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[0].val.programmaticStreamSerializationAllowed = 1;
    attrs[1].id = cudaLaunchAttributeClusterDimension;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    // CTAs per tile: the largest ks <= 8 (and <= S) whose tiles x ks CTAs fit
    // one wave, one per SM, with that many clusters co-resident
    static const int forced_ks = [] {
        const char *e = getenv("RSR_TC_KSPLIT");
        return e ? atoi(e) : 0;
    }();
    const int key_np = np + (I8 ? 1000 : 0) + (W2 ? 2000 : 0);
#define RSR_TC_LAUNCH(NPV)                                                                      \
    {                                                                                          \
        auto kern = rsr_tc_kernel<NPV, I8, W2>;                                                    \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
        int ks = tc_ks_cached(key_np, tiles, p.S, smem);                                       \
        if (ks == 0) { /* first launch of this shape: one CTA per SM, checked once */          \
            int per_sm = 0;                                                                    \
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TC_THREADS,       \
                                                              smem) != cudaSuccess ||          \
                per_sm != 1)                                                                   \
                return RSR_ERR_INVALID;                                                        \
        }                                                                                      \
        for (int c = 8; ks == 0 && c >= 2; --c) {                                              \
            if (forced_ks > 0 ? c != forced_ks : (c > p.S || tiles * c > sm_count())) continue; \
            attrs[1].val.clusterDim.x = c;                                                     \
            attrs[1].val.clusterDim.y = attrs[1].val.clusterDim.z = 1;                         \
            cfg.gridDim = dim3((unsigned)(tiles * c));                                         \
            int nc = 0;                                                                        \
            if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess &&              \
                (nc >= tiles || forced_ks > 0)) {                                               \
                ks = c;                                                                        \
                break;                                                                         \
            }                                                                                  \
            cudaGetLastError();                                                                \
        }                                                                                      \
        if (ks == 0) ks = 1;                                                                   \
        tc_ks_store(key_np, tiles, p.S, smem, ks);                                             \
        p.ks = ks;                                                                             \
        attrs[1].val.clusterDim.x = ks;                                                        \
        attrs[1].val.clusterDim.y = attrs[1].val.clusterDim.z = 1;                             \
        cfg.gridDim = dim3((unsigned)(tiles * ks));                                            \
        cudaLaunchKernelEx(&cfg, kern, p);                                                     \
    }
    if constexpr (W2) {
        if (np == 1) RSR_TC_LAUNCH(1) else RSR_TC_LAUNCH(2)
    } else {
        switch (np) {
            case 1: RSR_TC_LAUNCH(1) break;
            case 2: RSR_TC_LAUNCH(2) break;
            case 4: RSR_TC_LAUNCH(4) break;
            case 8: RSR_TC_LAUNCH(8) break;
            default: RSR_TC_LAUNCH(16) break;
        }
    }
#undef RSR_TC_LAUNCH
    return launch_status();
}

extern "C" {

rsr_status rsr_matmul_tc(const void *keymat, int64_t m, int64_t n, int32_t bitwidth, int32_t k,
                         int64_t block_begin, int64_t n_blocks, const void *V, int32_t v_dtype,
                         int64_t ldv, int32_t B, float *Y, int64_t ldy, void *workspace,
                         size_t workspace_bytes, rsr_stream_t stream) {
    (void)bitwidth;
    if (v_dtype != RSR_BF16) return RSR_ERR_INVALID;
    return tc_launch<false>(keymat, m, n, k, block_begin, n_blocks, V, ldv, B, Y, ldy, workspace,
                            workspace_bytes, stream);
}

// bf16 batches of B <= 32 over the wide code matrix (rsr_keymat_build_wide):
// 256-column steps, half the per-step commits and barriers
rsr_status rsr_matmul_tc_wide(const void *keymat_wide, int64_t m, int64_t n, int32_t bitwidth,
                              int32_t k, int64_t block_begin, int64_t n_blocks, const void *V,
                              int32_t v_dtype, int64_t ldv, int32_t B, float *Y, int64_t ldy,
                              void *workspace, size_t workspace_bytes, rsr_stream_t stream) {
    (void)bitwidth;
    if (v_dtype != RSR_BF16 || B > 32) return RSR_ERR_INVALID;
    return tc_launch<false, true>(keymat_wide, m, n, k, block_begin, n_blocks, V, ldv, B, Y, ldy,
                                  workspace, workspace_bytes, stream);
}

rsr_status rsr_matmul_tc_i8(const void *keymat_i8, int64_t m, int64_t n, int32_t bitwidth,
                            int32_t k, int64_t block_begin, int64_t n_blocks, const int8_t *V,
                            int64_t ldv, int32_t B, int32_t *Y, int64_t ldy, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream) {
    (void)bitwidth;
    return tc_launch<true>(keymat_i8, m, n, k, block_begin, n_blocks, V, ldv, B, Y, ldy,
                           workspace, workspace_bytes, stream);
}

rsr_status rsr_matmul_tc_i8_dequant(const void *keymat_i8, int64_t m, int64_t n,
                                    int32_t bitwidth, int32_t k, int64_t block_begin,
                                    int64_t n_blocks, const int8_t *Q, int64_t ldq, int32_t B,
                                    const double *scales, const double *row_beta, double beta,
                                    void *out, int32_t out_dtype, int64_t ldo, void *workspace,
                                    size_t workspace_bytes, rsr_stream_t stream) {
    (void)bitwidth;
    if (!scales || (out_dtype != RSR_F32 && out_dtype != RSR_BF16)) return RSR_ERR_INVALID;
    return tc_launch<true>(keymat_i8, m, n, k, block_begin, n_blocks, Q, ldq, B, out, ldo,
                           workspace, workspace_bytes, stream, scales, row_beta, beta,
                           out_dtype == RSR_BF16);
}

}  // extern "C"
