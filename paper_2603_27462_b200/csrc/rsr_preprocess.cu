// rsr_preprocess.cu -- GPU offline preprocessing, bit-exact with the reference.
//
// Replaces the per-cell counting sort of the reference
// (pkg/src/rsrmv/_native.py:25-161, driven by preproc.py:239-289).  One warp
// owns one (tile, block) cell:
//   1. pattern keys of the cell's columns (binary: 2^i weights; ternary:
//      base-3 digits, whose order equals the reference's 4^h code-key order),
//   2. a histogram in a warp-private table (shared memory, or global scratch
//      for the 3^9 / 3^10 / 2^13.. pattern spaces),
//   3. an ascending-key exclusive scan over the non-zero keys that emits the
//      group words in key order (ballot compaction),
//   4. a STABLE scatter of column ids: columns are visited in ascending order
//      32 at a time; __match_any_sync ranks equal keys inside the chunk and
//      the chunk leader advances the bucket cursor, so columns of one group
//      land in ascending order exactly as the serial counting sort puts them.
// Two launches (count, fill) bracket an int64 scan so outputs are sized
// exactly; the stream-layout builder for the multiply kernels lives here too.

#include "rsr_common.cuh"
#include "rsr_stream_layout.cuh"

namespace rsr {

constexpr int PP_WARPS = 8;                    // warps (cells in flight) per CTA
constexpr int64_t PP_SMEM_TABLE_MAX = 6144;    // buckets per warp kept in smem

// Pattern key of tile-local column j of the block starting at row r0.
// Ternary keys are base-3 (digit = 2-bit code); *bad is set on code 3.
__device__ __forceinline__ uint32_t column_key(const uint8_t *__restrict__ data,
                                               int64_t row_bytes, int64_t r0, int h,
                                               int64_t c, int bitwidth, bool *bad) {
    uint32_t key = 0;
    if (bitwidth == RSR_BINARY) {
        const uint8_t *p = data + r0 * row_bytes + (c >> 3);
        const int sh = (int)(c & 7);
        for (int i = 0; i < h; ++i) key |= (uint32_t)((__ldg(p + i * row_bytes) >> sh) & 1u) << i;
    } else {
        const uint8_t *p = data + r0 * row_bytes + (c >> 2);
        const int sh = (int)((c & 3) << 1);
        uint32_t w = 1;
        for (int i = 0; i < h; ++i) {
            uint32_t code = (__ldg(p + i * row_bytes) >> sh) & 3u;
            if (code == 3u) *bad = true;
            key += code * w;
            w *= 3u;
        }
    }
    return key;
}

// pos | neg<<16 of a pattern key (binary: key itself).
__device__ __forceinline__ uint32_t key_masks(uint32_t key, int bitwidth, int h) {
    if (bitwidth == RSR_BINARY) return key;
    uint32_t pos = 0, neg = 0;
    for (int i = 0; i < h; ++i) {
        uint32_t q = key / 3u, d = key - 3u * q;
        key = q;
        if (d == 1u) pos |= 1u << i;
        else if (d == 2u) neg |= 1u << i;
    }
    return pos | (neg << 16);
}

struct CellGeom {
    int64_t r0, c0, tn;
    int h;
};

__device__ __forceinline__ CellGeom cell_geom(int64_t cell, int64_t rows, int64_t cols, int k,
                                              int64_t tw, int64_t bc) {
    CellGeom g;
    const int64_t t = cell / bc, b = cell - t * bc;
    g.r0 = b * k;
    g.h = (int)min((int64_t)k, rows - g.r0);
    g.c0 = t * tw;
    g.tn = min(tw, cols - g.c0);
    return g;
}

__device__ __forceinline__ uint32_t *warp_table(uint32_t *smem_tab, uint32_t *gmem_tab,
                                                int64_t bk, int warp_in_cta) {
    if (smem_tab) return smem_tab + (int64_t)warp_in_cta * bk;
    const int64_t gw = (int64_t)blockIdx.x * PP_WARPS + warp_in_cta;
    return gmem_tab + gw * bk;
}

// Histogram of one cell into tab[0..B) (tab zeroed here first).
__device__ __forceinline__ void cell_histogram(const uint8_t *data, int64_t row_bytes,
                                               const CellGeom &g, int bitwidth, int64_t B,
                                               uint32_t *tab, uint32_t lane, bool *bad) {
    for (int64_t d = lane; d < B; d += 32) tab[d] = 0u;
    __syncwarp();
    for (int64_t j = lane; j < g.tn; j += 32) {
        uint32_t key = column_key(data, row_bytes, g.r0, g.h, g.c0 + j, bitwidth, bad);
        atomicAdd(tab + key, 1u);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(PP_WARPS * 32)
group_count_kernel(const uint8_t *__restrict__ data, int64_t rows, int64_t cols,
                   int64_t row_bytes, int bitwidth, int k, int64_t tw, int64_t bc,
                   int64_t cells, int64_t bk, uint32_t *gmem_tab, int64_t *go, int64_t *po,
                   int64_t *steps, int32_t *status) {
    extern __shared__ uint32_t pp_smem[];
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    uint32_t *tab = warp_table(gmem_tab ? nullptr : pp_smem, gmem_tab, bk, warp);
    for (int64_t cell = (int64_t)blockIdx.x * PP_WARPS + warp; cell < cells;
         cell += (int64_t)gridDim.x * PP_WARPS) {
        const CellGeom g = cell_geom(cell, rows, cols, k, tw, bc);
        const int64_t B = bucket_count(bitwidth, g.h);
        bool bad = false;
        cell_histogram(data, row_bytes, g, bitwidth, B, tab, lane, &bad);
        uint32_t ng = 0, over = 0;
        for (int64_t d = 1 + lane; d < B; d += 32) {
            const uint32_t c = tab[d];
            ng += c > 0u;
            over |= c > 0xFFFFu;
        }
        ng = warp_sum(ng);
        over = __any_sync(RSR_FULL_MASK, over != 0u);
        const bool anybad = __any_sync(RSR_FULL_MASK, bad);
        if (lane == 0) {
            const int64_t nret = g.tn - (int64_t)tab[0];
            go[cell + 1] = ng;
            po[cell + 1] = nret;
            // the reference's step tally (_native.py:45-81 / :109-153)
            const int64_t dsize = bitwidth == RSR_BINARY ? ((int64_t)1 << g.h)
                                                         : ((int64_t)1 << (2 * g.h));
            const int64_t per_group = bitwidth == RSR_BINARY ? 1 : 1 + g.h;
            steps[cell] = 3 * g.tn + 2 * dsize + nret + (int64_t)ng * per_group;
            if (over) atomicExch(status, (int32_t)RSR_ERR_TILE_TOO_WIDE);
            if (anybad) atomicCAS(status, 0, (int32_t)RSR_ERR_INVALID);
            if (cell == 0) {
                go[0] = 0;
                po[0] = 0;
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(PP_WARPS * 32)
group_fill_kernel(const uint8_t *__restrict__ data, int64_t rows, int64_t cols,
                  int64_t row_bytes, int bitwidth, int k, int64_t tw, int64_t bc,
                  int64_t cells, int64_t bk, uint32_t *gmem_tab, const int64_t *__restrict__ go,
                  const int64_t *__restrict__ po, uint64_t *__restrict__ words,
                  uint16_t *__restrict__ perm) {
    extern __shared__ uint32_t pp_smem[];
    const uint32_t lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    const int warp = threadIdx.x >> 5;
    uint32_t *tab = warp_table(gmem_tab ? nullptr : pp_smem, gmem_tab, bk, warp);
    for (int64_t cell = (int64_t)blockIdx.x * PP_WARPS + warp; cell < cells;
         cell += (int64_t)gridDim.x * PP_WARPS) {
        const CellGeom g = cell_geom(cell, rows, cols, k, tw, bc);
        const int64_t B = bucket_count(bitwidth, g.h);
        bool bad = false;
        cell_histogram(data, row_bytes, g, bitwidth, B, tab, lane, &bad);
        // ascending-key exclusive scan over non-zero keys; emit words.
        uint64_t *wout = words + go[cell];
        uint32_t running = 0, nw = 0;
        for (int64_t d0 = 0; d0 < B; d0 += 32) {
            const int64_t d = d0 + lane;
            const uint32_t c = (d < B && d != 0) ? tab[d] : 0u;
            const uint32_t incl = warp_inclusive_scan(c, lane);
            const uint32_t start = running + incl - c;
            const uint32_t ball = __ballot_sync(RSR_FULL_MASK, c > 0u);
            if (c > 0u) {
                const uint32_t m = key_masks((uint32_t)d, bitwidth, g.h);
                wout[nw + __popc(ball & lt)] =
                    (uint64_t)start | ((uint64_t)c << 16) | ((uint64_t)(m & 0xFFFFu) << 32) |
                    ((uint64_t)(m >> 16) << 48);
                tab[d] = start;  // becomes the scatter cursor of this key
            }
            running += __shfl_sync(RSR_FULL_MASK, incl, 31);
            nw += __popc(ball);
        }
        __syncwarp();
        // stable scatter of tile-local column ids
        uint16_t *pout = perm + po[cell];
        for (int64_t j0 = 0; j0 < g.tn; j0 += 32) {
            const int64_t j = j0 + lane;
            const bool valid = j < g.tn;
            uint32_t key = valid ? column_key(data, row_bytes, g.r0, g.h, g.c0 + j, bitwidth, &bad)
                                 : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(RSR_FULL_MASK, key);
            const bool live = valid && key != 0u;
            uint32_t base = 0;
            if (live) {
                base = tab[key];
                pout[base + __popc(peers & lt)] = (uint16_t)j;
            }
            __syncwarp();
            if (live && (peers & lt) == 0u) tab[key] = base + __popc(peers);
            __syncwarp();
        }
    }
}

// Single-CTA inclusive scan of a[1..cells] in place (a[0] already 0), for
// two int64 arrays at once.
__global__ void __launch_bounds__(1024)
scan2_kernel(int64_t *a, int64_t *b, int64_t cells) {
    __shared__ int64_t wa[32], wb[32];
    __shared__ int64_t carry_a, carry_b;
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        carry_a = 0;
        carry_b = 0;
        a[0] = 0;
        if (b) b[0] = 0;
    }
    __syncthreads();
    for (int64_t base = 0; base < cells; base += 1024) {
        const int64_t i = base + threadIdx.x;
        int64_t xa = i < cells ? a[i + 1] : 0, xb = (b && i < cells) ? b[i + 1] : 0;
        xa = warp_inclusive_scan(xa, lane);
        xb = warp_inclusive_scan(xb, lane);
        if (lane == 31) {
            wa[warp] = xa;
            wb[warp] = xb;
        }
        __syncthreads();
        if (warp == 0) {
            int64_t sa = wa[lane], sb = wb[lane];
            sa = warp_inclusive_scan(sa, lane);
            sb = warp_inclusive_scan(sb, lane);
            wa[lane] = sa;
            wb[lane] = sb;
        }
        __syncthreads();
        const int64_t pa = (warp ? wa[warp - 1] : 0) + carry_a;
        const int64_t pb = (warp ? wb[warp - 1] : 0) + carry_b;
        if (i < cells) {
            a[i + 1] = xa + pa;
            if (b) b[i + 1] = xb + pb;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry_a = xa + pa;
            carry_b = xb + pb;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// chunk stream: block-major cells, each a run of 32-byte chunks (see
// include/rsr_b200.h).  Two layouts:
//   u16 formats (0, 1) -- "quad" layout, rounds of 64 chunks, lane = chunk pair:
//     every pair (32 entries) starts with a key; keys only at slots = 0 mod 4;
//     inside a pair every key starts a new group (a group crossing a pair
//     boundary repeats its key at slot 0 of the next pair); padding is
//     column 0, whose staged v element is 0 -- the cell's real column 0 is not
//     in the stream, its pattern key is stored in col0_key[cell] instead.
//   u32 format (2) -- "even" layout: every chunk starts with a key, keys only at
//     even slots, padding key 0 / column 0 (bucket 0 is never reduced).

__global__ void stream_count_kernel(const uint64_t *__restrict__ words,
                                    const int64_t *__restrict__ go,
                                    const uint16_t *__restrict__ perm,
                                    const int64_t *__restrict__ po, int64_t bc, int64_t tc,
                                    int64_t CH, int layout, int64_t *e_off, int32_t *gslot) {
    // layout: 0 even (u32), 1 quad with the tile's column 0 carried outside
    // the stream (formats 0/1), 2 quad with every column in the stream (3)
    const bool quad = layout != 0;
    const int64_t cells = bc * tc;
    for (int64_t dc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; dc < cells;
         dc += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = dc / tc, t = dc - b * tc;
        const int64_t src = t * bc + b;
        int64_t p = 0;
        for (int64_t g = go[src]; g < go[src + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t L = (int64_t)((w >> 16) & 0xFFFFu);
            gslot[g] = (int32_t)p;
            if (quad) {
                // column 0 leads its group (columns ascend inside a group)
                const bool has0 = layout == 1 && perm[po[src] + (int64_t)(w & 0xFFFFu)] == 0;
                place_group_quad(p, L - has0, [](int64_t) {}, [](int64_t, int64_t) {},
                                 [](int64_t) {});
            } else {
                place_group(p, L, CH, [](int64_t) {}, [](int64_t, int64_t) {});
            }
        }
        e_off[dc + 1] = (p + 2 * CH - 1) / (2 * CH) * (2 * CH);  // whole chunk pairs
    }
}

template <typename E, bool SCALED>
__global__ void __launch_bounds__(256)
stream_build_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                    const uint16_t *__restrict__ perm, const int64_t *__restrict__ po, int64_t bc,
                    int64_t tc, int bitwidth, int64_t CH, const int64_t *__restrict__ e_off,
                    const int32_t *__restrict__ gslot, E *__restrict__ entries) {
    // scaled: column*4 / key*4|1 (byte offsets into 4-byte smem elements);
    // otherwise column / key with the top bit as the key flag
    constexpr E KEYFLAG = (E)1 << (8 * sizeof(E) - 1);
    auto enc_key = [](uint32_t k) -> E { return SCALED ? (E)((k << 2) | 1u) : (E)(KEYFLAG | k); };
    auto enc_col = [](uint32_t c) -> E { return SCALED ? (E)(c << 2) : (E)c; };
    const uint32_t lane = lane_id();
    const int64_t cells = bc * tc;
    for (int64_t dc = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; dc < cells;
         dc += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = dc / tc, t = dc - b * tc;
        const int64_t src = t * bc + b;
        const int64_t e0 = e_off[dc], elen = e_off[dc + 1] - e0;
        const int64_t nch = elen / CH;
        E *out = entries + e0;
        // padding: key 0 at even slots, column 0 at odd slots (both land in the
        // never-reduced bucket 0)
        for (int64_t i = lane; i < elen; i += 32) out[phys_slot(i, CH, nch)] = (i & 1) ? enc_col(0) : enc_key(0);
        __syncwarp();
        const int64_t p0 = po[src];
        for (int64_t g = go[src] + lane; g < go[src + 1]; g += 32) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu), L = (int64_t)((w >> 16) & 0xFFFFu);
            const E key = enc_key(dense_key(w, bitwidth));
            const uint16_t *cols = perm + p0 + ps;
            int64_t p = gslot[g];
            place_group(
                p, L, CH, [&](int64_t q) { out[phys_slot(q, CH, nch)] = key; },
                [&](int64_t q, int64_t j) { out[phys_slot(q, CH, nch)] = enc_col(cols[j]); });
        }
    }
}

// Bank-aware build of the u16 formats (quad layout).  The multiply gathers v
// from shared memory (4-byte elements, bank = column % 32); at slot j of a
// round the 32 lanes gather the columns at round positions 32L + j, and a
// key-sorted column order costs ~3.3 shared-memory wavefronts per gather
// instruction.  Columns of a group may be stored in any order (their sum is
// order-free up to float rounding), so one warp walks its cell's groups in key
// order and fills each column position with the window column (lane i holds
// one of the group's unplaced columns) whose bank is least used so far at that
// (round, slot): ~1.9 wavefronts per gather on random ternary cells
// (tools/bank_sim.py).  Also records the pattern key of the cell's column 0.
constexpr int BB_WARPS = 4;
constexpr int BB_PMAX = 32;    // rounds per cell tracked for bank use (beyond: no preference)
constexpr int BB_LSMAX = 256;  // groups up to this many stream columns get the local search
#ifndef BB_LSPASSES
#define BB_LSPASSES 1
#endif
constexpr size_t BB_WARP_SMEM = (size_t)BB_PMAX * 32 * 32 + BB_LSMAX * 8;

template <bool SCALED>
__global__ void __launch_bounds__(BB_WARPS * 32)
stream_build_banked_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                           const uint16_t *__restrict__ perm, const int64_t *__restrict__ po,
                           int64_t bc, int64_t tc, int bitwidth,
                           const int64_t *__restrict__ e_off, const int32_t *__restrict__ gslot,
                           uint16_t *__restrict__ entries, uint32_t *__restrict__ col0_key) {
    // per warp: gathers per (round, slot, bank) so far (u8), and the local
    // search's position / column lists of one group
    extern __shared__ __align__(16) unsigned char bb_smem[];
    constexpr uint16_t KEYFLAG = 0x8000u;
    auto enc_key = [](uint32_t k) -> uint16_t {
        return SCALED ? (uint16_t)((k << 2) | 1u) : (uint16_t)(KEYFLAG | k);
    };
    auto enc_col = [](uint32_t c) -> uint16_t { return SCALED ? (uint16_t)(c << 2) : (uint16_t)c; };
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    uint8_t *cnt = bb_smem + (size_t)warp * BB_WARP_SMEM;            // [BB_PMAX][32][32]
    uint32_t *lpos = reinterpret_cast<uint32_t *>(cnt + BB_PMAX * 32 * 32);  // [BB_LSMAX]
    uint32_t *lcol = lpos + BB_LSMAX;                                 // [BB_LSMAX]
    const int64_t cells = bc * tc;
    const uint32_t INVALID = 0xFFFFFFFFu;
    for (int64_t dc = (int64_t)blockIdx.x * BB_WARPS + warp; dc < cells;
         dc += (int64_t)gridDim.x * BB_WARPS) {
        const int64_t b = dc / tc, t = dc - b * tc;
        const int64_t src = t * bc + b;
        const int64_t e0 = e_off[dc], elen = e_off[dc + 1] - e0;
        const LaneRuns lr = lane_runs(elen >> 5);
        uint16_t *out = entries + e0;
        for (int64_t i = lane; i < elen; i += 32) out[i] = enc_col(0);  // pads everywhere
        const int64_t tracked_bytes = min(lr.P, (int64_t)BB_PMAX) * 1024;
        for (int64_t i = lane; i < tracked_bytes / 4; i += 32)
            reinterpret_cast<uint32_t *>(cnt)[i] = 0u;
        __syncwarp();
        uint32_t key0 = 0;
        // counter of (round, slot, bank) of logical slot q, or -1 if untracked
        auto cidx = [&](int64_t q, uint32_t bank) -> int {
            const int64_t j = q >> 5;
            const int64_t r = j - (j / lr.P) * lr.P;
            return r < BB_PMAX ? (int)((r * 32 + (q & 31)) * 32 + bank) : -1;
        };
        const int64_t p0 = po[src];
        for (int64_t g = go[src]; g < go[src + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu);
            int64_t L = (int64_t)((w >> 16) & 0xFFFFu);
            const uint32_t dk = dense_key(w, bitwidth);
            const uint16_t key = enc_key(dk);
            const uint16_t *cols = perm + p0 + ps;
            if (cols[0] == 0) {  // column 0 leads its group; it travels as col0_key
                key0 = dk;
                ++cols;
                --L;
            }
            // greedy: a window of 32 unplaced columns (one per lane, refilled
            // from a register batch); each position takes the window column
            // whose bank is least used at that (round, slot) so far
            uint32_t cand = (int64_t)lane < L ? cols[lane] : INVALID;
            int64_t nb = min(L, (int64_t)32);
            uint32_t batch = nb + lane < L ? cols[nb + lane] : INVALID;
            int bi = 0;
            int64_t p = gslot[g];
            place_group_quad(
                p, L,
                [&](int64_t q) {
                    if (lane == 0) out[run_slot(q, lr)] = key;  // key slots read no bank
                },
                [&](int64_t q, int64_t) {
                    const int ci = cand != INVALID ? cidx(q, cand & 31u) : -1;
                    const uint32_t mine = cand == INVALID ? 0x200u : (ci >= 0 ? cnt[ci] : 0u);
                    const uint32_t m = __reduce_min_sync(RSR_FULL_MASK, mine);
                    const int win = __ffs(__ballot_sync(RSR_FULL_MASK, mine == m)) - 1;
                    const uint32_t c = __shfl_sync(RSR_FULL_MASK, cand, win);
                    const uint32_t nxt = __shfl_sync(RSR_FULL_MASK, batch, bi);
                    if ((int)lane == win) cand = nxt;
                    if (++bi == 32) {
                        bi = 0;
                        nb += 32;
                        batch = nb + lane < L ? cols[nb + lane] : INVALID;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        const int k = cidx(q, c & 31u);
                        if (k >= 0 && cnt[k] < 255) ++cnt[k];
                        out[run_slot(q, lr)] = enc_col(c);
                    }
                    __syncwarp();
                },
                [&](int64_t q) {  // pad (column 0, pre-filled): reads bank 0
                    if (lane == 0) {
                        const int k = cidx(q, 0);
                        if (k >= 0 && cnt[k] == 0) cnt[k] = 1;  // one address: counted once
                    }
                    __syncwarp();
                });
        }
        // local search: swap two columns of one group when that lowers the sum
        // of squared bank loads over the (round, slot) sets they sit in
        for (int pass = 0; pass < BB_LSPASSES; ++pass)
        for (int64_t g = go[src]; g < go[src + 1]; ++g) {
            const uint64_t w = words[g];
            int64_t L = (int64_t)((w >> 16) & 0xFFFFu);
            if (perm[p0 + (int64_t)(w & 0xFFFFu)] == 0) --L;
            if (L < 2 || L > BB_LSMAX) continue;
            int64_t p = gslot[g];
            int n = 0;
            place_group_quad(
                p, L, [](int64_t) {},
                [&](int64_t q, int64_t) {
                    if (lane == 0) {
                        const uint32_t e = out[run_slot(q, lr)];
                        lpos[n] = (uint32_t)q;
                        lcol[n] = SCALED ? (e >> 2) : e;
                    }
                    ++n;
                },
                [](int64_t) {});
            __syncwarp();
            for (int i = 0; i < n; ++i) {
                const uint32_t qi = lpos[i], ci = lcol[i], bi_ = ci & 31u;
                const int ki = cidx(qi, bi_);
                int best = 1 << 30, bj = -1;
                for (int j = (int)lane; j < n; j += 32) {
                    const uint32_t qj = lpos[j], cj = lcol[j], bj_ = cj & 31u;
                    const int kj = cidx(qj, bj_);
                    if (j == i || bj_ == bi_ || ki < 0 || kj < 0) continue;
                    const int si = ki - (int)bi_, sj = kj - (int)bj_;  // set bases
                    if (si == sj) continue;
                    const int d = 2 * ((int)cnt[si + bj_] - (int)cnt[ki]) +
                                  2 * ((int)cnt[sj + bi_] - (int)cnt[kj]) + 4;
                    if (d < best) {
                        best = d;
                        bj = j;
                    }
                }
                const int m = __reduce_min_sync(RSR_FULL_MASK, best);
                if (m >= 0) continue;
                const int who = __ffs(__ballot_sync(RSR_FULL_MASK, best == m)) - 1;
                const int j = __shfl_sync(RSR_FULL_MASK, bj, who);
                if (lane == 0) {
                    const uint32_t qj = lpos[j], cj = lcol[j], bj_ = cj & 31u;
                    const int kj = cidx(qj, bj_);
                    const int si = ki - (int)bi_, sj = kj - (int)bj_;
                    --cnt[ki];
                    ++cnt[si + bj_];
                    --cnt[kj];
                    ++cnt[sj + bi_];
                    lcol[i] = cj;
                    lcol[j] = ci;
                    out[run_slot(qi, lr)] = enc_col(cj);
                    out[run_slot(qj, lr)] = enc_col(ci);
                }
                __syncwarp();
            }
        }
        if (lane == 0) col0_key[dc] = key0;
        __syncwarp();
    }
}

__global__ void count_ops_kernel(const uint64_t *__restrict__ words, int64_t n, int64_t *out3) {
    int64_t g = 0, s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t w = words[i];
        g += (int64_t)((w >> 16) & 0xFFFFu);
        s += __popcll(w >> 32);
    }
    g = warp_sum(g);
    s = warp_sum(s);
    if (lane_id() == 0) {
        atomicAdd((unsigned long long *)out3, (unsigned long long)g);
        atomicAdd((unsigned long long *)(out3 + 1), (unsigned long long)s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd((unsigned long long *)(out3 + 2), (unsigned long long)n);
}

struct GroupLaunch {
    int64_t bc, tc, cells, bk;
    bool smem;
    int grid;
    size_t smem_bytes;
};

static GroupLaunch group_launch(int64_t rows, int64_t cols, int32_t bitwidth, int32_t k,
                                int64_t tw) {
    GroupLaunch L;
    L.bc = (rows + k - 1) / k;
    L.tc = (cols + tw - 1) / tw;
    L.cells = L.bc * L.tc;
    L.bk = bucket_count(bitwidth, k);
    L.smem = L.bk <= PP_SMEM_TABLE_MAX;
    const int sms = sm_count();
    const int64_t need = (L.cells + PP_WARPS - 1) / PP_WARPS;
    if (L.smem) {
        L.grid = (int)std::min<int64_t>(need, (int64_t)sms * 16);
        L.smem_bytes = (size_t)L.bk * 4 * PP_WARPS;
    } else {
        L.grid = (int)std::min<int64_t>(need, (int64_t)sms * 2);
        L.smem_bytes = 0;
    }
    if (L.grid < 1) L.grid = 1;
    return L;
}

static rsr_status check_plan(int64_t rows, int64_t cols, int64_t row_bytes, int32_t bitwidth,
                             int32_t k, int64_t tw) {
    if (rows < 1 || cols < 1 || tw < 1) return RSR_ERR_INVALID;
    if (bitwidth != RSR_BINARY && bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    if (k < 1) return RSR_ERR_INVALID;
    if (k > (bitwidth == RSR_BINARY ? 16 : 10)) return RSR_ERR_K_TOO_LARGE;
    if (tw > 65536) return RSR_ERR_TILE_TOO_WIDE;
    const int64_t need = bitwidth == RSR_BINARY ? (cols + 7) / 8 : (cols + 3) / 4;
    if (row_bytes < need) return RSR_ERR_INVALID;
    return RSR_OK;
}

}  // namespace rsr

namespace rsr {
// halfword format builder (rsr_stream_h.cu)
rsr_status stream_build_h(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                          const int64_t *po, int64_t bc, int64_t tc, int64_t tw, int64_t ncols,
                          int32_t bitwidth, const int64_t *e_off, const int32_t *gslot,
                          uint16_t *entries, uint32_t *col0_key, cudaStream_t s);
}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_group_workspace_bytes(int64_t rows, int64_t cols, int32_t bitwidth, int32_t k,
                                 int64_t tile_width) {
    if (rows < 1 || cols < 1 || k < 1 || tile_width < 1) return 0;
    GroupLaunch L = group_launch(rows, cols, bitwidth, k, tile_width);
    if (L.smem) return 0;
    return (size_t)L.grid * PP_WARPS * (size_t)L.bk * 4;
}

rsr_status rsr_group_count(const uint8_t *data, int64_t rows, int64_t cols, int64_t row_bytes,
                           int32_t bitwidth, int32_t k, int64_t tile_width, int64_t *go,
                           int64_t *po, int64_t *sort_steps, int32_t *status_dev,
                           void *workspace, size_t workspace_bytes, rsr_stream_t stream) {
    rsr_status st = check_plan(rows, cols, row_bytes, bitwidth, k, tile_width);
    if (st != RSR_OK) return st;
    if (!data || !go || !po || !sort_steps || !status_dev) return RSR_ERR_INVALID;
    GroupLaunch L = group_launch(rows, cols, bitwidth, k, tile_width);
    uint32_t *gtab = nullptr;
    if (!L.smem) {
        if (workspace_bytes < rsr_group_workspace_bytes(rows, cols, bitwidth, k, tile_width) ||
            !workspace)
            return RSR_ERR_WORKSPACE;
        gtab = (uint32_t *)workspace;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (L.smem_bytes > 48 * 1024)
        cudaFuncSetAttribute(group_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L.smem_bytes);
    cudaMemsetAsync(status_dev, 0, sizeof(int32_t), s);
    group_count_kernel<<<L.grid, PP_WARPS * 32, L.smem_bytes, s>>>(
        data, rows, cols, row_bytes, bitwidth, k, tile_width, L.bc, L.cells, L.bk, gtab, go, po,
        sort_steps, status_dev);
    scan2_kernel<<<1, 1024, 0, s>>>(go, po, L.cells);
    return launch_status();
}

rsr_status rsr_group_fill(const uint8_t *data, int64_t rows, int64_t cols, int64_t row_bytes,
                          int32_t bitwidth, int32_t k, int64_t tile_width, const int64_t *go,
                          const int64_t *po, uint64_t *words, uint16_t *perm, void *workspace,
                          size_t workspace_bytes, rsr_stream_t stream) {
    rsr_status st = check_plan(rows, cols, row_bytes, bitwidth, k, tile_width);
    if (st != RSR_OK) return st;
    if (!data || !go || !po) return RSR_ERR_INVALID;
    GroupLaunch L = group_launch(rows, cols, bitwidth, k, tile_width);
    uint32_t *gtab = nullptr;
    if (!L.smem) {
        if (workspace_bytes < rsr_group_workspace_bytes(rows, cols, bitwidth, k, tile_width) ||
            !workspace)
            return RSR_ERR_WORKSPACE;
        gtab = (uint32_t *)workspace;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (L.smem_bytes > 48 * 1024)
        cudaFuncSetAttribute(group_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L.smem_bytes);
    group_fill_kernel<<<L.grid, PP_WARPS * 32, L.smem_bytes, s>>>(
        data, rows, cols, row_bytes, bitwidth, k, tile_width, L.bc, L.cells, L.bk, gtab, go, po,
        words, perm);
    return launch_status();
}

int32_t rsr_stream_format(int32_t bitwidth, int32_t k, int64_t tile_width) {
    const int64_t keys = bucket_count(bitwidth, k);
    if (tile_width <= 32704 && keys <= 2187) return 3;   // halfword u16 (bucket kernel)
    if (tile_width <= 32768 && keys <= 32768) return 0;  // u16
    return 2;                                            // u32
}

rsr_status rsr_stream_count(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int32_t format, int32_t chunk, int64_t *e_off, int32_t *gslot,
                            rsr_stream_t stream) {
    if (!go || !po || !e_off || block_count < 1 || tile_count < 1) return RSR_ERR_INVALID;
    if (format < 0 || format > 3 || chunk != (format == 2 ? 8 : 16)) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells + 127) / 128, 8192);
    stream_count_kernel<<<grid, 128, 0, s>>>(words, go, perm, po, block_count, tile_count, chunk,
                                             format == 2 ? 0 : (format == 3 ? 2 : 1), e_off,
                                             gslot);
    scan2_kernel<<<1, 1024, 0, s>>>(e_off, nullptr, cells);
    return launch_status();
}

rsr_status rsr_stream_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t format,
                            int32_t chunk, const int64_t *e_off, const int32_t *gslot,
                            void *entries, uint32_t *col0_key, rsr_stream_t stream) {
    if (!go || !po || !e_off || !entries || block_count < 1 || tile_count < 1)
        return RSR_ERR_INVALID;
    if (format < 0 || format > 3 || chunk != (format == 2 ? 8 : 16)) return RSR_ERR_INVALID;
    if (format != 2 && !col0_key) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (format == 3)
        return stream_build_h(words, go, perm, po, block_count, tile_count, tile_width, cols,
                              bitwidth, e_off, gslot, (uint16_t *)entries, col0_key, s);
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells * 32 + 255) / 256, (int64_t)sm_count() * 32);
    const int bgrid =
        (int)std::min<int64_t>((cells + BB_WARPS - 1) / BB_WARPS, (int64_t)sm_count() * 8);
    const size_t bsm = BB_WARPS * BB_WARP_SMEM;
    if (format == 1) {
        cudaFuncSetAttribute(stream_build_banked_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
        stream_build_banked_kernel<true><<<bgrid, BB_WARPS * 32, bsm, s>>>(
            words, go, perm, po, block_count, tile_count, bitwidth, e_off, gslot,
            (uint16_t *)entries, col0_key);
    } else if (format == 0) {
        cudaFuncSetAttribute(stream_build_banked_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
        stream_build_banked_kernel<false><<<bgrid, BB_WARPS * 32, bsm, s>>>(
            words, go, perm, po, block_count, tile_count, bitwidth, e_off, gslot,
            (uint16_t *)entries, col0_key);
    }
    else
        stream_build_kernel<uint32_t, false><<<grid, 256, 0, s>>>(words, go, perm, po, block_count,
                                                           tile_count, bitwidth, chunk, e_off,
                                                           gslot, (uint32_t *)entries);
    return launch_status();
}

rsr_status rsr_count_ops(const uint64_t *words, int64_t n_words, int64_t *out3,
                         rsr_stream_t stream) {
    if (!out3 || n_words < 0) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(out3, 0, 3 * sizeof(int64_t), s);
    if (n_words > 0) {
        const int grid = (int)std::min<int64_t>((n_words + 255) / 256, (int64_t)sm_count() * 4);
        count_ops_kernel<<<grid, 256, 0, s>>>(words, n_words, out3);
    }
    return launch_status();
}

}  // extern "C"
