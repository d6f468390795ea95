// rsr_stream_h.cu -- builder of the halfword chunk stream (format 3), the
// layout the hot multiply kernel reads (rsr_mv_kernel.cuh).
//
// Format 3 keeps the quad layout and lane runs of the u16 formats (see
// rsr_stream_layout.cuh) with different entry semantics:
//   column c  -> 2*c           byte offset of a 2-byte element (bf16 / int16 v)
//   key       -> key*4 | 1     byte offset of the key's 4-byte pattern bucket
//   padding   -> Z + 4*b       one of 32 zero words the kernel stages after the
//                              tile's image (Z = h_zero_b(tn)), one per bank b
// Every column of the tile is in the stream (no col0_key side channel), and
// padding can name a zero word in any bank.
//
// Column ORDER inside each group is free (a group's sum does not depend on
// it), and this builder uses that freedom to make the kernel's shared-memory
// gathers conflict-free.  At round r, slot s the 32 lanes gather the columns
// at logical slots (L*P + r)*32 + s; a 2-byte element c sits in bank
// (c >> 1) & 31.  The builder walks the instructions (r, s) in order; each
// lane holding a column slot offers the banks of its group's not-yet-placed
// columns, and a bipartite matching (lanes x banks) gives each lane a
// distinct bank: lanes with the fewest options choose first, each taking the
// free bank its group holds most columns of (keeping later slots flexible),
// with an augmenting-path search (Kuhn) when no free bank is left.  Padding
// takes a zero word in a bank no lane uses.  For float32 vectors the kernel
// stages 4-byte elements (bank c & 31); the two lanes of bf16 banks b and
// b ^ 16 then share an f32 bank pair, so the second of them prefers the
// column parity its partner did not take.  Random C2 cells (tools/banksim.c):
// ~1.2 wavefronts per gather vs ~3.3 for key order and 1.86 for the
// previous greedy + swap builder, whose zero padding sat in bank 0.
#include "rsr_mv_impl.cuh"
#include "rsr_stream_layout.cuh"

namespace rsr {

constexpr int SH_WARPS = 8;             // cells in flight per CTA (one warp each)
constexpr int64_t HB_MAX_TN = 32768;    // bitmap capacity (the format addresses <= 32704)

struct HWarpSmem {
    uint32_t used[HB_MAX_TN / 32];  // columns already placed (bitmap)
    uint8_t cnt[32][32];           // per lane: unplaced columns of its group per bank
    int8_t owner[32];              // matching: lane owning each bank (-1 free)
    int8_t lbank[32];              // matching: bank of each lane (-1 none)
    int8_t par[32];                // augmenting-path search: parent lane of a bank
    int8_t queue[32];
    uint32_t msk[32];              // per lane: banks its group can still offer
    int16_t pick16[16];            // f32 bank of the column taken by bf16 bank b < 16
};

// One stream lane's walk through its run: the quad layout of the cell's
// groups (place_group_quad) replayed one slot at a time.
struct HWalk {
    int64_t g, g1;      // current group (absolute word index), end of the cell's groups
    int64_t rem;        // columns of g still to lay out
    int phase;          // 0 group key next, 1 columns, 2 padding, 3 past the last group
};

enum : int { H_KEY = 0, H_COL = 1, H_PAD = 2, H_SINK = 3 };

__device__ __forceinline__ int walk_step(HWalk &w, int64_t p, const uint64_t *__restrict__ words) {
    switch (w.phase) {
        case 0:
            w.rem = (int64_t)((words[w.g] >> 16) & 0xFFFFu);
            w.phase = 1;
            return H_KEY;
        case 1:
            if ((p & 31) == 0) return H_KEY;  // pair start: the group continues
            if (--w.rem == 0) {
                if (((p + 1) & 3) == 0) {
                    ++w.g;
                    w.phase = w.g < w.g1 ? 0 : 3;
                } else {
                    w.phase = 2;
                }
            }
            return H_COL;
        case 2:
            if (((p + 1) & 3) == 0) {
                ++w.g;
                w.phase = w.g < w.g1 ? 0 : 3;
            }
            return H_PAD;
        default:
            return (p & 31) == 0 ? H_SINK : H_PAD;
    }
}

__global__ void __launch_bounds__(SH_WARPS * 32)
stream_build_h_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
                      const uint16_t *__restrict__ perm, const int64_t *__restrict__ po,
                      int64_t bc, int64_t tc, int64_t tw, int64_t ncols, int bitwidth,
                      const int64_t *__restrict__ e_off,
                      const int32_t *__restrict__ gslot, uint16_t *__restrict__ entries,
                      uint32_t *__restrict__ col0_key) {
    extern __shared__ __align__(16) unsigned char sh_smem[];
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    HWarpSmem &S = reinterpret_cast<HWarpSmem *>(sh_smem)[warp];
    const int64_t cells = bc * tc;
    for (int64_t dc = (int64_t)blockIdx.x * SH_WARPS + warp; dc < cells;
         dc += (int64_t)gridDim.x * SH_WARPS) {
        const int64_t b = dc / tc, t = dc - b * tc;
        const int64_t src = t * bc + b;
        const int64_t e0 = e_off[dc], elen = e_off[dc + 1] - e0;
        const LaneRuns lr = lane_runs(elen >> 5);
        uint16_t *out = entries + e0;
        const uint16_t *cperm = perm + po[src];
        const uint32_t zero_b = h_zero_b(min(tw, ncols - t * tw));
        const int64_t g0 = go[src], g1 = go[src + 1];
        for (int i = lane; i < HB_MAX_TN / 32; i += 32) S.used[i] = 0u;
        if (lane < 16) S.pick16[lane] = -1;
        if (lane == 0) col0_key[dc] = 0u;  // column 0 travels in the stream

        // lane L's run: pairs [L*P, L*P + len)
        const int64_t len = (int64_t)lane < lr.Lf ? lr.P
                            : ((int64_t)lane == lr.Lf ? lr.rem : 0);
        int64_t cached_g = -1;  // group whose bank counts S.cnt[lane] / gmask hold
        uint32_t gmask = 0u;
        HWalk w;
        w.g1 = g1;
        w.rem = 0;
        w.g = g1;
        w.phase = 3;
        if (len > 0 && g1 > g0) {
            // the group covering the run's first slot, then replay up to it
            const int64_t q0 = (int64_t)lane * lr.P * 32;
            int64_t lo = g0, hi = g1 - 1;
            while (lo < hi) {  // last group with gslot <= q0
                const int64_t mid = (lo + hi + 1) >> 1;
                if (gslot[mid] <= q0) lo = mid;
                else hi = mid - 1;
            }
            if ((int64_t)gslot[lo] <= q0) {
                w.g = lo;
                w.phase = 0;
                for (int64_t q = gslot[lo]; q < q0 && w.phase != 3; ++q) walk_step(w, q, words);
            } else {
                w.g = g0;  // (cannot happen: the first group starts at slot 0)
                w.phase = 0;
            }
        }
        __syncwarp();

        for (int64_t r = 0; r < lr.P; ++r) {
            const bool act = r < len;
            const int64_t pbase = ((int64_t)lane * lr.P + r) * 32;
            // slot 0 of the pair: a key (group start or continuation) or the sink
            int64_t gcur = w.g;
            if (act) {
                const int ty = walk_step(w, pbase, words);
                const uint16_t e = ty == H_KEY ? (uint16_t)((dense_key(words[gcur], bitwidth) << 2) | 1u)
                                               : (uint16_t)1u;  // sink: bucket 0, never reduced
                out[run_slot(pbase, lr)] = e;
            }
            for (int s = 1; s < 32; ++s) {
                const int64_t p = pbase + s;
                gcur = w.g;
                const int ty = act ? walk_step(w, p, words) : H_SINK;
                // ---- offers: banks of the group's unplaced columns, counted
                // when the lane enters the group and kept up to date by its
                // own picks (a group two lanes share at once -- a cell of one
                // round -- may leave a stale count; its pick then falls back)
                uint32_t mask = 0u;
                const uint16_t *gc = nullptr;
                int64_t glen = 0;
                if (ty == H_COL) {
                    const uint64_t wd = words[gcur];
                    gc = cperm + (int64_t)(wd & 0xFFFFu);
                    glen = (int64_t)((wd >> 16) & 0xFFFFu);
                    if (gcur != cached_g) {
                        cached_g = gcur;
                        uint32_t *row = reinterpret_cast<uint32_t *>(S.cnt[lane]);
#pragma unroll
                        for (int i = 0; i < 8; ++i) row[i] = 0u;
                        gmask = 0u;
                        for (int64_t j0 = 0; j0 < glen; j0 += 8) {
                            uint32_t cs[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) cs[u] = j0 + u < glen ? gc[j0 + u] : 0xFFFFu;
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const uint32_t c = cs[u];
                                if (c != 0xFFFFu && !((S.used[c >> 5] >> (c & 31)) & 1u)) {
                                    const uint32_t bk = (c >> 1) & 31u;
                                    S.cnt[lane][bk]++;
                                    gmask |= 1u << bk;
                                }
                            }
                        }
                    }
                    mask = gmask;
                }
                S.msk[lane] = mask;
                S.owner[lane] = -1;
                S.lbank[lane] = -1;
                __syncwarp();
                // ---- matching: fewest options first, most abundant free bank
                uint32_t taken = 0u;
                // the option counts present in this slot (bit c-1 for c options)
                uint32_t levels = __reduce_or_sync(RSR_FULL_MASK, mask ? 1u << (__popc(mask) - 1) : 0u);
                while (levels) {
                    const int lvl = __ffs(levels);
                    levels &= levels - 1u;
                    uint32_t cand = __ballot_sync(RSR_FULL_MASK, mask != 0u && __popc(mask) == lvl);
                    while (cand) {
                        const int i = __ffs(cand) - 1;
                        cand &= cand - 1u;
                        const uint32_t mi = __shfl_sync(RSR_FULL_MASK, mask, i);
                        const uint32_t fr = mi & ~taken;
                        if (fr) {
                            const uint32_t score =
                                ((fr >> lane) & 1u) ? (((uint32_t)S.cnt[i][lane] << 8) | (31u - lane)) : 0u;
                            const uint32_t best = __reduce_max_sync(RSR_FULL_MASK, score);
                            const int bk = 31 - (int)(best & 0xFFu);
                            taken |= 1u << bk;
                            if (lane == 0) {
                                S.owner[bk] = (int8_t)i;
                                S.lbank[i] = (int8_t)bk;
                            }
                        } else {
                            if (lane == 0) {  // augmenting path (Kuhn, BFS over banks)
                                uint32_t vis = 0u;
                                int qh = 0, qt = 0, endb = -1;
                                S.queue[qt++] = (int8_t)i;
                                while (qh < qt && endb < 0) {
                                    const int u = S.queue[qh++];
                                    uint32_t m = S.msk[u] & ~vis;
                                    while (m) {
                                        const int bb = __ffs(m) - 1;
                                        m &= m - 1u;
                                        vis |= 1u << bb;
                                        S.par[bb] = (int8_t)u;
                                        if (S.owner[bb] < 0) {
                                            endb = bb;
                                            break;
                                        }
                                        S.queue[qt++] = S.owner[bb];
                                    }
                                }
                                for (int bb = endb; bb >= 0;) {
                                    const int u = S.par[bb];
                                    const int ob = S.lbank[u];
                                    S.lbank[u] = (int8_t)bb;
                                    S.owner[bb] = (int8_t)u;
                                    if (u == i) break;
                                    bb = ob;
                                }
                            }
                            __syncwarp();
                            taken = __ballot_sync(RSR_FULL_MASK, S.owner[lane] >= 0);
                        }
                        __syncwarp();
                    }
                }
                const int mybank = S.lbank[lane];
                // ---- picks: bf16 banks < 16 first, then their partners b + 16
                // (preferring the f32 bank of the other parity), unmatched
                // lanes last (a bank no column of this slot uses, if any).
                // Test-and-set on the used bitmap: two lanes sharing a group
                // (a cell of one round) never take the same column.
                constexpr uint32_t NONE = 0xFFFFFFFFu;
                auto pick = [&](int want_bank, int avoid_f32, uint32_t occ) -> uint32_t {
                    for (int tries = 0; tries < 64; ++tries) {
                        uint32_t best = NONE;
                        int bestsc = 1 << 30;
                        for (int64_t j0 = 0; j0 < glen && bestsc > 0; j0 += 8) {
                            uint32_t cs[8];  // eight loads in flight
#pragma unroll
                            for (int u = 0; u < 8; ++u) cs[u] = j0 + u < glen ? gc[j0 + u] : 0xFFFFu;
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const uint32_t c = cs[u];
                                if (c == 0xFFFFu || bestsc == 0) continue;
                                if ((S.used[c >> 5] >> (c & 31)) & 1u) continue;
                                const int bk = (int)((c >> 1) & 31u);
                                int sc;
                                if (want_bank >= 0) {
                                    if (bk != want_bank) continue;
                                    sc = (int)(c & 31u) == avoid_f32 ? 1 : 0;
                                } else {
                                    sc = ((occ >> bk) & 1u) ? 1 : 0;
                                }
                                if (sc < bestsc) {
                                    bestsc = sc;
                                    best = c;
                                }
                            }
                        }
                        if (best == NONE) return NONE;
                        const uint32_t bit = 1u << (best & 31);
                        if (!(atomicOr(&S.used[best >> 5], bit) & bit)) {
                            const uint32_t bk = (best >> 1) & 31u;
                            if (--S.cnt[lane][bk] == 0) gmask &= ~(1u << bk);
                            return best;
                        }
                    }
                    return NONE;
                };
                uint32_t chosen = NONE;
                if (ty == H_COL && mybank >= 0 && mybank < 16) {
                    chosen = pick(mybank, -1, 0u);
                    if (chosen != NONE) S.pick16[mybank] = (int16_t)(chosen & 31u);
                }
                __syncwarp();
                if (ty == H_COL && mybank >= 16) chosen = pick(mybank, S.pick16[mybank - 16], 0u);
                __syncwarp();
                {
                    const uint32_t occ = __reduce_or_sync(
                        RSR_FULL_MASK, chosen != NONE ? 1u << ((chosen >> 1) & 31u) : 0u);
                    if (ty == H_COL && chosen == NONE) chosen = pick(-1, -1, occ);
                }
                // ---- padding: a zero word in a bank no column of this slot uses
                const uint32_t occ =
                    __reduce_or_sync(RSR_FULL_MASK, chosen != NONE ? 1u << ((chosen >> 1) & 31u) : 0u);
                const uint32_t freeb = ~occ;
                const int zb = freeb ? __ffs(freeb) - 1 : 0;
                if (act) {
                    uint16_t e;
                    if (ty == H_COL) e = (uint16_t)(chosen << 1);
                    else if (ty == H_KEY) e = (uint16_t)((dense_key(words[gcur], bitwidth) << 2) | 1u);
                    else e = (uint16_t)(zero_b + 4u * (uint32_t)zb);
                    out[run_slot(p, lr)] = e;
                }
                if (lane < 16) S.pick16[lane] = -1;
                __syncwarp();
            }
        }
        __syncwarp();
    }
}

rsr_status stream_build_h(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                          const int64_t *po, int64_t bc, int64_t tc, int64_t tw, int64_t ncols,
                          int32_t bitwidth, const int64_t *e_off, const int32_t *gslot,
                          uint16_t *entries, uint32_t *col0_key, cudaStream_t s) {
    if (tw > H_MAX_TN || ncols < 1) return RSR_ERR_INVALID;
    const int64_t cells = bc * tc;
    const size_t smem = SH_WARPS * sizeof(HWarpSmem);
    const int grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((cells + SH_WARPS - 1) / SH_WARPS,
                                                    (int64_t)sm_count() * 4));
    cudaFuncSetAttribute(stream_build_h_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    stream_build_h_kernel<<<grid, SH_WARPS * 32, smem, s>>>(words, go, perm, po, bc, tc, tw, ncols,
                                                             bitwidth, e_off, gslot, entries,
                                                             col0_key);
    return launch_status();
}

}  // namespace rsr
