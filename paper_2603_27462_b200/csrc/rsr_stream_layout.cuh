// rsr_stream_layout.cuh -- slot geometry of the device chunk stream, shared
// by the stream builders (rsr_preprocess.cu, rsr_stream_h.cu).
#pragma once

#include "rsr_common.cuh"

namespace rsr {

// Quad layout: slots of one group of R stream columns starting at slot p
// (p = 0 mod 4).  emit_key(slot) / emit_col(slot, j) / emit_pad(slot).
template <typename KeyFn, typename ColFn, typename PadFn>
__host__ __device__ __forceinline__ void place_group_quad(int64_t &p, int64_t R, KeyFn emit_key,
                                                         ColFn emit_col, PadFn emit_pad) {
    if (R == 0) return;
    emit_key(p++);
    for (int64_t j = 0; j < R; ++j) {
        if ((p & 31) == 0) emit_key(p++);  // pair start: the group continues
        emit_col(p++, j);
    }
    while (p & 3) emit_pad(p++);
}

// Even layout: slot placement of one group of L columns (the reference word's
// perm_len) starting at slot p (always even).  Keys only ever sit at EVEN slots: every
// segment that ends inside a chunk has odd length (an even remainder is split
// 1 + (R-1) with one repeated key), and a segment running to the chunk end
// has odd length automatically.  A group crossing a chunk boundary repeats its
// key at slot 0 of the next chunk.  emit_key(slot) / emit_col(slot, j).
template <typename KeyFn, typename ColFn>
__host__ __device__ __forceinline__ void place_group(int64_t &p, int64_t L, int64_t CH,
                                                    KeyFn emit_key, ColFn emit_col) {
    emit_key(p++);
    int64_t R = L, j = 0;
    while (true) {
        const int64_t room = CH - p % CH;  // odd
        if (R >= room) {
            for (int64_t i = 0; i < room; ++i) emit_col(p++, j++);
            R -= room;
            if (R == 0) break;
            emit_key(p++);
            continue;
        }
        if (R & 1) {
            for (int64_t i = 0; i < R; ++i) emit_col(p++, j++);
            break;
        }
        for (int64_t i = 0; i < R - 1; ++i) emit_col(p++, j++);
        emit_key(p++);
        emit_col(p++, j++);
        break;
    }
}

// Physical index of logical slot p inside a cell of nch chunks (nch even).
// A warp round is 64 chunks: lane L owns the consecutive chunk pair (2L,
// 2L+1), i.e. 64 bytes in four 16-byte quarters; the round is stored as
// [quarter 0 of every pair][quarter 1]...[quarter 3], so each of a lane's four
// 16-byte loads is one coalesced 512-byte access, and the round is one
// contiguous 2 KiB bulk copy.
__host__ __device__ __forceinline__ int64_t phys_slot(int64_t p, int64_t CH, int64_t nch) {
    const int64_t c = p / CH, js = p - c * CH;
    const int64_t pair = c >> 1, cin = c & 1;
    const int64_t r = pair >> 5, lanep = pair & 31;
    const int64_t npairs = nch >> 1;
    const int64_t np = min((int64_t)32, npairs - (r << 5));
    const int64_t qe = CH >> 1;  // entries per 16-byte quarter
    const int64_t q = cin * 2 + js / qe, within = js % qe;
    return r * 64 * CH + q * np * qe + lanep * qe + within;
}

// Quad layout physical placement ("lane runs").  A cell of N chunk pairs is
// processed in P = ceil(N / 32) rounds; lane L owns the CONTIGUOUS run of
// pairs [L*P, L*P + len_L) (len_L = P for L < Lf = N / P, rem = N - Lf*P for
// lane Lf, 0 beyond), so a lane carries its open group from round to round and
// lanes only meet at run boundaries.  Round r holds the pairs L*P + r of its
// np_r = Lf + (r < rem) active lanes, as four 16-byte quarters [q0 of the np_r
// pairs][q1][q2][q3] (every lane load coalesced), starting at pair R(r) =
// r*Lf + min(r, rem) of the cell.
struct LaneRuns {
    int64_t P, Lf, rem;
};
__host__ __device__ __forceinline__ LaneRuns lane_runs(int64_t npairs) {
    LaneRuns lr;
    lr.P = (npairs + 31) / 32;
    lr.Lf = lr.P ? npairs / lr.P : 0;
    lr.rem = npairs - lr.Lf * lr.P;
    return lr;
}
// Physical u16 index (inside the cell) of logical slot p.
__host__ __device__ __forceinline__ int64_t run_slot(int64_t p, const LaneRuns &lr) {
    const int64_t j = p >> 5, slot = p & 31;
    const int64_t L = j / lr.P, r = j - L * lr.P;
    const int64_t np = lr.Lf + (r < lr.rem ? 1 : 0);
    const int64_t R = r * lr.Lf + min(r, lr.rem);
    return R * 32 + (slot >> 3) * np * 8 + L * 8 + (slot & 7);
}

// Dense pattern key of a group from its masks: binary -> pos mask; ternary
// -> base-3 digits (1 = +1, 2 = -1).  Key 0 never occurs (zero patterns are
// dropped) and marks padding.
__device__ __forceinline__ uint32_t dense_key(uint64_t w, int bitwidth) {
    const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
    if (bitwidth == RSR_BINARY) return pos;
    uint32_t key = 0, p3 = 1;
    for (int i = 0; i < 16; ++i) {
        key += (((pos >> i) & 1u) + 2u * ((neg >> i) & 1u)) * p3;
        p3 *= 3u;
    }
    return key;
}

}  // namespace rsr
