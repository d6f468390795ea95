// rsr_audit.cu -- device audit and inverse of an RSR artifact.
//
// rsr_audit checks, one warp per (tile, block) cell, the per-cell invariants
// the reference's validate_artifact enforces (pkg/src/rsrmv/preproc.py:
// 305-372) on the reference arrays as they sit on the device: non-empty
// groups with consecutive perm ranges covering the cell, disjoint non-zero
// pos/neg masks without bits at or above the block height, no negative mask
// in a binary artifact, strictly ascending group keys (the reference's 4^h
// code keys), column ids inside the tile, unique per cell and ascending
// inside each group.  The result is the smallest (cell, check) pair that
// fails, so the host reports the same first failure a sequential audit in
// cell order would.  Header-level checks (shape, caps, offset arrays) run on
// the host before this kernel, which therefore never reads out of bounds.
//
// rsr_reconstruct is the lossless inverse (reference preproc.py:375-400):
// every group scatters its sign pattern back into the packed matrix.
#include "rsr_common.cuh"

namespace rsr {

constexpr int AU_WARPS = 4;
constexpr int AU_MAX_TN = 65536;

enum AuditCheck : unsigned {
    AU_EMPTY_GROUP = 1,
    AU_RANGES = 2,
    AU_COVER = 3,
    AU_OVERLAP = 4,
    AU_ZERO = 5,
    AU_HEIGHT = 6,
    AU_NEG_BINARY = 7,
    AU_KEY_ORDER = 8,
    AU_COLUMN_RANGE = 9,
    AU_DUPLICATE = 10,
    AU_COLUMN_ORDER = 11,
    AU_STRAY_PERM = 12
};

// reference pattern key: code(row i) * 4^i, code +1 -> 1, -1 -> 2
__device__ __forceinline__ uint64_t code_key(uint64_t w) {
    const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
    uint64_t key = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
        key |= (uint64_t)(((pos >> i) & 1u) | (((neg >> i) & 1u) << 1)) << (2 * i);
    return key;
}

__global__ void __launch_bounds__(AU_WARPS * 32)
audit_kernel(const uint64_t *__restrict__ words, const int64_t *__restrict__ go,
             const uint16_t *__restrict__ perm, const int64_t *__restrict__ po, int64_t m,
             int64_t n, int k, int bitwidth, int64_t tw, int64_t bc, int64_t tc,
             unsigned long long *result) {
    extern __shared__ uint32_t au_seen[];  // per warp: column bitmap of the cell
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    uint32_t *seen = au_seen + (size_t)warp * (AU_MAX_TN / 32);
    const int64_t cells = bc * tc;
    for (int64_t c = (int64_t)blockIdx.x * AU_WARPS + warp; c < cells;
         c += (int64_t)gridDim.x * AU_WARPS) {
        const int64_t t = c / bc, b = c - t * bc;
        const int64_t tn = min(tw, n - t * tw);
        const int h = (int)min((int64_t)k, m - b * k);
        const int64_t g0 = go[c], g1 = go[c + 1], p0 = po[c], plen = po[c + 1] - p0;
        unsigned worst = 0xFFu;
        auto fail = [&](unsigned code) { worst = code < worst ? code : worst; };
        if (g1 == g0) {
            if (plen != 0 && lane == 0) fail(AU_STRAY_PERM);
        } else {
            for (int64_t i = lane; i < (tn + 31) / 32; i += 32) seen[i] = 0u;
            __syncwarp();
            for (int64_t g = g0 + lane; g < g1; g += 32) {
                const uint64_t w = words[g];
                const int64_t ps = (int64_t)(w & 0xFFFFu), pl = (int64_t)((w >> 16) & 0xFFFFu);
                const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
                if (pl < 1) fail(AU_EMPTY_GROUP);
                if (g == g0 && ps != 0) fail(AU_RANGES);
                if (g + 1 < g1) {
                    const uint64_t wn = words[g + 1];
                    if ((int64_t)(wn & 0xFFFFu) != ps + pl) fail(AU_RANGES);
                    if (code_key(wn) <= code_key(w)) fail(AU_KEY_ORDER);
                } else if (ps + pl != plen) {
                    fail(AU_COVER);
                }
                if (pos & neg) fail(AU_OVERLAP);
                if ((pos | neg) == 0u) fail(AU_ZERO);
                if (h < 16 && ((pos | neg) >> h) != 0u) fail(AU_HEIGHT);
                if (bitwidth == RSR_BINARY && neg != 0u) fail(AU_NEG_BINARY);
                // columns of the group (only when its range lies inside the cell)
                if (pl >= 1 && ps + pl <= plen) {
                    int64_t prev = -1;
                    for (int64_t j = ps; j < ps + pl; ++j) {
                        const int64_t col = perm[p0 + j];
                        if (col >= tn) {
                            fail(AU_COLUMN_RANGE);
                            continue;
                        }
                        if (col <= prev) fail(AU_COLUMN_ORDER);
                        prev = col;
                        const uint32_t bit = 1u << (col & 31);
                        if (atomicOr(&seen[col >> 5], bit) & bit) fail(AU_DUPLICATE);
                    }
                }
            }
        }
        const unsigned cell_worst = __reduce_min_sync(RSR_FULL_MASK, worst);
        if (lane == 0 && cell_worst != 0xFFu)
            atomicMin(result, ((unsigned long long)c << 8) | cell_worst);
        __syncwarp();
    }
}

__global__ void reconstruct_kernel(const uint64_t *__restrict__ words,
                                   const int64_t *__restrict__ go,
                                   const uint16_t *__restrict__ perm,
                                   const int64_t *__restrict__ po, int64_t m, int64_t n, int k,
                                   int bitwidth, int64_t tw, int64_t bc, int64_t tc,
                                   int64_t row_bytes, uint32_t *__restrict__ packed32) {
    const uint32_t lane = lane_id();
    const int64_t cells = bc * tc;
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < cells;
         c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = c / bc, b = c - t * bc;
        const int64_t col0 = t * tw, r0 = b * k;
        const int h = (int)min((int64_t)k, m - r0);
        for (int64_t g = go[c]; g < go[c + 1]; ++g) {
            const uint64_t w = words[g];
            const int64_t ps = (int64_t)(w & 0xFFFFu), pl = (int64_t)((w >> 16) & 0xFFFFu);
            const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFFu), neg = (uint32_t)(w >> 48);
            for (int64_t j = lane; j < pl; j += 32) {
                const int64_t col = col0 + perm[po[c] + ps + j];
                for (int i = 0; i < h; ++i) {
                    uint32_t code = ((pos >> i) & 1u) ? 1u : (((neg >> i) & 1u) ? 2u : 0u);
                    if (!code) continue;
                    int64_t byte, sh;
                    if (bitwidth == RSR_BINARY) {
                        byte = (r0 + i) * row_bytes + (col >> 3);
                        sh = col & 7;
                    } else {
                        byte = (r0 + i) * row_bytes + (col >> 2);
                        sh = 2 * (col & 3);
                    }
                    atomicOr(packed32 + (byte >> 2), code << (8 * (byte & 3) + sh));
                }
            }
        }
    }
}

}  // namespace rsr

using namespace rsr;

extern "C" {

rsr_status rsr_audit(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                     const int64_t *po, int64_t m, int64_t n, int32_t k, int32_t bitwidth,
                     int64_t tile_width, int64_t block_count, int64_t tile_count,
                     unsigned long long *result, rsr_stream_t stream) {
    if (!go || !po || !result || m < 1 || n < 1 || k < 1 || k > 16 || tile_width < 1 ||
        tile_width > AU_MAX_TN || block_count < 1 || tile_count < 1)
        return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(result, 0xFF, sizeof(unsigned long long), s);
    const int64_t cells = block_count * tile_count;
    const size_t smem = (size_t)AU_WARPS * (AU_MAX_TN / 32) * 4;
    cudaFuncSetAttribute(audit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)std::min<int64_t>((cells + AU_WARPS - 1) / AU_WARPS,
                                            (int64_t)sm_count() * 4);
    audit_kernel<<<grid, AU_WARPS * 32, smem, s>>>(words, go, perm, po, m, n, k, bitwidth,
                                                   tile_width, block_count, tile_count, result);
    return launch_status();
}

size_t rsr_reconstruct_bytes(int64_t m, int64_t n, int32_t bitwidth) {
    const int64_t rb = bitwidth == RSR_BINARY ? (n + 7) / 8 : (n + 3) / 4;
    return (size_t)((m * rb + 3) & ~(int64_t)3);
}

rsr_status rsr_reconstruct(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                           const int64_t *po, int64_t m, int64_t n, int32_t k, int32_t bitwidth,
                           int64_t tile_width, int64_t block_count, int64_t tile_count,
                           uint8_t *packed, rsr_stream_t stream) {
    if (!go || !po || !packed || m < 1 || n < 1 || k < 1 || tile_width < 1) return RSR_ERR_INVALID;
    if (((uintptr_t)packed & 3) != 0) return RSR_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t rb = bitwidth == RSR_BINARY ? (n + 7) / 8 : (n + 3) / 4;
    cudaMemsetAsync(packed, 0, rsr_reconstruct_bytes(m, n, bitwidth), s);
    const int64_t cells = block_count * tile_count;
    const int grid = (int)std::min<int64_t>((cells * 32 + 255) / 256, (int64_t)sm_count() * 16);
    reconstruct_kernel<<<grid, 256, 0, s>>>(words, go, perm, po, m, n, k, bitwidth, tile_width,
                                            block_count, tile_count, rb, (uint32_t *)packed);
    return launch_status();
}

}  // extern "C"
