// rsr_pack.cu -- device-side weight ternarization and packing.
//
// Replaces matcore.ternarize_weights + encode for weights that already live
// on the GPU (reference matcore.py:151-173, :114-125): beta = mean|w| in
// float64 (1.0 for an all-zero matrix), q = clamp(round_half_away(w / beta),
// -1, 1), packed as 2-bit codes 0->00, +1->01, -1->10, four per byte,
// LSB-first, row-major.
#include "rsr_common.cuh"

namespace rsr {

__device__ __forceinline__ double ld_w(const void *w, int dt, int64_t i) {
    switch (dt) {
        case RSR_F32: return (double)__ldg((const float *)w + i);
        case RSR_BF16: return (double)bf16_bits_to_f32(__ldg((const uint16_t *)w + i));
        case RSR_F16: return (double)__half2float(__ldg((const __half *)w + i));
        default: return 0.0;
    }
}

// Per-block partial sums of |w| (fixed block/grid shape -> deterministic).
__global__ void abs_sum_partial_kernel(const void *w, int dt, int64_t n, double *partial) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += fabs(ld_w(w, dt, i));
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        s = warp_sum(s);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

__global__ void beta_finalize_kernel(const double *partial, int nb, int64_t n, double *beta) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nb; ++i) s += partial[i];
        const double b = s / (double)n;
        *beta = b == 0.0 ? 1.0 : b;
    }
}

// One thread per output byte (four columns of one row).
__global__ void ternarize_pack_kernel(const void *w, int dt, int64_t rows, int64_t cols,
                                      int64_t row_bytes, const double *beta_p, uint8_t *out) {
    const double beta = *beta_p;
    const int64_t total = rows * row_bytes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / row_bytes, cb = (i - r * row_bytes) * 4;
        uint32_t byte = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = cb + j;
            if (c < cols) {
                const double x = ld_w(w, dt, r * cols + c) / beta;
                const double rr = x >= 0.0 ? floor(x + 0.5) : -floor(-x + 0.5);
                const uint32_t code = rr >= 1.0 ? 1u : (rr <= -1.0 ? 2u : 0u);
                byte |= code << (2 * j);
            }
        }
        out[i] = (uint8_t)byte;
    }
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_ternarize_workspace_bytes(void) { return 1024 * sizeof(double); }

rsr_status rsr_ternarize_pack(const void *w, int32_t w_dtype, int64_t rows, int64_t cols,
                              uint8_t *packed, double *beta_out, void *workspace,
                              size_t workspace_bytes, rsr_stream_t stream) {
    if (!w || !packed || !beta_out || rows < 1 || cols < 1) return RSR_ERR_INVALID;
    if (w_dtype != RSR_F32 && w_dtype != RSR_BF16 && w_dtype != RSR_F16) return RSR_ERR_INVALID;
    if (!workspace || workspace_bytes < rsr_ternarize_workspace_bytes()) return RSR_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = 1024;
    double *partial = (double *)workspace;
    abs_sum_partial_kernel<<<nb, 256, 0, s>>>(w, w_dtype, rows * cols, partial);
    beta_finalize_kernel<<<1, 32, 0, s>>>(partial, nb, rows * cols, beta_out);
    const int64_t row_bytes = (cols + 3) / 4;
    const int64_t total = rows * row_bytes;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
    ternarize_pack_kernel<<<grid, 256, 0, s>>>(w, w_dtype, rows, cols, row_bytes, beta_out, packed);
    return launch_status();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Counter-based synthetic ternary generator for matrices too large for the
// reference's numpy generator (C5: 131072^2).  Entry (r, c) is +1 / -1 / 0
// with probabilities density/2, density/2, 1-density, decided by
// splitmix64(seed, r, c) -- restated bit-for-bit in oracle/rsr_oracle.c
// (oracle_random_ternary_rows) so sampled row strips can be checked on CPU.
namespace rsr {
__device__ __host__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__global__ void random_ternary_kernel(int64_t row0, int64_t rows, int64_t cols, int64_t row_bytes,
                                      uint64_t seed, uint64_t thr_half, uint8_t *out) {
    const int64_t total = rows * row_bytes;
    const uint64_t base = splitmix64(seed);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / row_bytes, cb = (i - r * row_bytes) * 4;
        const uint64_t rowkey = splitmix64(base ^ (uint64_t)(row0 + r));
        uint32_t byte = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = cb + j;
            if (c < cols) {
                const uint64_t h = splitmix64(rowkey + (uint64_t)c) >> 11;  // 53-bit uniform
                const uint32_t code = h < thr_half ? 1u : (h >= (1ull << 53) - thr_half ? 2u : 0u);
                byte |= code << (2 * j);
            }
        }
        out[i] = (uint8_t)byte;
    }
}
}  // namespace rsr

extern "C" rsr_status rsr_random_ternary(int64_t row0, int64_t rows, int64_t cols, uint64_t seed,
                                         double density, uint8_t *packed, rsr_stream_t stream) {
    if (!packed || rows < 1 || cols < 1 || !(density >= 0.0 && density <= 1.0))
        return RSR_ERR_INVALID;
    const int64_t row_bytes = (cols + 3) / 4;
    const uint64_t thr_half = (uint64_t)(density / 2.0 * 9007199254740992.0);  // * 2^53
    const int64_t total = rows * row_bytes;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)rsr::sm_count() * 32);
    rsr::random_ternary_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(row0, rows, cols, row_bytes,
                                                                        seed, thr_half, packed);
    return rsr::launch_status();
}

// ---- two-plane decomposition of a ternary matrix ------------
// M = P - N with P = [M == +1], N = [M == -1], both binary, written stacked:
// rows [0, rows) of `planes` are P, rows [rows, 2 rows) are N (1 bit per
// entry, LSB-first, ceil(cols/8) bytes per row: the reference's binary
// packing, matcore.py:114-125).  One thread per output byte of P and N.
namespace rsr {
__global__ void split_planes_kernel(const uint8_t *__restrict__ tern, int64_t rows, int64_t cols,
                                    int64_t tern_row_bytes, int64_t bin_row_bytes,
                                    uint8_t *__restrict__ planes) {
    const int64_t total = rows * bin_row_bytes;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / bin_row_bytes, cb = (i - r * bin_row_bytes) * 8;
        uint32_t pos = 0, neg = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = cb + j;
            if (c < cols) {
                const uint32_t code = (__ldg(tern + r * tern_row_bytes + (c >> 2)) >> (2 * (c & 3))) & 3u;
                pos |= (code == 1u ? 1u : 0u) << j;
                neg |= (code == 2u ? 1u : 0u) << j;
            }
        }
        planes[i] = (uint8_t)pos;
        planes[total + i] = (uint8_t)neg;
    }
}
}  // namespace rsr

extern "C" rsr_status rsr_split_planes(const uint8_t *ternary, int64_t rows, int64_t cols,
                                       int64_t row_bytes, uint8_t *planes, rsr_stream_t stream) {
    if (!ternary || !planes || rows < 1 || cols < 1 || row_bytes < (cols + 3) / 4)
        return RSR_ERR_INVALID;
    const int64_t brb = (cols + 7) / 8;
    const int64_t total = rows * brb;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)rsr::sm_count() * 32);
    rsr::split_planes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ternary, rows, cols, row_bytes,
                                                                      brb, planes);
    return rsr::launch_status();
}
