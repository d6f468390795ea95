/*
 * rsr_b200.h -- C ABI of the B200-native (sm_100a) RSR matvec library.
 *
 * Drop-in boundary for the reference package `rsrmv`'s native seam
 * (pkg/src/rsrmv/_native.py): the reference binds flat numpy arrays and
 * scalars into numba cores; this library takes flat DEVICE arrays, sizes and
 * a cudaStream_t.  No torch types cross this boundary.  Every entry point is
 * stream-ordered and never allocates; all but the *_host round trips (which
 * synchronize the stream before returning host results) never synchronize.
 * Each returns an rsr_status (0 = success).  The Python shim (paper_2603_27462_b200/_lib.py)
 * maps status codes onto the reference's exception kinds
 * (pkg/src/rsrmv/errors.py:23-74).
 *
 * Layout conventions follow the reference exactly:
 *   packed matrix : uint8[rows][row_bytes], row-major, LSB-first;
 *                   binary 1 bit/entry, ternary 2-bit codes 0->00 +1->01 -1->10
 *                   (matcore.py:24-26, :77-78, :114-125)
 *   group word    : u64 = perm_start | perm_len<<16 | pos_mask<<32 | neg_mask<<48
 *                   (_native.py:4-9, preproc.py:31-41)
 *   cells         : tile-major, cell = t * block_count + b (preproc.py:120-122)
 *
 * The multiply kernels consume a device-only "chunk stream" derived from the
 * reference arrays once per artifact (rsr_stream_build): cells in block-major
 * order, each a run of 32-byte chunks.  An entry is either a tile-local
 * column to gather or the pattern KEY of the group whose columns follow
 * (binary: pos mask; ternary: base-3 digits).  A warp round is 64 chunks and
 * lane L owns the chunk pair (2L, 2L+1), so any lane can start decoding at a
 * pair boundary without knowing what came before it.  See DESIGN.md.
 */
#ifndef RSR_B200_H
#define RSR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *rsr_stream_t; /* a cudaStream_t */

typedef enum {
    RSR_OK = 0,
    RSR_ERR_TILE_TOO_WIDE = 1,  /* a group longer than 65535 columns (preproc.py:271-276) */
    RSR_ERR_K_TOO_LARGE = 2,    /* k above 16 binary / 10 ternary (preproc.py:102-103) */
    RSR_ERR_INVALID = 3,        /* bad argument (shape, null pointer, dtype) */
    RSR_ERR_DIMENSION = 4,      /* vector length != columns (kernels.py:52-56) */
    RSR_ERR_CUDA = 5,           /* a CUDA launch failed; see rsr_last_cuda_error() */
    RSR_ERR_WORKSPACE = 6       /* workspace smaller than the *_workspace_bytes() query */
} rsr_status;

typedef enum { RSR_BINARY = 0, RSR_TERNARY = 1 } rsr_bitwidth;

/* Element types of vectors crossing the boundary. */
typedef enum {
    RSR_F32 = 0,
    RSR_BF16 = 1,
    RSR_F16 = 2,
    RSR_I8 = 3,
    RSR_I32 = 4,
    RSR_F64 = 5   /* rsr_absmax_quantize only (reference float64 activations) */
} rsr_dtype;

/* Device view of a matrix's chunk stream (built by rsr_stream_build). */
typedef struct {
    int64_t m, n;              /* rows, cols */
    int32_t k, bitwidth;       /* block height, rsr_bitwidth */
    int64_t tile_width, block_count, tile_count;
    int32_t format;            /* rsr_stream_format(): 0 u16, 1 u16 scaled, 2 u32 */
    int32_t chunk;             /* entries per 32-byte chunk: 16 (u16) or 8 (u32) */
    const void *entries;       /* device chunk stream */
    const int64_t *e_off;      /* device, cells+1 entry offsets, block-major cell order */
    int64_t row_begin_block;   /* first block this view covers (row-block sharding) */
    int64_t n_blocks;          /* blocks covered (== block_count unless sharded) */
    const uint32_t *col0_key;  /* device, per cell (block-major): pattern key of the
                                  tile's column 0 (u16 formats; NULL for format 2) */
    int32_t device;            /* CUDA device ordinal holding the arrays; launches
                                  switch to it (and back) when it is not current;
                                  -1 = the current device */
} rsr_stream_view;

/* ---- library info ---------------------------------------------------- */
const char *rsr_version(void);
const char *rsr_last_cuda_error(void);
int rsr_device_sm_count(int device);

/* ---- offline preprocessing ------------------------------------------------
 * Replaces preproc.preprocess's per-cell loop over
 * _native.group_block_{binary,ternary} (preproc.py:239-289,
 * _native.py:25-161).  Two phases so the caller can size the outputs:
 *   1. rsr_group_count: per-cell group / retained counts, exclusive-scanned
 *      into go[cells+1] and po[cells+1] (int64, device), plus per-cell
 *      sort_steps exactly as the reference tallies them.  *status_dev
 *      (int32, device) receives RSR_ERR_TILE_TOO_WIDE when any group would
 *      exceed 65535 columns.
 *   2. rsr_group_fill: words[go[cells]] and perm[po[cells]], byte-identical to
 *      the reference artifact.
 * data is the packed matrix on the device (uint8[rows][row_bytes]).       */
size_t rsr_group_workspace_bytes(int64_t rows, int64_t cols, int32_t bitwidth, int32_t k,
                                 int64_t tile_width);
rsr_status rsr_group_count(const uint8_t *data, int64_t rows, int64_t cols, int64_t row_bytes,
                           int32_t bitwidth, int32_t k, int64_t tile_width,
                           int64_t *go, int64_t *po, int64_t *sort_steps, int32_t *status_dev,
                           void *workspace, size_t workspace_bytes, rsr_stream_t stream);
rsr_status rsr_group_fill(const uint8_t *data, int64_t rows, int64_t cols, int64_t row_bytes,
                          int32_t bitwidth, int32_t k, int64_t tile_width,
                          const int64_t *go, const int64_t *po, uint64_t *words, uint16_t *perm,
                          void *workspace, size_t workspace_bytes, rsr_stream_t stream);

/* ---- chunk stream (device-only multiply format) ------------------------------
 * rsr_stream_count: per-cell entry counts exclusive-scanned into e_off
 * (cells+1, block-major) and each group's first slot inside its cell into
 * gslot (int32, one per reference word).  The caller reads e_off[cells] to
 * size the entries, then rsr_stream_build writes them.
 * Formats (rsr_stream_format picks one per plan):
 *   3  u16, "halfword": column*2 (byte offset of a 2-byte element), KEY*4|1,
 *      or a zero word Z + 4*bank (Z = 2*roundup(tile columns, 64)); every
 *      column in the stream, bank-matched column order (rsr_stream_h.cu)
 *                                              (tiles <= 32704, keys <= 2187)
 *   0  u16, flag bit 15: column, or KEY|0x8000   (tiles <= 32768, other k)
 *   1  u16, "scaled": column*4, or KEY*4|1 -- byte offsets straight into
 *      4-byte shared-memory elements (round-1 format; still decodable)
 *   2  u32, flag bit 31                          (anything wider / larger)
 * u16 formats use the QUAD layout: every chunk pair starts with a key, keys
 * sit only at slots = 0 mod 4, inside a pair each key starts a new group,
 * padding is column 0 (staged as zero; the tile's real column 0 is carried
 * as col0_key[cell], 0 = none), and inside each group the columns are
 * ordered to spread each round's shared-memory gathers over the 32 banks.
 * Format 2 uses the EVEN layout: every chunk starts with a key, keys at even
 * slots, padding key 0 / column 0.
 * Each warp round (64 chunks) is stored as four 16-byte quarters per chunk
 * pair, [quarter 0 of all pairs][quarter 1][quarter 2][quarter 3].           */
int32_t rsr_stream_format(int32_t bitwidth, int32_t k, int64_t tile_width);
rsr_status rsr_stream_count(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int32_t format, int32_t chunk, int64_t *e_off, int32_t *gslot,
                            rsr_stream_t stream);
/* col0_key: device u32[cells] (u16 formats; may be NULL for format 2).       */
rsr_status rsr_stream_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t format,
                            int32_t chunk, const int64_t *e_off, const int32_t *gslot,
                            void *entries, uint32_t *col0_key, rsr_stream_t stream);

/* ---- online multiply --------------------------------------------------------
 * rsr_matvec: y (+)= A . v  over the view's row blocks.
 *   v dtype RSR_I8  -> y int32, exact   (replaces _native.matvec_i8 /
 *                                        matvec_i8_par, _native.py:167-285)
 *   v dtype F32/BF16/F16 -> y float32, fp32 accumulation (replaces
 *                                        _native.matvec_f32, _native.py:214-242)
 * y holds rows [row_begin_block*k, ...) of the full output; accumulate=0
 * overwrites, 1 adds (the reference cores add into caller-zeroed y).
 * workspace: rsr_matvec_workspace_bytes(view) bytes of device scratch
 * (only needed when tile_count > 1).                                         */
size_t rsr_matvec_workspace_bytes(const rsr_stream_view *view);
rsr_status rsr_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype, void *y,
                      int32_t accumulate, void *workspace, size_t workspace_bytes,
                      rsr_stream_t stream);

/* rsr_matvec_peers: rsr_matvec fused with the sharded path's all-gather
 * (SURVEY 8e): the multiply's epilogue (or, with tile_count > 1, its tile
 * finalize) stores every output row of the view to each of npeers buffers
 * instead of one y.  y_peers is a DEVICE array of npeers pointers, each to
 * this view's first row inside one rank's full output buffer -- peer memory
 * mapped into this device's address space (e.g. torch symmetric memory),
 * this rank's own buffer included.  No accumulate.  Stream-ordered like
 * rsr_matvec; the caller synchronizes the ranks (a barrier over the same
 * peers) before any rank reads its full output.  Replaces rsr_matvec +
 * ncclAllGather of the y slices.                                            */
rsr_status rsr_matvec_peers(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                            void *const *y_peers, int32_t npeers, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream);

/* rsr_matvec_host: the synchronous host-buffer form behind the Python API's
 * numpy path -- copies v_host (n elements of v_dtype; pinned memory for full
 * speed) to dev_v, multiplies into dev_y, copies the view's rows back to
 * y_host and synchronizes the stream.  Page-locked (device-mapped) host
 * buffers are copied by small kernels over the host link; pageable ones by
 * cudaMemcpyAsync.                                                          */
rsr_status rsr_matvec_host(const rsr_stream_view *view, const void *v_host, int32_t v_dtype,
                           void *y_host, void *dev_v, void *dev_y, void *workspace,
                           size_t workspace_bytes, rsr_stream_t stream);

/* rsr_fused_matvec_host: rsr_fused_matvec (float32 output) with host
 * buffers, as rsr_matvec_host -- the numpy path of rsr_matvec_fused and of
 * Multiplier("RsrTernary").multiply (reference kernels.py:105-125, :215).    */
rsr_status rsr_fused_matvec_host(const rsr_stream_view *view, const void *v_host, int32_t v_dtype,
                                 double beta, void *y_host, void *dev_v, void *dev_y,
                                 void *workspace, size_t workspace_bytes, rsr_stream_t stream);

/* rsr_fused_matvec: absmax-quantize v (float64 math, half away from zero,
 * +-127), exact int32 multiply, out[i] = f32(f64(y_i) * (beta / scale)).
 * Bit-identical to _native.fused_matvec (_native.py:339-353).  The
 * quantization is fused into every CTA's prologue (no separate pass).
 * row_beta (device f64[m], may be NULL): per-row beta for stacked siblings
 * (kernels.batched_preprocess, kernels.py:128-160) -- each sibling's rows get
 * exactly its own f32(f64(y_i) * (beta_j / scale)).  out_dtype RSR_F32 or
 * RSR_BF16 (bf16 = round-to-nearest-even of that f32).  scale_out (device
 * f64, may be NULL) receives the activation scale.                         */
rsr_status rsr_fused_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                            double beta, const double *row_beta, void *out, int32_t out_dtype,
                            double *scale_out, void *workspace, size_t workspace_bytes,
                            rsr_stream_t stream);

/* rsr_fused_matvec_norm: rsr_fused_matvec of the RMS-normalized vector
 * (BitNet's BitLinear = RMSNorm + absmax quantization + ternary product, with
 * the norm of HF BitNetRMSNorm: x * rsqrt(mean(x^2) + eps) rounded to bf16,
 * times the bf16 weight norm_w, rounded to bf16) in ONE launch.  bf16 v of
 * one tile (n % 8 == 0, 16-byte aligned v and norm_w); the mean of squares
 * is an fp32 sum in a fixed order (it may differ from torch's reduction in
 * the last bit).  Out: as rsr_fused_matvec; no scale output.              */
rsr_status rsr_fused_matvec_norm(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                                 const void *norm_w, float norm_eps, double beta,
                                 const double *row_beta, void *out, int32_t out_dtype,
                                 void *workspace, size_t workspace_bytes, rsr_stream_t stream);

/* rsr_rmsnorm_rows: out[r] = the norm of rsr_fused_matvec_norm applied to
 * each bf16 row x[r] (rows x n, contiguous) with bf16 weight w -- a single
 * launch per norm (the dense arm of the decode comparison uses it).        */
rsr_status rsr_rmsnorm_rows(const void *x, const void *w, int64_t rows, int64_t n, float eps,
                            void *out, rsr_stream_t stream);

/* ---- batched multi-vector multiply (not in the reference) ----
 * rsr_matmul: Y[b] = A . V[b] for b < B, over the view's row blocks.
 *   V: B vectors, element (b, col) at V[b*ldv + col] (ldv >= n);
 *   Y: element (b, row) at Y[b*ldy + row], rows of the view (ldy >= rows).
 *   v_dtype RSR_I8 -> Y int32 (exact); F32/BF16/F16 -> Y float32 (fp32 sums,
 *   the single-vector float tolerance).  u16 stream formats only (tiles <=
 *   32768 columns, <= 2187 pattern keys); other views return
 *   RSR_ERR_INVALID and the caller multiplies column by column.
 * workspace: rsr_matmul_workspace_bytes(view, B) (only when tile_count > 1). */
size_t rsr_matmul_workspace_bytes(const rsr_stream_view *view, int32_t B);
rsr_status rsr_matmul(const rsr_stream_view *view, const void *V, int32_t v_dtype, int64_t ldv,
                      int32_t B, void *Y, int64_t ldy, void *workspace, size_t workspace_bytes,
                      rsr_stream_t stream);

/* ---- batched fused path (prefill: T activation rows, one stacked linear) -----
 * rsr_absmax_quantize_rows: Q[t] (int8, row stride ldq) and scales[t] (f64)
 * = the reference absmax quantization of each row V[t] (_native.py:313-336).
 * rsr_matmul then gives the exact int32 products; rsr_dequant_rows writes
 * out[t][i] = f32(f64(Y[t][i]) * (beta_i / scales[t])) (beta_i = row_beta[i]
 * when row_beta is non-NULL, else beta; bf16 = RNE of that f32) -- row by row
 * the single-vector rsr_fused_matvec result, bit for bit.  norm_w (bf16
 * rows only, may be NULL): each row first goes through the fused RMSNorm of
 * rsr_fused_matvec_norm.                                                    */
rsr_status rsr_absmax_quantize_rows(const void *V, int32_t v_dtype, int64_t ldv, int64_t rows,
                                    int64_t n, const void *norm_w, float norm_eps, int8_t *Q,
                                    int64_t ldq, double *scales, rsr_stream_t stream);
rsr_status rsr_dequant_rows(const int32_t *Y, int64_t ldy, int64_t rows, int64_t m,
                            const double *scales, const double *row_beta, double beta, void *out,
                            int32_t out_dtype, int64_t ldo, rsr_stream_t stream);

/* ---- batched multiply on the tensor cores (tcgen05) ---------------------------
 * For bf16 batches the pattern-table expansion runs on the tensor cores: the
 * code matrix holds every column's pattern key as 2-bit row codes (the
 * reference pattern_key code form, preproc.py:183-197: +1 -> 01, -1 -> 10;
 * k <= 16), one row at a time: u32 [ceil(cols/128)][round8(bc*k)][8], word q
 * of a (step, row) = columns 16q .. 16q + 15, the codes of column pair j at
 * bits 2 (j % 4) of bytes 2 (j / 4) (even column) and 2 (j / 4) + 1 (odd);
 * built once from the reference arrays (tile-major cells, as rsr_group_fill
 * writes them; rsr_keymat_bytes / rsr_keymat_build; 16-byte aligned).
 * rsr_matmul_tc: Y[b] (f32, rows of blocks [block_begin, +n_blocks)) =
 * A . V[b] for bf16 V[b*ldv + col], B <= 256, V 16-byte aligned and ldv a
 * multiple of 8 (the B tiles are TMA boxes of V; RSR_ERR_INVALID otherwise);
 * fp32 accumulation of exact +-1 products (the float-path tolerance; the
 * split-K sum order is fixed, so results are deterministic).  Split-K runs
 * inside thread-block clusters (partials summed through distributed shared
 * memory); the workspace argument is kept for ABI stability and not used
 * (rsr_matmul_tc_workspace_bytes returns 256).                              */
size_t rsr_keymat_bytes(int64_t block_count, int64_t cols, int32_t bitwidth, int32_t k);
rsr_status rsr_keymat_build(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                            const int64_t *po, int64_t block_count, int64_t tile_count,
                            int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                            void *keymat, rsr_stream_t stream);
size_t rsr_matmul_tc_workspace_bytes(int64_t m, int64_t n, int32_t k, int64_t block_begin,
                                     int64_t n_blocks, int32_t B);
/* int8 batches on tcgen05 kind::i8 (s8 x s8 -> s32, exact): the same code
 * matrix in the int8 path's order (rsr_keymat_build_i8, the size
 * rsr_keymat_bytes gives -- it is sized for this layout): 256-column steps,
 * u32 [ceil(cols/256)][round8(bc*k)][16], column 4w + i of a 16-column word
 * in nibble i + 4 (w / 2) at bit offset 2 (w % 2) (the bf16 layout uses a
 * prefix of the same size); rsr_matmul_tc_i8: Y[b] (int32) = A . V[b] for int8
 * V[b*ldv + col] (V 16-byte aligned, ldv a multiple of 16), bit-exact with
 * the integer path of rsr_matvec per column.                                */
/* rsr_keymat_build_wide / rsr_matmul_tc_wide: bf16 batches of B <= 32 with
 * 256-column pipeline steps (half the per-step commits and barriers of
 * rsr_matmul_tc): the code matrix in the int8 path's layout (256-column
 * steps, rsr_keymat_bytes) with the bf16 path's bit order.  Same arguments,
 * results and determinism as rsr_matmul_tc.                                 */
rsr_status rsr_keymat_build_wide(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                                 const int64_t *po, int64_t block_count, int64_t tile_count,
                                 int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                                 void *keymat_wide, rsr_stream_t stream);
rsr_status rsr_matmul_tc_wide(const void *keymat_wide, int64_t m, int64_t n, int32_t bitwidth,
                              int32_t k, int64_t block_begin, int64_t n_blocks, const void *V,
                              int32_t v_dtype, int64_t ldv, int32_t B, float *Y, int64_t ldy,
                              void *workspace, size_t workspace_bytes, rsr_stream_t stream);

rsr_status rsr_keymat_build_i8(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                               const int64_t *po, int64_t block_count, int64_t tile_count,
                               int64_t tile_width, int64_t cols, int32_t bitwidth, int32_t k,
                               void *keymat_i8, rsr_stream_t stream);
rsr_status rsr_matmul_tc_i8(const void *keymat_i8, int64_t m, int64_t n, int32_t bitwidth,
                            int32_t k, int64_t block_begin, int64_t n_blocks, const int8_t *V,
                            int64_t ldv, int32_t B, int32_t *Y, int64_t ldy, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream);
/* The same multiply with rsr_dequant_rows fused into its epilogue (batched
 * fused prefill: rsr_absmax_quantize_rows -> this): out[t][i] =
 * f32(f64(y[t][i]) * (beta_i / scales[t])) (beta_i = row_beta[i] or beta;
 * out f32 or bf16 = RNE of that f32), row for row the single-vector
 * rsr_fused_matvec result.                                                  */
rsr_status rsr_matmul_tc_i8_dequant(const void *keymat_i8, int64_t m, int64_t n,
                                    int32_t bitwidth, int32_t k, int64_t block_begin,
                                    int64_t n_blocks, const int8_t *Q, int64_t ldq, int32_t B,
                                    const double *scales, const double *row_beta, double beta,
                                    void *out, int32_t out_dtype, int64_t ldo, void *workspace,
                                    size_t workspace_bytes, rsr_stream_t stream);
rsr_status rsr_matmul_tc(const void *keymat, int64_t m, int64_t n, int32_t bitwidth, int32_t k,
                         int64_t block_begin, int64_t n_blocks, const void *V, int32_t v_dtype,
                         int64_t ldv, int32_t B, float *Y, int64_t ldy, void *workspace,
                         size_t workspace_bytes, rsr_stream_t stream);

/* ---- device weight conversion ------------------------------------------------
 * matcore.ternarize_weights + encode (matcore.py:151-173, :114-125) for a
 * weight matrix already on the device (f32/bf16/f16, row-major rows x cols):
 * *beta_out (device f64) = mean|w| (1.0 if zero); packed (device u8,
 * rows x ceil(cols/4)) = 2-bit codes of clamp(round_half_away(w/beta), -1, 1).
 * The |w| sum is a fixed-shape two-level reduction (deterministic; its
 * rounding may differ from numpy's pairwise sum in the last bits).          */
size_t rsr_ternarize_workspace_bytes(void);
rsr_status rsr_ternarize_pack(const void *w, int32_t w_dtype, int64_t rows, int64_t cols,
                              uint8_t *packed, double *beta_out, void *workspace,
                              size_t workspace_bytes, rsr_stream_t stream);

/* Two-plane decomposition M = P - N of a packed ternary matrix (SURVEY 8a
 * P7): planes (device u8, 2*rows x ceil(cols/8)) receives P = [M == +1] in
 * rows [0, rows) and N = [M == -1] in rows [rows, 2*rows), binary-packed as
 * the reference packs binary matrices (matcore.py:114-125).                */
rsr_status rsr_split_planes(const uint8_t *ternary, int64_t rows, int64_t cols, int64_t row_bytes,
                            uint8_t *planes, rsr_stream_t stream);

/* Synthetic ternary rows [row0, row0+rows) of a cols-wide matrix, packed, for
 * configs too large for the reference's numpy generator (C5, 131072^2):
 * entry (r, c) = +1/-1/0 with p = density/2, density/2, 1-density from
 * splitmix64(seed, r, c).  Restated in oracle/rsr_oracle.c for CPU checks.  */
rsr_status rsr_random_ternary(int64_t row0, int64_t rows, int64_t cols, uint64_t seed,
                              double density, uint8_t *packed, rsr_stream_t stream);

/* Debug: when non-NULL, subsequent multiply launches record a per-CTA
 * %globaltimer timeline into probe[cta*4 + {0: start, 1: prologue done,
 * 2: first warp done (min), 3: last warp done (max)}] (device u64; slots 2/3
 * must be pre-set to UINT64_MAX / 0).  NULL (default) disables it.          */
void rsr_debug_set_probe(unsigned long long *probe);

/* ---- artifact audit and inverse ---------------------------------------------
 * rsr_audit: the per-cell invariants of preproc.validate_artifact
 * (preproc.py:305-372) over the device reference arrays (tile-major cells;
 * the caller has checked the offset arrays span words / perm and never
 * decrease).  *result (device u64) = (cell << 8 | check) of the first
 * failure in cell order (check numbering: csrc/rsr_audit.cu AuditCheck), or
 * UINT64_MAX when the artifact is sound.
 * rsr_reconstruct: the packed matrix the artifact encodes (preproc.py:
 * 375-400) into `packed` (rsr_reconstruct_bytes() bytes, 4-byte aligned;
 * row-major, ceil(n/8) or ceil(n/4) bytes per row).                         */
rsr_status rsr_audit(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                     const int64_t *po, int64_t m, int64_t n, int32_t k, int32_t bitwidth,
                     int64_t tile_width, int64_t block_count, int64_t tile_count,
                     unsigned long long *result, rsr_stream_t stream);
size_t rsr_reconstruct_bytes(int64_t m, int64_t n, int32_t bitwidth);
rsr_status rsr_reconstruct(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                           const int64_t *po, int64_t m, int64_t n, int32_t k, int32_t bitwidth,
                           int64_t tile_width, int64_t block_count, int64_t tile_count,
                           uint8_t *packed, rsr_stream_t stream);

/* ---- helpers ---------------------------------------------------------------- */
/* _native.count_ops (_native.py:288-307): out3 (device int64[3]) =
 * gather adds, scatter adds, groups.                                         */
rsr_status rsr_count_ops(const uint64_t *words, int64_t n_words, int64_t *out3,
                         rsr_stream_t stream);
/* _native.absmax_quantize (_native.py:313-336) / matcore.quantize_activations
 * (matcore.py:176-194): q int8[n], *scale_out f64.  v_dtype F32/BF16/F16 or
 * F64 (float64 vectors keep their float64 values, as the reference does). */
rsr_status rsr_absmax_quantize(const void *v, int32_t v_dtype, int64_t n, int8_t *q,
                               double *scale_out, rsr_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RSR_B200_H */
