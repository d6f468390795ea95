/*
 * rsr_oracle.c -- CPU restatement of the reference RSR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package may link or call
 * this file; it is the checker (tests/, __graft_entry__.smoke()) and the CPU
 * baseline arm of bench.py.  Each function restates one numba core of the
 * reference package `rsrmv` (pkg/src/rsrmv/_native.py) in plain C so the
 * parity tests can run at full size in seconds and so the CPU baseline can be
 * timed on the GPU box's host cores (the reference itself cannot travel).
 *
 * Parity is pinned against golden vectors produced by importing the reference
 * (tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 *
 * Conventions (reference _native.py:1-12): group words pack four u16 fields,
 * bits [0,16) perm_start, [16,32) perm_len, [32,48) pos_mask, [48,64)
 * neg_mask.  Cells are (tile, block) pairs flattened tile-major:
 * cell = t * bc + b.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Offline grouping: reference _native.py:25-88 (binary), :91-161 (ternary). */

/* Column pattern key of one column inside a block.  Binary: bit of row i is
 * weighted 2^i (_native.py:37-44).  Ternary: 2-bit code of row i weighted 4^i
 * (_native.py:100-108).  data is row-major with row_bytes per row. */
static inline uint32_t col_key(const uint8_t *data, int64_t row_bytes, int64_t r0,
                               int h, int64_t c, int ternary)
{
    uint32_t key = 0;
    if (!ternary) {
        const int64_t byte_i = c >> 3;
        const int sh = (int)(c & 7);
        for (int i = 0; i < h; ++i)
            key |= (uint32_t)((data[(r0 + i) * row_bytes + byte_i] >> sh) & 1u) << i;
    } else {
        const int64_t byte_i = c >> 2;
        const int sh = (int)((c & 3) << 1);
        for (int i = 0; i < h; ++i)
            key |= (uint32_t)((data[(r0 + i) * row_bytes + byte_i] >> sh) & 3u) << (2 * i);
    }
    return key;
}

/* Group one (tile, block) cell by a stable counting sort over the pattern
 * space.  Scratch: keys[tn], tkeys[tn], tidx[tn] (u16), counts[buckets]
 * (zeroed on entry, left zeroed).  Outputs words_out[ng], perm_out[nret].
 * Returns ng, or -1 when one group would exceed a u16 perm_len
 * (_native.py:83-84 / :155-156).  *nret_out and *steps_out receive the
 * retained-column count and the elementary step count exactly as the
 * reference tallies them (_native.py:45-81 / :109-153). */
int64_t oracle_group_block(const uint8_t *data, int64_t row_bytes, int64_t r0, int h,
                           int64_t c0, int64_t tn, int ternary,
                           uint32_t *keys, uint32_t *tkeys, uint16_t *tidx,
                           uint32_t *counts, uint64_t *words_out, uint16_t *perm_out,
                           int64_t *nret_out, int64_t *steps_out)
{
    int64_t steps = 0;
    for (int64_t j = 0; j < tn; ++j)
        keys[j] = col_key(data, row_bytes, r0, h, c0 + j, ternary);
    steps += tn;

    const int64_t dsize = ternary ? ((int64_t)1 << (2 * h)) : ((int64_t)1 << h);
    for (int64_t j = 0; j < tn; ++j)
        counts[keys[j]]++;
    steps += tn;
    uint32_t run = 0;
    for (int64_t d = 0; d < dsize; ++d) {
        uint32_t c = counts[d];
        counts[d] = run;
        run += c;
    }
    steps += dsize;
    for (int64_t j = 0; j < tn; ++j) {
        uint32_t p = counts[keys[j]]++;
        tkeys[p] = keys[j];
        tidx[p] = (uint16_t)j;
    }
    steps += tn;
    memset(counts, 0, (size_t)dsize * sizeof(uint32_t));
    steps += dsize;

    int64_t zn = 0;
    while (zn < tn && tkeys[zn] == 0) ++zn;
    int64_t ng = 0, nret = 0, j = zn;
    while (j < tn) {
        const uint32_t key = tkeys[j];
        const int64_t start = j;
        while (j < tn && tkeys[j] == key) perm_out[nret++] = tidx[j++];
        uint64_t pos, neg = 0;
        if (!ternary) {
            pos = key;
            steps += j - start + 1;
        } else {
            pos = 0;
            for (int i = 0; i < h; ++i) {
                uint32_t code = (key >> (2 * i)) & 3u;
                if (code == 1) pos |= 1ull << i;
                else if (code == 2) neg |= 1ull << i;
            }
            steps += j - start + 1 + h;
        }
        const int64_t pl = j - start;
        if (pl > 0xFFFF) {
            *nret_out = 0;
            *steps_out = steps;
            return -1;
        }
        words_out[ng++] = (uint64_t)(start - zn) | ((uint64_t)pl << 16) | (pos << 32) | (neg << 48);
    }
    *nret_out = nret;
    *steps_out = steps;
    return ng;
}

/* Whole-matrix preprocessing driver: reference preproc.py:239-289.  The
 * caller sizes words/perm by upper bounds (per cell: words <= min(tn,
 * buckets-1), perm <= tn); go/po/steps have cells+1 / cells+1 / cells
 * entries.  Returns 0, or -1 on a too-long group (TileTooWide). */
int oracle_preprocess(const uint8_t *data, int64_t rows, int64_t cols, int64_t row_bytes,
                      int ternary, int k, int64_t tw,
                      uint64_t *words, uint16_t *perm, int64_t *go, int64_t *po,
                      int64_t *steps)
{
    const int64_t bc = (rows + k - 1) / k;
    const int64_t tc = (cols + tw - 1) / tw;
    const int64_t tn_max = tw < cols ? tw : cols;
    const int64_t buckets = ternary ? ((int64_t)1 << (2 * k)) : ((int64_t)1 << k);
    uint32_t *keys = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)tn_max);
    uint32_t *tkeys = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)tn_max);
    uint16_t *tidx = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)tn_max);
    uint32_t *counts = (uint32_t *)calloc((size_t)buckets, sizeof(uint32_t));
    int rc = 0;
    int64_t cell = 0;
    go[0] = 0;
    po[0] = 0;
    for (int64_t t = 0; t < tc && rc == 0; ++t) {
        const int64_t c0 = t * tw;
        const int64_t tn = (cols - c0) < tw ? (cols - c0) : tw;
        for (int64_t b = 0; b < bc; ++b, ++cell) {
            const int64_t r0 = b * k;
            const int h = (int)((rows - r0) < k ? (rows - r0) : k);
            int64_t nret = 0, st = 0;
            int64_t ng = oracle_group_block(data, row_bytes, r0, h, c0, tn, ternary, keys, tkeys,
                                            tidx, counts, words + go[cell], perm + po[cell],
                                            &nret, &st);
            if (ng < 0) { rc = -1; break; }
            go[cell + 1] = go[cell] + ng;
            po[cell + 1] = po[cell] + nret;
            steps[cell] = st;
        }
    }
    free(keys); free(tkeys); free(tidx); free(counts);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Online multiply.  y += artifact . v (callers zero y).                     */

/* One cell of the int path: reference _native.py:185-211.  Integer sums are
 * order-free so a single accumulator gives the reference's result. */
static inline void cell_i8(const uint64_t *words, const uint16_t *perm, int64_t g0, int64_t g1,
                           int64_t p0, const int8_t *vt, int32_t *yb, int h)
{
    for (int64_t g = g0; g < g1; ++g) {
        const uint64_t w = words[g];
        const int64_t ps = (int64_t)(w & 0xFFFF), pl = (int64_t)((w >> 16) & 0xFFFF);
        const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFF), neg = (uint32_t)((w >> 48) & 0xFFFF);
        int32_t s = 0;
        const uint16_t *pp = perm + p0 + ps;
        for (int64_t j = 0; j < pl; ++j) s += (int32_t)vt[pp[j]];
        for (int i = 0; i < h; ++i)
            yb[i] += ((int32_t)((pos >> i) & 1u) - (int32_t)((neg >> i) & 1u)) * s;
    }
}

/* Reference matvec_i8 (_native.py:167-211): tiles outer, blocks inner. */
void oracle_matvec_i8(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                      const int64_t *po, const int8_t *v, int64_t n, int32_t *y, int64_t m,
                      int k, int64_t bc, int64_t tc, int64_t tw)
{
    for (int64_t t = 0; t < tc; ++t)
        for (int64_t b = 0; b < bc; ++b) {
            const int64_t base = b * k;
            const int h = (int)(base + k <= m ? k : m - base);
            const int64_t cell = t * bc + b;
            cell_i8(words, perm, go[cell], go[cell + 1], po[cell], v + t * tw, y + base, h);
        }
    (void)n;
}

/* Reference matvec_i8_par (_native.py:245-285): blocks in parallel, tiles
 * ascending inside each block, so the result is bit-identical to serial. */
void oracle_matvec_i8_par(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                          const int64_t *po, const int8_t *v, int64_t n, int32_t *y, int64_t m,
                          int k, int64_t bc, int64_t tc, int64_t tw, int threads)
{
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
    for (int64_t b = 0; b < bc; ++b) {
        const int64_t base = b * k;
        const int h = (int)(base + k <= m ? k : m - base);
        for (int64_t t = 0; t < tc; ++t) {
            const int64_t cell = t * bc + b;
            cell_i8(words, perm, go[cell], go[cell + 1], po[cell], v + t * tw, y + base, h);
        }
    }
    (void)n; (void)threads;
}

/* One cell of the float path: reference _native.py:230-242 -- float64 group
 * sums accumulated sequentially, float64 y. */
static inline void cell_f64(const uint64_t *words, const uint16_t *perm, int64_t g0, int64_t g1,
                            int64_t p0, const float *vt, double *yb, int h)
{
    for (int64_t g = g0; g < g1; ++g) {
        const uint64_t w = words[g];
        const int64_t ps = (int64_t)(w & 0xFFFF), pl = (int64_t)((w >> 16) & 0xFFFF);
        const uint32_t pos = (uint32_t)((w >> 32) & 0xFFFF), neg = (uint32_t)((w >> 48) & 0xFFFF);
        double s = 0.0;
        const uint16_t *pp = perm + p0 + ps;
        for (int64_t j = 0; j < pl; ++j) s += (double)vt[pp[j]];
        for (int i = 0; i < h; ++i)
            yb[i] += (double)((int32_t)((pos >> i) & 1u) - (int32_t)((neg >> i) & 1u)) * s;
    }
}

/* Reference matvec_f32 (_native.py:214-242).  y is float64; the caller casts
 * to float32 (kernels.py:98-102). */
void oracle_matvec_f32(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                       const int64_t *po, const float *v, int64_t n, double *y, int64_t m,
                       int k, int64_t bc, int64_t tc, int64_t tw)
{
    for (int64_t t = 0; t < tc; ++t)
        for (int64_t b = 0; b < bc; ++b) {
            const int64_t base = b * k;
            const int h = (int)(base + k <= m ? k : m - base);
            const int64_t cell = t * bc + b;
            cell_f64(words, perm, go[cell], go[cell + 1], po[cell], v + t * tw, y + base, h);
        }
    (void)n;
}

/* Block-parallel twin of oracle_matvec_f32 (no reference counterpart; the
 * reference float path is serial).  Each block's rows see the identical
 * sequence of float64 operations (tiles ascending, groups ascending), so the
 * output is bit-identical to the serial port.  Used as the multi-core CPU
 * baseline for the float metric. */
void oracle_matvec_f32_par(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                           const int64_t *po, const float *v, int64_t n, double *y, int64_t m,
                           int k, int64_t bc, int64_t tc, int64_t tw, int threads)
{
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads)
#endif
    for (int64_t b = 0; b < bc; ++b) {
        const int64_t base = b * k;
        const int h = (int)(base + k <= m ? k : m - base);
        for (int64_t t = 0; t < tc; ++t) {
            const int64_t cell = t * bc + b;
            cell_f64(words, perm, go[cell], go[cell + 1], po[cell], v + t * tw, y + base, h);
        }
    }
    (void)n; (void)threads;
}

/* Reference count_ops (_native.py:288-307): gather = sum perm_len, scatter =
 * popcount of bits 32..63, groups = number of words. */
void oracle_count_ops(const uint64_t *words, const int64_t *go, int64_t cells,
                      int64_t *gather, int64_t *scatter, int64_t *groups)
{
    int64_t g = 0, s = 0;
    for (int64_t i = 0; i < go[cells]; ++i) {
        g += (int64_t)((words[i] >> 16) & 0xFFFF);
        s += __builtin_popcountll(words[i] >> 32);
    }
    *gather = g;
    *scatter = s;
    *groups = go[cells];
}

/* Reference absmax_quantize (_native.py:313-336): float64 amax and scale,
 * round half away from zero, clamp to +-127.  Returns the scale. */
double oracle_absmax_quantize(const float *v, int64_t n, int8_t *q)
{
    double amax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs((double)v[i]);
        if (a > amax) amax = a;
    }
    const double scale = amax == 0.0 ? 1.0 : 127.0 / amax;
    for (int64_t i = 0; i < n; ++i) {
        const double x = (double)v[i] * scale;
        double r = x >= 0.0 ? floor(x + 0.5) : -floor(-x + 0.5);
        if (r > 127.0) r = 127.0;
        else if (r < -127.0) r = -127.0;
        q[i] = (int8_t)r;
    }
    return scale;
}

/* Reference fused_matvec (_native.py:339-353): quantize, serial int matvec,
 * out[i] = f32(f64(y[i]) * (beta / scale)). */
void oracle_fused_matvec(const uint64_t *words, const int64_t *go, const uint16_t *perm,
                         const int64_t *po, const float *v, int64_t n, float *out, int64_t m,
                         int k, int64_t bc, int64_t tc, int64_t tw, double beta, int threads)
{
    int8_t *q = (int8_t *)malloc((size_t)(n > 0 ? n : 1));
    int32_t *y = (int32_t *)calloc((size_t)(m > 0 ? m : 1), sizeof(int32_t));
    const double scale = oracle_absmax_quantize(v, n, q);
    if (threads == 1)
        oracle_matvec_i8(words, go, perm, po, q, n, y, m, k, bc, tc, tw);
    else /* integer sums: bit-identical to the serial reference */
        oracle_matvec_i8_par(words, go, perm, po, q, n, y, m, k, bc, tc, tw, threads);
    const double factor = beta / scale;
    for (int64_t i = 0; i < m; ++i) out[i] = (float)((double)y[i] * factor);
    free(q);
    free(y);
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Counter-based synthetic ternary rows (the device generator of
 * paper_2603_27462_b200/csrc/rsr_pack.cu, restated for sampled-strip checks
 * of the C5 config; not a reference function). */
static inline uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void oracle_random_ternary_rows(int64_t row0, int64_t rows, int64_t cols, uint64_t seed,
                                double density, uint8_t *out)
{
    const int64_t row_bytes = (cols + 3) / 4;
    const uint64_t thr_half = (uint64_t)(density / 2.0 * 9007199254740992.0);
    const uint64_t base = splitmix64(seed);
    for (int64_t r = 0; r < rows; ++r) {
        const uint64_t rowkey = splitmix64(base ^ (uint64_t)(row0 + r));
        for (int64_t b = 0; b < row_bytes; ++b) {
            uint32_t byte = 0;
            for (int j = 0; j < 4; ++j) {
                const int64_t c = b * 4 + j;
                if (c < cols) {
                    const uint64_t h = splitmix64(rowkey + (uint64_t)c) >> 11;
                    const uint32_t code = h < thr_half ? 1u : (h >= (1ull << 53) - thr_half ? 2u : 0u);
                    byte |= code << (2 * j);
                }
            }
            out[r * row_bytes + b] = (uint8_t)byte;
        }
    }
}
