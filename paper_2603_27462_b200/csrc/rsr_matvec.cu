// rsr_matvec.cu -- launch logic and C ABI of the online multiply.
// The kernel itself is in rsr_mv_impl.cuh (instantiated in rsr_mv_fmt*.cu).

#include <cstdio>

#include "rsr_mv_impl.cuh"

namespace rsr {

// tc > 1: sum the tile partials in ascending tile order (the reference order).
template <int MODE>
__global__ void tile_finalize_kernel(MvParams p, int64_t rows_view) {
    using Acc = typename std::conditional<MODE == MODE_FLOAT, float, int32_t>::type;
    const Acc *part = reinterpret_cast<const Acc *>(p.part);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows_view;
         r += (int64_t)gridDim.x * blockDim.x) {
        if (p.blk0 * p.k + r >= p.m_rows) continue;
        Acc s = (Acc)0;
        for (int64_t t = 0; t < p.tc; ++t) s += part[t * rows_view + r];
        if (MODE == MODE_FLOAT) {
            float *y = reinterpret_cast<float *>(p.y);
            put_row<float>(p, r, p.accumulate ? y[r] + (float)s : (float)s);
        } else if (MODE == MODE_INT) {
            int32_t *y = reinterpret_cast<int32_t *>(p.y);
            put_row<int32_t>(p, r, p.accumulate ? y[r] + (int32_t)s : (int32_t)s);
        } else {
            const double beta = p.row_beta ? p.row_beta[p.blk0 * p.k + r] : p.beta;
            const float o = (float)((double)s * (beta / *p.scale_dev));
            if (p.out_bf16) put_row<__nv_bfloat16>(p, r, __float2bfloat16_rn(o));
            else put_row<float>(p, r, o);
        }
    }
}

// FMT_U32 (tiles wider than 32768 columns): v converted/quantized once into
// global scratch; the multiply gathers it through L1/L2.
__global__ void stage_global_kernel(const void *v, int dtype, int64_t n, int mode, void *out,
                                    double *scale_dev) {
    double scale = 1.0;
    if (mode == MODE_FUSED) {
        const double amax = cta_absmax(v, dtype, n);
        scale = amax == 0.0 ? 1.0 : 127.0 / amax;
        if (blockIdx.x == 0 && threadIdx.x == 0) *scale_dev = scale;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (mode == MODE_FLOAT) ((float *)out)[i] = load_as_f32(v, dtype, i);
        else if (mode == MODE_INT) ((int8_t *)out)[i] = ((const int8_t *)v)[i];
        else ((int8_t *)out)[i] = quantize_one(load_as_f32(v, dtype, i), scale);
    }
}

// float64 vectors (matcore.quantize_activations keeps numpy float64 values).
__global__ void absmax_quantize_f64_kernel(const double *v, int64_t n, int8_t *q,
                                           double *scale_out) {
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x = fabs(v[i]);
        a = x > a ? x : a;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
        a = o > a ? o : a;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a = red[w] > a ? red[w] : a;
    const double scale = a == 0.0 ? 1.0 : 127.0 / a;
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double xs = v[i] * scale;
        double r = xs >= 0.0 ? floor(xs + 0.5) : -floor(-xs + 0.5);
        r = r > 127.0 ? 127.0 : (r < -127.0 ? -127.0 : r);
        q[i] = (int8_t)(int)r;
    }
}

__global__ void absmax_quantize_kernel(const void *v, int dtype, int64_t n, int8_t *q,
                                       double *scale_out) {
    const double amax = cta_absmax(v, dtype, n);
    const double scale = amax == 0.0 ? 1.0 : 127.0 / amax;
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        q[i] = quantize_one(load_as_f32(v, dtype, i), scale);
}

// ---------------------------------------------------------------------------
// host-side dispatch

static unsigned long long *g_probe = nullptr;  // debug timeline buffer (off by default)

static rsr_status check_view(const rsr_stream_view *vw) {
    if (!vw || !vw->entries || !vw->e_off) return RSR_ERR_INVALID;
    if (vw->k < 1 || vw->k > 16 || vw->m < 1 || vw->n < 1 || vw->tile_count < 1 ||
        vw->n_blocks < 0 || vw->tile_width < 1)
        return RSR_ERR_INVALID;
    if (vw->bitwidth != RSR_BINARY && vw->bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    if (vw->format != rsr_stream_format(vw->bitwidth, vw->k, vw->tile_width))
        return RSR_ERR_INVALID;
    if (vw->chunk != (vw->format == FMT_U32 ? 8 : 16)) return RSR_ERR_INVALID;
    if (vw->format != FMT_U32 && !vw->col0_key) return RSR_ERR_INVALID;
    return RSR_OK;
}

// workspace: [tile partials][16B: fused scale][staged v (FMT_U32)]
static size_t part_bytes(const rsr_stream_view *vw) {
    return vw->tile_count <= 1 ? 0
                               : (((size_t)vw->tile_count * vw->n_blocks * vw->k * 4 + 15) & ~15);
}
static size_t ws_bytes_for(const rsr_stream_view *vw) {
    size_t b = part_bytes(vw) + 16;
    if (vw->format == FMT_U32) b += (size_t)vw->n * 4;
    return b;
}

template <int MODE>
static rsr_status launch_mv(const rsr_stream_view *vw, const void *v, int vdtype, void *y,
                            int accumulate, double beta, double *scale_out, void *ws,
                            size_t ws_bytes, cudaStream_t s, const double *row_beta = nullptr,
                            int out_bf16 = 0, const uint16_t *norm_w = nullptr,
                            float norm_eps = 0.f, void *const *y_peers = nullptr,
                            int npeers = 0) {
    rsr_status st = check_view(vw);
    if (st != RSR_OK) return st;
    if (!v || (!y && !npeers)) return RSR_ERR_INVALID;
    if (npeers && (!y_peers || npeers < 0 || accumulate)) return RSR_ERR_INVALID;
    if (vw->n_blocks == 0) return RSR_OK;
    DeviceGuard guard(vw->device);
    const bool need_ws = vw->tile_count > 1 || vw->format == FMT_U32;
    if (need_ws && (ws_bytes < ws_bytes_for(vw) || !ws)) return RSR_ERR_WORKSPACE;
    MvParams p;
    p.entries = vw->entries;
    p.e_off = vw->e_off;
    p.col0_key = vw->col0_key;
    p.m_rows = vw->m;
    p.n = vw->n;
    p.tw = vw->tile_width;
    p.tc = vw->tile_count;
    p.blk0 = vw->row_begin_block;
    p.nblk = vw->n_blocks;
    p.k = vw->k;
    p.bitwidth = vw->bitwidth;
    p.nkeys = (int)bucket_count(vw->bitwidth, vw->k);
    p.v = v;
    p.vdtype = vdtype;
    p.y = y;
    p.accumulate = accumulate;
    p.part = ws;
    p.beta = beta;
    p.row_beta = row_beta;
    p.out_bf16 = out_bf16;
    p.norm_w = norm_w;
    p.norm_eps = norm_eps;
    p.y_peers = y_peers;
    p.npeers = npeers;
    p.scale_dev = scale_out;
    p.probe = g_probe;
    {
        static const int dbg = getenv("RSR_MV_DEBUG") ? atoi(getenv("RSR_MV_DEBUG")) : 0;
        p.dbg = dbg;
        static const int pf = getenv("RSR_MV_PF") ? atoi(getenv("RSR_MV_PF")) : 0;
        p.pf = pf;
    }
    if (MODE == MODE_FUSED && !p.scale_dev && need_ws)
        p.scale_dev = (double *)((char *)ws + part_bytes(vw));
    p.vstaged = nullptr;
    if (vw->format == FMT_U32) {
        void *stg = (char *)ws + part_bytes(vw) + 16;
        p.vstaged = stg;
        // the fused scale is computed by one CTA so every element sees it
        stage_global_kernel<<<MODE == MODE_FUSED ? 1 : 256, 1024, 0, s>>>(v, vdtype, vw->n, MODE,
                                                                          stg, p.scale_dev);
    }
    const bool bucket = vw->format != FMT_U32 && p.nkeys <= BUCKET_MAX_KEYS;
    // format 3 stages v by kind: bf16 halfwords for bf16 vectors, f32 words
    // for f32/f16 vectors, int16 for the integer and fused paths
    const int vk = MODE == MODE_FLOAT ? (vdtype == RSR_BF16 ? VK_BF16 : VK_F32X2) : VK_I16;
    if (vw->format == FMT_H && !bucket) return RSR_ERR_INVALID;
    KernelFn fn = vw->format == FMT_H            ? pick_fmt3(MODE, vk, vw->k)
                  : vw->format == FMT_U16_SCALED ? pick_fmt1(MODE, vw->k)
                  : vw->format == FMT_U16        ? pick_fmt0(MODE, vw->k, bucket)
                                                 : pick_fmt2(MODE, vw->k);
    if (!fn) return RSR_ERR_INVALID;

    // One persistent CTA per SM (per tile) with as many warps as fit and are
    // needed.  Small matrices (few cells per SM) put a team of 2-8 warps on
    // each cell so the whole grid stays busy.
    const int sms = sm_count();
    const int64_t tn = std::min(vw->tile_width, vw->n);
    const bool ring = bucket && vw->format != FMT_U32;
    const size_t vsz = (vw->format == FMT_U16_SCALED || MODE == MODE_FLOAT) ? 4 : 1;
    size_t fixed = 0;
    if (vw->format == FMT_H) fixed += (h_image_bytes(vk, tn) + 15) & ~(size_t)15;
    else if (vw->format != FMT_U32) fixed += ((size_t)tn * vsz + 15) & ~(size_t)15;
    if (bucket) fixed += ((size_t)p.nkeys * vw->k * 4 + 15) & ~(size_t)15;
    size_t per_warp = bucket ? (size_t)p.nkeys * 4 : 0;
    if (ring) per_warp += 16 * 4;  // team exchange
    const size_t smem_cap = 227 * 1024;
    const int64_t cells_per_tile = vw->n_blocks;
    static const int ctas_per_sm = getenv("RSR_MV_CTAS_PER_SM") ? atoi(getenv("RSR_MV_CTAS_PER_SM")) : 1;
    const int64_t cta_cap = std::max<int64_t>(1, (int64_t)sms * ctas_per_sm / vw->tile_count);
    int team = 1;
    if (ring) {
        const int64_t est_rounds = std::max<int64_t>(1, (tn * 9 / 8 + 1023) / 1024);
        // (a member needs about a round of its own: est_rounds >= team + 1;
        // measured at the BitNet o-projection, 2560^2 k=5 fused: 3 rounds,
        // teams of 4 5.75 us/call vs 6.73 with teams of 2)
        while (team < 8 && cells_per_tile * team * 2 <= cta_cap * MV_MAX_WARPS &&
               est_rounds >= team + 1)
            team *= 2;
        // More cells than one wave of warps: a team size that shortens the
        // longest warp's share (makespan in cells, teams of t warps take 1/t
        // of a cell each) -- e.g. 3277 cells on 2960 warps: 2 cells per warp
        // alone, 1.25 with teams of 4.
        if (cells_per_tile > cta_cap * MV_MAX_WARPS) {
            double best = 1e30;
            for (int t = 1; t <= 8 && est_rounds >= 2 * t; t *= 2) {
                if (fixed + t * per_warp > smem_cap) break;
                const int64_t slots = cta_cap * (MV_MAX_WARPS / t * t);
                const double span = (double)((cells_per_tile * t + slots - 1) / slots) / t +
                                    0.15 * (t - 1);  // measured cost of each extra member
                if (span < best) {
                    best = span;
                    team = t;
                }
            }
        }
        static const int force_team = getenv("RSR_MV_TEAM") ? atoi(getenv("RSR_MV_TEAM")) : 0;
        if (force_team > 0) team = force_team;  // experiment knob
        while (team > 1 && fixed + team * per_warp > smem_cap) team /= 2;
    }
    int64_t warps = (cells_per_tile * team + cta_cap - 1) / cta_cap;
    warps = (warps + team - 1) / team * team;
    warps = std::max<int64_t>(team, std::min<int64_t>(warps, MV_MAX_WARPS / team * team));
    if (norm_w) {
        // the fused RMSNorm runs in the register-staged prologue: one tile,
        // bf16, 8-aligned, at most 16 elements per thread
        if (vw->tile_count != 1 || vdtype != RSR_BF16 || (tn & 7) != 0 ||
            ((uintptr_t)v & 15) != 0 || ((uintptr_t)norm_w & 15) != 0 || tn > 16 * 32 * MV_MAX_WARPS)
            return RSR_ERR_INVALID;
        const int64_t need = (tn + 511) / 512;
        if (warps < need) warps = std::min<int64_t>((need + team - 1) / team * team, MV_MAX_WARPS);
    }
    while (warps > team && fixed + warps * per_warp > smem_cap) warps -= team;
    if (fixed + warps * per_warp > smem_cap) return RSR_ERR_INVALID;
    const size_t smem = fixed + warps * per_warp;
    const int64_t teams_per_cta = warps / team;
    const int64_t ctas_per_tile =
        std::min<int64_t>(cta_cap, (cells_per_tile + teams_per_cta - 1) / teams_per_cta);
    p.team = team;
    {
        // raise the dynamic-smem limit once per (device, kernel), not on every launch
        static thread_local KernelFn last_fn[64];
        static thread_local size_t last_smem[64];
        static thread_local int last_dev[64];
        int dev = 0;
        cudaGetDevice(&dev);
        const size_t slot = (((uintptr_t)fn >> 4) + (size_t)dev * 7) & 63;
        // the default cap is 48 KiB minus the kernel's static shared memory
        // (the fused kernels keep 512 B of reduction scratch): raise it early
        if (smem > 46 * 1024 &&
            (last_fn[slot] != fn || last_dev[slot] != dev || last_smem[slot] < smem)) {
            const cudaError_t e =
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return launch_status();
            last_fn[slot] = fn;
            last_dev[slot] = dev;
            last_smem[slot] = smem;
        }
    }
    dim3 grid((unsigned)ctas_per_tile, (unsigned)vw->tile_count);
    static const bool dbg_launch = getenv("RSR_DEBUG_LAUNCH") != nullptr;
    if (dbg_launch) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, fn);
        fprintf(stderr,
                "rsr launch mode=%d fmt=%d k=%d grid=(%u,%u) block=%d smem=%zu team=%d | "
                "maxThreads=%d static=%zu maxDyn=%d regs=%d local=%zu\n",
                MODE, vw->format, vw->k, grid.x, grid.y, (int)(warps * 32), smem, team,
                fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.numRegs,
                fa.localSizeBytes);
    }
    static const bool use_pdl = !getenv("RSR_MV_PDL") || atoi(getenv("RSR_MV_PDL")) != 0;
    static const int pdl_stream = getenv("RSR_MV_PDL_STREAM") ? atoi(getenv("RSR_MV_PDL_STREAM")) : -1;
    p.pdl = !use_pdl ? 0 : (pdl_stream >= 0 ? (pdl_stream ? 2 : 1) : (tn > 8192 ? 2 : 1));
    if (use_pdl) {
        // programmatic dependent launch: overlaps this launch's pre-wait
        // prologue with the tail of the previous multiply in the stream
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3((unsigned)(warps * 32));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, fn, p);
    } else {
        fn<<<grid, (unsigned)(warps * 32), smem, s>>>(p);
    }
    if (vw->tile_count > 1) {
        const int64_t rows_view = vw->n_blocks * vw->k;
        const int g2 = (int)std::min<int64_t>((rows_view + 255) / 256, 4096);
        tile_finalize_kernel<MODE><<<g2, 256, 0, s>>>(p, rows_view);
    }
    return launch_status();
}

}  // namespace rsr

using namespace rsr;

extern "C" {

size_t rsr_matvec_workspace_bytes(const rsr_stream_view *view) {
    if (!view) return 0;
    if (view->tile_count <= 1 && view->format != FMT_U32) return 0;
    return ws_bytes_for(view);
}

rsr_status rsr_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype, void *y,
                      int32_t accumulate, void *workspace, size_t workspace_bytes,
                      rsr_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (v_dtype == RSR_I8)
        return launch_mv<MODE_INT>(view, v, v_dtype, y, accumulate, 1.0, nullptr, workspace,
                                   workspace_bytes, s);
    if (v_dtype == RSR_F32 || v_dtype == RSR_BF16 || v_dtype == RSR_F16)
        return launch_mv<MODE_FLOAT>(view, v, v_dtype, y, accumulate, 1.0, nullptr, workspace,
                                     workspace_bytes, s);
    return RSR_ERR_INVALID;
}

rsr_status rsr_matvec_peers(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                            void *const *y_peers, int32_t npeers, void *workspace,
                            size_t workspace_bytes, rsr_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (npeers < 1 || !y_peers) return RSR_ERR_INVALID;
    if (v_dtype == RSR_I8)
        return launch_mv<MODE_INT>(view, v, v_dtype, nullptr, 0, 1.0, nullptr, workspace,
                                   workspace_bytes, s, nullptr, 0, nullptr, 0.f, y_peers, npeers);
    if (v_dtype == RSR_F32 || v_dtype == RSR_BF16 || v_dtype == RSR_F16)
        return launch_mv<MODE_FLOAT>(view, v, v_dtype, nullptr, 0, 1.0, nullptr, workspace,
                                     workspace_bytes, s, nullptr, 0, nullptr, 0.f, y_peers,
                                     npeers);
    return RSR_ERR_INVALID;
}

rsr_status rsr_fused_matvec_norm(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                                 const void *norm_w, float norm_eps, double beta,
                                 const double *row_beta, void *out, int32_t out_dtype,
                                 void *workspace, size_t workspace_bytes, rsr_stream_t stream) {
    if (!norm_w || out_dtype != RSR_F32 && out_dtype != RSR_BF16) return RSR_ERR_INVALID;
    if (view && view->bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    return launch_mv<MODE_FUSED>(view, v, v_dtype, out, 0, beta, nullptr, workspace,
                                 workspace_bytes, (cudaStream_t)stream, row_beta,
                                 out_dtype == RSR_BF16, (const uint16_t *)norm_w, norm_eps);
}

rsr_status rsr_fused_matvec(const rsr_stream_view *view, const void *v, int32_t v_dtype,
                            double beta, const double *row_beta, void *out, int32_t out_dtype,
                            double *scale_out, void *workspace, size_t workspace_bytes,
                            rsr_stream_t stream) {
    if (v_dtype != RSR_F32 && v_dtype != RSR_BF16 && v_dtype != RSR_F16) return RSR_ERR_INVALID;
    if (out_dtype != RSR_F32 && out_dtype != RSR_BF16) return RSR_ERR_INVALID;
    if (view && view->bitwidth != RSR_TERNARY) return RSR_ERR_INVALID;
    return launch_mv<MODE_FUSED>(view, v, v_dtype, out, 0, beta, scale_out, workspace,
                                 workspace_bytes, (cudaStream_t)stream, row_beta,
                                 out_dtype == RSR_BF16);
}

// Host-buffer multiply for the synchronous API: H2D copy of v, the multiply,
// D2H copy of y, stream sync -- one call instead of one per step.
//
// Page-locked host buffers are mapped into the device address space (UVA),
// so the two copies run as small kernels over the host link instead of DMA
// memcpys: a kernel launch costs less than a copy-engine round trip at 64 KB,
// and the copy-in kernel releases the multiply early (PDL), whose pre-wait
// prologue (sign table, bucket zeroing, first stream round) then overlaps it.
// Pageable buffers keep the cudaMemcpyAsync path.
static const void *mapped_device_ptr(const void *h, int dir) {
    // experiment knob RSR_HOST_COPY_DMA: 1 both copies DMA, 2 input only, 3 output only
    static const int dma = getenv("RSR_HOST_COPY_DMA") ? atoi(getenv("RSR_HOST_COPY_DMA")) : 0;
    if (dma == 1 || (dma == 2 && dir == 0) || (dma == 3 && dir == 1)) return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return at.devicePointer;
}

// nbytes copied with 16-byte accesses when both sides allow it, bytes otherwise.
__global__ void host_link_copy_kernel(const void *__restrict__ src, void *__restrict__ dst,
                                      int64_t nbytes, int wait_prev) {
    if (wait_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
    else asm volatile("griddepcontrol.launch_dependents;");
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool vec = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
    if (vec) {
        const int64_t nv = nbytes >> 4;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int64_t i = tid; i < nv; i += stride) d4[i] = s4[i];
        const unsigned char *s1 = reinterpret_cast<const unsigned char *>(src);
        unsigned char *d1 = reinterpret_cast<unsigned char *>(dst);
        for (int64_t i = (nv << 4) + tid; i < nbytes; i += stride) d1[i] = s1[i];
    } else {
        const unsigned char *s1 = reinterpret_cast<const unsigned char *>(src);
        unsigned char *d1 = reinterpret_cast<unsigned char *>(dst);
        for (int64_t i = tid; i < nbytes; i += stride) d1[i] = s1[i];
    }
}

static void launch_host_link_copy(const void *src, void *dst, int64_t nbytes, bool after_prev,
                                  cudaStream_t s) {
    const int threads = 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nbytes / 16 + threads - 1) / threads, 64));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = after_prev ? 1 : 0;
    cudaLaunchKernelEx(&cfg, host_link_copy_kernel, src, dst, nbytes, after_prev ? 1 : 0);
}

}  // extern "C"

// copy-in, the multiply (`mv`), copy-out, stream sync
template <class Mv>
static rsr_status host_round_trip(const rsr_stream_view *view, const void *v_host, size_t vbytes,
                                  void *y_host, void *dev_v, void *dev_y, cudaStream_t s,
                                  Mv &&mv) {
    DeviceGuard guard(view->device);
    const int64_t rows =
        std::min(view->n_blocks * view->k, view->m - view->row_begin_block * view->k);
    const size_t ybytes = (size_t)rows * 4;
    const void *v_map = mapped_device_ptr(v_host, 0);
    void *y_map = const_cast<void *>(mapped_device_ptr(y_host, 1));
    if (v_map) {
        launch_host_link_copy(v_map, dev_v, (int64_t)vbytes, false, s);
    } else if (cudaMemcpyAsync(dev_v, v_host, vbytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
        return launch_status();
    }
    // (the multiply's epilogue storing y straight into the mapped buffer
    // measured slower end to end: its scattered 4-byte host writes cost the
    // host's read of the result more than the copy kernel saves)
    const rsr_status st = mv(dev_y);
    if (st != RSR_OK) return st;
    if (y_map) {
        launch_host_link_copy(dev_y, y_map, (int64_t)ybytes, true, s);
    } else if (cudaMemcpyAsync(y_host, dev_y, ybytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        return launch_status();
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return launch_status();
    return RSR_OK;
}

static size_t dtype_bytes(int32_t d) {
    return d == RSR_F32 || d == RSR_I32 ? 4 : (d == RSR_I8 ? 1 : 2);
}

extern "C" {

rsr_status rsr_matvec_host(const rsr_stream_view *view, const void *v_host, int32_t v_dtype,
                           void *y_host, void *dev_v, void *dev_y, void *workspace,
                           size_t workspace_bytes, rsr_stream_t stream) {
    if (!view || !v_host || !y_host || !dev_v || !dev_y) return RSR_ERR_INVALID;
    return host_round_trip(view, v_host, (size_t)view->n * dtype_bytes(v_dtype), y_host, dev_v,
                           dev_y, (cudaStream_t)stream, [&](void *yt) {
                               return rsr_matvec(view, dev_v, v_dtype, yt, 0, workspace,
                                                 workspace_bytes, stream);
                           });
}

rsr_status rsr_fused_matvec_host(const rsr_stream_view *view, const void *v_host, int32_t v_dtype,
                                 double beta, void *y_host, void *dev_v, void *dev_y,
                                 void *workspace, size_t workspace_bytes, rsr_stream_t stream) {
    if (!view || !v_host || !y_host || !dev_v || !dev_y) return RSR_ERR_INVALID;
    return host_round_trip(view, v_host, (size_t)view->n * dtype_bytes(v_dtype), y_host, dev_v,
                           dev_y, (cudaStream_t)stream, [&](void *yt) {
                               return rsr_fused_matvec(view, dev_v, v_dtype, beta, nullptr, yt,
                                                       RSR_F32, nullptr, workspace,
                                                       workspace_bytes, stream);
                           });
}

void rsr_debug_set_probe(unsigned long long *probe) { g_probe = probe; }

rsr_status rsr_absmax_quantize(const void *v, int32_t v_dtype, int64_t n, int8_t *q,
                               double *scale_out, rsr_stream_t stream) {
    if (!v || !q || n < 0) return RSR_ERR_INVALID;
    if (v_dtype != RSR_F32 && v_dtype != RSR_BF16 && v_dtype != RSR_F16 && v_dtype != RSR_F64)
        return RSR_ERR_INVALID;
    if (n == 0) return RSR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (int)std::min<int64_t>((n + 1023) / 1024, 64);
    if (v_dtype == RSR_F64)
        absmax_quantize_f64_kernel<<<grid, 1024, 0, s>>>((const double *)v, n, q, scale_out);
    else
        absmax_quantize_kernel<<<grid, 1024, 0, s>>>(v, v_dtype, n, q, scale_out);
    return launch_status();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Batched fused path (prefill: T activation rows through one stacked linear).
// rsr_absmax_quantize_rows quantizes each row with the reference rule
// (_native.py:313-336, float64 math, per-row scale); the int8 batch then goes
// through rsr_matmul (exact int32); rsr_dequant_rows applies
// f32(f64(y) * (beta_i / scale_t)) per (row i, vector t) -- the fused
// kernel's epilogue, so every row equals the single-vector fused result.
namespace rsr {
// element i of row vr, through the fused RMSNorm when norm_w is set (bf16 rows)
__device__ __forceinline__ float row_elem(const char *vr, int dtype, int64_t i,
                                          const uint16_t *norm_w, float rs) {
    const float x = load_as_f32(vr, dtype, i);
    if (!norm_w) return x;
    const float nx = __bfloat162float(__float2bfloat16_rn(x * rs));
    return __bfloat162float(__float2bfloat16_rn(bf16_bits_to_f32(__ldg(norm_w + i)) * nx));
}

// one CTA (1024 threads) per row; the element loops are unrolled so a
// thread's loads are in flight together (a row is only n / 1024 elements per
// thread).  max |x| is taken in f32 (exact: the conversion to f64 is exact),
// the scale in f64 (the reference rule)
constexpr int QROWS_THREADS = 1024;
__global__ void __launch_bounds__(QROWS_THREADS) absmax_quantize_rows_kernel(
    const void *V, int dtype, int64_t ldv, int64_t n, int8_t *Q, int64_t ldq, double *scales,
    const uint16_t *norm_w, float norm_eps) {
    __shared__ float red[32];
    const int64_t row = blockIdx.x;
    const char *vr = reinterpret_cast<const char *>(V) +
                     row * ldv * (dtype == RSR_F32 ? 4 : 2);
    float rs = 0.f;
    if (norm_w) {
        float ss = 0.f;
#pragma unroll 8
        for (int64_t i = threadIdx.x; i < n; i += QROWS_THREADS) {
            const float x = load_as_f32(vr, dtype, i);
            ss += x * x;
        }
        rs = rsqrtf(cta_reduce_sum_f32(ss) * (1.0f / (float)n) + norm_eps);
    }
    float a = 0.f;
#pragma unroll 8
    for (int64_t i = threadIdx.x; i < n; i += QROWS_THREADS)
        a = fmaxf(a, fabsf(row_elem(vr, dtype, i, norm_w, rs)));
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) a = fmaxf(a, __shfl_xor_sync(RSR_FULL_MASK, a, d));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    a = 0.f;
#pragma unroll
    for (int w = 0; w < QROWS_THREADS / 32; ++w) a = fmaxf(a, red[w]);
    const double amax = (double)a;
    const double scale = amax == 0.0 ? 1.0 : 127.0 / amax;
    if (threadIdx.x == 0) scales[row] = scale;
#pragma unroll 8
    for (int64_t i = threadIdx.x; i < n; i += QROWS_THREADS)
        Q[row * ldq + i] = quantize_one(row_elem(vr, dtype, i, norm_w, rs), scale);
}

__global__ void dequant_rows_kernel(const int32_t *Y, int64_t ldy, int64_t rows, int64_t m,
                                    const double *scales, const double *row_beta, double beta,
                                    void *out, int out_bf16, int64_t ldo) {
    const int64_t total = rows * m;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / m, i = e - t * m;
        const double b = row_beta ? row_beta[i] : beta;
        const float o = (float)((double)Y[t * ldy + i] * (b / scales[t]));
        if (out_bf16) reinterpret_cast<__nv_bfloat16 *>(out)[t * ldo + i] = __float2bfloat16_rn(o);
        else reinterpret_cast<float *>(out)[t * ldo + i] = o;
    }
}
}  // namespace rsr

extern "C" {

rsr_status rsr_absmax_quantize_rows(const void *V, int32_t v_dtype, int64_t ldv, int64_t rows,
                                    int64_t n, const void *norm_w, float norm_eps, int8_t *Q,
                                    int64_t ldq, double *scales, rsr_stream_t stream) {
    if (!V || !Q || !scales || rows < 0 || n < 1 || ldv < n || ldq < n) return RSR_ERR_INVALID;
    if (v_dtype != RSR_F32 && v_dtype != RSR_BF16 && v_dtype != RSR_F16) return RSR_ERR_INVALID;
    if (norm_w && v_dtype != RSR_BF16) return RSR_ERR_INVALID;
    if (rows == 0) return RSR_OK;
    absmax_quantize_rows_kernel<<<(unsigned)rows, QROWS_THREADS, 0, (cudaStream_t)stream>>>(
        V, v_dtype, ldv, n, Q, ldq, scales, (const uint16_t *)norm_w, norm_eps);
    return launch_status();
}

rsr_status rsr_dequant_rows(const int32_t *Y, int64_t ldy, int64_t rows, int64_t m,
                            const double *scales, const double *row_beta, double beta, void *out,
                            int32_t out_dtype, int64_t ldo, rsr_stream_t stream) {
    if (!Y || !scales || !out || rows < 0 || m < 1 || ldy < m || ldo < m) return RSR_ERR_INVALID;
    if (out_dtype != RSR_F32 && out_dtype != RSR_BF16) return RSR_ERR_INVALID;
    if (rows == 0) return RSR_OK;
    const int grid = (int)std::min<int64_t>((rows * m + 255) / 256, (int64_t)sm_count() * 8);
    dequant_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(Y, ldy, rows, m, scales, row_beta,
                                                                 beta, out, out_dtype == RSR_BF16,
                                                                 ldo);
    return launch_status();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Standalone fused RMSNorm (one launch per norm), the same arithmetic as the
// prologue of rsr_fused_matvec_norm: used for the dense comparison arm of the
// decode benchmark so both arms run their norms as single kernels.
namespace rsr {
__global__ void rmsnorm_rows_kernel(const uint16_t *x, const uint16_t *w, int64_t n, float eps,
                                    uint16_t *out) {
    const int64_t row = blockIdx.x;
    const uint16_t *xr = x + row * n;
    float ss = 0.f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float v = bf16_bits_to_f32(xr[i]);
        ss += v * v;
    }
    const float rs = rsqrtf(cta_reduce_sum_f32(ss) * (1.0f / (float)n) + eps);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float nx = __bfloat162float(__float2bfloat16_rn(bf16_bits_to_f32(xr[i]) * rs));
        out[row * n + i] =
            __bfloat16_as_ushort(__float2bfloat16_rn(bf16_bits_to_f32(w[i]) * nx));
    }
}
}  // namespace rsr

extern "C" rsr_status rsr_rmsnorm_rows(const void *x, const void *w, int64_t rows, int64_t n,
                                       float eps, void *out, rsr_stream_t stream) {
    if (!x || !w || !out || rows < 0 || n < 1) return RSR_ERR_INVALID;
    if (rows == 0) return RSR_OK;
    rsr::rmsnorm_rows_kernel<<<(unsigned)rows, 512, 0, (cudaStream_t)stream>>>(
        (const uint16_t *)x, (const uint16_t *)w, n, eps, (uint16_t *)out);
    return rsr::launch_status();
}
