// rsr_mv_kernel.cuh -- the sm_100a RSR multiply kernel (included by
// rsr_mv_impl.cuh; see that file's header for the algorithm).
#pragma once

// Experiment knobs (RSR_MV_DEBUG bits) are compiled in only with
// -DRSR_MV_EXPERIMENTS; production builds carry no extra instructions.
#ifdef RSR_MV_EXPERIMENTS
#define RSR_DBG(p, bit) ((p).dbg & (bit))
#else
#define RSR_DBG(p, bit) 0
#endif

namespace rsr {

// Streaming 16-byte load of the chunk stream: read once, not kept in L1.
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// CTA-wide max of a per-thread double (result broadcast to every thread).
__device__ __forceinline__ double cta_reduce_max(double a) {
    __shared__ double red[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
        a = o > a ? o : a;
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[warp] = a;
    __syncthreads();
    if (warp == 0) {
        a = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double o = __shfl_xor_sync(RSR_FULL_MASK, a, d);
            a = o > a ? o : a;
        }
        if (threadIdx.x == 0) red[0] = a;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}


template <int K, int MODE, int FMT, bool BUCKET, int VK = VK_DEFAULT>
__global__ void __launch_bounds__(MV_MAX_WARPS * 32)
rsr_mv_kernel(MvParams p) {
    using T = MvTypes<MODE, FMT, VK>;
    constexpr bool FH = FMT == FMT_H;
    using Acc = typename T::Acc;
    constexpr int VSZ = T::VSZ;
    constexpr bool SMEM_V = T::SMEM_V;
    constexpr int CH = FMT == FMT_U32 ? 8 : 16;  // entries per 32-byte chunk
    constexpr bool RING = FMT != FMT_U32 && BUCKET;

    extern __shared__ __align__(128) unsigned char mv_smem[];
    const int nwarps = blockDim.x >> 5;
    const int64_t t = blockIdx.y;
    const int64_t c0 = t * p.tw;
    const int64_t tn = min(p.tw, p.n - c0);
    const uint32_t lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const uint4 *__restrict__ ent4 = reinterpret_cast<const uint4 *>(p.entries);
    const int64_t bstride = (int64_t)gridDim.x * nwarps;
    const int64_t cta_id = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    auto probe = [&](int slot) {  // debug timeline: globaltimer per CTA
        if (p.probe && threadIdx.x == 0) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            p.probe[cta_id * 4 + slot] = tnow;
        }
    };
    probe(0);

    // smem: [v tile][sign table K x NB][buckets W x NB][team exchange W x 16]
    size_t off = 0;
    unsigned char *vsm = mv_smem + off;
    if constexpr (FH) off += (h_image_bytes(VK, tn) + 15) & ~(size_t)15;
    else if constexpr (SMEM_V) off += ((size_t)tn * VSZ + 15) & ~(size_t)15;
    Acc *__restrict__ stab = reinterpret_cast<Acc *>(mv_smem + off);
    if constexpr (BUCKET) off += ((size_t)p.nkeys * K * sizeof(Acc) + 15) & ~(size_t)15;
    Acc *__restrict__ buckets = reinterpret_cast<Acc *>(mv_smem + off);
    if constexpr (BUCKET) off += (size_t)nwarps * p.nkeys * sizeof(Acc);
    Acc *__restrict__ xch = reinterpret_cast<Acc *>(mv_smem + off);  // team exchange [W][16]
    Acc *bk = buckets + (size_t)warp * p.nkeys;
    const uint32_t vbase = (uint32_t)__cvta_generic_to_shared(vsm);
    // Format 3 with f32 staging (VK_F32X2): column c's word at byte
    // 4*(c/2) + (c odd ? x2h_bytes : 0), i.e. entry e = 2c maps to
    // (e & ~3) + (e & 2) * x2h_bytes / 2.  Word bits 2-6 then equal the
    // entry's, so the f32 gathers hit the banks the stream builder matched
    // for 2-byte staging (a plain 4*c image would put c and c + 32 on one
    // bank).  x2h_bytes = the zero words' byte + 128 (a multiple of 128).
    constexpr bool X2S = FH && VK == VK_F32X2;
    const uint32_t x2h_bytes = X2S ? h_zero_b(tn) + 128u : 0u;
    auto f32_slot = [&](int64_t c) -> size_t {
        return X2S ? (size_t)((c >> 1) << 2) + (size_t)(c & 1) * x2h_bytes : (size_t)c * 4;
    };
    uint32_t bkbase = (uint32_t)__cvta_generic_to_shared(bk);

    // Teams (bucket path): `team` consecutive warps share one cell; warp `sub`
    // of the team takes rounds sub, sub+team, ... with its own buckets, and
    // the team's k-row partials are combined in a fixed order at the end.
    const int team = RING ? p.team : 1;
    const int tpc = nwarps / team;               // teams per CTA
    const int tid_team = warp / team, sub = warp % team;
    int64_t b = RING ? (int64_t)blockIdx.x * tpc + tid_team : (int64_t)blockIdx.x * nwarps + warp;
    const int64_t cstride = RING ? (int64_t)gridDim.x * tpc : bstride;
    // Integer paths flush with native shared atomics, so a team shares one set
    // of buckets and splits the pattern-table reduction; the float path keeps
    // per-warp buckets (plain read-modify-write flushes).
    const bool shbk = RING && MODE != MODE_FLOAT && team > 1;
    if (shbk) {
        bk = buckets + (size_t)(tid_team * team) * p.nkeys;
        bkbase = (uint32_t)__cvta_generic_to_shared(bk);
    }

    // ---- stream fetch (bucket path) ------------------------------------------
    // Lane-run layout (run_slot in rsr_preprocess.cu): a cell of N chunk pairs
    // takes P = ceil(N/32) rounds; lane L owns pairs [L*P, L*P + len_L), and
    // round r holds np_r = Lf + (r < rem) pairs as four coalesced 16-byte
    // quarters.  A team of warps splits a cell's rounds into contiguous
    // ranges.  Each warp fetches its next round one round ahead straight into
    // registers (no shared-memory staging: the L1 data pipe is the bottleneck
    // resource of this kernel).  Lanes past np_r read zeros (key 0 / column 0).
    struct Cell {
        int64_t b;          // cell (block index in the view)
        uint32_t c0;        // first chunk
        uint32_t P, Lf, rem;
        uint32_t r0, r1;    // this warp's rounds
    };
    constexpr int CSH = CH == 16 ? 4 : 3;  // log2(CH); chunk indices are 32-bit
    auto cell_at = [&](int64_t cb, int64_t e0, int64_t e1) {
        Cell c;
        c.b = cb;
        c.c0 = (uint32_t)(e0 >> CSH);
        const uint32_t N = ((uint32_t)(e1 >> CSH) - c.c0) >> 1;
        c.P = (N + 31u) >> 5;
        c.Lf = c.P ? N / c.P : 0u;
        c.rem = N - c.Lf * c.P;
        c.r0 = (uint32_t)(((uint64_t)c.P * sub) / team);
        c.r1 = (uint32_t)(((uint64_t)c.P * (sub + 1)) / team);
        return c;
    };
    Cell fc;          // cell of the prefetched round
    uint32_t fr = 0;  // the prefetched round
    uint4 qa[4], qb[4];  // ping-pong round buffers (the prefetched round is in qa)
    auto seek = [&](int64_t cb) {  // first round of this warp in cells cb, cb + cstride, ...
        fc.b = cb;
        while (cb < p.nblk) {
            const int64_t dc = cb * p.tc + t;
            fc = cell_at(cb, p.e_off[dc], p.e_off[dc + 1]);
            if (fc.r0 < fc.r1) break;
            cb += cstride;
            fc.b = cb;
        }
        fr = fc.r0;
    };
    auto load_round = [&](uint4 (&nq)[4]) {
        if (fc.b >= p.nblk) return;  // nothing left: the stale registers are never consumed
        const uint32_t np = fc.Lf + (fr < fc.rem ? 1u : 0u);
        const uint32_t R = fr * fc.Lf + min(fr, fc.rem);
        const uint4 *src = ent4 + 2 * ((size_t)fc.c0 + 2 * (size_t)R) + lane;
        if (np == 32u) {
#pragma unroll
            for (int j = 0; j < 4; ++j) nq[j] = ld_stream(src + 32 * j);
        } else {
            // lanes past the round's pairs: slot 0 = the sink key, the rest
            // padding (format 3: the bank-0 zero word; else column 0)
            const uint32_t zb = FH ? h_zero_b(tn) : 0u;
            const uint32_t PW = zb | (zb << 16);
            const uint32_t P0 = FH ? (1u | (zb << 16)) : 0u;
            nq[0] = make_uint4(P0, PW, PW, PW);
#pragma unroll
            for (int j = 1; j < 4; ++j) nq[j] = make_uint4(PW, PW, PW, PW);
            if (lane < np) {
#pragma unroll
                for (int j = 0; j < 4; ++j) nq[j] = ld_stream(src + j * np);
            }
        }
    };
    // the first cell's offsets are requested up front (consumed by start_stream)
    int64_t pre0 = 0, pre1 = 0;
    if (RING && b < p.nblk) {
        pre0 = __ldg(p.e_off + b * p.tc + t);
        pre1 = __ldg(p.e_off + b * p.tc + t + 1);
    }
    bool stream_started = false;
    auto start_stream = [&]() {
        if (stream_started) return;
        stream_started = true;
        if constexpr (RING) {
            fc.b = p.nblk;
            if (b < p.nblk) {
                fc = cell_at(b, pre0, pre1);
                fr = fc.r0;
                if (fc.r0 >= fc.r1) seek(b + cstride);
            }
            load_round(qa);
        }
    };
    // sign table + zeroed buckets (no global loads: issued while v is in flight)
    bool tables_done = false;
    auto init_tables = [&]() {
        if (tables_done) return;
        tables_done = true;
        if constexpr (BUCKET) {
            // the sign table serves only the shared-bucket (integer team) and
            // k = 1 reductions; the others use the digit-split reduction
            const bool need_stab = K < 2 || shbk;
            for (int key = threadIdx.x; key < (need_stab ? p.nkeys : 0); key += blockDim.x) {
                uint32_t kk = (uint32_t)key;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    int sg = 0;
                    if (p.bitwidth == RSR_BINARY) {
                        sg = (int)((kk >> i) & 1u);
                    } else {
                        const uint32_t q3 = kk / 3u, d = kk - 3u * q3;
                        kk = q3;
                        sg = d == 1u ? 1 : (d == 2u ? -1 : 0);
                    }
                    stab[i * p.nkeys + key] = (Acc)sg;  // row-major: lanes read consecutive keys
                }
            }
            for (int i = threadIdx.x; i < nwarps * p.nkeys; i += blockDim.x) buckets[i] = (Acc)0;
        }
    };
    const bool fine = RSR_DBG(p, 256);  // debug: finer prologue timeline

    // ---- programmatic dependent launch ----------------------------------
    // The next multiply in the stream may start its pre-wait prologue as soon
    // as SMs free up.  Everything touched before griddepcontrol.wait (the
    // chunk stream, e_off, the shared tables) is never written by a multiply;
    // v, y and the workspace are touched only after it.  Without a PDL launch
    // the wait returns at once and the stream is requested after v (below).
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.pdl) {
        init_tables();
        // requesting the stream pre-wait pays off for long cells (its e_off
        // round trip is exposed otherwise); short cells request it after v
        if (p.pdl == 2) start_stream();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- prologue -------------------------------------------------------
    // The float path's v loads are issued first (vectorized, into registers);
    // the sign table and buckets are initialised while they are in flight;
    // v is converted into shared memory and only then is the first stream
    // round requested.
    double scale = 1.0;
    bool vstaged_float = false;
    if constexpr (MODE == MODE_FLOAT && FH && VK == VK_BF16) {
        // bf16 v copied as halfwords (16-byte loads and stores); the stream
        // was requested once they are issued
        const uint16_t *src = reinterpret_cast<const uint16_t *>(p.v) + c0;
        const int64_t nt = blockDim.x;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const int64_t nvec = tn >> 3;
            constexpr int U = 4;
            bool started = false;
            for (int64_t i0 = threadIdx.x; i0 < nvec; i0 += U * nt) {
                uint4 r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t i = i0 + u * nt;
                    r[u] = i < nvec ? __ldg(reinterpret_cast<const uint4 *>(src) + i)
                                    : make_uint4(0, 0, 0, 0);
                }
                init_tables();
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t i = i0 + u * nt;
                    if (i < nvec) reinterpret_cast<uint4 *>(vsm)[i] = r[u];
                }
                if (!started) {
                    start_stream();
                    started = true;
                }
            }
            for (int64_t i = (nvec << 3) + threadIdx.x; i < tn; i += nt)
                reinterpret_cast<uint16_t *>(vsm)[i] = __ldg(src + i);
        } else {
            for (int64_t i = threadIdx.x; i < tn; i += nt)
                reinterpret_cast<uint16_t *>(vsm)[i] = __ldg(src + i);
        }
        vstaged_float = true;
    } else if constexpr (MODE == MODE_FLOAT && SMEM_V && VSZ == 4) {
        // (format 3, f32 staging: even columns' words from byte 0, odd
        // columns' from byte x2h_bytes -- see f32x2_byte)
        const int esz = p.vdtype == RSR_F32 ? 4 : 2;
        const int epv = 16 / esz;  // elements per 16-byte load
        const char *src = reinterpret_cast<const char *>(p.v) + c0 * esz;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const int64_t nvec = tn / epv;
            constexpr int U = 4;
            const int64_t nt = blockDim.x;
            bool started = false;
            for (int64_t i0 = threadIdx.x; i0 < nvec; i0 += U * nt) {
                uint4 r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t i = i0 + u * nt;
                    r[u] = i < nvec ? __ldg(reinterpret_cast<const uint4 *>(src) + i)
                                    : make_uint4(0, 0, 0, 0);
                }
                init_tables();  // ALU + shared stores while v is in flight
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t i = i0 + u * nt;
                    if (i < nvec && X2S) {
                        // elements c = i*epv ..: evens to byte 2c, odds to
                        // x2h_bytes + 2c (c even)
                        const uint32_t w4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
                        unsigned char *ev = vsm + 2 * i * epv;
                        unsigned char *od = ev + x2h_bytes;
                        if (esz == 4) {
                            *reinterpret_cast<float2 *>(ev) =
                                make_float2(__uint_as_float(w4[0]), __uint_as_float(w4[2]));
                            *reinterpret_cast<float2 *>(od) =
                                make_float2(__uint_as_float(w4[1]), __uint_as_float(w4[3]));
                        } else {
                            float e4[4], o4[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (p.vdtype == RSR_BF16) {
                                    e4[q] = __uint_as_float(w4[q] << 16);
                                    o4[q] = __uint_as_float(w4[q] & 0xFFFF0000u);
                                } else {
                                    const __half2 h2 = *reinterpret_cast<const __half2 *>(&w4[q]);
                                    e4[q] = __low2float(h2);
                                    o4[q] = __high2float(h2);
                                }
                            }
                            *reinterpret_cast<float4 *>(ev) = make_float4(e4[0], e4[1], e4[2], e4[3]);
                            *reinterpret_cast<float4 *>(od) = make_float4(o4[0], o4[1], o4[2], o4[3]);
                        }
                    } else if (i < nvec) {
                        float *d = reinterpret_cast<float *>(vsm) + i * epv;
                        const uint32_t w4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
                        if (esz == 4) {
                            reinterpret_cast<float4 *>(d)[0] = make_float4(
                                __uint_as_float(w4[0]), __uint_as_float(w4[1]),
                                __uint_as_float(w4[2]), __uint_as_float(w4[3]));
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                float lo, hi;
                                if (p.vdtype == RSR_BF16) {
                                    lo = __uint_as_float(w4[q] << 16);
                                    hi = __uint_as_float(w4[q] & 0xFFFF0000u);
                                } else {
                                    const __half2 h2 = *reinterpret_cast<const __half2 *>(&w4[q]);
                                    lo = __low2float(h2);
                                    hi = __high2float(h2);
                                }
                                reinterpret_cast<float2 *>(d)[q] = make_float2(lo, hi);
                            }
                        }
                    }
                }
                if (!started) {  // v has arrived: now request the stream
                    start_stream();
                    started = true;
                }
            }
            for (int64_t i = nvec * epv + threadIdx.x; i < tn; i += nt)  // tail
                *reinterpret_cast<float *>(vsm + f32_slot(i)) = load_as_f32(p.v, p.vdtype, c0 + i);
            vstaged_float = true;
        }
    }
    init_tables();  // (no-op when the vectorized staging already did it)
    if (fine) probe(1);
    // Fused path with one tile and 4-byte staging: a single pass over v stages
    // it as f32 while tracking |v|max, then quantizes in place.
    bool staged = false;
    if constexpr (MODE == MODE_FUSED && SMEM_V && (VSZ == 4 || FH)) {
        // Decode-sized bf16 vectors: the whole vector in registers (<= two
        // 16-byte loads per thread), |v|max from registers, quantize straight
        // from registers -- no f32 round trip through shared memory.
        const int64_t nt = blockDim.x;
        if (p.tc == 1 && p.vdtype == RSR_BF16 && (tn & 7) == 0 && tn <= nt * 16 &&
            (reinterpret_cast<uintptr_t>(p.v) & 15) == 0) {
            const int64_t nvec = tn >> 3;
            uint4 r[2];
            float mx = 0.f;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int64_t i = threadIdx.x + u * nt;
                r[u] = i < nvec ? __ldg(reinterpret_cast<const uint4 *>(p.v) + i)
                                : make_uint4(0, 0, 0, 0);
            }
            if (p.norm_w) {
                // fused RMSNorm (BitLinear): mean of squares in fp32 over the
                // whole vector, then bf16(w * bf16(x * rsqrt(mean + eps)))
                float ss = 0.f;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t w4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float lo = __uint_as_float(w4[q] << 16);
                        const float hi = __uint_as_float(w4[q] & 0xFFFF0000u);
                        ss += lo * lo;
                        ss += hi * hi;
                    }
                }
                const float tot = cta_reduce_sum_f32(ss);
                const float rs = rsqrtf(tot * (1.0f / (float)tn) + p.norm_eps);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int64_t i = threadIdx.x + u * nt;
                    if (i < nvec) rmsnorm8(r[u], __ldg(reinterpret_cast<const uint4 *>(p.norm_w) + i), rs);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t w4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    mx = fmaxf(mx, fabsf(__uint_as_float(w4[q] << 16)));
                    mx = fmaxf(mx, fabsf(__uint_as_float(w4[q] & 0xFFFF0000u)));
                }
            }
            const double amax = cta_reduce_max((double)mx);  // exact: max of floats
            scale = amax == 0.0 ? 1.0 : 127.0 / amax;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int64_t i = threadIdx.x + u * nt;
                if (i < nvec) {
                    const uint32_t w4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
                    int32_t qv[8];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        qv[2 * q] = quantize_one(__uint_as_float(w4[q] << 16), scale);
                        qv[2 * q + 1] = quantize_one(__uint_as_float(w4[q] & 0xFFFF0000u), scale);
                    }
                    if constexpr (FH) {  // eight int16 halfwords
                        auto pk = [](int32_t lo, int32_t hi) {
                            return (uint32_t)(uint16_t)lo | ((uint32_t)(uint16_t)hi << 16);
                        };
                        reinterpret_cast<uint4 *>(vsm)[i] =
                            make_uint4(pk(qv[0], qv[1]), pk(qv[2], qv[3]), pk(qv[4], qv[5]),
                                       pk(qv[6], qv[7]));
                    } else {
                        int4 *d = reinterpret_cast<int4 *>(vsm) + 2 * i;
                        d[0] = make_int4(qv[0], qv[1], qv[2], qv[3]);
                        d[1] = make_int4(qv[4], qv[5], qv[6], qv[7]);
                    }
                }
            }
            if (p.scale_dev && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
                *p.scale_dev = scale;
            staged = true;
        }
        if (!staged && p.tc == 1 && !FH) {  // (format 3's int16 image has no room for f32)
            double a = 0.0;
            for_each_v_real(p.v, p.vdtype, 0, tn, [&](int64_t i, float x) {
                reinterpret_cast<float *>(vsm)[i] = x;
                const double ax = fabs((double)x);
                a = ax > a ? ax : a;
            });
            const double amax = cta_reduce_max(a);
            scale = amax == 0.0 ? 1.0 : 127.0 / amax;
            for (int64_t i = threadIdx.x; i < tn; i += blockDim.x)  // same thread wrote i
                reinterpret_cast<int32_t *>(vsm)[i] =
                    quantize_one(reinterpret_cast<float *>(vsm)[i], scale);
            if (p.scale_dev && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
                *p.scale_dev = scale;
            staged = true;
        }
    }
    if constexpr (MODE == MODE_FUSED) {
        if (!staged) {
            if constexpr (SMEM_V) {
                const double amax = cta_absmax_fast(p.v, p.vdtype, p.n);
                scale = amax == 0.0 ? 1.0 : 127.0 / amax;
                if (p.scale_dev && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
                    *p.scale_dev = scale;
            } else {
                scale = *p.scale_dev;  // written by the staging kernel
            }
        }
    }
    if (!staged && !vstaged_float) if constexpr (SMEM_V) {
        if constexpr (MODE == MODE_FLOAT && VK == VK_BF16) {
            // (not reached: the bf16 copy above always stages)
        } else if constexpr (MODE == MODE_FLOAT) {
            for_each_v_real(p.v, p.vdtype, c0, tn,
                       [&](int64_t i, float x) { *reinterpret_cast<float *>(vsm + f32_slot(i)) = x; });
        } else {
            auto put = [&](int64_t i, float x) {
                const int8_t q = MODE == MODE_INT ? (int8_t)x : quantize_one(x, scale);
                if constexpr (VSZ == 4) reinterpret_cast<int32_t *>(vsm)[i] = q;
                else if constexpr (VSZ == 2) reinterpret_cast<int16_t *>(vsm)[i] = q;
                else reinterpret_cast<int8_t *>(vsm)[i] = q;
            };
            if constexpr (MODE == MODE_INT) for_each_v_t<RSR_I8>(p.v, c0, tn, put);
            else for_each_v_real(p.v, p.vdtype, c0, tn, put);
        }
    }
    if (fine) probe(2);
    // The stream is requested once v is in (its burst would otherwise queue
    // ahead of the v loads); its first round's latency overlaps the rest.
    start_stream();
    // Quad layout: column 0 is the zero padding entry.  The tile's real
    // column-0 value (as staged: f32 / int8 / quantized) is added in the
    // epilogue to the bucket of col0_key[cell].  Thread 0 staged element 0.
    Acc v0 = (Acc)0;
    if constexpr (FH) {
        // format 3: every column is in the stream; padding names one of 32
        // zero words after the image (one per bank)
        // (f32 staging: the padding entries' words sit right after the
        // even-column image, at the same byte -- f32x2_byte(zero entry))
        for (int i = threadIdx.x; i < 32; i += blockDim.x)  // (a CTA may have a single warp)
            reinterpret_cast<uint32_t *>(vsm + h_zero_b(tn))[i] = 0u;
    } else if constexpr (SMEM_V) {
        if constexpr (MODE == MODE_FLOAT) v0 = load_as_f32(p.v, p.vdtype, c0);
        else if constexpr (MODE == MODE_INT) v0 = (Acc)__ldg(reinterpret_cast<const int8_t *>(p.v) + c0);
        else v0 = (Acc)quantize_one(load_as_f32(p.v, p.vdtype, c0), scale);
        if (threadIdx.x == 0) {
            if constexpr (VSZ == 4) reinterpret_cast<uint32_t *>(vsm)[0] = 0u;
            else vsm[0] = 0;
        }
    }
    __syncthreads();
    probe(fine ? 3 : 1);

    using VG = typename std::conditional<MODE == MODE_FLOAT, float, int8_t>::type;
    const VG *__restrict__ vglob = reinterpret_cast<const VG *>(p.vstaged) + c0;

    // ---- per-cell epilogue: pattern-table reduction + warp reduce + store ----
    auto finish_cell = [&](int64_t bb, Acc (&acc)[K]) {
        // the tile's column 0 (not in the u16 stream)
        uint32_t key0 = 0;
        if constexpr (SMEM_V && !FH) key0 = p.col0_key[bb * p.tc + t];
        // y_i = sum_key sgn_i(key) * bucket[key]  (bucket 0 is never reduced)
        if constexpr (BUCKET) {
            if (key0 && sub == 0 && lane == 0) {
                if (shbk) bucket_flush_final(bkbase + key0 * 4u, v0);  // native red
                else bk[key0] += v0;
            }
            __syncwarp();
            int kfirst = (int)lane, kstep = 32;
            if (shbk) {  // whole team has flushed; split the keys across it
                asm volatile("bar.sync %0, %1;" ::"r"(1 + tid_team), "r"(team * 32) : "memory");
                kfirst += 32 * sub;
                kstep *= team;
            }
            // buckets are re-zeroed for the warp's next cell only
            const bool rezero = bb + cstride < p.nblk;
            if (!shbk && K >= 2 && !RSR_DBG(p, 4)) {
                // Digit-split reduction (no sign table): key = lane + NL * l
                // with NL = 3^KH (ternary) or 2^KH (binary) lanes.  Rows below
                // KH take their sign from the lane's own digits, so they need
                // only the lane's total T = sum_l bucket; rows KH.. take it
                // from the digits of l, compile-time constants of the
                // unrolled loop (an add, a subtract or nothing).
                if (p.bitwidth == RSR_TERNARY) {
                    constexpr int KH = K >= 3 ? 3 : K;
                    constexpr int NL = KH == 3 ? 27 : (KH == 2 ? 9 : 3);
                    constexpr int NI = (K - KH) == 0 ? 1 : ((K - KH) == 1 ? 3 : ((K - KH) == 2 ? 9
                                       : ((K - KH) == 3 ? 27 : ((K - KH) == 4 ? 81 : 243))));
                    if ((int)lane < NL) {
                        Acc tsum = (Acc)0;
#pragma unroll
                        for (int l = 0; l < NI; ++l) {
                            const int key = (int)lane + NL * l;
                            const Acc bv = key ? bk[key] : (Acc)0;
                            if (rezero) bk[key] = (Acc)0;
                            tsum += bv;
                            int q = l;
#pragma unroll
                            for (int i = KH; i < K; ++i) {
                                const int d = q % 3;
                                q /= 3;
                                if (d == 1) acc[i] += bv;
                                else if (d == 2) acc[i] -= bv;
                                else acc[i] += bv * (Acc)0;  // 0 * NaN: the reference's y += sgn * s
                            }
                        }
                        uint32_t q = lane;
#pragma unroll
                        for (int i = 0; i < KH; ++i) {
                            const uint32_t d = q % 3u;
                            q /= 3u;
                            acc[i] += d == 1u ? tsum : (d == 2u ? -tsum : tsum * (Acc)0);
                        }
                    }
                } else {
                    constexpr int KH = K >= 5 ? 5 : K;
                    constexpr int NL = 1 << KH;
                    constexpr int NI = 1 << (K - KH);
                    if ((int)lane < NL) {
                        Acc tsum = (Acc)0;
#pragma unroll
                        for (int l = 0; l < NI; ++l) {
                            const int key = (int)lane + NL * l;
                            const Acc bv = key ? bk[key] : (Acc)0;
                            if (rezero) bk[key] = (Acc)0;
                            tsum += bv;
#pragma unroll
                            for (int i = KH; i < K; ++i)
                                acc[i] += ((l >> (i - KH)) & 1) ? bv : bv * (Acc)0;
                        }
#pragma unroll
                        for (int i = 0; i < KH; ++i)
                            acc[i] += ((lane >> i) & 1u) ? tsum : tsum * (Acc)0;
                    }
                }
            } else {
                for (int key = kfirst; key < (RSR_DBG(p, 4) ? 0 : p.nkeys); key += kstep) {
                    const Acc bv = key ? bk[key] : (Acc)0;
                    bk[key] = (Acc)0;
#pragma unroll
                    for (int i = 0; i < K; ++i) acc[i] += stab[i * p.nkeys + key] * bv;
                }
            }
            __syncwarp();
        } else if constexpr (SMEM_V) {
            if (key0 && lane == 0) reg_flush<K, Acc>(acc, key0, v0, p.bitwidth);
        }
        const int64_t row0 = bb * p.k;  // row within the view
        const int64_t grow0 = (p.blk0 + bb) * p.k;
        Acc mine = (Acc)0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const Acc r = warp_sum(acc[i]);
            if (lane == (uint32_t)i) mine = r;
        }
        if (team > 1) {
            // combine the team's partials in warp order (deterministic)
            if (lane < (uint32_t)K) xch[warp * 16 + lane] = mine;
            asm volatile("bar.sync %0, %1;" ::"r"(1 + tid_team), "r"(team * 32) : "memory");
            if (sub == 0 && lane < (uint32_t)K) {
                mine = (Acc)0;
                for (int j = 0; j < team; ++j) mine += xch[(tid_team * team + j) * 16 + lane];
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + tid_team), "r"(team * 32) : "memory");
            if (sub != 0) return;
        }
        if (lane < (uint32_t)K && grow0 + lane < p.m_rows) {
            const int64_t r = row0 + lane;
            if (p.tc > 1) {
                const int64_t rows_view = p.nblk * p.k;
                reinterpret_cast<Acc *>(p.part)[t * rows_view + r] = mine;
            } else if constexpr (MODE == MODE_FLOAT) {
                float *y = reinterpret_cast<float *>(p.y);
                put_row<float>(p, r, p.accumulate ? y[r] + (float)mine : (float)mine);
            } else if constexpr (MODE == MODE_INT) {
                int32_t *y = reinterpret_cast<int32_t *>(p.y);
                put_row<int32_t>(p, r, p.accumulate ? y[r] + (int32_t)mine : (int32_t)mine);
            } else {
                const double beta = p.row_beta ? p.row_beta[grow0 + lane] : p.beta;
                const float o = (float)((double)(int32_t)mine * (beta / scale));
                if (p.out_bf16) put_row<__nv_bfloat16>(p, r, __float2bfloat16_rn(o));
                else put_row<float>(p, r, o);
            }
        }
    };

    if constexpr (RING) {
        // ===== bucket path =====================================================
        // A round gives each lane the next chunk pair (32 slots) of its run, as
        // four 16-byte quarters.  Quad layout: slot 4q (low half of word 2q) is
        // a key or a column, slots 4q+1..4q+3 are columns; slot 0 is always a
        // key (a repeat of the open group's key when the group continues), and
        // inside a pair every other key starts a new group.  The open group
        // (cur, s) is carried from round to round.  Scaled format: entries are
        // byte offsets (column*4; key*4|1) straight into v and the buckets.
        // entry decoding: scaled (byte offsets of 4-byte elements), format 3
        // (byte offsets of 2-byte elements, doubled for f32 staging, keys
        // key*4|1), else column | key flag 0x8000
        constexpr bool SC = FMT == FMT_U16_SCALED || FH;
        constexpr bool X2 = FH && VK == VK_F32X2;
        auto is_key = [](uint32_t x) -> uint32_t { return SC ? (x & 1u) : (x & 0x8000u); };
        auto key_off = [](uint32_t x) -> uint32_t { return SC ? (x & 0xFFFCu) : (x & 0x7FFFu) * 4u; };
        const uint32_t x2h = x2h_bytes >> 1;
        auto lo_off = [x2h](uint32_t x) -> uint32_t {
            return X2 ? (x & 0xFFFCu) + (x & 2u) * x2h
                      : (FH ? (x & 0xFFFFu) : (SC ? (x & 0xFFFCu) : (x & 0x7FFFu) * VSZ));
        };
        auto hi_off = [x2h](uint32_t x) -> uint32_t {
            if constexpr (X2) {
                const uint32_t e = x >> 16;
                return (e & 0xFFFCu) + (e & 2u) * x2h;
            }
            return SC ? (x >> 16) : (x >> 16) * VSZ;
        };
        auto gat = [&](uint32_t off) -> Acc {
            if constexpr (FH && VK == VK_I16) return lds_s16(vbase + off);
            else return lds_v<Acc, VSZ == 2 ? 4 : VSZ>(vbase + off);
        };
        // sum of three gathers (bf16 halfwords: f32 += bf16 adds)
        auto gat3 = [&](uint32_t oa, uint32_t ob, uint32_t oc) -> Acc {
            if constexpr (FH && VK == VK_BF16) {
                const uint16_t a = lds_u16(vbase + oa), b = lds_u16(vbase + ob),
                               c = lds_u16(vbase + oc);
                return (Acc)add_bf16(add_bf16(add_bf16(0.0f, c), b), a);
            } else {
                return gat(oa) + (gat(ob) + gat(oc));
            }
        };
        // a predicated gather added to the open group's sum (key slots: no load)
        auto gat_unless_add = [&](uint32_t skip, uint32_t off, Acc s0) -> Acc {
            if constexpr (FH && VK == VK_BF16) {
                return (Acc)add_bf16((float)s0, lds_u16_unless(skip, vbase + off));
            } else if constexpr (FH && VK == VK_I16) {
                return s0 + (Acc)lds_s16_unless(skip, vbase + off);
            } else {
                return s0 + lds_v_unless<Acc, VSZ == 2 ? 4 : VSZ>(skip, vbase + off);
            }
        };
        for (; b < p.nblk; b += cstride) {
            const int64_t dc = b * p.tc + t;
            const Cell c = cell_at(b, p.e_off[dc], p.e_off[dc + 1]);
            Acc acc[K];
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] = (Acc)0;
            // open group: its bucket's shared address (bkbase = bucket 0, the
            // never-reduced sink) and its partial sum
            uint32_t cur = bkbase;
            Acc s = (Acc)0;
            auto do_round = [&](const uint4 (&q)[4]) {
                const uint4 a0 = q[0], a1 = q[1], a2 = q[2], a3 = q[3];
                // Pairs past a lane's run are zeros: key 0 (the sink) at slot 0,
                // then column-0 (zero) gathers -- no divergence.
                const uint32_t w[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                                        a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
                if (RSR_DBG(p, 32)) {  // experiment: stream only
                    uint32_t x = 0;
#pragma unroll
                    for (int i = 0; i < 16; ++i) x ^= w[i];
                    acc[0] += (Acc)x;
                    return;
                }
                if constexpr (MODE == MODE_FLOAT) {
                    // The bucket addresses of the groups this round closes follow
                    // from the keys alone, so their eight bucket loads are issued
                    // before the gathers (latency hidden); the adds and stores
                    // follow the sums.  The keys of one round's completed groups
                    // are distinct (a group completes once, in the lane holding
                    // its end), bucket 0 (the sink) aside.
                    uint32_t fk[8];
                    bool kk[8];
                    uint32_t cc = cur;
                    {
                        const uint32_t k0 = bkbase + key_off(w[0]);
                        kk[0] = k0 != cc;
                        fk[0] = kk[0] ? cc : bkbase;
                        cc = k0;
                    }
#pragma unroll
                    for (int qd = 1; qd < 8; ++qd) {
                        const uint32_t x = w[2 * qd];
                        kk[qd] = is_key(x) != 0u;
                        fk[qd] = kk[qd] ? cc : bkbase;
                        cc = kk[qd] ? bkbase + key_off(x) : cc;
                    }
                    float tb[8];
                    if (!RSR_DBG(p, 1)) lds_bucket8(fk, tb);
                    float fs[8];
                    fs[0] = s;
                    s = (kk[0] ? (Acc)0 : s) + gat3(hi_off(w[0]), lo_off(w[1]), hi_off(w[1]));
#pragma unroll
                    for (int qd = 1; qd < 8; ++qd) {
                        const uint32_t x = w[2 * qd], y = w[2 * qd + 1];
                        // slot 4q: a column unless it is a key (predicated-off
                        // lanes of a key slot take no shared-memory bank)
                        const Acc t3 = gat3(hi_off(x), lo_off(y), hi_off(y));
                        fs[qd] = s;
                        s = gat_unless_add(kk[qd], lo_off(x), kk[qd] ? (Acc)0 : s) + t3;
                    }
                    cur = cc;
                    if (!RSR_DBG(p, 1)) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) sts_bucket(fk[i], tb[i] + fs[i]);
                    }
                } else {
                    {   // slot 0: always a key; a new one closes the open group
                        const uint32_t k0 = bkbase + key_off(w[0]);
                        const bool ns = k0 != cur;
                        bucket_flush_pred(ns, cur, s);  // native shared red
                        cur = k0;
                        s = (ns ? (Acc)0 : s) + gat3(hi_off(w[0]), lo_off(w[1]), hi_off(w[1]));
                    }
#pragma unroll
                    for (int qd = 1; qd < 8; ++qd) {
                        const uint32_t x = w[2 * qd], y = w[2 * qd + 1];
                        const bool isk = is_key(x) != 0u;
                        const uint32_t ko = key_off(x);
                        const Acc t3 = gat3(hi_off(x), lo_off(y), hi_off(y));
                        bucket_flush_pred(isk, cur, s);
                        cur = isk ? bkbase + ko : cur;
                        s = gat_unless_add(isk, lo_off(x), isk ? (Acc)0 : s) + t3;
                    }
                }
            };
            auto advance = [&](uint4 (&nq)[4]) {  // prefetch this warp's next round
                if (++fr >= fc.r1) seek(fc.b + cstride);
                load_round(nq);
            };
            if constexpr (MODE != MODE_FUSED) {
                // two rounds per iteration (ping-pong: no register copies)
                uint32_t r = c.r0;
                while (r < c.r1) {
                    advance(qb);
                    do_round(qa);
                    if (++r >= c.r1) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) qa[j] = qb[j];
                        break;
                    }
                    advance(qa);
                    do_round(qb);
                    ++r;
                }
            } else {
                // the fused kernel serves small decode-time matrices, launched
                // between other kernels: one copy of the round body (smaller
                // i-cache footprint) at the price of 16 register moves a round
                for (uint32_t r = c.r0; r < c.r1; ++r) {
                    advance(qb);
                    do_round(qa);
#pragma unroll
                    for (int j = 0; j < 4; ++j) qa[j] = qb[j];
                }
            }
            // Close every lane's open group.  A group spanning whole runs leaves
            // equal open keys in consecutive lanes (contiguous lane runs): a
            // segmented suffix sum lets each run's first lane flush alone (no
            // CAS loop, fixed summation order).  Integer: native shared red.
            if constexpr (MODE == MODE_FLOAT) {
                float sj = s;
                const uint32_t kj = cur;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const float os = __shfl_down_sync(RSR_FULL_MASK, sj, d);
                    const uint32_t ok = __shfl_down_sync(RSR_FULL_MASK, kj, d);
                    if (lane + d < 32 && ok == kj) sj += os;
                }
                const uint32_t pk = __shfl_up_sync(RSR_FULL_MASK, kj, 1);
                if (lane == 0 || pk != kj) sts_bucket(kj, lds_bucket(kj) + sj);
            } else {
                bucket_flush_final(cur, s);
            }
            __syncwarp();
            finish_cell(b, acc);
        }
        if (p.probe && lane == 0 && !fine) {  // debug timeline: first / last warp done
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            atomicMin(p.probe + cta_id * 4 + 2, tnow);
            atomicMax(p.probe + cta_id * 4 + 3, tnow);
        }
    } else {
        // ===== generic path (register flush and/or u32 entries) ================
        for (; b < p.nblk; b += bstride) {
            const int64_t dc = b * p.tc + t;
            Acc acc[K];
#pragma unroll
            for (int i = 0; i < K; ++i) acc[i] = (Acc)0;
            if constexpr (FMT == FMT_U16) {
                // quad layout in lane runs (see the bucket path), register flush
                const Cell c = cell_at(b, p.e_off[dc], p.e_off[dc + 1]);
                auto gat = [&](uint32_t col) -> Acc { return lds_v<Acc, VSZ>(vbase + col * VSZ); };
                uint32_t cur = 0;
                Acc s = (Acc)0;
                for (uint32_t r = 0; r < c.P; ++r) {
                    const uint32_t np = c.Lf + (r < c.rem ? 1u : 0u);
                    const uint32_t R = r * c.Lf + min(r, c.rem);
                    uint4 a[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[j] = make_uint4(0, 0, 0, 0);
                    if (lane < np) {
                        const uint4 *src = ent4 + 2 * ((size_t)c.c0 + 2 * (size_t)R) + lane;
#pragma unroll
                        for (int j = 0; j < 4; ++j) a[j] = ld_stream(src + j * np);
                    }
                    const uint32_t w[16] = {a[0].x, a[0].y, a[0].z, a[0].w, a[1].x, a[1].y,
                                            a[1].z, a[1].w, a[2].x, a[2].y, a[2].z, a[2].w,
                                            a[3].x, a[3].y, a[3].z, a[3].w};
                    const uint32_t k0 = w[0] & 0x7FFFu;
                    if (k0 != cur) {
                        reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                        cur = k0;
                        s = (Acc)0;
                    }
                    s += gat(w[0] >> 16) + (gat(w[1] & 0xFFFFu) + gat(w[1] >> 16));
#pragma unroll
                    for (int qd = 1; qd < 8; ++qd) {
                        const uint32_t x = w[2 * qd], y = w[2 * qd + 1];
                        const uint32_t lo = x & 0xFFFFu;
                        const uint32_t isk = lo & 0x8000u;
                        const Acc g = lds_v_unless<Acc, VSZ>(isk, vbase + (lo & 0x7FFFu) * VSZ);
                        const Acc t3 = gat(x >> 16) + (gat(y & 0xFFFFu) + gat(y >> 16));
                        if (isk) reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                        cur = isk ? (lo & 0x7FFFu) : cur;
                        s = (isk ? (Acc)0 : s) + g + t3;
                    }
                }
                reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
            } else {  // FMT_U32 (even layout, round-major), v gathered from global scratch
                const int64_t cch0 = p.e_off[dc] / CH, cch1 = p.e_off[dc + 1] / CH;
                // rounds of 64 chunks, lane L owns the chunk pair (2L, 2L+1): four
                // coalesced 16-byte quarters (see phys_slot in rsr_preprocess.cu)
                auto load_pair = [&](int64_t base, uint4 (&q)[4]) {
                    const int64_t np = min((int64_t)64, cch1 - base) >> 1;
#pragma unroll
                    for (int j = 0; j < 4; ++j) q[j] = make_uint4(0, 0, 0, 0);
                    if ((int64_t)lane < np) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) q[j] = __ldg(ent4 + 2 * base + j * np + lane);
                    }
                };
                uint4 q[4];
                load_pair(cch0, q);
                for (int64_t base = cch0; base < cch1; base += 64) {
                    const bool valid_pair = (int64_t)lane < (min((int64_t)64, cch1 - base) >> 1);
                    uint4 a[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[j] = q[j];
                    if (base + 64 < cch1) load_pair(base + 64, q);  // prefetch the next round
                    if (!valid_pair) continue;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const uint4 a0 = a[2 * half], a1 = a[2 * half + 1];
                        const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                        constexpr uint32_t KF = 1u << 31;
                        uint32_t cur = w[0] & ~KF;
                        Acc s = (Acc)__ldg(vglob + w[1]);
#pragma unroll
                        for (int i = 2; i < 8; i += 2) {
                            const Acc h = (Acc)__ldg(vglob + w[i + 1]);
                            if (w[i] & KF) {
                                reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                                cur = w[i] & ~KF;
                                s = (Acc)0;
                            } else {
                                s += (Acc)__ldg(vglob + w[i]);
                            }
                            s += h;
                        }
                        reg_flush<K, Acc>(acc, cur, s, p.bitwidth);
                    }
                }
            }
            finish_cell(b, acc);
        }
    }
}

}  // namespace rsr
