// K6: per-tile forward multimodal blend.  Replaces the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187).
//
// One CTA per 16x16 tile, one thread per pixel; warps own 8x4 pixel blocks and
// run INDEPENDENTLY (no block barrier): each warp streams the tile list front
// to back in 32-entry chunks, culls each chunk against its block with the
// conservative alpha-support boxes (one ballot), and walks the surviving
// entries exactly as the reference walks the list: alpha test, skip below
// 1/255, blend, T *= 1-alpha, break after blending once T < early_stop_T.  A
// culled entry would have failed the alpha test, so results are the
// reference's.
//
// Phase A (per (warp, Gaussian) event, sequential per pixel): alpha, w = alpha T,
//   colour / k accumulation, T update, contributor count and terminus.  Each
//   blended pair is enqueued (pixel, Gaussian, w).  Semantic logits:
//   - FP64: channel-parallel into shared rows s_O[lane][C] (lane ch adds
//     w_L * sem_j[ch] for each blending lane L, in list order per pixel);
//   - FP32: events are batched 8 at a time and O[32 px][C] += W[32 px][8 ev] .
//     S[8 ev][C] runs on the tensor cores (mma.sync m16n8k8 TF32 with a hi/lo
//     split: FP32-level accuracy), accumulators in shared memory in fragment
//     order.  An event blends ~9 of the 32 pixels, so the dense product is ~7x
//     fewer instructions than the per-pair scalar update.
// Phase B (flush, 32 pairs per warp vector): the ray-ellipsoid midpoint depth
//   (fallback: centre depth) of every queued pair with all lanes busy, and
//   w * depth added to the owning pixel's depth sum.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kThreads = 256;
#ifndef K6_BCHUNK
#define K6_BCHUNK 4  // semantic n-tiles whose B values are loaded together
#endif
#ifndef K6_NEXT_PREFETCH
#define K6_NEXT_PREFETCH 1  // next chunk ids one chunk ahead + L1 prefetch of their records: 2.05 ms vs 2.11
#endif
constexpr int kQueue = 64;
// The semantics-free blend: 4-warp CTAs (half a tile) at 5 CTAs / SM = 96
// registers, 20 warps / SM: 1.74 ms vs 1.80 with 8-warp CTAs at 3 / SM (80
// registers, 24 warps, more spills) or 4 / SM (128 registers, 16 warps).
#ifndef K6_SPLIT_WARPS
#define K6_SPLIT_WARPS 4  // warps per CTA of the semantics-free variant
#endif
#ifndef K6_SPLIT_MINB
#define K6_SPLIT_MINB 5  // its CTAs per SM
#endif

__host__ __device__ inline int sem_pitch(int C) { return C | 1; }  // odd pitch: conflict-free rows

template <typename Real>
struct FwdWarpSmem {
    AlphaRec<Real> rec[32];
    float zoff;  // FP32: the camera's z offset (midpoint depth = zoff - h / a~)
    uint32_t gid[32];
    uint32_t q_lane[kQueue];
    uint32_t q_gid[kQueue];
    Real q_w[kQueue];
    Real q_wd[kQueue];
    float q_dx[kQueue], q_dy[kQueue];  // FP32: the pixel's offset from the splat centre (DepthRec)
};

// FP32 semantic tiles: per warp W[32 px][8 ev] (1 KB), the batch's Gaussian ids,
// and the accumulators, one float4 per lane per (m-tile, n-tile).
struct SemTC {
    float w[32 * 8];
    uint32_t gid[8];
};
__host__ __device__ inline int sem_ntiles(int C) { return (C + 7) / 8; }

template <typename Real>
size_t forward_smem_bytes(int C, int warps = 8) {
    size_t per_warp = sizeof(FwdWarpSmem<Real>);
    if (C > 0) {
        if constexpr (sizeof(Real) == 4)
            per_warp += sizeof(SemTC) + size_t(sem_ntiles(C)) * 2 * 32 * sizeof(float4);
        else
            per_warp += sizeof(Real) * 32 * size_t(sem_pitch(C));
    }
    return size_t(warps) * per_warp + 64;
}

// W is stored per pixel row with the event index permuted (k -> 2(k&3) + k/4)
// so that a lane's A-fragment pair (k = t, t + 4) is one 8-byte word, and the
// pair position XOR-swizzled by the row to spread the per-event stores.
__device__ __forceinline__ int semtc_wpos(int row, int k) {
    return (((k & 3) << 1) | (k >> 2)) ^ (((row >> 2) & 3) << 1);
}

// O += W S for the nb (<= 8) batched events of this warp.
__device__ __forceinline__ void semtc_batch(SemTC* st, float4* acc, const float* __restrict__ semantics, int C,
                                            int nb, int lane) {
    __syncwarp();
    const int g4 = lane >> 2, t = lane & 3, NT = sem_ntiles(C);
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int r0 = mi * 16 + g4, r1 = r0 + 8;
        const float2 v0 = *reinterpret_cast<const float2*>(st->w + r0 * 8 + semtc_wpos(r0, t));
        const float2 v1 = *reinterpret_cast<const float2*>(st->w + r1 * 8 + semtc_wpos(r1, t));
        split_tf32(v0.x, ah[mi][0], al[mi][0]);
        split_tf32(v1.x, ah[mi][1], al[mi][1]);
        split_tf32(v0.y, ah[mi][2], al[mi][2]);
        split_tf32(v1.y, ah[mi][3], al[mi][3]);
    }
    // Rows of events beyond the batch stay zero (their W columns are zero too,
    // but 0 * garbage could be NaN).
    const float* s0 = t < nb ? semantics + size_t(st->gid[t]) * C : nullptr;
    const float* s1 = t + 4 < nb ? semantics + size_t(st->gid[t + 4]) * C : nullptr;
    for (int n0 = 0; n0 < NT; n0 += K6_BCHUNK) {
        float b[K6_BCHUNK][2];
#pragma unroll
        for (int j = 0; j < K6_BCHUNK; ++j) {  // all loads of the chunk in flight together
            const int ch = (n0 + j) * 8 + g4;
            b[j][0] = s0 && ch < C ? __ldg(s0 + ch) : 0.f;
            b[j][1] = s1 && ch < C ? __ldg(s1 + ch) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < K6_BCHUNK; ++j) {
            if (n0 + j >= NT) break;
            uint32_t bh[2], bl[2];
            split_tf32(b[j][0], bh[0], bl[0]);
            split_tf32(b[j][1], bh[1], bl[1]);
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                float4* cp = acc + (size_t(mi) * NT + n0 + j) * 32 + lane;
                float4 cv = *cp;
                float d[4] = {cv.x, cv.y, cv.z, cv.w};
                mma_tf32(d, al[mi], bh);
                mma_tf32(d, ah[mi], bl);
                mma_tf32(d, ah[mi], bh);
                *cp = make_float4(d[0], d[1], d[2], d[3]);
            }
        }
    }
    __syncwarp();
}

// Phase B on the first n queue entries (n <= 32).  `own` has bit e set when
// queue entry e belongs to this lane's pixel.
template <typename Real>
__device__ __forceinline__ void flush_depth(const ForwardArgs<Real>& a, FwdWarpSmem<Real>* ws, int n, int bx, int by,
                                         Real& dep, unsigned own) {
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        const int L = int(ws->q_lane[lane]);
        const uint32_t g = ws->q_gid[lane];
        const int xL = bx + (L & 7), yL = by + (L >> 3);
        Real d;
        if constexpr (sizeof(Real) == 4) {
            // the quadratic forms of DepthRec (common.cuh) at this pixel's offset
            const float4* const q4 = reinterpret_cast<const float4*>(a.drec + g);
            const float4 e0 = q4[0], e1 = q4[1], e2 = q4[2], e3 = q4[3];  // E0..3 | E4 E5 H0 H1 | H2 zc A0 A1 | A2..5
            const float dx = ws->q_dx[lane], dy = ws->q_dy[lane];
            const float xx = dx * dx, xy = dx * dy, yy = dy * dy;
            const float t1 = e0.y * dx, t2 = e0.z * dy, t3 = e0.w * xx, t4 = e1.x * xy, t5 = e1.y * yy;
            const float disc = ((e0.x + t1) + (t2 + t3)) + (t4 + t5);
            const float sdisc = ((fabsf(e0.x) + fabsf(t1)) + (fabsf(t2) + fabsf(t3))) + (fabsf(t4) + fabsf(t5));
            const float u1 = e1.w * dx, u2 = e2.x * dy;
            const float h = e1.z + u1 + u2;
            const float sh = fabsf(e1.z) + fabsf(u1) + fabsf(u2);
            if (fabsf(disc) <= 1e-5f * sdisc || fabsf(h) <= 1e-5f * sh) {  // near a decision boundary
                double t, aa, bb, ds[3], dep;
                const bool ok = intersect_fp64<float>(a.cam, a.raw, g, float(xL) + 0.5f, float(yL) + 0.5f, &t, &aa,
                                                      &bb, ds, &dep);
                d = ok ? float(dep) : e2.y;
            } else if (disc >= 0.f && h < 0.f) {
                const float at = ((e2.z + e2.w * dx) + (e3.x * dy + e3.y * xx)) + (e3.z * xy + e3.w * yy);
                d = ws->zoff - __fdividef(h, at);
            } else {
                d = e2.y;
            }
        } else {
            const BlendRec<Real>& br = a.brec[g];
            const PixelRay<Real> ray = make_ray<Real>(a.cam, xL, yL);
            const HitEval<Real> h = intersect<Real>(br, ray, a.cam, a.raw, g);
            d = !h.hit ? br.zc : (h.depth_fp64 >= Real(0) ? h.depth_fp64 : midpoint_depth<Real>(a.cam, ray, h.t_mid));
        }
        if (!isfinite(d)) raise_error(a.err, kErrNonFiniteBlend, (long long)yL * a.W + xL, g);
        ws->q_wd[lane] = ws->q_w[lane] * d;
    }
    __syncwarp();
    while (own) {  // this pixel's entries, in queue (= list) order
        const int e = __ffs(own) - 1;
        own &= own - 1;
        dep += ws->q_wd[e];
    }
    __syncwarp();
}

}  // namespace

// kSplit (FP32): semantics are left to the separate tensor-core pass
// (forward_split.cu, K6b), which replays the event log with the blend weights
// this kernel writes (one 32-float row per event); nothing semantic is live
// here.
// A CTA covers one tile with 8 warps, or (kSplit, K6_SPLIT_WARPS = 4) half a
// tile with 4: the warps never synchronise, so smaller CTAs only change how
// registers and shared memory are granted per SM.
constexpr int kSplitWarps = K6_SPLIT_WARPS;
// kWsum: the replay records weight sums (capture flag 2; parity checks only) --
// a compile-time switch keeps its per-event test out of the hot loop.
template <typename Real, bool kSplit, bool kWsum = true>
__global__ void __launch_bounds__(kSplit ? 32 * kSplitWarps : kThreads, kSplit ? K6_SPLIT_MINB : 2)
    forward_kernel(const __grid_constant__ ForwardArgs<Real> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp: the CTA's shared-memory slot
    constexpr int kParts = kSplit ? 8 / kSplitWarps : 1;            // CTAs per tile
    const int wq = kParts > 1 ? int(blockIdx.x % kParts) * kSplitWarps + warp : warp;  // 8x4 block of the tile
    const int C = kSplit ? 0 : a.C, pitch = sem_pitch(C);
    constexpr bool kTC = sizeof(Real) == 4;  // tensor-core semantic accumulation (FP32)
    FwdWarpSmem<Real>* ws = reinterpret_cast<FwdWarpSmem<Real>*>(smem_raw) + warp;
    unsigned char* const sem_base = reinterpret_cast<unsigned char*>(reinterpret_cast<FwdWarpSmem<Real>*>(smem_raw) + 8);
    const int NT = sem_ntiles(C);
    // FP64: per-pixel rows.  FP32: SemTC + fragment-ordered accumulators.
    Real* const warp_O = reinterpret_cast<Real*>(sem_base) + size_t(warp) * 32 * pitch;
    Real* const my_O = warp_O + size_t(lane) * pitch;
    SemTC* const st = reinterpret_cast<SemTC*>(sem_base + size_t(warp) * (sizeof(SemTC) + size_t(NT) * 1024));
    float4* const acc = reinterpret_cast<float4*>(st + 1);
    if constexpr (kTC) {
        for (int i = lane; i < 2 * NT * 32; i += 32) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
        for (int ch = 0; ch < C; ++ch) my_O[ch] = Real(0);
    }
    int nb = 0;  // FP32: events in the open semantic batch

    const int tile = kParts > 1 ? int(blockIdx.x / kParts) : int(blockIdx.x);
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (wq & 1) * 8, by = ty * kTile + (wq >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    if constexpr (kTC) {
        if (lane == 0) ws->zoff = make_ray<Real>(a.cam, x, y).zoff;
    }
    const Real pxf = Real(x) + Real(0.5), pyf = Real(y) + Real(0.5);
    const uint2 range = a.tile_range[tile];
    const int len = int(range.y - range.x);

    Real T = Real(1), col0 = 0, col1 = 0, col2 = 0, dep = 0, kk = 0;
    int count = 0, last = 0;
    bool done = !inside;
    const Real early = Real(a.rp.early_stop_T);
    const bool c0 = lane < C, c1 = lane + 32 < C;
    int qn = 0;
    unsigned long long own = 0;  // queue entries owned by this pixel
    uint4* const evl = a.ev_list ? a.ev_list + size_t(8) * range.x + size_t(wq) * len : nullptr;
    float* const wd = kSplit ? a.ev_w + (size_t(8) * range.x + size_t(wq) * len) * 32 + lane : nullptr;
    uint32_t n_ev = 0, n_pairs = 0;
    if (kSplit && int64_t(size_t(8) * range.x + size_t(wq) * len + len) * 32 > a.ev_w_cap) {
        // a captured replay outgrew the weight rows (sized by the last eager render)
        if (lane == 0) raise_error(a.err, kErrInstanceOverflow, int64_t(size_t(8) * range.x + size_t(wq) * len + len) * 32,
                                   a.ev_w_cap);
        done = true;
    }

#if K6_NEXT_PREFETCH
    uint32_t g_next = lane < len ? a.inst_gauss[range.x + lane] : 0u;
#endif
    for (int c = 0; c * 32 < len; ++c) {
        // Cull against the bounding box of the block's still-active pixels: a
        // Gaussian whose alpha-support box misses it cannot blend any pixel
        // that is not done (saturated or outside the image).
        const unsigned live = __ballot_sync(0xffffffffu, !done);
        if (live == 0u) break;
        const unsigned cols = (live | (live >> 8) | (live >> 16) | (live >> 24)) & 0xffu;
        const int r0 = (__ffs(live) - 1) >> 3, r1 = (31 - __clz(live)) >> 3;
        const Real rx0 = Real(bx + __ffs(cols) - 1) + Real(0.5), rx1 = Real(bx + 31 - __clz(cols)) + Real(0.5);
        const Real ry0 = Real(by + r0) + Real(0.5), ry1 = Real(by + r1) + Real(0.5);
        const int pos = c * 32 + lane;
        bool hit = false;
#if K6_NEXT_PREFETCH
        const uint32_t g_cur = g_next;
        if (pos + 32 < len) {  // the next chunk's ids now, its records into L1 once they arrive
            g_next = a.inst_gauss[range.x + pos + 32];
        }
#endif
        if (pos < len) {
#if K6_NEXT_PREFETCH
            const uint32_t g = g_cur;
#else
            const uint32_t g = a.inst_gauss[range.x + pos];
#endif
            const AlphaRec<Real> r = a.arec[g];
            ws->rec[lane] = r;
            ws->gid[lane] = g;
            hit = !(r.bx1 < rx0 || r.bx0 > rx1 || r.by1 < ry0 || r.by0 > ry1);
            if (hit) {
                if constexpr (kTC)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.drec + g)));
                else
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.brec + g)));
            }
        }
        unsigned bits = __ballot_sync(0xffffffffu, hit);
        __syncwarp();
#if K6_NEXT_PREFETCH
        if (pos + 32 < len) asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.arec + g_next)));
#endif
        while (bits) {
            const int slot = __ffs(bits) - 1;
            bits &= bits - 1;
            AlphaEval<Real> ae;
            ae.pass = false;
            if (!done) ae = eval_alpha<Real>(ws->rec[slot], pxf, pyf);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            if (kSplit || evl) {  // the backward replays exactly these events (always logged when split)
                if (lane == 0) evl[n_ev] = make_uint4(uint32_t(c * 32 + slot), mask, ws->gid[slot], 0u);
                if constexpr (kSplit) {  // w = alpha T; negated when alpha was clamped at 0.99 (for the backward)
                    const Real w = ae.alpha * T;
                    wd[n_ev * 32u] = ae.pass ? (ae.clamped ? -w : w) : Real(0);
                }
                ++n_ev;
                n_pairs += __popc(mask);
            }
            const uint32_t g = ws->gid[slot];
            Real w = Real(0);
            if (ae.pass) {
                if (!isfinite(ae.alpha)) {
                    raise_error(a.err, kErrNonFiniteBlend, (long long)y * a.W + x, g);
                    done = true;
                }
                const AlphaRec<Real>& br = ws->rec[slot];
                w = ae.alpha * T;
                col0 += w * br.rgb[0];
                col1 += w * br.rgb[1];
                col2 += w * br.rgb[2];
                kk += w * br.k;
                if constexpr (kWsum) {
                    if (a.weight_sums) atomicAdd(a.weight_sums + g, w);
                }
                const int e = qn + __popc(mask & ((1u << lane) - 1u));
                own |= 1ull << e;
                ws->q_lane[e] = uint32_t(lane);
                ws->q_gid[e] = g;
                ws->q_w[e] = w;
                if constexpr (kTC) {
                    ws->q_dx[e] = float(ae.dx);
                    ws->q_dy[e] = float(ae.dy);
                }
                T *= (Real(1) - ae.alpha);
                ++count;
                last = c * 32 + slot + 1;
                if (a.rp.early_termination && T < early) done = true;
            }
            __syncwarp();
            const int npairs = __popc(mask);
            if constexpr (kTC) {
                if (C > 0) {
                    st->w[lane * 8 + semtc_wpos(lane, nb)] = float(w);
                    if (lane == 0) st->gid[nb] = g;
                    if (lane * 32 < C) {  // pull the row into L1 ahead of the batch
                        const float* row = reinterpret_cast<const float*>(a.semantics) + size_t(g) * C;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(row + lane * 32));
                    }
                    if (++nb == 8) {
                        semtc_batch(st, acc, reinterpret_cast<const float*>(a.semantics), C, 8, lane);
                        nb = 0;
                    }
                }
            } else if (C > 0) {  // semantic logits, channel-parallel, list order per pixel
                const Real* semg = a.semantics + size_t(g) * C;
                const Real sv0 = c0 ? semg[lane] : Real(0);
                const Real sv1 = c1 ? semg[lane + 32] : Real(0);
                // The event's rows are distinct pixels: batch the loads before the
                // stores so the shared-memory round trips overlap.
                const int cc0 = c0 ? lane : 0, cc1 = c1 ? lane + 32 : 0;
                int e = qn;
                for (; e + 4 <= qn + npairs; e += 4) {
                    Real* r0 = warp_O + int(ws->q_lane[e]) * pitch;
                    Real* r1 = warp_O + int(ws->q_lane[e + 1]) * pitch;
                    Real* r2 = warp_O + int(ws->q_lane[e + 2]) * pitch;
                    Real* r3 = warp_O + int(ws->q_lane[e + 3]) * pitch;
                    const Real w0 = ws->q_w[e], w1 = ws->q_w[e + 1], w2 = ws->q_w[e + 2], w3 = ws->q_w[e + 3];
                    const Real a0 = r0[cc0], a1 = r1[cc0], a2 = r2[cc0], a3 = r3[cc0];
                    const Real b0 = r0[cc1], b1 = r1[cc1], b2 = r2[cc1], b3 = r3[cc1];
                    if (c0) {
                        r0[lane] = a0 + w0 * sv0;
                        r1[lane] = a1 + w1 * sv0;
                        r2[lane] = a2 + w2 * sv0;
                        r3[lane] = a3 + w3 * sv0;
                    }
                    if (c1) {
                        r0[lane + 32] = b0 + w0 * sv1;
                        r1[lane + 32] = b1 + w1 * sv1;
                        r2[lane + 32] = b2 + w2 * sv1;
                        r3[lane + 32] = b3 + w3 * sv1;
                    }
                }
                for (; e < qn + npairs; ++e) {
                    const Real wL = ws->q_w[e];
                    Real* row = warp_O + int(ws->q_lane[e]) * pitch;
                    if (c0) row[lane] += wL * sv0;
                    if (c1) row[lane + 32] += wL * sv1;
                }
                for (int ch = lane + 64; ch < C; ch += 32) {  // C > 64
                    const Real sv = semg[ch];
                    for (int e = qn; e < qn + npairs; ++e) warp_O[int(ws->q_lane[e]) * pitch + ch] += ws->q_w[e] * sv;
                }
                __syncwarp();
            }
            qn += npairs;
            if (qn >= 32) {
                flush_depth<Real>(a, ws, 32, bx, by, dep, unsigned(own));
                own >>= 32;
                const int rest = qn - 32;
                if (lane < rest) {  // reads >= 32, writes < 32
                    ws->q_lane[lane] = ws->q_lane[32 + lane];
                    ws->q_gid[lane] = ws->q_gid[32 + lane];
                    ws->q_w[lane] = ws->q_w[32 + lane];
                    if constexpr (kTC) {
                        ws->q_dx[lane] = ws->q_dx[32 + lane];
                        ws->q_dy[lane] = ws->q_dy[32 + lane];
                    }
                }
                qn = rest;
                __syncwarp();
            }
        }
    }
    if (qn > 0) flush_depth<Real>(a, ws, qn, bx, by, dep, unsigned(own));
    if constexpr (kTC) {
        if (nb > 0) {
            for (int k = nb; k < 8; ++k) st->w[lane * 8 + semtc_wpos(lane, k)] = 0.f;
            semtc_batch(st, acc, reinterpret_cast<const float*>(a.semantics), C, nb, lane);
        }
    }
    if (a.ev_count && lane == 0) {
        a.ev_count[size_t(tile) * 8 + wq] = n_ev;
        a.ev_npairs[size_t(tile) * 8 + wq] = n_pairs;
    }
    if constexpr (kTC) {
        if (a.sem_out) {  // straight from the fragments: lane (g4, t) holds rows g4, g4 + 8 x cols 2t, 2t + 1
            const size_t HW = size_t(a.W) * a.H;
            const int g4 = lane >> 2, t = lane & 3;
            for (int i = 0; i < 2 * NT; ++i) {
                const int mi = i / NT, nj = i - mi * NT;
                const float4 v = acc[size_t(i) * 32 + lane];
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int row = mi * 16 + g4 + (q >> 1) * 8, ch = nj * 8 + 2 * t + (q & 1);
                    const int px = bx + (row & 7), py = by + (row >> 3);
                    if (ch < C && px < a.W && py < a.H) a.sem_out[size_t(ch) * HW + size_t(py) * a.W + px] = Real(vv[q]);
                }
            }
        }
    }
    if (!inside) return;
    col0 += T * Real(a.rp.bg[0]);
    col1 += T * Real(a.rp.bg[1]);
    col2 += T * Real(a.rp.bg[2]);
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    if (a.color) {
        a.color[p] = col0;
        a.color[HW + p] = col1;
        a.color[2 * HW + p] = col2;
    }
    if (a.depth) a.depth[p] = dep;
    if (a.kmap) a.kmap[p] = kk;
    a.T[p] = T;
    if (a.contributors) a.contributors[p] = count;
    if (a.terminus) a.terminus[p] = last;
    if (!kTC && a.sem_out)
        for (int ch = 0; ch < C; ++ch) a.sem_out[size_t(ch) * HW + p] = my_O[ch];
    if (!isfinite(col0) || !isfinite(col1) || !isfinite(col2) || !isfinite(dep) || !isfinite(T))
        raise_error(a.err, kErrNonFiniteOutput, (long long)p, -1);
}

template <typename Real>
void launch_forward(const ForwardArgs<Real>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    const size_t smem = forward_smem_bytes<Real>(a.C);
    static std::atomic<unsigned long long> attr{0};  // per instantiation, per device
    opt_in_smem(reinterpret_cast<const void*>(forward_kernel<Real, false>), attr);
    forward_kernel<Real, false><<<ntiles, kThreads, smem, s>>>(a);
    count_launches(1);
}

void launch_forward_blend_split(const ForwardArgs<float>& a, int ntiles, cudaStream_t s) {
    if (ntiles == 0) return;
    const size_t smem = forward_smem_bytes<float>(0, kSplitWarps);
    static std::atomic<unsigned long long> attr{0};
    static std::atomic<unsigned long long> attr_nw{0};
    if (a.weight_sums) {
        opt_in_smem(reinterpret_cast<const void*>(forward_kernel<float, true, true>), attr);
        forward_kernel<float, true, true><<<ntiles * (8 / kSplitWarps), 32 * kSplitWarps, smem, s>>>(a);
    } else {
        opt_in_smem(reinterpret_cast<const void*>(forward_kernel<float, true, false>), attr_nw);
        forward_kernel<float, true, false><<<ntiles * (8 / kSplitWarps), 32 * kSplitWarps, smem, s>>>(a);
    }
    count_launches(1);
}

template void launch_forward<float>(const ForwardArgs<float>&, int, cudaStream_t);
template void launch_forward<double>(const ForwardArgs<double>&, int, cudaStream_t);

}  // namespace msplat_cuda
