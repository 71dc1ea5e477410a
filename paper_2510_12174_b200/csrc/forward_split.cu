// K6 (FP32, C <= 64) as two kernels -- the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187) split at the blend-event log.
//
// K6a forward_alpha_kernel: the sequential part.  One CTA per 16x16 tile,
//   warps own 8x4 pixel blocks and stream the tile list independently in
//   32-entry chunks exactly as the fused kernel did: conservative
//   alpha-support culling (one ballot), alpha test, skip below 1/255, blend,
//   T *= 1 - alpha, break once T < early_stop_T.  Outputs colour, k map, T,
//   contributor count and terminus, the event log (list position, lane mask)
//   and the BLEND WEIGHTS of every event as one 32-float row (w = alpha T for
//   the blending lanes, 0 elsewhere).  Nothing else is live across the loop,
//   so it runs at 4 CTAs / SM.
// K6b forward_pairs_kernel: the per-pair part, replayed from the log.  One
//   warp per (tile, 8x4 block) segment walks its events front to back in
//   batches of 8, software-pipelined one batch ahead (the batch's weight rows
//   and semantic rows staged into shared memory by cp.async while the
//   previous batch computes; Gaussian ids fetched two batches ahead):
//   - semantic logits O[32 px][C] += W[32 px][8 ev] . S[8 ev][C] on the tensor
//     cores (mma.sync m16n8k8 TF32 with a hi/lo split: FP32-level accuracy),
//     accumulators in REGISTERS (the fused kernel had to keep them in shared
//     memory);
//   - the ray-ellipsoid midpoint depth (fallback: centre depth) of every
//     blended pair, 32 pairs at a time through a queue (all lanes busy), and
//     w * depth added to the pixel's depth sum in list order.
// Both read identical decisions (the log), so the outputs are the fused
// kernel's: same per-pixel summation order for colour, k, depth and
// semantics.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kThreads = 256;
constexpr int kNtMax = 8;  // semantic n-tiles in registers: C <= 64
constexpr int kQueue = 64;
#ifndef K6B_TILE_ORDER
#define K6B_TILE_ORDER 0  // 1: the semantic pass in tile order (L2 sharing between neighbouring tiles)
#endif
#ifndef K6_SPLIT_DEPTH
#define K6_SPLIT_DEPTH 0  // 1: depth in its own pass after a depth-free blend (measured slower)
#endif
#ifndef K6C_MINB
#define K6C_MINB 3  // depth-pass CTAs per SM
#endif


// ---------------------------------------------------------------- K6a
__global__ void __launch_bounds__(kThreads, 4) forward_alpha_kernel(const __grid_constant__ ForwardArgs<float> a) {
    __shared__ AlphaRec<float> s_rec[8][32];
    __shared__ uint32_t s_gid[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    AlphaRec<float>* const rec = s_rec[warp];
    uint32_t* const gids = s_gid[warp];
    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (warp & 1) * 8, by = ty * kTile + (warp >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const float pxf = float(x) + 0.5f, pyf = float(y) + 0.5f;
    const float rx0 = float(bx) + 0.5f, rx1 = rx0 + 7.f;
    const float ry0 = float(by) + 0.5f, ry1 = ry0 + 3.f;
    const uint2 range = a.tile_range[tile];
    const int len = int(range.y - range.x);

    float T = 1.f, col0 = 0.f, col1 = 0.f, col2 = 0.f, kk = 0.f;
    int count = 0, last = 0;
    bool done = !inside;
    const float early = float(a.rp.early_stop_T);
    const size_t ev0 = size_t(8) * range.x + size_t(warp) * len;  // this warp's event-log region
    uint2* const evl = a.ev_list + ev0;
    float* const wd = a.ev_w + ev0 * 32;  // its weight rows: event e's lane L at wd[32 e + L]
    uint32_t n_ev = 0, n_pairs = 0;
    if (int64_t(ev0 + len) * 32 > a.ev_w_cap) {  // a captured replay outgrew the weight buffer
        if (lane == 0) raise_error(a.err, kErrInstanceOverflow, int64_t(ev0 + len) * 32, a.ev_w_cap);
        done = true;
    }

    uint32_t g_next = lane < len ? a.inst_gauss[range.x + lane] : 0u;
    for (int c = 0; c * 32 < len; ++c) {
        if (__all_sync(0xffffffffu, done)) break;
        const int pos = c * 32 + lane;
        bool hit = false;
        const uint32_t g_cur = g_next;
        if (pos + 32 < len) g_next = a.inst_gauss[range.x + pos + 32];  // the next chunk's ids, one chunk ahead
        if (pos < len) {
            const AlphaRec<float> r = a.arec[g_cur];
            rec[lane] = r;
            gids[lane] = g_cur;
            hit = !(r.bx1 < rx0 || r.bx0 > rx1 || r.by1 < ry0 || r.by0 > ry1);
        }
        unsigned bits = __ballot_sync(0xffffffffu, hit);
        __syncwarp();
        if (pos + 32 < len) asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(a.arec + g_next)));
        while (bits) {
            const int slot = __ffs(bits) - 1;
            bits &= bits - 1;
            AlphaEval<float> ae;
            ae.pass = false;
            if (!done) ae = eval_alpha<float>(rec[slot], pxf, pyf);
            const unsigned mask = __ballot_sync(0xffffffffu, ae.pass);
            if (mask == 0) continue;
            if (lane == 0) evl[n_ev] = make_uint2(uint32_t(c * 32 + slot), mask);
            float w = 0.f;
            if (ae.pass) {
                const uint32_t g = gids[slot];
                if (!isfinite(ae.alpha)) {
                    raise_error(a.err, kErrNonFiniteBlend, (long long)y * a.W + x, g);
                    done = true;
                }
                const AlphaRec<float>& br = rec[slot];
                w = ae.alpha * T;
                col0 += w * br.rgb[0];
                col1 += w * br.rgb[1];
                col2 += w * br.rgb[2];
                kk += w * br.k;
                if (a.weight_sums) atomicAdd(a.weight_sums + g, w);
                T *= (1.f - ae.alpha);
                ++count;
                last = c * 32 + slot + 1;
                if (a.rp.early_termination && T < early) done = true;
            }
            wd[size_t(n_ev) * 32 + lane] = w;  // one coalesced 128-byte row per event
            ++n_ev;
            n_pairs += __popc(mask);
        }
    }
    if (lane == 0) {
        a.ev_count[size_t(tile) * 8 + warp] = n_ev;
        a.ev_npairs[size_t(tile) * 8 + warp] = n_pairs;
    }
    if (!inside) return;
    col0 += T * float(a.rp.bg[0]);
    col1 += T * float(a.rp.bg[1]);
    col2 += T * float(a.rp.bg[2]);
    const size_t HW = size_t(a.W) * a.H, p = size_t(y) * a.W + x;
    if (a.color) {
        a.color[p] = col0;
        a.color[HW + p] = col1;
        a.color[2 * HW + p] = col2;
    }
    if (a.kmap) a.kmap[p] = kk;
    a.T[p] = T;
    if (a.contributors) a.contributors[p] = count;
    if (a.terminus) a.terminus[p] = last;
    // rasterizer.cpp:179-183 (the depth sum is checked by K6b)
    if (!isfinite(col0) || !isfinite(col1) || !isfinite(col2) || !isfinite(T))
        raise_error(a.err, kErrNonFiniteOutput, (long long)p, -1);
}

// ---------------------------------------------------------------- K6b
constexpr int kSemPitch = 72;  // staged semantic rows: (t * 72) mod 32 = 8 t, conflict-free B fragments

constexpr int kWPitch = 40;  // W tile rows: (k * 40) mod 32 = 8 k, conflict-free A fragments

struct PairSmem {
    float wt[2][8][kWPitch];        // W^T[8 ev][32 px] tiles (the weight rows as written), double-buffered
    float srow[2][8][kSemPitch];    // the batch's semantic rows, double-buffered
    uint32_t gid[2][8];             // the batch's Gaussian ids, double-buffered
    float4 ray[32];                 // the block's pixel rays (cached_ray)
    uint32_t q_lane[kQueue];
    uint32_t q_gid[kQueue];
    float q_w[kQueue];
    float q_wd[kQueue];
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}

// Issues the cp.async staging of batch b (nb events; ids already in
// ws->gid[b & 1]): this lane's weight of each event into the W tile, and the
// events' semantic rows (8-byte pieces when sem_vec).  One commit group.
template <bool kSem>
__device__ __forceinline__ void stage_batch(const ForwardArgs<float>& a, PairSmem* ws, const float* wrows, int b, int nb,
                                            int lane) {
    const int buf = b & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // 8 rows x 8 16-byte pieces
        const int i = lane + 32 * h, k = i >> 3, q = i & 7;
        float* const dst = &ws->wt[buf][k][4 * q];
        if (k < nb) cp_async16(dst, wrows + size_t(8 * b + k) * 32 + 4 * q);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if constexpr (kSem) {  // a lane owns a piece column and walks the rows
        const int C = a.C;
        if (a.sem_vec) {
            for (int j = lane; j < (C >> 1); j += 32)
                for (int k = 0; k < nb; ++k)
                    cp_async8(&ws->srow[buf][k][2 * j], a.semantics + size_t(ws->gid[buf][k]) * C + 2 * j);
        } else {
            for (int j = lane; j < C; j += 32)
                for (int k = 0; k < nb; ++k)
                    cp_async4(&ws->srow[buf][k][j], a.semantics + size_t(ws->gid[buf][k]) * C + j);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// O += W S for a staged batch (events beyond nb: zero W columns, rows never read).
template <int NT>
__device__ __forceinline__ void sem_batch(const PairSmem* ws, int buf, float (&acc)[2][NT][4], int C, int nb,
                                          int lane) {
    const int g4 = lane >> 2, t = lane & 3;
    const float* const w0 = ws->wt[buf][t];      // event t's weights over the 32 pixels
    const float* const w1 = ws->wt[buf][t + 4];  // event t + 4
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {  // A[px][ev]: rows px = 16 mi + g4 (+ 8), cols ev = t (+ 4)
        const int r0 = mi * 16 + g4, r1 = r0 + 8;
        split_tf32(fabsf(w0[r0]), ah[mi][0], al[mi][0]);  // (the sign marks a clamped alpha)
        split_tf32(fabsf(w0[r1]), ah[mi][1], al[mi][1]);
        split_tf32(fabsf(w1[r0]), ah[mi][2], al[mi][2]);
        split_tf32(fabsf(w1[r1]), ah[mi][3], al[mi][3]);
    }
    const float* const s0 = ws->srow[buf][t];
    const float* const s1 = ws->srow[buf][t + 4];
    const bool e0 = t < nb, e1 = t + 4 < nb;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int ch = j * 8 + g4;
        const float b0 = (e0 && ch < C) ? s0[ch] : 0.f;
        const float b1 = (e1 && ch < C) ? s1[ch] : 0.f;
        uint32_t bh[2], bl[2];
        split_tf32(b0, bh[0], bl[0]);
        split_tf32(b1, bh[1], bl[1]);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            mma_tf32(acc[mi][j], al[mi], bh);
            mma_tf32(acc[mi][j], ah[mi], bl);
            mma_tf32(acc[mi][j], ah[mi], bh);
        }
    }
}

// The ray-ellipsoid midpoint depth of the first n (<= 32) queued pairs, w * d
// added to the owning pixels in queue (= list) order.
__device__ __forceinline__ void flush_depth(const ForwardArgs<float>& a, PairSmem* ws, float zoff, int n, int bx,
                                            int by, float& dep, unsigned own) {
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        const int L = int(ws->q_lane[lane]);
        const uint32_t g = ws->q_gid[lane];
        const BlendRec<float>& br = a.brec[g];
        const int xL = bx + (L & 7), yL = by + (L >> 3);
        const PixelRay<float> ray = cached_ray(ws->ray[L], zoff, xL, yL);
        const HitEval<float> h = intersect<float>(br, ray, a.cam, a.raw, g);
        const float d = !h.hit ? br.zc : (h.depth_fp64 >= 0.f ? h.depth_fp64 : midpoint_depth<float>(a.cam, ray, h.t_mid));
        if (!isfinite(d)) raise_error(a.err, kErrNonFiniteBlend, (long long)yL * a.W + xL, g);
        ws->q_wd[lane] = ws->q_w[lane] * d;
    }
    __syncwarp();
    while (own) {
        const int e = __ffs(own) - 1;
        own &= own - 1;
        dep += ws->q_wd[e];
    }
    __syncwarp();
}

// NT > 0: the semantic pass, NT = ceil(C / 8) n-tiles of accumulators in
// registers.  NT == 0: the depth pass.  (Two passes over the log: together,
// the accumulators and the depth chain's registers would spill.)
template <int NT>
__global__ void __launch_bounds__(kThreads, NT > 0 ? 2 : K6C_MINB) forward_pairs_kernel(const __grid_constant__ ForwardArgs<float> a) {
    constexpr bool kSem = NT > 0;
    constexpr bool kDepth = NT == 0;
    extern __shared__ __align__(16) unsigned char k6b_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PairSmem* const ws = reinterpret_cast<PairSmem*>(k6b_smem) + warp;
    const int seg = a.work_order ? int(a.work_order[blockIdx.x * 8 + warp]) : int(blockIdx.x) * 8 + warp;
    const int tile = seg >> 3, wl = seg & 7;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (wl & 1) * 8, by = ty * kTile + (wl >> 1) * 4;
    const int x = bx + (lane & 7), y = by + (lane >> 3);
    const int C = a.C;
    float zoff = 0.f;
    if constexpr (kDepth) {
        ws->ray[lane] = ray_cache_entry(make_ray<float>(a.cam, x, y));
        zoff = make_ray<float>(a.cam, bx, by).zoff;
    }
    const uint2 range = a.tile_range[tile];
    const size_t ev0 = size_t(8) * range.x + size_t(wl) * (range.y - range.x);
    const uint2* const evl = a.ev_list + ev0;
    const float* const wrows = a.ev_w + ev0 * 32;
    const int n_ev = int(a.ev_count[seg]);
    const int nbatch = (n_ev + 7) / 8;
    const unsigned lt = (1u << lane) - 1u;

    float acc[2][kSem ? NT : 1][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int j = 0; j < (kSem ? NT : 1); ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[mi][j][q] = 0.f;
    float dep = 0.f;
    int qn = 0;
    unsigned long long own = 0;

    // ids of batch b are fetched at iteration b - 2 (lanes < 8), stored and
    // staged at iteration b - 1, consumed at iteration b
    auto fetch_gid = [&](int b) -> uint32_t {
        const int e = 8 * b + lane;
        return (lane < 8 && e < n_ev) ? a.inst_gauss[range.x + evl[e].x] : 0u;
    };
    uint32_t g_next = 0u;  // ids of batch b + 1
    if (nbatch > 0) {
        const uint32_t g0 = fetch_gid(0);
        if (lane < 8) ws->gid[0][lane] = g0;
        g_next = fetch_gid(1);
        __syncwarp();
        stage_batch<kSem>(a, ws, wrows, 0, n_ev < 8 ? n_ev : 8, lane);
    }
    for (int b = 0; b < nbatch; ++b) {
        const int nb = n_ev - 8 * b < 8 ? n_ev - 8 * b : 8;
        const int buf = b & 1;
        // stage batch b + 1 (its ids arrived during the previous batch)
        if (b + 1 < nbatch) {
            if (lane < 8) {
                ws->gid[buf ^ 1][lane] = g_next;
                if (kDepth) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.brec + g_next)));
            }
            g_next = fetch_gid(b + 2);
            __syncwarp();
            const int nb1 = n_ev - 8 * (b + 1) < 8 ? n_ev - 8 * (b + 1) : 8;
            stage_batch<kSem>(a, ws, wrows, b + 1, nb1, lane);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        if constexpr (kSem) sem_batch<NT>(ws, buf, acc, C, nb, lane);
        // depth: enqueue each event's blending lanes, flush 32 at a time
#pragma unroll 1
        for (int k = 0; kDepth && k < nb; ++k) {
            const float wk = fabsf(ws->wt[buf][k][lane]);
            const unsigned m = __ballot_sync(0xffffffffu, wk != 0.f);
            if (wk != 0.f) {
                const int e = qn + __popc(m & lt);
                own |= 1ull << e;
                ws->q_lane[e] = uint32_t(lane);
                ws->q_gid[e] = ws->gid[buf][k];
                ws->q_w[e] = wk;
            }
            qn += __popc(m);
            __syncwarp();
            if (qn >= 32) {
                flush_depth(a, ws, zoff, 32, bx, by, dep, unsigned(own));
                own >>= 32;
                const int rest = qn - 32;
                if (lane < rest) {  // reads >= 32, writes < 32
                    ws->q_lane[lane] = ws->q_lane[32 + lane];
                    ws->q_gid[lane] = ws->q_gid[32 + lane];
                    ws->q_w[lane] = ws->q_w[32 + lane];
                }
                qn = rest;
                __syncwarp();
            }
        }
        __syncwarp();  // batch b's buffers are free for batch b + 2
    }
    if (kDepth && qn > 0) flush_depth(a, ws, zoff, qn, bx, by, dep, unsigned(own));
    const size_t HW = size_t(a.W) * a.H;
    if constexpr (kSem) {
        if (a.sem_out) {  // straight from the fragments: lane (g4, t) holds rows g4, g4 + 8 x cols 2t, 2t + 1
            const int g4 = lane >> 2, t = lane & 3;
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int row = mi * 16 + g4 + (q >> 1) * 8, ch = j * 8 + 2 * t + (q & 1);
                        const int px = bx + (row & 7), py = by + (row >> 3);
                        if (ch < C && px < a.W && py < a.H)
                            a.sem_out[size_t(ch) * HW + size_t(py) * a.W + px] = acc[mi][j][q];
                    }
        }
    }
    if (!kDepth || x >= a.W || y >= a.H) return;
    const size_t p = size_t(y) * a.W + x;
    if (a.depth) a.depth[p] = dep;
    if (!isfinite(dep)) raise_error(a.err, kErrNonFiniteOutput, (long long)p, -1);  // rasterizer.cpp:179-183
}

}  // namespace

bool forward_split_supported(int C) { return C <= 8 * kNtMax; }

void launch_forward_split(const ForwardArgs<float>& a, int ntiles, cudaStream_t s, const uint32_t* seg_order,
                          uint32_t* order_scratch) {
    if (ntiles == 0) return;
#if K6_SPLIT_DEPTH
    forward_alpha_kernel<<<ntiles, kThreads, 0, s>>>(a);
    count_launches(1);
#else
    launch_forward_blend_split(a, ntiles, s);  // blend + depth fused; semantics below
#endif
    ForwardArgs<float> b = a;
    b.work_order = nullptr;
#if !K6B_TILE_ORDER
    if (seg_order && order_scratch) {  // longest-first segment order (by event count)
        launch_work_order(a.ev_count, ntiles * 8, const_cast<uint32_t*>(seg_order), order_scratch, s);
        b.work_order = seg_order;
    }
#endif
    const size_t smem = 8 * sizeof(PairSmem);
    static std::atomic<unsigned long long> attr[9];  // per instantiation, per device
#define K6B_LAUNCH(NT_)                                                                               \
    opt_in_smem(reinterpret_cast<const void*>(forward_pairs_kernel<NT_>), attr[NT_], int(smem));      \
    forward_pairs_kernel<NT_><<<ntiles, kThreads, smem, s>>>(b);
    switch ((a.C + 7) / 8) {
        case 0: break;
        case 1: K6B_LAUNCH(1) break;
        case 2: K6B_LAUNCH(2) break;
        case 3: K6B_LAUNCH(3) break;
        case 4: K6B_LAUNCH(4) break;
        case 5: K6B_LAUNCH(5) break;
        case 6: K6B_LAUNCH(6) break;
        case 7: K6B_LAUNCH(7) break;
        default: K6B_LAUNCH(8) break;
    }
#if K6_SPLIT_DEPTH
    K6B_LAUNCH(0)
    count_launches(1);
#endif
#undef K6B_LAUNCH
    if (a.C > 0) count_launches(1);
}

}  // namespace msplat_cuda
