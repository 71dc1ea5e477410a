// K6 (FP32, C <= 64) as two kernels -- the tile loop of rasterize
// (core/src/rasterizer.cpp:112-187) split at the blend-event log.
//
// 1. forward_kernel<float, kSplit = true> (forward.cu): the blend without
//    semantics -- alpha test, colour, k, T, early termination, contributor
//    count / terminus and the ray-ellipsoid depth of every blended pair --
//    which also writes the event log and the BLEND WEIGHTS of every event as
//    one 32-float row (w = alpha T for the blending lanes, 0 elsewhere,
//    negated where alpha was clamped at 0.99: the backward reads the same
//    rows).  Without the semantic accumulators it runs at 3 CTAs / SM.
// 2. forward_pairs_kernel<NT> (here): the semantic logits, replayed from the
//    log.  One warp per (tile, 8x4 block) segment walks its events front to
//    back in batches of 8, software-pipelined one batch ahead (the batch's
//    weight rows and semantic rows staged into shared memory by cp.async
//    while the previous batch computes; Gaussian ids fetched two batches
//    ahead), and accumulates O[32 px][C] += W[32 px][8 ev] . S[8 ev][C] on
//    the tensor cores (mma.sync m16n8k8 TF32 with a hi/lo split:
//    FP32-level accuracy) into REGISTER accumulators (the fused kernel had to
//    keep them in shared memory).
// Same per-pixel summation order as the fused kernel for colour, k, depth;
// the semantic sums run in the same 8-event batches.
// Measured alternative (cfg3): a depth-free alpha pass (0.53 ms) + a separate
// depth pass (1.0-1.14 ms) + this pass was slower (2.18 ms) than the blend
// with depth + this pass (1.78 ms): the depth pass re-walks the log and its
// BlendRec gathers lose the L1 prefetch the blend issues at box-hit time.
#include "blend_common.cuh"
#include "kernels.h"

namespace msplat_cuda {

namespace {

constexpr int kNtMax = 8;  // semantic n-tiles in registers: C <= 64


// ---------------------------------------------------------------- K6b
constexpr int kWPitch = 40;    // W tile rows: (k * 40) mod 32 = 8 k, conflict-free A fragments
constexpr int kSemPitch = 72;  // staged semantic rows: (t * 72) mod 32 = 8 t, conflict-free B fragments

constexpr int kOutPitch = 36;   // epilogue tile [channel][36]: conflict-free fragment stores and pixel reads

struct PairStage {
    float wt[2][8][kWPitch];      // W^T[8 ev][32 px] tiles (the weight rows as written), double-buffered
    float srow[2][8][kSemPitch];  // the batch's semantic rows (16-byte chunks: the row starts at soff)
    uint32_t gid[2][8];           // the batch's Gaussian ids, double-buffered
    uint32_t soff[2][8];          // float offset of each semantic row inside its staged chunks
};
// The staging buffers, then (after the last batch) the output tile.
union PairSmem {
    PairStage st;
    float out[8 * kNtMax][kOutPitch];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src)
                 : "memory");
}

// Issues the cp.async staging of batch b (nb events; ids already in
// ws->st.gid[b & 1]): the events' weight rows (16-byte pieces) and semantic
// rows (16-byte chunks, four lanes per event).  One commit group.
__device__ __forceinline__ void stage_batch(const ForwardArgs<float>& a, PairSmem* ws, const float* wrows, int b, int nb,
                                            int lane) {
    const int buf = b & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // 8 rows x 8 16-byte pieces
        const int i = lane + 32 * h, kk = i >> 3, q = i & 7;
        float* const dst = &ws->st.wt[buf][kk][4 * q];
        if (kk < nb) cp_async16(dst, wrows + size_t(8 * b + kk) * 32 + 4 * q);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // semantic rows: the 16-byte chunks covering each row (any 4-byte
    // alignment; a chunk never straddles a page, so reading whole chunks is
    // safe), 4 lanes per event, the row's float offset in soff
    const int C = a.C;
    const int k = lane >> 2, part = lane & 3;
    if (k < nb) {
        const uintptr_t r0 = reinterpret_cast<uintptr_t>(a.semantics + size_t(ws->st.gid[buf][k]) * C);
        const uintptr_t c0 = r0 & ~uintptr_t(15);
        const int nch = int(((r0 + uintptr_t(4 * C) + 15) & ~uintptr_t(15)) - c0) >> 4;
        if (part == 0) ws->st.soff[buf][k] = uint32_t(r0 - c0) >> 2;
        const float* src = reinterpret_cast<const float*>(c0) + 4 * part;
        float* dst = ws->st.srow[buf][k] + 4 * part;
        for (int q = part; q < nch; q += 4, src += 16, dst += 16) cp_async16(dst, src);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// O += W S for a staged batch (events beyond nb: zero W rows, S rows never read).
template <int NT>
__device__ __forceinline__ void sem_batch(const PairSmem* ws, int buf, float (&acc)[2][NT][4], int C, int nb,
                                          int lane) {
    const int g4 = lane >> 2, t = lane & 3;
    const float* const w0 = ws->st.wt[buf][t];      // event t's weights over the 32 pixels
    const float* const w1 = ws->st.wt[buf][t + 4];  // event t + 4
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {  // A[px][ev]: rows px = 16 mi + g4 (+ 8), cols ev = t (+ 4)
        const int r0 = mi * 16 + g4, r1 = r0 + 8;
        split_tf32(fabsf(w0[r0]), ah[mi][0], al[mi][0]);  // (the sign marks a clamped alpha)
        split_tf32(fabsf(w0[r1]), ah[mi][1], al[mi][1]);
        split_tf32(fabsf(w1[r0]), ah[mi][2], al[mi][2]);
        split_tf32(fabsf(w1[r1]), ah[mi][3], al[mi][3]);
    }
    const float* const s0 = ws->st.srow[buf][t] + ws->st.soff[buf][t];
    const float* const s1 = ws->st.srow[buf][t + 4] + ws->st.soff[buf][t + 4];
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

#ifndef K6B_WARPS
#define K6B_WARPS 4  // warps per CTA of the semantic pass (4 x 4 CTAs/SM: 285 us vs 295 at 8 x 2)
#endif
#ifndef K6B_MINB
#define K6B_MINB (16 / K6B_WARPS)
#endif
constexpr int kSemWarps = K6B_WARPS;

// NT = ceil(C / 8) semantic n-tiles of accumulators in registers.
template <int NT>
__global__ void __launch_bounds__(32 * kSemWarps, K6B_MINB) forward_pairs_kernel(const __grid_constant__ ForwardArgs<float> a) {
    extern __shared__ __align__(16) unsigned char k6b_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PairSmem* const ws = reinterpret_cast<PairSmem*>(k6b_smem) + warp;
    const int item = int(blockIdx.x) * kSemWarps + warp;
    if (item >= a.nseg) return;
    const int seg = a.work_order ? int(a.work_order[item]) : item;
    const int tile = seg >> 3, wl = seg & 7;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = tx * kTile + (wl & 1) * 8, by = ty * kTile + (wl >> 1) * 4;
    const int C = a.C;
    const uint2 range = a.tile_range[tile];
    const size_t ev0 = size_t(8) * range.x + size_t(wl) * (range.y - range.x);
    const float* const wrows = a.ev_w + ev0 * 32;
    const int n_ev = int(a.ev_count[seg]);
    const int nbatch = (n_ev + 7) / 8;

    float acc[2][NT][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[mi][j][q] = 0.f;

    // ids of batch b are fetched at iteration b - 2 (lanes < 8), stored and
    // staged at iteration b - 1, consumed at iteration b
    const uint4* const evl = a.ev_list + ev0;  // the blend logs each event's Gaussian id
    auto fetch_gid = [&](int b) -> uint32_t {
        const int e = 8 * b + lane;
        return (lane < 8 && e < n_ev) ? evl[e].z : 0u;
    };
    uint32_t g_next = 0u;  // ids of batch b + 1
    if (nbatch > 0) {
        const uint32_t g0 = fetch_gid(0);
        if (lane < 8) ws->st.gid[0][lane] = g0;
        g_next = fetch_gid(1);
        __syncwarp();
        stage_batch(a, ws, wrows, 0, n_ev < 8 ? n_ev : 8, lane);
    }
    for (int b = 0; b < nbatch; ++b) {
        const int nb = n_ev - 8 * b < 8 ? n_ev - 8 * b : 8;
        const int buf = b & 1;
        if (b + 1 < nbatch) {  // stage batch b + 1 (its ids arrived during the previous batch)
            if (lane < 8) ws->st.gid[buf ^ 1][lane] = g_next;
            g_next = fetch_gid(b + 2);
            __syncwarp();
            const int nb1 = n_ev - 8 * (b + 1) < 8 ? n_ev - 8 * (b + 1) : 8;
            stage_batch(a, ws, wrows, b + 1, nb1, lane);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        sem_batch<NT>(ws, buf, acc, C, nb, lane);
        __syncwarp();  // batch b's buffers are free for batch b + 2
    }
    if (!a.sem_out) return;
    // through shared memory: the fragments (lane (g4, t) holds pixel rows g4,
    // g4 + 8 x channels 2t, 2t + 1) into [channel][pixel], then each lane
    // writes its own pixel of every channel plane (4 x 32-byte rows per plane)
    __syncwarp();  // the staging buffers are free
    const int g4 = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                ws->out[j * 8 + 2 * t + (q & 1)][mi * 16 + g4 + (q >> 1) * 8] = acc[mi][j][q];
    __syncwarp();
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    if (px < a.W && py < a.H) {
        const size_t HW = size_t(a.W) * a.H;
        float* dst = a.sem_out + size_t(py) * a.W + px;
        for (int ch = 0; ch < C; ++ch, dst += HW) *dst = ws->out[ch][lane];
    }
}

}  // namespace

bool forward_split_supported(int C) { return C <= 8 * kNtMax; }

void launch_forward_split(const ForwardArgs<float>& a, int ntiles, cudaStream_t s, const uint32_t* seg_order,
                          uint32_t* order_scratch) {
    if (ntiles == 0) return;
    launch_forward_blend_split(a, ntiles, s);  // blend + depth; semantics below
    if (a.C == 0) return;
    ForwardArgs<float> b = a;
    b.work_order = nullptr;
    if (seg_order && order_scratch) {  // longest-first segment order (by event count)
        launch_work_order(a.ev_count, ntiles * 8, const_cast<uint32_t*>(seg_order), order_scratch, s);
        b.work_order = seg_order;
    }
    b.nseg = ntiles * 8;
    const unsigned ctas = unsigned((ntiles * 8 + kSemWarps - 1) / kSemWarps);
    const size_t smem = kSemWarps * sizeof(PairSmem);
    static std::atomic<unsigned long long> attr[kNtMax + 1];  // per instantiation, per device
#define K6B_LAUNCH(NT_)                                                                          \
    opt_in_smem(reinterpret_cast<const void*>(forward_pairs_kernel<NT_>), attr[NT_], int(smem)); \
    forward_pairs_kernel<NT_><<<ctas, 32 * kSemWarps, smem, s>>>(b);
    switch ((a.C + 7) / 8) {
        case 1: K6B_LAUNCH(1) break;
        case 2: K6B_LAUNCH(2) break;
        case 3: K6B_LAUNCH(3) break;
        case 4: K6B_LAUNCH(4) break;
        case 5: K6B_LAUNCH(5) break;
        case 6: K6B_LAUNCH(6) break;
        case 7: K6B_LAUNCH(7) break;
        default: K6B_LAUNCH(8) break;
    }
#undef K6B_LAUNCH
    count_launches(1);
}

}  // namespace msplat_cuda
