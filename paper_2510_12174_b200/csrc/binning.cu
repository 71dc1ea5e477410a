// K2-K5: binning.  Replaces bin_and_sort (core/src/rasterizer.cpp:14-45).
//
// The reference sorts visible splats by (sort_depth, index) with std::sort and
// pushes each one into every tile of its rect, so each tile list ascends by
// (depth, index).  Only that per-tile order is observable, so the B200 path
// never sorts globally by depth:
//   K2  tile histogram: every (Gaussian, tile) instance bumps its tile's
//       counter (global atomics; 3.2k counters at cfg3);
//   K3  one CTA scans the counters into the per-tile [start, end) ranges
//       (the instance total and the longest list with them);
//   K4  scatter: every instance claims a slot of its tile by an atomic cursor
//       and writes (depth key, Gaussian id) there -- the order inside a tile
//       is arbitrary at this point;
//   K5  one CTA per tile sorts its list by (depth key, id) with a bitonic
//       network in shared memory (lists longer than the shared-memory
//       capacity run the same network in place in global memory).  The
//       (key, id) order is total, so the result is the reference's list bit
//       for bit whatever order the atomics produced.
// The round-1 pipeline (global LSD radix sort by depth, emission in depth
// order, stable radix sort by tile) is kept behind MSPLAT_RADIX_BINNING=1 for
// A/B timing.  All counts stay on the device: no host round trip.
#include "common.cuh"
#include "kernels.h"
#include "radix_sort.cuh"

#include <algorithm>
#include <cstdlib>

namespace msplat_cuda {

namespace {

constexpr int kDepthBits = 9;   // 7 passes x 9 bits = bits 0..62 (bit 63 is 0 for z > 0)
constexpr int kTileBits = 8;

__global__ void gather_counts_kernel(int64_t n, const uint32_t* __restrict__ order_sorted,
                                     const uint32_t* __restrict__ tile_count,
                                     uint32_t* __restrict__ count_sorted) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) count_sorted[r] = tile_count[order_sorted[r]];
}

__global__ void finalize_count_kernel(const uint32_t* __restrict__ total32, int64_t cap,
                                      int64_t* __restrict__ d_count, DeviceError* err) {
    const int64_t total = int64_t(*total32);
    if (total > cap) {
        raise_error(err, kErrInstanceOverflow, total, cap);
        *d_count = 0;  // render nothing; the host grows the buffers and re-runs
    } else {
        *d_count = total;
    }
}

// One thread per depth-sorted Gaussian emits its (usually 1-4) instances; the
// rare Gaussian covering more than 32 tiles (a near-plane splat: SURVEY.md
// App. C saw 2.9k of them produce 94% of instances) is emitted by its whole
// warp instead, so no thread serialises a huge rect.  Consecutive threads own
// consecutive output ranges (the scan is in depth order): coalesced writes.
__global__ void __launch_bounds__(256) emit_instances_kernel(int64_t n, const uint32_t* __restrict__ order_sorted,
                                                             const uint2* __restrict__ tile_rect,
                                                             const uint32_t* __restrict__ count_sorted,
                                                             const uint32_t* __restrict__ offset_sorted, int tiles_x,
                                                             const int64_t* __restrict__ d_count,
                                                             uint32_t* __restrict__ inst_tile,
                                                             uint32_t* __restrict__ inst_gauss) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool overflow = *d_count == 0;  // nothing is emitted; the host grows the buffers
    uint32_t cnt = 0, g = 0, off = 0;
    uint2 rect = make_uint2(0, 0);
    if (r < n && !overflow) {
        cnt = count_sorted[r];
        if (cnt) {
            g = order_sorted[r];
            rect = tile_rect[g];
            off = offset_sorted[r];
        }
    }
    const bool big = cnt > 32u;
    if (cnt && !big) {
        const int tx0 = int(rect.x & 0xffffu), tx1 = int(rect.x >> 16), ty0 = int(rect.y & 0xffffu);
        int tx = tx0, ty = ty0;
        for (uint32_t j = 0; j < cnt; ++j) {
            inst_tile[off + j] = uint32_t(ty * tiles_x + tx);
            inst_gauss[off + j] = g;
            if (++tx > tx1) {
                tx = tx0;
                ++ty;
            }
        }
    }
    unsigned bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {
        const int src = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        const uint32_t bc = __shfl_sync(0xffffffffu, cnt, src), bg = __shfl_sync(0xffffffffu, g, src);
        const uint32_t bo = __shfl_sync(0xffffffffu, off, src);
        const uint32_t rx = __shfl_sync(0xffffffffu, rect.x, src), ry = __shfl_sync(0xffffffffu, rect.y, src);
        const int tx0 = int(rx & 0xffffu), tx1 = int(rx >> 16), ty0 = int(ry & 0xffffu);
        const int w = tx1 - tx0 + 1;
        for (uint32_t j = lane; j < bc; j += 32) {
            inst_tile[bo + j] = uint32_t((ty0 + int(j) / w) * tiles_x + tx0 + int(j) % w);
            inst_gauss[bo + j] = bg;
        }
    }
}

__global__ void tile_ranges_kernel(const int64_t* __restrict__ d_count,
                                   const uint32_t* __restrict__ tile_sorted,
                                   uint2* __restrict__ range) {
    const int64_t count = *d_count;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t t = tile_sorted[i];
    if (i == 0 || tile_sorted[i - 1] != t) range[t].x = uint32_t(i);
    if (i == count - 1 || tile_sorted[i + 1] != t) range[t].y = uint32_t(i + 1);
}

// ---------------------------------------------------------------- per-tile path
// Calls f(g, tile) for every tile of Gaussian r's rect (r < end): one thread
// per Gaussian, or the whole warp for the rare splat covering more than 32
// tiles.  Must be called by full warps with consecutive r.
template <typename F>
__device__ __forceinline__ void for_each_instance(int64_t r, int64_t end, const uint32_t* __restrict__ tile_count,
                                                  const uint2* __restrict__ tile_rect, int tiles_x, F&& f) {
    const int lane = threadIdx.x & 31;
    uint32_t cnt = 0;
    uint2 rect = make_uint2(0, 0);
    if (r < end) {
        cnt = tile_count[r];
        if (cnt) rect = tile_rect[r];
    }
    const bool big = cnt > 32u;
    if (cnt && !big) {
        const int tx0 = int(rect.x & 0xffffu), tx1 = int(rect.x >> 16), ty0 = int(rect.y & 0xffffu);
        int tx = tx0, ty = ty0;
        for (uint32_t j = 0; j < cnt; ++j) {
            f(uint32_t(r), uint32_t(ty * tiles_x + tx));
            if (++tx > tx1) {
                tx = tx0;
                ++ty;
            }
        }
    }
    unsigned bigs = __ballot_sync(0xffffffffu, big);
    while (bigs) {
        const int src = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        const uint32_t bc = __shfl_sync(0xffffffffu, cnt, src);
        const uint32_t rx = __shfl_sync(0xffffffffu, rect.x, src), ry = __shfl_sync(0xffffffffu, rect.y, src);
        const uint32_t bg = uint32_t(r - lane + src);
        const int tx0 = int(rx & 0xffffu), tx1 = int(rx >> 16), ty0 = int(ry & 0xffffu);
        const int w = tx1 - tx0 + 1;
        for (uint32_t j = lane; j < bc; j += 32) f(bg, uint32_t((ty0 + int(j) / w) * tiles_x + tx0 + int(j) % w));
    }
}

// K2 / K4 grid: kBinCtas CTAs per SM, each over a contiguous chunk of
// Gaussians.  With kPriv the CTA counts its instances per tile in shared
// memory first (all atomics on 3.2k global counters would queue on a few L2
// slices), then flushes one coalesced atomic per non-empty tile.
constexpr int kBinThreads = 512;
constexpr int kBinCtas = 2;
constexpr int64_t kPrivMaxTiles = 24576;  // 2 x 96 KB of shared bins (scatter)

// Also reduces the depth-key range of the binned Gaussians into
// key_range[0] = max ~key, key_range[1] = max key (zeroed beforehand).
template <bool kPriv>
__global__ void __launch_bounds__(kBinThreads) tile_hist_kernel(int64_t n, int64_t chunk,
                                                                const uint32_t* __restrict__ tile_count,
                                                                const uint2* __restrict__ tile_rect, int tiles_x,
                                                                int64_t tiles, const uint64_t* __restrict__ depth_key,
                                                                uint32_t* __restrict__ tile_cnt,
                                                                unsigned long long* __restrict__ key_range) {
    extern __shared__ uint32_t s_bin[];
    __shared__ unsigned long long s_range[2];
    if (threadIdx.x < 2) s_range[threadIdx.x] = 0ull;
    if constexpr (kPriv)
        for (int64_t t = threadIdx.x; t < tiles; t += kBinThreads) s_bin[t] = 0u;
    __syncthreads();
    const int64_t b0 = int64_t(blockIdx.x) * chunk, b1 = min(n, b0 + chunk);
    unsigned long long kmin_c = 0ull, kmax = 0ull;  // kmin_c: max of ~key
    for (int64_t base = b0 + (threadIdx.x & ~31); base < b1; base += kBinThreads) {
        const int64_t r = base + (threadIdx.x & 31);
        if (r < b1 && tile_count[r]) {
            const unsigned long long k = depth_key[r];
            kmin_c = max(kmin_c, ~k);
            kmax = max(kmax, k);
        }
        for_each_instance(r, b1, tile_count, tile_rect, tiles_x, [&](uint32_t, uint32_t t) {
            if constexpr (kPriv)
                atomicAdd(s_bin + t, 1u);
            else
                atomicAdd(tile_cnt + t, 1u);
        });
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin_c = max(kmin_c, __shfl_xor_sync(0xffffffffu, kmin_c, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(s_range, kmin_c);
        atomicMax(s_range + 1, kmax);
    }
    __syncthreads();
    if (threadIdx.x < 2 && s_range[threadIdx.x]) atomicMax(key_range + threadIdx.x, s_range[threadIdx.x]);
    if constexpr (kPriv) {
        for (int64_t t = threadIdx.x; t < tiles; t += kBinThreads) {
            const uint32_t v = s_bin[t];
            if (v) atomicAdd(tile_cnt + t, v);
        }
    }
}

// K3: one CTA scans the per-tile counters into the [start, end) ranges and
// the scatter cursors; the instance total and the longest list go to
// d_total[0..1]; tiles whose list exceeds kSortSmall are listed in
// big[1..big[0]] for the large-list sort.  On overflow every range is left
// empty and the latched error makes the host grow the buffers and re-run.
constexpr int kTileScanThreads = 1024;
constexpr int kSortE = 8;                              // keys per thread of the register sort
constexpr int kSortSmallThreads = 256;
constexpr int kSortSmall = kSortSmallThreads * kSortE;  // 2048: one CTA per tile
constexpr int kSortMediumThreads = 512;                   // lists up to 4096
constexpr int kSortLargeThreads = 1024;                   // up to 8192 in registers, beyond in global memory
__global__ void __launch_bounds__(kTileScanThreads) tile_scan_kernel(int64_t tiles, const uint32_t* __restrict__ tile_cnt,
                                                                     int64_t cap, uint2* __restrict__ range,
                                                                     uint32_t* __restrict__ cursor,
                                                                     int64_t* __restrict__ d_count,
                                                                     uint32_t* __restrict__ d_total,
                                                                     uint32_t* __restrict__ big, DeviceError* err) {
    __shared__ uint32_t s_max[kTileScanThreads / 32];
    __shared__ uint32_t s_nbig;
    if (threadIdx.x == 0) s_nbig = 0;
    __syncthreads();
    uint32_t carry = 0, mx = 0;
    for (int64_t base = 0; base < tiles; base += kTileScanThreads) {
        const int64_t t = base + threadIdx.x;
        const uint32_t c = t < tiles ? tile_cnt[t] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<uint32_t, kTileScanThreads>(c, tot);
        if (t < tiles) {
            range[t] = make_uint2(carry + ex, carry + ex + c);
            cursor[t] = carry + ex;
            if (c > uint32_t(kSortSmall)) big[1 + atomicAdd(&s_nbig, 1u)] = uint32_t(t);
        }
        carry += tot;  // CTA-uniform
        mx = max(mx, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    const bool overflow = int64_t(carry) > cap;
    if (overflow)
        for (int64_t t = threadIdx.x; t < tiles; t += kTileScanThreads) range[t] = make_uint2(0u, 0u);
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int w = 0; w < kTileScanThreads / 32; ++w) m = max(m, s_max[w]);
        d_total[0] = carry;
        d_total[1] = m;
        big[0] = overflow ? 0u : s_nbig;
        if (overflow) raise_error(err, kErrInstanceOverflow, int64_t(carry), cap);
        *d_count = overflow ? 0 : int64_t(carry);
    }
}

// Sort item of an instance: a 32-bit monotone image of its 64-bit depth key
// over the Gaussian id.  The image is (key - min) >> shift with the shift
// that fits this view's key range into 32 bits (about 31 significant bits of
// depth at cfg3 instead of the IEEE high word's 20), so sorting items puts
// every tile list in (depth, index) order except inside runs of equal images,
// which the sort settles with the full keys (sort_tile_regs).
struct KeyMap {
    uint64_t kmin;
    int shift;
};
__device__ __forceinline__ KeyMap key_map(const unsigned long long* key_range) {
    KeyMap m;
    m.kmin = ~key_range[0];
    const uint64_t span = key_range[1] > m.kmin ? key_range[1] - m.kmin : 0ull;
    m.shift = span >> 32 ? 32 - __clzll(span) : 0;
    return m;
}
__device__ __forceinline__ uint64_t sort_item(const KeyMap& m, uint64_t key, uint32_t g) {
    return (((key - m.kmin) >> m.shift) << 32) | g;
}

// K4: every instance claims a slot of its tile and writes its sort item
// there (the order inside a tile is arbitrary until K5).  kPriv: the CTA
// counts per tile in shared memory, reserves one block of slots per
// non-empty tile with a single global atomic, then hands the block out with
// shared atomics.
template <bool kPriv>
__global__ void __launch_bounds__(kBinThreads) tile_scatter_kernel(int64_t n, int64_t chunk,
                                                                   const uint32_t* __restrict__ tile_count,
                                                                   const uint2* __restrict__ tile_rect, int tiles_x,
                                                                   int64_t tiles, const uint64_t* __restrict__ depth_key,
                                                                   const int64_t* __restrict__ d_count,
                                                                   const unsigned long long* __restrict__ key_range,
                                                                   uint32_t* __restrict__ cursor,
                                                                   uint64_t* __restrict__ items) {
    extern __shared__ uint32_t s_bin[];
    uint32_t* const s_base = s_bin + tiles;
    if (*d_count == 0) return;  // empty, or overflow (no slot is valid)
    const KeyMap km = key_map(key_range);
    const int64_t b0 = int64_t(blockIdx.x) * chunk, b1 = min(n, b0 + chunk);
    if constexpr (kPriv) {
        for (int64_t t = threadIdx.x; t < tiles; t += kBinThreads) s_bin[t] = 0u;
        __syncthreads();
        for (int64_t base = b0 + (threadIdx.x & ~31); base < b1; base += kBinThreads)
            for_each_instance(base + (threadIdx.x & 31), b1, tile_count, tile_rect, tiles_x,
                              [&](uint32_t, uint32_t t) { atomicAdd(s_bin + t, 1u); });
        __syncthreads();
        for (int64_t t = threadIdx.x; t < tiles; t += kBinThreads) {
            const uint32_t v = s_bin[t];
            if (v) s_base[t] = atomicAdd(cursor + t, v);
            s_bin[t] = 0u;
        }
        __syncthreads();
    }
    for (int64_t base = b0 + (threadIdx.x & ~31); base < b1; base += kBinThreads) {
        const int64_t r = base + (threadIdx.x & 31);
        const uint64_t key = r < b1 ? depth_key[r] : 0ull;
        for_each_instance(r, b1, tile_count, tile_rect, tiles_x, [&](uint32_t g, uint32_t t) {
            uint32_t pos;
            if constexpr (kPriv)
                pos = s_base[t] + atomicAdd(s_bin + t, 1u);
            else
                pos = atomicAdd(cursor + t, 1u);
            items[pos] = sort_item(km, g == uint32_t(r) ? key : depth_key[g], g);
        });
    }
}

// ---- K5: per-tile sort of the items (bitonic network, flip form: every
// compare-exchange leaves the minimum at the lower index).  Thread t of the
// sorting group holds items t*E .. t*E+E-1 in registers; partners inside a
// thread are exchanged in registers, inside a warp by shuffles, across warps
// through shared memory (8-byte slots, index skewed by i/8: conflict-free).
// Positions >= L hold ~0 (above every real item: ids are < 2^31).
__device__ __forceinline__ int skew(int i) { return i + (i >> 3); }

template <int S>  // flip step of size S <= E inside the thread: pairs (j, j ^ (S-1))
__device__ __forceinline__ void reg_flip(uint64_t (&v)[kSortE]) {
#pragma unroll
    for (int j = 0; j < kSortE; ++j) {
        const int p = j ^ (S - 1);
        if (p > j) {
            const uint64_t lo = min(v[j], v[p]), hi = max(v[j], v[p]);
            v[j] = lo;
            v[p] = hi;
        }
    }
}
template <int ST>  // half-cleaner step of stride ST < E inside the thread
__device__ __forceinline__ void reg_step(uint64_t (&v)[kSortE]) {
#pragma unroll
    for (int j = 0; j < kSortE; ++j) {
        if (!(j & ST)) {
            const uint64_t lo = min(v[j], v[j + ST]), hi = max(v[j], v[j + ST]);
            v[j] = lo;
            v[j + ST] = hi;
        }
    }
}
// Strides 4, 2, 1: the tail of every merge of size >= 16.
__device__ __forceinline__ void reg_tail(uint64_t (&v)[kSortE]) {
    reg_step<4>(v);
    reg_step<2>(v);
    reg_step<1>(v);
}

__device__ __forceinline__ void group_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Sorts the group's P (power of two, <= nthreads * E) items in v.  t: thread
// index in the group; sm: >= skew(P) slots (used when P > 32 E).
__device__ __forceinline__ void bitonic_regs(uint64_t (&v)[kSortE], int P, int t, int nthreads, uint64_t* sm) {
    for (int s = 2; s <= P; s <<= 1) {
        // flip step: partner i ^ (s - 1)
        if (s == 2) {
            reg_flip<2>(v);
            continue;
        } else if (s == 4) {
            reg_flip<4>(v);
            reg_step<1>(v);
            continue;
        } else if (s == 8) {
            reg_flip<8>(v);
            reg_step<2>(v);
            reg_step<1>(v);
            continue;
        } else {
            const int m = s / kSortE - 1;     // partner thread t ^ m, item E-1-j
            const bool lower = !(t & ((s / kSortE) >> 1));
            uint64_t o[kSortE];
            if (s <= 32 * kSortE) {
#pragma unroll
                for (int j = 0; j < kSortE; ++j) o[j] = __shfl_xor_sync(0xffffffffu, v[kSortE - 1 - j], m);
            } else {
#pragma unroll
                for (int j = 0; j < kSortE; ++j) sm[skew(t * kSortE + j)] = v[j];
                group_sync(nthreads);
                const int pt = t ^ m;
#pragma unroll
                for (int j = 0; j < kSortE; ++j) o[j] = sm[skew(pt * kSortE + kSortE - 1 - j)];
                group_sync(nthreads);
            }
#pragma unroll
            for (int j = 0; j < kSortE; ++j) v[j] = lower ? min(v[j], o[j]) : max(v[j], o[j]);
        }
        // half-cleaner steps, stride s/4 .. 1
        for (int st = s >> 2; st >= kSortE; st >>= 1) {
            const int m = st / kSortE;
            const bool lower = !(t & m);
            uint64_t o[kSortE];
            if (st < 32 * kSortE) {
#pragma unroll
                for (int j = 0; j < kSortE; ++j) o[j] = __shfl_xor_sync(0xffffffffu, v[j], m);
            } else {
#pragma unroll
                for (int j = 0; j < kSortE; ++j) sm[skew(t * kSortE + j)] = v[j];
                group_sync(nthreads);
#pragma unroll
                for (int j = 0; j < kSortE; ++j) o[j] = sm[skew((t ^ m) * kSortE + j)];
                group_sync(nthreads);
            }
#pragma unroll
            for (int j = 0; j < kSortE; ++j) v[j] = lower ? min(v[j], o[j]) : max(v[j], o[j]);
        }
        reg_tail(v);
    }
}

// Runs of equal high words: (full key, id) order by insertion sort (the run
// is id-ordered already, so this is linear unless full keys differ).  at(i)
// addresses item i; every item is rewritten as its id's final position.
template <typename At>
__device__ __forceinline__ void sort_fixup(At at, int i, int L, const uint64_t* __restrict__ depth_key) {
    const uint64_t it = at(i);
    const bool head = (i == 0 || (at(i - 1) >> 32) != (it >> 32)) && i + 1 < L && (at(i + 1) >> 32) == (it >> 32);
    if (!head) return;
    int e = i + 1;
    while (e < L && (at(e) >> 32) == (it >> 32)) ++e;
    for (int k = i + 1; k < e; ++k) {
        const uint64_t x = at(k);
        const uint64_t kx = depth_key[uint32_t(x)];
        int p = k - 1;
        while (p >= i) {
            const uint64_t y = at(p);
            const uint64_t ky = depth_key[uint32_t(y)];
            if (ky < kx || (ky == kx && uint32_t(y) < uint32_t(x))) break;
            at(p + 1) = y;
            --p;
        }
        at(p + 1) = x;
    }
}

// Register sort of one tile list of L <= nthreads * E items by a group of
// nthreads threads (warps beyond the list's power of two return early).
// sm, fk: >= skew(L) slots each.  After the item sort, runs of equal high
// words are in id order; they are also in (full key, id) order unless some
// full key decreases along the run.  The members' full keys are gathered in
// parallel and checked pairwise; only when a run is out of order (distinct
// depths sharing a high word: rare, while exactly equal depths -- e.g. a
// wall facing the camera -- are common and already in order) do the run
// heads insertion-sort their runs.
__device__ __forceinline__ void sort_tile_regs(const uint64_t* __restrict__ items, int L, int nthreads,
                                               uint64_t* sm, uint64_t* fk, int* s_flag,
                                               const uint64_t* __restrict__ depth_key, uint32_t* __restrict__ out) {
    int P = 1;
    while (P < L) P <<= 1;
    const int active = max(32, ((P + kSortE - 1) / kSortE + 31) & ~31);
    const int t = threadIdx.x;
    if (t >= active) return;
    uint64_t v[kSortE];
#pragma unroll
    for (int j = 0; j < kSortE; ++j) {
        const int i = t * kSortE + j;
        v[j] = i < L ? items[i] : ~0ull;
    }
    bitonic_regs(v, P, t, active, sm);
    if (t == 0) *s_flag = 0;
#pragma unroll
    for (int j = 0; j < kSortE; ++j) sm[skew(t * kSortE + j)] = v[j];
    group_sync(active);
    // full keys of run members (one parallel gather)
#pragma unroll
    for (int j = 0; j < kSortE; ++j) {
        const int i = t * kSortE + j;
        if (i >= L) break;
        const uint32_t h = uint32_t(v[j] >> 32);
        const bool run = (i > 0 && uint32_t(sm[skew(i - 1)] >> 32) == h) ||
                         (i + 1 < L && uint32_t(sm[skew(i + 1)] >> 32) == h);
        if (run) fk[skew(i)] = depth_key[uint32_t(v[j])];
    }
    group_sync(active);
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kSortE; ++j) {
        const int i = t * kSortE + j;
        if (i >= L) break;
        if (i > 0 && uint32_t(sm[skew(i - 1)] >> 32) == uint32_t(v[j] >> 32) && fk[skew(i - 1)] > fk[skew(i)])
            bad = true;
    }
    if (bad) *s_flag = 1;
    group_sync(active);
    if (*s_flag) {
#pragma unroll 1
        for (int j = 0; j < kSortE; ++j) {
            const int i = t * kSortE + j;
            if (i >= L) break;
            const uint32_t h = uint32_t(sm[skew(i)] >> 32);
            if (!((i == 0 || uint32_t(sm[skew(i - 1)] >> 32) != h) && i + 1 < L &&
                  uint32_t(sm[skew(i + 1)] >> 32) == h))
                continue;
            int e = i + 1;
            while (e < L && uint32_t(sm[skew(e)] >> 32) == h) ++e;
            for (int k = i + 1; k < e; ++k) {  // (full key, id) insertion sort
                const uint64_t x = sm[skew(k)], kx = fk[skew(k)];
                int p = k - 1;
                while (p >= i) {
                    const uint64_t y = sm[skew(p)], ky = fk[skew(p)];
                    if (ky < kx || (ky == kx && uint32_t(y) < uint32_t(x))) break;
                    sm[skew(p + 1)] = y;
                    fk[skew(p + 1)] = ky;
                    --p;
                }
                sm[skew(p + 1)] = x;
                fk[skew(p + 1)] = kx;
            }
        }
        group_sync(active);
    }
    // coalesced output: thread t writes ids t, t + active, ...
    for (int i = t; i < L; i += active) out[i] = uint32_t(sm[skew(i)]);
}

__global__ void __launch_bounds__(kSortSmallThreads) tile_sort_small_kernel(const uint2* __restrict__ range,
                                                                            const uint64_t* __restrict__ items,
                                                                            const uint64_t* __restrict__ depth_key,
                                                                            uint32_t* __restrict__ out) {
    __shared__ uint64_t sm[kSortSmall + kSortSmall / 8], fk[kSortSmall + kSortSmall / 8];
    __shared__ int s_flag;
    const uint2 rg = range[blockIdx.x];
    const int L = int(rg.y - rg.x);
    if (L <= 0 || L > kSortSmall) return;
    if (L == 1) {
        if (threadIdx.x == 0) out[rg.x] = uint32_t(items[rg.x]);
        return;
    }
    sort_tile_regs(items + rg.x, L, kSortSmallThreads, sm, fk, &s_flag, depth_key, out + rg.x);
}

// Lists longer than kSortSmall: persistent CTAs over big[1..big[0]], each
// variant taking the lists in (LO, THREADS * E] (medium: 512 threads, up to
// 4096; large: 1024 threads, up to 8192 in registers and, beyond that, the
// flip-form network in place in global memory -- positions >= L are virtual
// +inf and never touched).
template <int THREADS, int LO, bool kGlobal>
__global__ void __launch_bounds__(THREADS) tile_sort_big_kernel(const uint2* __restrict__ range,
                                                                const uint32_t* __restrict__ big,
                                                                uint64_t* __restrict__ items,
                                                                const uint64_t* __restrict__ depth_key,
                                                                uint32_t* __restrict__ out) {
    constexpr int HI = THREADS * kSortE;
    extern __shared__ uint64_t sml[];
    __shared__ int s_flag;
    uint64_t* const fkl = sml + HI + HI / 8;
    const uint32_t nbig = big[0];
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
        const uint32_t tile = big[1 + b];
        const uint2 rg = range[tile];
        const int L = int(rg.y - rg.x);
        if (L <= LO || (!kGlobal && L > HI)) continue;
        if (L <= HI) {
            sort_tile_regs(items + rg.x, L, THREADS, sml, fkl, &s_flag, depth_key, out + rg.x);
            __syncthreads();  // warps that returned early are back: next tile
            continue;
        }
        uint64_t* const k = items + rg.x;
        int P = 1;
        while (P < L) P <<= 1;
        for (int s = 2; s <= P; s <<= 1) {
            for (int st = s >> 1; st > 0; st >>= 1) {
                for (int i = threadIdx.x; i < P / 2; i += THREADS) {
                    int lo, hi;
                    if (st == s >> 1) {  // flip
                        const int pos = i & (st - 1);
                        lo = (i - pos) * 2 + pos;
                        hi = lo + s - 1 - 2 * pos;
                    } else {
                        lo = ((i & ~(st - 1)) << 1) | (i & (st - 1));
                        hi = lo + st;
                    }
                    if (hi < L) {
                        const uint64_t a = k[lo], c = k[hi];
                        if (a > c) {
                            k[lo] = c;
                            k[hi] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        auto at = [&](int i) -> uint64_t& { return k[i]; };
        for (int i = threadIdx.x; i < L; i += THREADS) sort_fixup(at, i, L, depth_key);
        __syncthreads();
        for (int i = threadIdx.x; i < L; i += THREADS) out[rg.x + i] = uint32_t(k[i]);
        __syncthreads();
    }
}

int bits_for(int64_t v) {
    int b = 1;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

}  // namespace

size_t binning_scratch_elems(int64_t n_cap, int64_t inst_cap) {
    const size_t h1 = size_t(1 << kDepthBits) * sort_tiles_for(n_cap);
    const size_t h2 = size_t(1 << kTileBits) * sort_tiles_for(inst_cap);
    return h1 > h2 ? h1 : h2;
}

bool radix_binning() {
    static const bool on = [] {
        const char* e = std::getenv("MSPLAT_RADIX_BINNING");
        return e && e[0] == '1';
    }();
    return on;
}

void run_binning_radix(BinningBuffers& b, cudaStream_t s);

void run_binning(BinningBuffers& b, cudaStream_t s) {
    if (radix_binning()) return run_binning_radix(b, s);
    const int64_t n = b.n;
    const int64_t tiles = int64_t(b.tiles_x) * b.tiles_y;
    cudaMemsetAsync(b.tile_cnt, 0, sizeof(uint32_t) * size_t(tiles), s);
    cudaMemsetAsync(b.key_range, 0, 2 * sizeof(unsigned long long), s);
    const bool priv = tiles <= kPrivMaxTiles;
    const int64_t ctas_max = int64_t(kBinCtas) * device_sm_count();
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(ctas_max, (n + kBinThreads - 1) / kBinThreads));
    const int64_t chunk = (n + ctas - 1) / ctas;
    if (n > 0) {
        if (priv) {
            static std::atomic<unsigned long long> attr{0};
            opt_in_smem(reinterpret_cast<const void*>(tile_hist_kernel<true>), attr, 100 * 1024);
            tile_hist_kernel<true><<<unsigned(ctas), kBinThreads, size_t(tiles) * 4, s>>>(
                n, chunk, b.tile_count, b.tile_rect, b.tiles_x, tiles, b.depth_key, b.tile_cnt, b.key_range);
        } else {
            tile_hist_kernel<false><<<unsigned(ctas), kBinThreads, 0, s>>>(
                n, chunk, b.tile_count, b.tile_rect, b.tiles_x, tiles, b.depth_key, b.tile_cnt, b.key_range);
        }
        count_launches(1);
    }
    tile_scan_kernel<<<1, kTileScanThreads, 0, s>>>(tiles, b.tile_cnt, b.inst_cap, b.tile_range, b.tile_cur,
                                                    b.d_inst_count, b.d_inst_total32, b.big_tiles, b.err);
    count_launches(1);
    if (n > 0) {
        if (priv) {
            static std::atomic<unsigned long long> attr{0};
            opt_in_smem(reinterpret_cast<const void*>(tile_scatter_kernel<true>), attr, 200 * 1024);
            tile_scatter_kernel<true><<<unsigned(ctas), kBinThreads, size_t(tiles) * 8, s>>>(
                n, chunk, b.tile_count, b.tile_rect, b.tiles_x, tiles, b.depth_key, b.d_inst_count, b.key_range,
                b.tile_cur, b.inst_key);
        } else {
            tile_scatter_kernel<false><<<unsigned(ctas), kBinThreads, 0, s>>>(
                n, chunk, b.tile_count, b.tile_rect, b.tiles_x, tiles, b.depth_key, b.d_inst_count, b.key_range,
                b.tile_cur, b.inst_key);
        }
        count_launches(1);
    }
    if (tiles > 0) {
        tile_sort_small_kernel<<<unsigned(tiles), kSortSmallThreads, 0, s>>>(b.tile_range, b.inst_key, b.depth_key,
                                                                            b.inst_gauss);
        constexpr int kMed = kSortMediumThreads * kSortE, kLarge = kSortLargeThreads * kSortE;
        static std::atomic<unsigned long long> attr_m{0}, attr_l{0};
        const size_t smem_m = size_t(kMed + kMed / 8) * 8 * 2, smem_l = size_t(kLarge + kLarge / 8) * 8 * 2;
        auto* km = tile_sort_big_kernel<kSortMediumThreads, kSortSmall, false>;
        auto* kl = tile_sort_big_kernel<kSortLargeThreads, kMed, true>;
        opt_in_smem(reinterpret_cast<const void*>(km), attr_m, int(smem_m));
        opt_in_smem(reinterpret_cast<const void*>(kl), attr_l, int(smem_l));
        km<<<unsigned(2 * device_sm_count()), kSortMediumThreads, smem_m, s>>>(b.tile_range, b.big_tiles, b.inst_key,
                                                                            b.depth_key, b.inst_gauss);
        kl<<<unsigned(device_sm_count()), kSortLargeThreads, smem_l, s>>>(b.tile_range, b.big_tiles, b.inst_key,
                                                                         b.depth_key, b.inst_gauss);
        count_launches(3);
    }
    b.sorted_gauss = b.inst_gauss;
}

void run_binning_radix(BinningBuffers& b, cudaStream_t s) {
    const int64_t n = b.n;
    const int64_t tiles = int64_t(b.tiles_x) * b.tiles_y;
    SortScratch sc{b.hist, b.hist_scanned, b.scan_tiles};

    // K2: depth sort (values = Gaussian ids, initially 0..n-1 from K1).
    const bool depth_in_b = radix_sort_pairs<uint64_t, kDepthBits>(
        b.depth_key, b.order, b.depth_key_alt, b.order_alt, nullptr, n, b.depth_key_bits,
        sc, s);
    const uint32_t* order_sorted = depth_in_b ? b.order_alt : b.order;

    // K3: counts in depth order -> exclusive scan -> instance emission.
    if (n > 0) {
        gather_counts_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(n, order_sorted, b.tile_count,
                                                                       b.count_sorted);
        count_launches(1);
        device_exclusive_scan<uint32_t>(b.count_sorted, b.offset_sorted, nullptr, n, b.scan_tiles,
                                        b.d_inst_total32, s);
    } else {
        cudaMemsetAsync(b.d_inst_total32, 0, sizeof(uint32_t), s);
    }
    finalize_count_kernel<<<1, 1, 0, s>>>(b.d_inst_total32, b.inst_cap, b.d_inst_count, b.err);
    count_launches(1);
    if (n > 0)
        emit_instances_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(
            n, order_sorted, b.tile_rect, b.count_sorted, b.offset_sorted, b.tiles_x,
            b.d_inst_count, b.inst_tile, b.inst_gauss);
        count_launches(1);

    // K4: stable sort of the instances by tile id.
    const bool tile_in_b = radix_sort_pairs<uint32_t, kTileBits>(
        b.inst_tile, b.inst_gauss, b.inst_tile_alt, b.inst_gauss_alt, b.d_inst_count, b.inst_cap,
        bits_for(tiles), sc, s);
    const uint32_t* tile_sorted = tile_in_b ? b.inst_tile_alt : b.inst_tile;
    b.sorted_gauss = tile_in_b ? b.inst_gauss_alt : b.inst_gauss;

    // K5: per-tile ranges.
    cudaMemsetAsync(b.tile_range, 0, sizeof(uint2) * tiles, s);
    if (b.inst_cap > 0)
        tile_ranges_kernel<<<unsigned((b.inst_cap + 255) / 256), 256, 0, s>>>(b.d_inst_count,
                                                                              tile_sorted, b.tile_range);
        count_launches(1);
}

}  // namespace msplat_cuda
