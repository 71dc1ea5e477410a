// Device-wide exclusive scan and stable LSD radix sort, hand-written for the
// binning stage (K2 depth sort, K4 tile sort).  Element counts may live in
// device memory so the whole render can be enqueued (and graph-captured)
// without a host round trip; grids are sized by a host-side capacity.
//
// Radix pass = 3 launches:
//   upsweep   : per-tile digit histogram, warp-aggregated with __match_any_sync
//   rowscan   : per digit, exclusive scan along the tiles (one warp per digit)
//               and the digit total
//   downsweep : digit bases (block scan of the RADIX totals, redundantly per
//               CTA), stable rank (per-warp match_any multisplit, warps in
//               order) and scatter to base[digit] + row prefix[digit][tile] +
//               warp prefix + lane rank.
// Stability: items are processed in global index order (tile-major, then
// warp-major, then item-row, then lane), which is what makes the composition
// of passes an exact (key, original index) order -- the tie-break the
// reference's std::sort comparator uses (rasterizer.cpp:25-28).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace msplat_cuda {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef K_SORT_ITEMS
#define K_SORT_ITEMS 8  // 2048 keys per CTA: 490 CTAs for 1M keys (binning 0.357 ms vs 0.369 at 4096)
#endif
constexpr int kSortItems = K_SORT_ITEMS;
constexpr int kSortTileItems = kSortThreads * kSortItems;

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;  // 1024 elements per CTA: >= 1 CTA per SM for the histogram scans

// --------------------------------------------------------------- block scan
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) >= o) v += n;
    }
    return v;
}

// Exclusive scan of one value per thread across the CTA; returns the CTA total.
template <typename T, int THREADS>
__device__ __forceinline__ T block_exclusive_scan(T v, T& total) {
    __shared__ T warp_sums[THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T s = lane < THREADS / 32 ? warp_sums[lane] : T(0);
        s = warp_inclusive_scan(s);
        if (lane < THREADS / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const T base = warp > 0 ? warp_sums[warp - 1] : T(0);
    total = warp_sums[THREADS / 32 - 1];
    __syncthreads();
    return base + inc - v;
}

// ------------------------------------------------------- device-wide scan
// Pass 1: per-CTA sums of kScanTile elements.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const T* __restrict__ in,
                                                                  const int64_t* __restrict__ d_n,
                                                                  int64_t n_host,
                                                                  T* __restrict__ tile_sums) {
    const int64_t n = d_n ? *d_n : n_host;
    const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    T total;
    block_exclusive_scan<T, kScanThreads>(s, total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Pass 2: single CTA scans the tile sums in place (exclusive); writes the grand
// total to *d_total when given.
template <typename T>
__global__ void __launch_bounds__(1024) scan_tiles_kernel(T* __restrict__ tile_sums, int ntiles,
                                                         T* __restrict__ d_total) {
    T carry = 0;
    for (int start = 0; start < ntiles; start += 1024) {
        const int i = start + threadIdx.x;
        const T v = i < ntiles ? tile_sums[i] : T(0);
        T total;
        const T ex = block_exclusive_scan<T, 1024>(v, total);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

// Pass 3: per-CTA exclusive scan plus the tile offset.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const T* __restrict__ in,
                                                                 const int64_t* __restrict__ d_n,
                                                                 int64_t n_host,
                                                                 const T* __restrict__ tile_offsets,
                                                                 T* __restrict__ out) {
    const int64_t n = d_n ? *d_n : n_host;
    const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    T v[kScanItems];
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : T(0);
        s += v[i];
    }
    T total;
    T run = block_exclusive_scan<T, kScanThreads>(s, total) + tile_offsets[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

// ---------------------------------------------------------------- radix sort
template <typename Key, int BITS>
__device__ __forceinline__ uint32_t digit_of(Key k, int shift) {
    return uint32_t(k >> shift) & ((1u << BITS) - 1u);
}

// Global item index of (tile, warp, row, lane): warp-striped inside a warp.
__device__ __forceinline__ int64_t sort_item_index(int64_t tile, int warp, int row, int lane) {
    return tile * kSortTileItems + int64_t(warp) * 32 * kSortItems + row * 32 + lane;
}

template <typename Key, int BITS>
__global__ void __launch_bounds__(kSortThreads) radix_upsweep_kernel(
    const Key* __restrict__ keys, const int64_t* __restrict__ d_n, int64_t n_host, int shift,
    uint32_t* __restrict__ hist, int ntiles) {
    constexpr int RADIX = 1 << BITS;
    __shared__ uint32_t h[RADIX];
    for (int d = threadIdx.x; d < RADIX; d += kSortThreads) h[d] = 0;
    __syncthreads();
    const int64_t n = d_n ? *d_n : n_host;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t dig[kSortItems];  // all loads in flight before the first match
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int64_t i = sort_item_index(blockIdx.x, warp, r, lane);
        dig[r] = i < n ? digit_of<Key, BITS>(keys[i], shift) : 0xffffffffu;
    }
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint32_t d = dig[r];
        const bool ok = d != 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        if (ok && lane == leader) atomicAdd(&h[d], __popc(peers));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += kSortThreads) hist[int64_t(d) * ntiles + blockIdx.x] = h[d];
}

// Per digit (one warp each): exclusive scan of hist[d][0 .. ntiles) into
// out[d][.] and the row total into totals[d].  A lane scans a contiguous
// chunk of the row (loads in flight together), then the warp scans the chunk sums.
template <int RADIX>
__global__ void __launch_bounds__(256) radix_rowscan_kernel(const uint32_t* __restrict__ hist, int ntiles,
                                                           uint32_t* __restrict__ out, uint32_t* __restrict__ totals) {
    const int d = int((blockIdx.x * 256u + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (d >= RADIX) return;
    const uint32_t* __restrict__ row = hist + int64_t(d) * ntiles;
    uint32_t* __restrict__ orow = out + int64_t(d) * ntiles;
    const int per = (ntiles + 31) >> 5, t0 = lane * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
    uint32_t s = 0;
#pragma unroll 8
    for (int t = t0; t < t1; ++t) s += row[t];
    const uint32_t inc = warp_inclusive_scan(s);
    uint32_t run = inc - s;
#pragma unroll 8
    for (int t = t0; t < t1; ++t) {
        const uint32_t v = row[t];
        orow[t] = run;
        run += v;
    }
    if (lane == 31) totals[d] = inc;
}

template <typename Key, int BITS>
__global__ void __launch_bounds__(kSortThreads) radix_downsweep_kernel(
    const Key* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, Key* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const int64_t* __restrict__ d_n, int64_t n_host, int shift,
    const uint32_t* __restrict__ offsets /* row-scanned [RADIX][ntiles] */, const uint32_t* __restrict__ totals,
    int ntiles) {
    constexpr int RADIX = 1 << BITS;
    static_assert(RADIX % kSortThreads == 0, "digits per thread");
    constexpr int PER = RADIX / kSortThreads;
    __shared__ uint32_t wh[kSortWarps][RADIX];
    __shared__ uint32_t base[RADIX];
    {  // digit bases: exclusive scan of the totals (thread t owns digits [t PER, t PER + PER))
        uint32_t tv[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            tv[j] = totals[threadIdx.x * PER + j];
            sum += tv[j];
        }
        uint32_t all;
        uint32_t ex = block_exclusive_scan<uint32_t, kSortThreads>(sum, all);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int d = threadIdx.x * PER + j;
            base[d] = ex + offsets[int64_t(d) * ntiles + blockIdx.x];
            ex += tv[j];
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) wh[w][d] = 0;
        }
    }
    __syncthreads();
    const int64_t n = d_n ? *d_n : n_host;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    Key k[kSortItems];
    uint32_t v[kSortItems];
    uint32_t rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int64_t i = sort_item_index(blockIdx.x, warp, r, lane);
        if (i < n) {
            k[r] = keys_in[i];
            v[r] = vals_in[i];
        } else {
            k[r] = Key(0);
            v[r] = 0;
        }
    }
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int64_t i = sort_item_index(blockIdx.x, warp, r, lane);
        const bool ok = i < n;
        const uint32_t d = ok ? digit_of<Key, BITS>(k[r], shift) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t before = 0;
        if (ok && lane == leader) {
            before = wh[warp][d];
            wh[warp][d] = before + __popc(peers);
        }
        before = __shfl_sync(0xffffffffu, before, leader);
        rank[r] = before + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
    // Exclusive prefix over warps per digit (warp order == global order).
    for (int d = threadIdx.x; d < RADIX; d += kSortThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t t = wh[w][d];
            wh[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int64_t i = sort_item_index(blockIdx.x, warp, r, lane);
        if (i < n) {
            const uint32_t d = digit_of<Key, BITS>(k[r], shift);
            const uint32_t dst = base[d] + wh[warp][d] + rank[r];
            keys_out[dst] = k[r];
            vals_out[dst] = v[r];
        }
    }
}

// Host-side driver.  Scratch requirements (elements): hist RADIX * tiles(cap)
// uint32, hist_scanned RADIX * tiles(cap) + RADIX uint32 (row prefixes, then
// the digit totals).
struct SortScratch {
    uint32_t* hist = nullptr;
    uint32_t* hist_scanned = nullptr;
    uint32_t* scan_tiles = nullptr;
};

inline int sort_tiles_for(int64_t cap) { return int((cap + kSortTileItems - 1) / kSortTileItems); }

template <typename T>
inline void device_exclusive_scan(const T* in, T* out, const int64_t* d_n, int64_t n_cap,
                                  T* tile_sums, T* d_total, cudaStream_t s) {
    const int ntiles = int((n_cap + kScanTile - 1) / kScanTile);
    if (ntiles == 0) return;
    scan_reduce_kernel<T><<<ntiles, kScanThreads, 0, s>>>(in, d_n, n_cap, tile_sums);
    count_launches(1);
    scan_tiles_kernel<T><<<1, 1024, 0, s>>>(tile_sums, ntiles, d_total);
    count_launches(1);
    scan_apply_kernel<T><<<ntiles, kScanThreads, 0, s>>>(in, d_n, n_cap, tile_sums, out);
    count_launches(1);
}

// Sorts (keys, vals) by bits [0, total_bits) of the key.  Ping-pongs between
// the *_a and *_b buffers; returns true when the result ends in the b buffers.
template <typename Key, int BITS>
inline bool radix_sort_pairs(Key* keys_a, uint32_t* vals_a, Key* keys_b, uint32_t* vals_b,
                             const int64_t* d_n, int64_t n_cap, int total_bits,
                             const SortScratch& sc, cudaStream_t s) {
    constexpr int RADIX = 1 << BITS;
    const int ntiles = sort_tiles_for(n_cap);
    bool in_b = false;
    if (ntiles == 0) return false;
    for (int shift = 0; shift < total_bits; shift += BITS) {
        const Key* kin = in_b ? keys_b : keys_a;
        const uint32_t* vin = in_b ? vals_b : vals_a;
        Key* kout = in_b ? keys_a : keys_b;
        uint32_t* vout = in_b ? vals_a : vals_b;
        radix_upsweep_kernel<Key, BITS><<<ntiles, kSortThreads, 0, s>>>(kin, d_n, n_cap, shift,
                                                                       sc.hist, ntiles);
        count_launches(1);
        uint32_t* const totals = sc.hist_scanned + int64_t(RADIX) * ntiles;
        radix_rowscan_kernel<RADIX><<<(RADIX * 32 + 255) / 256, 256, 0, s>>>(sc.hist, ntiles, sc.hist_scanned, totals);
        radix_downsweep_kernel<Key, BITS><<<ntiles, kSortThreads, 0, s>>>(
            kin, vin, kout, vout, d_n, n_cap, shift, sc.hist_scanned, totals, ntiles);
        count_launches(2);
        in_b = !in_b;
    }
    return in_b;
}

}  // namespace msplat_cuda
