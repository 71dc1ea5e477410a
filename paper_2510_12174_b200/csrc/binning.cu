// K2-K5: binning.  Replaces bin_and_sort (core/src/rasterizer.cpp:14-45).
//
// The reference sorts visible splats by (sort_depth, index) with std::sort and
// pushes each one into every tile of its rect, so each tile list ascends by
// (depth, index).  Here:
//   K2  stable LSD radix sort of the 64-bit IEEE pattern of the FP64 depth
//       (positive doubles order like their bits; values start as the index, so
//       ties keep index order) -- 7 passes of 9 bits cover bits 0..62;
//   K3  exclusive scan of the per-Gaussian tile counts in depth order, then
//       emission of (tile id, Gaussian id) instances in that order;
//   K4  stable radix sort of the instances by tile id alone: within a tile the
//       emission (= depth, index) order survives, which is the reference list;
//   K5  per-tile [start, end) ranges from the tile-id boundaries.
// All counts stay on the device, so the sequence needs no host round trip.
#include "common.cuh"
#include "kernels.h"
#include "radix_sort.cuh"

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

void run_binning(BinningBuffers& b, cudaStream_t s) {
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
