// Single-pass exclusive scan with decoupled look-back, fused with the producer of the
// scanned values and the consumer of the prefixes (one launch instead of a flag kernel,
// a library scan (init + scan kernels) and a compaction kernel).
//
//   value(i) -> uint32_t           computed once per item (may have side effects)
//   emit(i, value, prefix)         called once per item with its exclusive prefix
//   *total = sum of all values     written by the last tile
//
// Tiles of 256 threads x kItems items (strided, so loads coalesce; one item per thread for
// values behind dependent random loads, so more tiles hide the latency); a tile publishes its
// aggregate, then warp 0 walks back over the predecessors' states 32 at a time until it
// meets an inclusive prefix (the CUB/Merrill-Garland scheme). Tile states carry the
// launch's epoch, so nothing has to be reset between launches.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace sfb {

struct ScanTiles {
  uint64_t* state = nullptr;  // [max_tiles]: epoch << 34 | status << 32 | value
  int64_t max_tiles = 0;
  uint32_t epoch = 0;
  void init(int64_t max_items);
  void release();
};

constexpr int kScanThreads = 256;
constexpr int kScanItemsMax = 8;  // items per thread: 8 for streaming values, fewer for
                                  // latency-bound ones (dependent random loads per item)

#ifdef __CUDACC__
namespace scan_detail {
constexpr uint64_t kAgg = 1, kPre = 2;
__device__ __forceinline__ void publish(uint64_t* p, uint32_t epoch, uint64_t status, uint32_t v) {
  const uint64_t w = (static_cast<uint64_t>(epoch) << 34) | (status << 32) | v;
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ uint64_t peek(const uint64_t* p) {
  uint64_t w;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
}  // namespace scan_detail

template <int kScanItems, typename ValueFn, typename EmitFn>
__global__ void __launch_bounds__(kScanThreads) lookback_scan_kernel(int64_t n, ValueFn value,
                                                                     EmitFn emit,
                                                                     uint64_t* __restrict__ state,
                                                                     uint32_t epoch,
                                                                     int32_t* __restrict__ total,
                                                                     const int32_t* __restrict__ live) {
  __shared__ uint32_t warp_sum[kScanThreads / 32];
  __shared__ uint32_t tile_prefix;
  pdl_wait();  // launched with launch_pdl: the producer of the scanned values must be done
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int64_t kScanTile = kScanThreads * kScanItems;
  // live (device count, nullable): items [live, n) are empty; tiles past the last live one
  // exit at once (no successor reads their state) and the last live tile writes the total
  if (live) n = min(n, static_cast<int64_t>(max(0, *live)));
  const int64_t ntiles = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
  const int64_t last_tile = ntiles - 1;
  // persistent: CTA b scans tiles b, b + G, b + 2G, ... in order (G = gridDim.x, capped by
  // mgr_grid); a tile's look-back only waits on lower tiles, which their CTAs reach first
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kScanTile;
    uint32_t v[kScanItems], ex[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + tid;
      v[k] = i < n ? value(i) : 0u;
    }
    uint32_t run = 0;  // tile-local running total (uniform)
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      uint32_t x = v[k];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
      }
      if (lane == 31) warp_sum[wid] = x;
      __syncthreads();
      uint32_t before = 0, all = 0;
#pragma unroll
      for (int w = 0; w < kScanThreads / 32; ++w) {
        const uint32_t s = warp_sum[w];
        before += w < wid ? s : 0u;
        all += s;
      }
      ex[k] = run + before + x - v[k];
      run += all;
      __syncthreads();
    }
    using namespace scan_detail;
    if (tile == 0) {
      if (tid == 0) {
        publish(state, epoch, kPre, run);
        tile_prefix = 0;
      }
    } else if (wid == 0) {
      if (lane == 0) publish(state + tile, epoch, kAgg, run);
      uint32_t excl = 0;
      int64_t look = tile - 1;
      for (;;) {
        const int64_t t = look - lane;
        uint64_t w = t >= 0 ? peek(state + t)
                            : ((static_cast<uint64_t>(epoch) << 34) | (kPre << 32));
        uint64_t st = (w >> 34) == epoch ? ((w >> 32) & 3u) : 0u;
        while (__any_sync(0xFFFFFFFFu, st == 0)) {  // a predecessor has not published yet
          if (st == 0) {
            w = peek(state + t);
            st = (w >> 34) == epoch ? ((w >> 32) & 3u) : 0u;
          }
        }
        const unsigned pre = __ballot_sync(0xFFFFFFFFu, st == kPre);
        const int stop = pre ? __ffs(pre) - 1 : 31;  // closest predecessor with a full prefix
        uint32_t val = lane <= stop ? static_cast<uint32_t>(w) : 0u;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, off);
        excl += val;
        if (pre) break;
        look -= 32;
      }
      if (lane == 0) {
        publish(state + tile, epoch, kPre, excl + run);
        tile_prefix = excl;
      }
    }
    __syncthreads();
    const uint32_t pfx = tile_prefix;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + tid;
      if (i < n) emit(i, v[k], pfx + ex[k]);
    }
    if (total && tile == last_tile && tid == 0) *total = static_cast<int32_t>(pfx + run);
    __syncthreads();  // warp_sum / tile_prefix are reused by the next tile
  }
}

// launches the fused scan over n items (n >= 1) on stream s, kItems items per thread;
// live (nullable): a device count <= n of the items that exist (the grid covers n)
template <int kItems = kScanItemsMax, typename ValueFn, typename EmitFn>
void lookback_scan(ScanTiles& st, int64_t n, ValueFn value, EmitFn emit, int32_t* total,
                   cudaStream_t s, const int32_t* live = nullptr) {
  static_assert(kItems >= 1 && kItems <= kScanItemsMax, "items per thread");
  const int64_t tiles = (n + kScanThreads * kItems - 1) / (kScanThreads * kItems);
  SFB_CHECK(tiles <= st.max_tiles, "scan larger than its tile state");
  if (++st.epoch >= (1u << 30)) {  // 30-bit epochs wrap: clear every state (epoch 0 = invalid)
    CUDA_CHECK(cudaMemsetAsync(st.state, 0, sizeof(uint64_t) * st.max_tiles, s));
    st.epoch = 1;
  }
  launch_pdl(lookback_scan_kernel<kItems, ValueFn, EmitFn>, dim3(mgr_grid(tiles)),
             dim3(kScanThreads), 0, s, n, value, emit, st.state, st.epoch, total, live);
  CUDA_LAUNCH_CHECK();
}
#endif

}  // namespace sfb
