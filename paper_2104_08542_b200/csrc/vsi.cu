// Virtual Sparse Id on the device, bit-exact with virtual_sparse_id
// (core/src/vsi.cpp:23-54): global_ids in FIRST-APPEARANCE order and every
// position remapped to its index in that list.
//
// A sort-unique would give sorted order, so the kernels use the
// min-position formulation instead (SURVEY §7 hard part (i)):
//   1. first[f] = min position of f    (direct-mapped table over the
//      vocabulary in HBM; read-before-atomicMin skips the contended atomics)
//   2. one fused decoupled look-back scan (scan.cuh) over flag[i] = (first[f_i] == i):
//      a flagged i writes global_ids[rank] = f_i and re-tags first[f_i] = rank | 2^31
//      (safe: no other position ever equals the first position, so the tag cannot make
//      another flag true, and the first position reads first[f_i] before it tags it);
//      the last tile writes U
//   3. vid[i] = first[f_i] & (2^31 - 1)
//   4. first[global_ids[k]] = unseen   (reset only the touched entries)
// The direct-mapped table (4 B per vocabulary id: 135 MB at 33.8M ids) is the HBM-rich
// choice: no probing, no tombstones, one sector per access.
//
// Arbitrary u64 ids (the reference accepts any FeatureId, vsi.cpp:41-46): the same three
// passes over an open-addressing hash table (keys u64, linear probing) instead of the
// direct-mapped one. A warp first merges equal ids with __match_any_sync so only the
// lowest lane of each group (its smallest position) inserts; every position keeps its
// table slot, so the scan and the remap read the slot directly.
#include <cub/device/device_radix_sort.cuh>

#include "ops.h"
#include "scan.cuh"

namespace sfb {

namespace {

constexpr uint32_t kUnseen = 0xFFFFFFFFu;

__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

// first[f] = min position of f. Consecutive positions of a warp are consecutive fields of
// one row (disjoint vocabulary shards), so a warp rarely holds one id twice and a
// __match_any_sync pre-dedup costs more than it saves; instead the word is read first and
// the atomic skipped when an earlier position is already recorded (first[] only decreases),
// which removes the contended atomics on hot ids.
__global__ void vsi_first_kernel(const uint32_t* __restrict__ ids, int64_t n,
                                 uint32_t* __restrict__ first) {
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t f = __ldg(ids + i);
    if (__ldcg(first + f) > static_cast<uint32_t>(i))
      atomicMin(first + f, static_cast<uint32_t>(i));
  }
}

constexpr uint32_t kTag = 0x80000000u;

struct VsiFlag {  // first appearance?
  const uint32_t* ids;
  const uint32_t* first;
  __device__ uint32_t operator()(int64_t i) const {
    return __ldcg(first + __ldg(ids + i)) == static_cast<uint32_t>(i) ? 1u : 0u;
  }
};
struct VsiEmit {
  const uint32_t* ids;
  uint32_t* first;
  uint32_t* gids;
  __device__ void operator()(int64_t i, uint32_t flag, uint32_t rank) const {
    if (!flag) return;
    const uint32_t f = __ldg(ids + i);
    gids[rank] = f;
    first[f] = rank | kTag;
  }
};

__global__ void vsi_vid_kernel(const uint32_t* __restrict__ ids, int64_t n,
                               const uint32_t* __restrict__ first, uint32_t* __restrict__ vids) {
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    vids[i] = __ldcg(first + __ldg(ids + i)) & ~kTag;
}

// ---- hashed path (arbitrary u64 ids, or u32 ids with an L2-resident table) ----
// KeyT = unsigned long long (any FeatureId) or uint32_t (device ids below the vocabulary: a
// table of 2 x cap slots fits in L2, where the direct-mapped table over the vocabulary does
// not, so its random accesses are L2 hits instead of DRAM sectors)
template <typename KeyT>
__device__ __forceinline__ KeyT hash_empty() {
  return static_cast<KeyT>(~0ull);
}
__device__ __forceinline__ uint64_t hmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}
// keys[mask + 1] is the dedicated slot of the id equal to the empty marker
template <typename KeyT, typename IdT>
__global__ void vsi_hash_insert_kernel(const IdT* __restrict__ ids, int64_t n,
                                       KeyT* __restrict__ keys, uint32_t* __restrict__ pos,
                                       uint64_t mask, uint32_t* __restrict__ hslot) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  // grid-stride in warp-aligned steps (the ballot / match below need whole warps)
  for (int64_t i0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) & ~31ll;
       i0 < n; i0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
  const int64_t i = i0 + lane;
  const bool live = i < n;
  const KeyT f = live ? static_cast<KeyT>(ids[i]) : hash_empty<KeyT>();
  const unsigned act = __ballot_sync(0xFFFFFFFFu, live);
  if (!live) continue;
  const unsigned peers = __match_any_sync(act, f);
  const int leader = __ffs(peers) - 1;  // the group's smallest position
  uint32_t slot = 0;
  if (lane == leader) {
    if (f == hash_empty<KeyT>()) {
      slot = static_cast<uint32_t>(mask + 1);
    } else {
      uint64_t h = hmix64(static_cast<uint64_t>(f)) & mask;
      for (;;) {
        const KeyT cur = __ldcg(keys + h);  // read first: repeated ids skip the CAS
        if (cur == f) break;
        if (cur == hash_empty<KeyT>()) {
          const KeyT prev = atomicCAS(keys + h, hash_empty<KeyT>(), f);
          if (prev == hash_empty<KeyT>() || prev == f) break;
        }
        h = (h + 1) & mask;
      }
      slot = static_cast<uint32_t>(h);
    }
    if (__ldcg(pos + slot) > static_cast<uint32_t>(i)) atomicMin(pos + slot, static_cast<uint32_t>(i));
  }
  slot = __shfl_sync(act, slot, leader);
  hslot[i] = slot;
  }
}
struct VsiHashFlag {
  const uint32_t* hslot;
  const uint32_t* pos;
  __device__ uint32_t operator()(int64_t i) const {
    return __ldcg(pos + __ldg(hslot + i)) == static_cast<uint32_t>(i) ? 1u : 0u;
  }
};
template <typename IdT>
struct VsiHashEmit {
  const IdT* ids;
  const uint32_t* hslot;
  uint32_t* pos;
  IdT* gids;
  uint32_t* uslot;
  __device__ void operator()(int64_t i, uint32_t flag, uint32_t rank) const {
    if (!flag) return;
    const uint32_t sl = __ldg(hslot + i);
    gids[rank] = ids[i];
    uslot[rank] = sl;
    pos[sl] = rank | kTag;
  }
};
__global__ void vsi_hash_vid_kernel(const uint32_t* __restrict__ hslot, int64_t n,
                                    const uint32_t* __restrict__ pos, uint32_t* __restrict__ vids) {
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    vids[i] = __ldcg(pos + __ldg(hslot + i)) & ~kTag;
}
template <typename KeyT>
__global__ void vsi_hash_reset_kernel(const uint32_t* __restrict__ uslot,
                                      const int32_t* __restrict__ unique, KeyT* __restrict__ keys,
                                      uint32_t* __restrict__ pos) {
  pdl_wait();
  const int32_t u = *unique;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < u;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t sl = uslot[k];
    keys[sl] = hash_empty<KeyT>();
    pos[sl] = kUnseen;
  }
}

__global__ void vsi_reset_kernel(const uint32_t* __restrict__ gids,
                                 const int32_t* __restrict__ unique, uint32_t* __restrict__ first) {
  pdl_wait();
  const int32_t u = *unique;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < u;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    first[gids[k]] = kUnseen;
}

__global__ void ids_to_u32_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                  int64_t n, uint64_t limit, int32_t* bad) {
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = in[i];
    if (v >= limit) {
      *bad = 1;
      out[i] = 0;
    } else {
      out[i] = static_cast<uint32_t>(v);
    }
  }
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                  int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace

size_t sort_pairs_temp_bytes(int64_t n) {
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint64_t*>(nullptr),
                                             static_cast<uint64_t*>(nullptr),
                                             static_cast<const uint32_t*>(nullptr),
                                             static_cast<uint32_t*>(nullptr), static_cast<int>(n)));
  return bytes;
}

void sort_pairs_u64_u32(void* temp, size_t temp_bytes, const uint64_t* keys_in, uint64_t* keys_out,
                        const uint32_t* vals_in, uint32_t* vals_out, int64_t n, int end_bit,
                        cudaStream_t s) {
  CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out,
                                             static_cast<int>(n), 0, end_bit, s));
  g_launches += 1 + (end_bit + 7) / 8;  // histogram + one onesweep pass per 8 bits
}

void ScanTiles::init(int64_t max_items) {
  release();
  max_tiles = std::max<int64_t>(1, (max_items + kScanThreads - 1) / kScanThreads);
  CUDA_CHECK(cudaMalloc(&state, sizeof(uint64_t) * max_tiles));
  CUDA_CHECK(cudaMemset(state, 0, sizeof(uint64_t) * max_tiles));
  epoch = 0;
}

void ScanTiles::release() {
  if (state) cudaFree(state);
  state = nullptr;
  max_tiles = 0;
}

void VsiScratch::init(uint64_t ks, int64_t c, bool hash32) {
  release();
  key_space = ks;
  cap = c > 0 ? c : 1;
  hashed32 = hash32 && ks > 0;
  tiles.init(cap);
  if (hashed32) {  // u32 keys in a table of at least 2 cap slots (+1 for the empty marker)
    hmask = 1;
    while (hmask + 1 < static_cast<uint64_t>(2 * cap)) hmask = 2 * hmask + 1;
    CUDA_CHECK(cudaMalloc(&d_hkeys32, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMemset(d_hkeys32, 0xFF, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMalloc(&d_first, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMemset(d_first, 0xFF, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMalloc(&d_hslot, sizeof(uint32_t) * cap));
    CUDA_CHECK(cudaMalloc(&d_uslot, sizeof(uint32_t) * cap));
  } else if (key_space) {
    CUDA_CHECK(cudaMalloc(&d_first, sizeof(uint32_t) * key_space));
    fill_u32_kernel<<<1184, 256>>>(d_first, static_cast<int64_t>(key_space), kUnseen);
    CUDA_LAUNCH_CHECK();
  } else {  // hashed: a power-of-two table of at least 2 cap slots (+1 for the empty marker)
    hmask = 1;
    while (hmask + 1 < static_cast<uint64_t>(2 * cap)) hmask = 2 * hmask + 1;
    CUDA_CHECK(cudaMalloc(&d_hkeys, sizeof(unsigned long long) * (hmask + 2)));
    CUDA_CHECK(cudaMemset(d_hkeys, 0xFF, sizeof(unsigned long long) * (hmask + 2)));
    CUDA_CHECK(cudaMalloc(&d_first, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMemset(d_first, 0xFF, sizeof(uint32_t) * (hmask + 2)));
    CUDA_CHECK(cudaMalloc(&d_hslot, sizeof(uint32_t) * cap));
    CUDA_CHECK(cudaMalloc(&d_uslot, sizeof(uint32_t) * cap));
  }
  CUDA_CHECK(cudaDeviceSynchronize());
}

void VsiScratch::release() {
  tiles.release();
  for (void* p : {static_cast<void*>(d_first), static_cast<void*>(d_hkeys),
                  static_cast<void*>(d_hkeys32), static_cast<void*>(d_hslot),
                  static_cast<void*>(d_uslot)})
    if (p) cudaFree(p);
  d_first = d_hslot = d_uslot = d_hkeys32 = nullptr;
  d_hkeys = nullptr;
  hmask = 0;
  hashed32 = false;
}

void vsi_device(VsiScratch& v, const uint32_t* d_ids, int64_t n, uint32_t* d_gids,
                uint32_t* d_vids, int32_t* d_unique, cudaStream_t s, bool reset) {
  SFB_CHECK(n > 0 && n <= v.cap, "vsi batch exceeds scratch capacity");
  SFB_CHECK(v.key_space > 0, "direct-mapped VSI needs a key space");
  const int grid = mgr_grid(ceil_div(n, 256));  // manager stage: capped, grid-stride kernels
  if (v.hashed32) {  // L2-resident hashed table; always reset behind the batch
    launch_pdl(vsi_hash_insert_kernel<uint32_t, uint32_t>, dim3(grid), dim3(256), 0, s, d_ids, n, v.d_hkeys32,
                                                                    v.d_first, v.hmask, v.d_hslot);
    CUDA_LAUNCH_CHECK();
    lookback_scan<2>(v.tiles, n, VsiHashFlag{v.d_hslot, v.d_first},
                     VsiHashEmit<uint32_t>{d_ids, v.d_hslot, v.d_first, d_gids, v.d_uslot},
                     d_unique, s);
    launch_pdl(vsi_hash_vid_kernel, dim3(grid), dim3(256), 0, s, v.d_hslot, n, v.d_first, d_vids);
    CUDA_LAUNCH_CHECK();
    launch_pdl(vsi_hash_reset_kernel<uint32_t>, dim3(std::min(grid, num_sms() * 8)), dim3(256), 0, s, v.d_uslot, d_unique, v.d_hkeys32, v.d_first);
    CUDA_LAUNCH_CHECK();
    return;
  }
  launch_pdl(vsi_first_kernel, dim3(grid), dim3(256), 0, s, d_ids, n, v.d_first);
  CUDA_LAUNCH_CHECK();
  lookback_scan<2>(v.tiles, n, VsiFlag{d_ids, v.d_first}, VsiEmit{d_ids, v.d_first, d_gids},
                   d_unique, s);
  launch_pdl(vsi_vid_kernel, dim3(grid), dim3(256), 0, s, d_ids, n, v.d_first, d_vids);
  CUDA_LAUNCH_CHECK();
  if (reset) {
    launch_pdl(vsi_reset_kernel, dim3(std::min(grid, num_sms() * 8)), dim3(256), 0, s, d_gids, d_unique, v.d_first);
    CUDA_LAUNCH_CHECK();
  }
}

void vsi_device_hashed(VsiScratch& v, const uint64_t* d_ids, int64_t n, uint64_t* d_gids,
                       uint32_t* d_vids, int32_t* d_unique, cudaStream_t s) {
  SFB_CHECK(n > 0 && n <= v.cap, "vsi batch exceeds scratch capacity");
  SFB_CHECK(v.key_space == 0, "hashed VSI needs a context created with key_space 0");
  const int grid = mgr_grid(ceil_div(n, 256));
  launch_pdl(vsi_hash_insert_kernel<unsigned long long, uint64_t>, dim3(grid), dim3(256), 0, s, d_ids, n, v.d_hkeys, v.d_first, v.hmask, v.d_hslot);
  CUDA_LAUNCH_CHECK();
  lookback_scan<2>(v.tiles, n, VsiHashFlag{v.d_hslot, v.d_first},
                   VsiHashEmit<uint64_t>{d_ids, v.d_hslot, v.d_first, d_gids, v.d_uslot},
                   d_unique, s);
  launch_pdl(vsi_hash_vid_kernel, dim3(grid), dim3(256), 0, s, v.d_hslot, n, v.d_first, d_vids);
  CUDA_LAUNCH_CHECK();
  launch_pdl(vsi_hash_reset_kernel<unsigned long long>, dim3(std::min(grid, num_sms() * 8)), dim3(256), 0, s, v.d_uslot, d_unique, v.d_hkeys, v.d_first);
  CUDA_LAUNCH_CHECK();
}

void ids_to_u32(const uint64_t* d_in, uint32_t* d_out, int64_t n, uint64_t limit, int32_t* d_bad,
                cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(ids_to_u32_kernel, dim3(mgr_grid(ceil_div(n, 256))), dim3(256), 0, s, d_in, d_out, n, limit, d_bad);
  CUDA_LAUNCH_CHECK();
}

void u32_to_u64(const uint32_t* d_in, uint64_t* d_out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  u32_to_u64_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_in, d_out, n);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
