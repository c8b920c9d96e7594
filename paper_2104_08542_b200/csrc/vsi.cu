// Virtual Sparse Id on the device, bit-exact with virtual_sparse_id
// (core/src/vsi.cpp:23-54): global_ids in FIRST-APPEARANCE order and every
// position remapped to its index in that list.
//
// A sort-unique would give sorted order, so the kernels use the
// min-position formulation instead (SURVEY §7 hard part (i)):
//   1. first[f] = min position of f    (direct-mapped table over the
//      vocabulary in HBM; read-before-atomicMin skips the contended atomics)
//   2. flag[i]  = (first[f_i] == i)    (i is a first appearance; evaluated inside
//   3. rank     = exclusive scan(flag)  the CUB scan; U = rank[n-1] + flag[n-1])
//   4. global_ids[rank[i]] = f_i for flagged i;  vid[i] = rank[first[f_i]]
//   5. first[global_ids[k]] = unseen   (reset only the touched entries)
// The direct-mapped table (4 B per vocabulary id: 135 MB at 33.8M ids) is the
// HBM-rich choice: no probing, no tombstones, one sector per access.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "ops.h"

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
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = __ldg(ids + i);
  if (__ldcg(first + f) > static_cast<uint32_t>(i)) atomicMin(first + f, static_cast<uint32_t>(i));
}

__global__ void vsi_emit_kernel(const uint32_t* __restrict__ ids, int64_t n,
                                const uint32_t* __restrict__ first,
                                const uint32_t* __restrict__ rank, uint32_t* __restrict__ gids,
                                uint32_t* __restrict__ vids, int32_t* __restrict__ unique) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = ids[i];
  const uint32_t r = rank[i];
  const uint32_t fi = __ldg(first + f);
  const uint32_t flag = fi == static_cast<uint32_t>(i) ? 1u : 0u;
  if (flag) gids[r] = f;
  vids[i] = __ldg(rank + fi);
  if (i == n - 1) *unique = static_cast<int32_t>(r + flag);
}

__global__ void vsi_reset_kernel(const uint32_t* __restrict__ gids,
                                 const int32_t* __restrict__ unique, uint32_t* __restrict__ first) {
  const int32_t u = *unique;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < u;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    first[gids[k]] = kUnseen;
}

__global__ void ids_to_u32_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                  int64_t n, uint64_t limit, int32_t* bad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t v = in[i];
  if (v >= limit) {
    *bad = 1;
    out[i] = 0;
  } else {
    out[i] = static_cast<uint32_t>(v);
  }
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                  int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// flag[i] = (first[ids[i]] == i), evaluated inside the scan (no flag array / kernel)
struct FirstFlag {
  const uint32_t* ids;
  const uint32_t* first;
  __device__ uint32_t operator()(int i) const {
    return __ldg(first + __ldg(ids + i)) == static_cast<uint32_t>(i) ? 1u : 0u;
  }
};
using FlagIt = thrust::transform_iterator<FirstFlag, thrust::counting_iterator<int>>;

size_t flag_scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  FlagIt it(thrust::counting_iterator<int>(0), FirstFlag{nullptr, nullptr});
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, static_cast<uint32_t*>(nullptr),
                                           static_cast<int>(n)));
  return bytes;
}

}  // namespace

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr), static_cast<int>(n)));
  return bytes;
}

void exclusive_scan_u32(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out,
                        int64_t n, cudaStream_t s) {
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, static_cast<int>(n), s));
  g_launches += 2;  // init + decoupled look-back scan
}

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

void VsiScratch::init(uint64_t ks, int64_t c) {
  release();
  key_space = ks;
  cap = c > 0 ? c : 1;
  CUDA_CHECK(cudaMalloc(&d_first, sizeof(uint32_t) * key_space));
  CUDA_CHECK(cudaMalloc(&d_flag, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&d_rank, sizeof(uint32_t) * cap));
  cub_bytes = std::max(scan_temp_bytes(cap), flag_scan_temp_bytes(cap));
  CUDA_CHECK(cudaMalloc(&d_cub, cub_bytes));
  fill_u32_kernel<<<1184, 256>>>(d_first, static_cast<int64_t>(key_space), kUnseen);
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cudaDeviceSynchronize());
}

void VsiScratch::release() {
  cudaFree(d_first);
  cudaFree(d_flag);
  cudaFree(d_rank);
  cudaFree(d_cub);
  d_first = d_flag = d_rank = nullptr;
  d_cub = nullptr;
}

void vsi_device(VsiScratch& v, const uint32_t* d_ids, int64_t n, uint32_t* d_gids,
                uint32_t* d_vids, int32_t* d_unique, cudaStream_t s, bool reset) {
  SFB_CHECK(n > 0 && n <= v.cap, "vsi batch exceeds scratch capacity");
  const int grid = ceil_div(n, 256);
  vsi_first_kernel<<<grid, 256, 0, s>>>(d_ids, n, v.d_first);
  CUDA_LAUNCH_CHECK();
  {
    FlagIt it(thrust::counting_iterator<int>(0), FirstFlag{d_ids, v.d_first});
    size_t bytes = v.cub_bytes;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(v.d_cub, bytes, it, v.d_rank, static_cast<int>(n), s));
    g_launches += 2;  // init + decoupled look-back scan
  }
  vsi_emit_kernel<<<grid, 256, 0, s>>>(d_ids, n, v.d_first, v.d_rank, d_gids, d_vids, d_unique);
  CUDA_LAUNCH_CHECK();
  if (reset) {
    vsi_reset_kernel<<<std::min(grid, num_sms() * 8), 256, 0, s>>>(d_gids, d_unique, v.d_first);
    CUDA_LAUNCH_CHECK();
  }
}

void ids_to_u32(const uint64_t* d_in, uint32_t* d_out, int64_t n, uint64_t limit, int32_t* d_bad,
                cudaStream_t s) {
  if (n <= 0) return;
  ids_to_u32_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_in, d_out, n, limit, d_bad);
  CUDA_LAUNCH_CHECK();
}

void u32_to_u64(const uint32_t* d_in, uint64_t* d_out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  u32_to_u64_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_in, d_out, n);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
