// PCIe microbenchmark for the MixCache write-back / fill paths (not shipped; evidence for
// DESIGN.md §9). Rows are [emb | m | v] fp32, 3*d floats, scattered in a large pinned,
// mapped host table; device side is SoA (emb, m, v separate [C x d] arrays) as in cache.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_rows pcie_rows.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

constexpr int D = 80;
constexpr int D4 = D / 4;

// one warp per row, float4 stores (the shipped evict kernel)
__global__ void write_warp(int n, const uint32_t* rows, const uint32_t* slots, const float4* emb,
                           const float4* mom, const float4* vel, float4* host) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const size_t r = rows[w], s = slots[w];
  float4* dst = host + r * 3 * D4;
  for (int c = lane; c < 3 * D4; c += 32) {
    const int which = c / D4, cc = c - which * D4;
    dst[c] = (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc];
  }
}

// flat (row, chunk) items, grid-stride
__global__ void write_flat(int n, const uint32_t* rows, const uint32_t* slots, const float4* emb,
                           const float4* mom, const float4* vel, float4* host) {
  const int64_t items = static_cast<int64_t>(n) * 3 * D4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < items;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / (3 * D4)), c = static_cast<int>(i - k * 3 * D4);
    const int which = c / D4, cc = c - which * D4;
    const size_t r = rows[k], s = slots[k];
    host[r * 3 * D4 + c] = (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc];
  }
}

// gather rows into a contiguous HBM staging buffer (then one copy-engine D2H)
__global__ void gather_stage(int n, const uint32_t* slots, const float4* emb, const float4* mom,
                             const float4* vel, float4* stage) {
  const int64_t items = static_cast<int64_t>(n) * 3 * D4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < items;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / (3 * D4)), c = static_cast<int>(i - k * 3 * D4);
    const int which = c / D4, cc = c - which * D4;
    const size_t s = slots[k];
    stage[i] = (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc];
  }
}

// one warp per row, zero-copy reads (the shipped admit fill)
__global__ void read_warp(int n, const uint32_t* rows, const uint32_t* slots, const float4* host,
                          float4* emb, float4* mom, float4* vel) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const size_t r = rows[w], s = slots[w];
  const float4* src = host + r * 3 * D4;
  for (int c = lane; c < 3 * D4; c += 32) {
    const int which = c / D4, cc = c - which * D4;
    (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc] = src[c];
  }
}

__global__ void read_flat(int n, const uint32_t* rows, const uint32_t* slots, const float4* host,
                          float4* emb, float4* mom, float4* vel) {
  const int64_t items = static_cast<int64_t>(n) * 3 * D4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < items;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / (3 * D4)), c = static_cast<int>(i - k * 3 * D4);
    const int which = c / D4, cc = c - which * D4;
    const size_t r = rows[k], s = slots[k];
    (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc] = host[r * 3 * D4 + c];
  }
}

// fused: warp v writes back victim v and then fills admitted row v into the same slot
__global__ void swap_warp(int n, const uint32_t* wrows, const uint32_t* rrows, const uint32_t* slots,
                          float4* emb, float4* mom, float4* vel, float4* host) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  const size_t s = slots[w];
  float4* dst = host + static_cast<size_t>(wrows[w]) * 3 * D4;
  const float4* src = host + static_cast<size_t>(rrows[w]) * 3 * D4;
  float4 a[2], b[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = lane + 32 * q;
    if (c < 3 * D4) {
      const int which = c / D4, cc = c - which * D4;
      a[q] = (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc];
      b[q] = src[c];
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int c = lane + 32 * q;
    if (c < 3 * D4) {
      const int which = c / D4, cc = c - which * D4;
      dst[c] = a[q];
      (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc] = b[q];
    }
  }
}


// TMA bulk stores: each warp stages a row (SoA -> AoS) in shared memory and lane 0 issues
// one cp.async.bulk shared->global (host) of the whole 960 B row; 4 stages per warp
constexpr int kStages = 4;
__global__ void write_tma(int n, const uint32_t* rows, const uint32_t* slots, const float4* emb,
                          const float4* mom, const float4* vel, float4* host) {
  __shared__ __align__(128) float4 sm[8][kStages][3 * D4];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = gridDim.x * 8;
  int it = 0;
  for (int w = blockIdx.x * 8 + wib; w < n; w += nw, ++it) {
    const int st = it % kStages;
    if (it >= kStages) {  // the bulk store that used this stage must have read smem
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1) : "memory");
      __syncwarp();
    }
    const size_t r = rows[w], s = slots[w];
    for (int c = lane; c < 3 * D4; c += 32) {
      const int which = c / D4, cc = c - which * D4;
      sm[wib][st][c] = (which == 0 ? emb : which == 1 ? mom : vel)[s * D4 + cc];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(&sm[wib][st][0]));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(host + r * 3 * D4),
                   "r"(sa), "n"(3 * D4 * 16)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 94000;
  const size_t host_rows = argc > 2 ? strtoull(argv[2], 0, 10) : 8000000;  // 7.7 GB
  const size_t C = 524288;
  const size_t row_b = 3 * D * 4;
  printf("n=%d rows x %zu B = %.1f MB; host table %.1f GB\n", n, row_b, n * row_b / 1e6,
         host_rows * row_b / 1e9);
  float4* host;
  CK(cudaHostAlloc(&host, host_rows * row_b, cudaHostAllocMapped | cudaHostAllocPortable));
  float4 *emb, *mom, *vel, *stage, *hstage;
  CK(cudaMalloc(&emb, C * D * 4));
  CK(cudaMalloc(&mom, C * D * 4));
  CK(cudaMalloc(&vel, C * D * 4));
  CK(cudaMalloc(&stage, n * row_b));
  CK(cudaHostAlloc(&hstage, n * row_b, 0));
  std::mt19937_64 rng(1);
  std::vector<uint32_t> rows(n), rrows(n), slots(n);
  for (int i = 0; i < n; ++i) {
    rows[i] = rng() % host_rows;
    rrows[i] = rng() % host_rows;
    slots[i] = rng() % C;
  }
  uint32_t *d_rows, *d_rrows, *d_slots;
  CK(cudaMalloc(&d_rows, n * 4));
  CK(cudaMalloc(&d_rrows, n * 4));
  CK(cudaMalloc(&d_slots, n * 4));
  CK(cudaMemcpy(d_rows, rows.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rrows, rrows.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_slots, slots.data(), n * 4, cudaMemcpyHostToDevice));
  // touch the host pages once
  for (size_t i = 0; i < host_rows * row_b / 16; i += 256) host[i] = make_float4(0, 0, 0, 0);
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  cudaEvent_t fork, join;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  const double mb = n * row_b / 1e6;
  auto timeit = [&](const char* name, double bytes_mb, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    CK(cudaDeviceSynchronize());
    const int reps = 10;
    CK(cudaEventRecord(e0, s1));
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(e1, s1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("%-34s %8.3f ms  %7.1f GB/s\n", name, ms, bytes_mb / ms);
  };
  for (int bpw : {256, 512}) {
    char nm[64];
    snprintf(nm, sizeof nm, "write_warp (block %d)", bpw);
    timeit(nm, mb, [&] {
      write_warp<<<(n * 32 + bpw - 1) / bpw, bpw, 0, s1>>>(n, d_rows, d_slots, emb, mom, vel, host);
    });
  }
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "write_flat (grid %d)", g);
    timeit(nm, mb, [&] {
      write_flat<<<g, 256, 0, s1>>>(n, d_rows, d_slots, emb, mom, vel, host);
    });
  }
  for (int g : {148, 148 * 2, 148 * 4, 148 * 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "write_tma (grid %d)", g);
    timeit(nm, mb, [&] { write_tma<<<g, 256, 0, s1>>>(n, d_rows, d_slots, emb, mom, vel, host); });
  }
  timeit("stage+CE D2H (contiguous)", mb, [&] {
    gather_stage<<<148 * 8, 256, 0, s1>>>(n, d_slots, emb, mom, vel, stage);
    cudaMemcpyAsync(hstage, stage, n * row_b, cudaMemcpyDeviceToHost, s1);
  });
  timeit("CE D2H only (contiguous)", mb, [&] {
    cudaMemcpyAsync(hstage, stage, n * row_b, cudaMemcpyDeviceToHost, s1);
  });
  timeit("CE H2D only (contiguous)", mb, [&] {
    cudaMemcpyAsync(stage, hstage, n * row_b, cudaMemcpyHostToDevice, s1);
  });
  timeit("read_warp", mb, [&] {
    read_warp<<<(n * 32 + 255) / 256, 256, 0, s1>>>(n, d_rows, d_slots, host, emb, mom, vel);
  });
  for (int g : {148 * 8, 148 * 16, 148 * 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "read_flat (grid %d)", g);
    timeit(nm, mb, [&] {
      read_flat<<<g, 256, 0, s1>>>(n, d_rows, d_slots, host, emb, mom, vel);
    });
  }
  timeit("swap_warp (write n + read n)", 2 * mb, [&] {
    swap_warp<<<(n * 32 + 255) / 256, 256, 0, s1>>>(n, d_rows, d_rrows, d_slots, emb, mom, vel, host);
  });
  // concurrent write (s1) and read (s2)
  timeit("write_flat || read_flat (2 streams)", 2 * mb, [&] {
    CK(cudaEventRecord(fork, s1));
    CK(cudaStreamWaitEvent(s2, fork));
    write_flat<<<148 * 8, 256, 0, s1>>>(n, d_rows, d_slots, emb, mom, vel, host);
    read_flat<<<148 * 8, 256, 0, s2>>>(n, d_rrows, d_slots, host, emb, mom, vel);
    CK(cudaEventRecord(join, s2));
    CK(cudaStreamWaitEvent(s1, join));
  });
  printf("done\n");
  return 0;
}
