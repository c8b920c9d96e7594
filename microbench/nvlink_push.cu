// NVLink all-to-all push microbenchmark (not shipped; evidence for DESIGN.md §9/§10).
// One process drives W GPUs with peer access; every GPU pushes `mb` MB split evenly over
// its W-1 peers at the same time (the owner-routed exchange's pattern), by
//   st   : SM 16 B stores, grid-stride (the shipped push_blocks kernel)
//   tma  : rows staged in shared memory, cp.async.bulk shared -> peer global (8 KB per op)
//   ce   : cudaMemcpyPeerAsync per peer (copy engines)
// and reports the per-GPU outbound rate (max over GPUs of the time).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_push nvlink_push.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

struct Dst {
  float4* p[8];
  int64_t n4;  // float4 per peer
};

__global__ void push_st(const float4* __restrict__ src, Dst d, int W, int me, int unroll) {
  const int o = blockIdx.y;
  if (o == me) return;
  const float4* s = src + static_cast<int64_t>(o) * d.n4;
  float4* t = d.p[o] + static_cast<int64_t>(me) * d.n4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < d.n4;
       i0 += 2 * stride) {
    float4 v0 = s[i0];
    float4 v1 = i0 + stride < d.n4 ? s[i0 + stride] : make_float4(0, 0, 0, 0);
    t[i0] = v0;
    if (i0 + stride < d.n4) t[i0 + stride] = v1;
  }
}

constexpr int kChunk = 8192;  // bytes per bulk op
__global__ void push_tma(const float4* __restrict__ src, Dst d, int W, int me) {
  __shared__ __align__(128) float4 sm[4][kChunk / 16];
  const int o = blockIdx.y;
  if (o == me) return;
  const char* s = reinterpret_cast<const char*>(src + static_cast<int64_t>(o) * d.n4);
  char* t = reinterpret_cast<char*>(d.p[o] + static_cast<int64_t>(me) * d.n4);
  const int64_t bytes = d.n4 * 16;
  int it = 0;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kChunk; c < bytes;
       c += static_cast<int64_t>(gridDim.x) * kChunk, ++it) {
    const int st = it & 3;
    if (it >= 4) {
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      __syncthreads();
    }
    const int n = static_cast<int>(bytes - c < kChunk ? bytes - c : kChunk);
    for (int i = threadIdx.x; i < n / 16; i += blockDim.x)
      sm[st][i] = reinterpret_cast<const float4*>(s + c)[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(&sm[st][0]));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(t + c),
                   "r"(sa), "r"(n)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int W = argc > 1 ? atoi(argv[1]) : 2;
  const double mb = argc > 2 ? atof(argv[2]) : 36.0;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (W > ndev) W = ndev;
  const int64_t per = static_cast<int64_t>(mb * 1e6 / (W - 1)) / 16 * 16;  // bytes per peer
  printf("W=%d, %.1f MB out per GPU (%.2f MB per peer)\n", W, per * (W - 1) / 1e6, per / 1e6);
  std::vector<float4*> src(W), dst(W);
  std::vector<cudaStream_t> st(W);
  std::vector<cudaEvent_t> e0(W), e1(W);
  for (int g = 0; g < W; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < W; ++h)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src[g], per * W));
    CK(cudaMalloc(&dst[g], per * W));
    CK(cudaMemset(src[g], 1, per * W));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  auto run = [&](const char* name, int mode, int grid) {
    for (int rep = 0; rep < 6; ++rep) {
      for (int g = 0; g < W; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < W; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        Dst d{};
        for (int h = 0; h < W; ++h) d.p[h] = dst[h];
        d.n4 = per / 16;
        if (mode == 0) push_st<<<dim3(grid, W), 256, 0, st[g]>>>(src[g], d, W, g, 2);
        else if (mode == 1) push_tma<<<dim3(grid, W), 256, 0, st[g]>>>(src[g], d, W, g);
        else
          for (int h = 0; h < W; ++h)
            if (h != g)
              CK(cudaMemcpyPeerAsync(reinterpret_cast<char*>(dst[h]) + per * g, h,
                                     reinterpret_cast<char*>(src[g]) + per * h, g, per, st[g]));
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float mx = 0;
      for (int g = 0; g < W; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        mx = ms > mx ? ms : mx;
      }
      if (rep == 5)
        printf("%-26s grid %5d  %8.3f ms  %7.1f GB/s out per GPU\n", name, grid, mx,
               per * (W - 1) / (mx * 1e-3) / 1e9);
    }
  };
  for (int grid : {148, 296, 592, 1184}) run("SM st.v4", 0, grid);
  for (int grid : {74, 148, 296}) run("TMA bulk 8 KB", 1, grid);
  run("copy engine (peer memcpy)", 2, 0);
  printf("done\n");
  return 0;
}
