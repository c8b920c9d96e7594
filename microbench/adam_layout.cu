// Lazy-Adam row update layout microbenchmark (not shipped; DESIGN.md §9 evidence):
// U random slots of a C-slot table, d = 80 fp32. SoA = emb / m / v in three [C x d] arrays
// (the shipped layout); AoS = one [C x 3d] array (emb | m | v contiguous per slot);
// SoA96 = three arrays with rows padded to 96 floats (384 B, 128 B aligned).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o adam_layout adam_layout.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int D4 = 20;

template <int LD4, bool AOS>
__global__ void adam(int n_rows, const uint32_t* __restrict__ slot, const float4* __restrict__ g,
                     float4* __restrict__ emb, float4* __restrict__ mom, float4* __restrict__ vel) {
  const int64_t n = static_cast<int64_t>(n_rows) * D4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i / D4;
    const int c = static_cast<int>(i - j * D4);
    const uint32_t s = __ldg(slot + j);
    float4 gg = __ldg(g + i);
    float4 *pe, *pm, *pv;
    if (AOS) {
      pe = emb + static_cast<int64_t>(s) * 3 * D4 + c;
      pm = pe + D4;
      pv = pe + 2 * D4;
    } else {
      pe = emb + static_cast<int64_t>(s) * LD4 + c;
      pm = mom + static_cast<int64_t>(s) * LD4 + c;
      pv = vel + static_cast<int64_t>(s) * LD4 + c;
    }
    float4 m = *pm, v = *pv, e = *pe;
#define A(X)                              \
  m.X = 0.9f * m.X + 0.1f * gg.X;         \
  v.X = 0.999f * v.X + 0.001f * gg.X * gg.X; \
  e.X -= 1e-3f * m.X / (sqrtf(v.X) + 1e-8f);
    A(x) A(y) A(z) A(w)
#undef A
    *pm = m;
    *pv = v;
    *pe = e;
  }
}

int main() {
  const int64_t C = 33800000;
  const int U = 147000;
  std::vector<uint32_t> h(U);
  std::mt19937_64 rng(3);
  for (auto& x : h) x = rng() % C;
  uint32_t* slot;
  float4 *g, *a, *b, *c;
  cudaMalloc(&slot, U * 4);
  cudaMemcpy(slot, h.data(), U * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&g, static_cast<size_t>(U) * D4 * 16);
  cudaMalloc(&a, C * 24 * 16 * 3 / 3 * 3 / 3 * 1ull);  // placeholder, replaced below
  cudaFree(a);
  const size_t rows_bytes = static_cast<size_t>(C) * 96 * 4;  // 384 B per row (covers d=80 too)
  cudaMalloc(&a, rows_bytes);
  cudaMalloc(&b, rows_bytes);
  cudaMalloc(&c, rows_bytes);
  float4* aos;
  cudaMalloc(&aos, static_cast<size_t>(C) * 240 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = static_cast<double>(U) * (80 * 4 * 6 + 80 * 4);  // r/w e,m,v + g
  auto run = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("%-28s %7.2f us  %7.1f GB/s  (%s)\n", name, ms * 1e3, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int grid : {148 * 8, 148 * 16}) {
    printf("grid %d\n", grid);
    run("SoA d=80 (shipped)", [&] { adam<20, false><<<grid, 256>>>(U, slot, g, a, b, c); });
    run("SoA rows padded to 96", [&] { adam<24, false><<<grid, 256>>>(U, slot, g, a, b, c); });
    run("AoS emb|m|v per slot", [&] { adam<20, true><<<grid, 256>>>(U, slot, g, aos, nullptr, nullptr); });
  }
  return 0;
}
