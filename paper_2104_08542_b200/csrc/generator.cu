// Synthetic Criteo-shaped Zipf batches on the device, bit-exact with the
// reference SyntheticGenerator (core/src/generator.cpp:32-115).
//
// The reference draws ONE sequential splitmix stream per batch
// (generator.cpp:92), F+1 draws per row. splitmix64 is counter based — draw k
// of a stream seeded s is mix(s + (k+1)*golden) — so every (row, field) draw
// is computed independently here and each rank synthesises only its rows.
// Zipf CDFs are built on the host with std::pow exactly as generator.cpp:52-61
// does (glibc pow), uploaded once, and sampled by an upper_bound binary search
// per id (generator.cpp:70-75). All fp64 arithmetic uses __d*_rn intrinsics
// so no FMA contraction can change a rounding.
#include <cmath>
#include <vector>

#include "ops.h"

namespace sfb {

namespace {

__device__ __forceinline__ uint64_t upper_bound_cdf(const double* __restrict__ cdf, uint64_t k,
                                                    double unit) {
  uint64_t lo = 0, hi = k;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(cdf + mid) > unit) hi = mid;
    else lo = mid + 1;
  }
  return lo == k ? k - 1 : lo;  // generator.cpp:73
}

// One thread per (row, field): feature id and its hidden truth weight.
__global__ void gen_features_kernel(uint64_t seed_b, uint64_t seed, uint64_t truth_hash, int F,
                                    int32_t row0, int32_t nrows,
                                    const uint64_t* __restrict__ shard_starts, uint64_t base,
                                    const double* __restrict__ cdf_base,
                                    const double* __restrict__ cdf_big,
                                    uint64_t* __restrict__ features, double* __restrict__ tw) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(nrows) * F) return;
  const int64_t r = row0 + i / F;
  const int f = static_cast<int>(i % F);
  const uint64_t k = static_cast<uint64_t>(r) * (F + 1) + f;  // draw index within the batch stream
  const double unit = unit_from(splitmix_mix(seed_b + (k + 1) * kGolden));
  const uint64_t s0 = shard_starts[f], sz = shard_starts[f + 1] - s0;
  const uint64_t feat = s0 + upper_bound_cdf(sz == base ? cdf_base : cdf_big, sz, unit);
  features[i] = feat;
  // truth_weight (generator.cpp:77-80): Rng(derive_seed(seed,"truth",f)).next_uniform(-1,1)
  uint64_t st = derive_seed_h(seed, truth_hash, feat);
  tw[i] = uniform_from(splitmix_next(st), -1.0, 1.0);
}

// One thread per row: ordered logit sum, logistic probability, Bernoulli label
// (generator.cpp:94-105).
__global__ void gen_labels_kernel(uint64_t seed_b, int F, int32_t row0, int32_t nrows,
                                  double truth_scale, const double* __restrict__ tw,
                                  uint8_t* __restrict__ labels) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int64_t r = row0 + i;
  const double* t = tw + static_cast<int64_t>(i) * F;
  double logit = 0;
  for (int f = 0; f < F; ++f) logit = __dadd_rn(logit, t[f]);
  const double p = __ddiv_rn(1.0, __dadd_rn(1.0, exp(__dmul_rn(-truth_scale, logit))));
  const uint64_t k = static_cast<uint64_t>(r) * (F + 1) + F;
  const double u = unit_from(splitmix_mix(seed_b + (k + 1) * kGolden));
  labels[i] = u < p ? 1 : 0;
}

__global__ void init_embedding_kernel(uint64_t seed_e, int dim, double* out) {
  // generator.cpp:110-115: Rng(derive_seed(seed,"embed",f)), dim next_uniform(-0.01,0.01)
  const int c = threadIdx.x;
  if (c < dim) out[c] = uniform_from(splitmix_mix(seed_e + (c + 1) * kGolden), -0.01, 0.01);
}

std::vector<double> build_cdf(uint64_t k, double s) {  // generator.cpp:52-61
  std::vector<double> cdf(k);
  double total = 0;
  for (uint64_t i = 0; i < k; ++i) {
    total += std::pow(static_cast<double>(i + 1), -s);
    cdf[i] = total;
  }
  for (auto& v : cdf) v /= total;
  return cdf;
}

}  // namespace

void GenTables::build(int F, uint64_t V, uint64_t sd, double z) {
  release();
  if (V < static_cast<uint64_t>(F)) fail(kLogic, "vocabulary smaller than field count");
  fields = F;
  vocab = V;
  seed = sd;
  zipf = z;
  truth_scale = 2.5 / std::sqrt(static_cast<double>(F));  // generator.cpp:28,93
  shard_starts.assign(F + 1, 0);
  base = V / F;
  const uint64_t rem = V % F;
  for (int f = 0; f < F; ++f)
    shard_starts[f + 1] = shard_starts[f] + base + (static_cast<uint64_t>(f) < rem ? 1 : 0);
  CUDA_CHECK(cudaMalloc(&d_shard_starts, sizeof(uint64_t) * (F + 1)));
  CUDA_CHECK(cudaMemcpy(d_shard_starts, shard_starts.data(), sizeof(uint64_t) * (F + 1),
                        cudaMemcpyHostToDevice));
  auto cb = build_cdf(base, z);
  CUDA_CHECK(cudaMalloc(&d_cdf_base, sizeof(double) * cb.size()));
  CUDA_CHECK(cudaMemcpy(d_cdf_base, cb.data(), sizeof(double) * cb.size(), cudaMemcpyHostToDevice));
  if (rem) {
    auto cg = build_cdf(base + 1, z);
    CUDA_CHECK(cudaMalloc(&d_cdf_big, sizeof(double) * cg.size()));
    CUDA_CHECK(cudaMemcpy(d_cdf_big, cg.data(), sizeof(double) * cg.size(), cudaMemcpyHostToDevice));
  }
}

void GenTables::release() {
  cudaFree(d_shard_starts);
  cudaFree(d_cdf_base);
  cudaFree(d_cdf_big);
  cudaFree(d_tw);
  d_shard_starts = nullptr;
  d_cdf_base = d_cdf_big = d_tw = nullptr;
  tw_cap = 0;
}

void generate_rows(GenTables& g, int64_t step, int32_t row0, int32_t nrows, uint64_t* d_features,
                   uint8_t* d_labels, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(nrows) * g.fields;
  if (n > g.tw_cap) {
    CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(g.d_tw);
    CUDA_CHECK(cudaMalloc(&g.d_tw, sizeof(double) * n));
    g.tw_cap = n;
  }
  const uint64_t seed_b = derive_seed_h(g.seed, fnv1a64("batch"), static_cast<uint64_t>(step));
  gen_features_kernel<<<ceil_div(n, 256), 256, 0, s>>>(seed_b, g.seed, fnv1a64("truth"), g.fields,
                                                        row0, nrows, g.d_shard_starts, g.base,
                                                        g.d_cdf_base, g.d_cdf_big, d_features,
                                                        g.d_tw);
  CUDA_LAUNCH_CHECK();
  gen_labels_kernel<<<ceil_div(nrows, 128), 128, 0, s>>>(seed_b, g.fields, row0, nrows,
                                                          g.truth_scale, g.d_tw, d_labels);
  CUDA_LAUNCH_CHECK();
}

void initial_embedding_device(uint64_t seed, uint64_t feature, int dim, double* d_out,
                              cudaStream_t s) {
  init_embedding_kernel<<<1, ((dim + 31) / 32) * 32, 0, s>>>(
      derive_seed_h(seed, fnv1a64("embed"), feature), dim, d_out);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
