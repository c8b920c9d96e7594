// Worker ops on the virtual table: the forward gathers and
// the backward scatter-add are HBM-bound byte movers, so every kernel moves
// 128-bit vectors with consecutive threads on consecutive 16 B of one
// embedding row (d=80 -> 20 lanes cover a 320 B row; rows are 16 B aligned).
#include <cub/device/device_radix_sort.cuh>

#include "kernels.h"

namespace sfb {

namespace {

template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
  return __ldcs(p);
}

__global__ void gather_cache_v4(const uint32_t* __restrict__ own_k,
                                const uint32_t* __restrict__ own_slot,
                                const int32_t* __restrict__ n_ptr, int32_t n_bound, int d4,
                                const float4* __restrict__ emb, float4* __restrict__ G,
                                float4* __restrict__ dG_zero, float* __restrict__ B_zero) {
  pdl_wait();
  const int32_t n_own = n_ptr ? *n_ptr : n_bound;
  const int64_t n = static_cast<int64_t>(n_own) * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = idiv(i, d4);
    const int c = static_cast<int>(i - j * d4);
    const int64_t g = static_cast<int64_t>(own_k[j]) * d4 + c;
    G[g] = emb[static_cast<int64_t>(own_slot[j]) * 3 * d4 + c];  // cache rows: [emb | m | v]
    if (dG_zero) dG_zero[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (B_zero && c == 0) B_zero[own_k[j]] = 0.f;
  }
}

// one worker without a materialised G: only dG[0:U) and B[0:U) need clearing
__global__ void zero_rows_b_kernel(const int32_t* __restrict__ n_ptr, int d4,
                                   float4* __restrict__ dG, float* __restrict__ B) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(*n_ptr) * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    dG[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t j = idiv(i, d4);
    if (i == j * d4) B[j] = 0.f;
  }
}

__global__ void gather_cache_s(const uint32_t* __restrict__ own_k,
                               const uint32_t* __restrict__ own_slot, const int32_t* __restrict__ n_ptr, int32_t n_bound, int d,
                               const float* __restrict__ emb, float* __restrict__ G) {
  const int32_t n_own = n_ptr ? *n_ptr : n_bound;
  const int64_t n = static_cast<int64_t>(n_own) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = idiv(i, d);
    const int c = static_cast<int>(i - j * d);
    G[static_cast<int64_t>(own_k[j]) * d + c] = emb[static_cast<int64_t>(own_slot[j]) * 3 * d + c];
  }
}

// Thread per (row, 16 B column chunk); loops over the F fields of the row.
// Writes X (streaming store: it is consumed once by the tower) and the FM
// partial sums.
// slot_of != nullptr (one worker): G is not materialised; unique k's row is read from the
// cache slot slot_of[k] (= own_slot, an L2-resident table) instead.
// Two threads per (row, 16 B chunk), adjacent lanes, each gathering half of the F fields
// (8 row loads in flight), the FM partial sums combined with one shuffle: twice the
// threads of a whole-row loop, so the kernel reaches two waves and hides the HBM latency.
__global__ void __launch_bounds__(256, 5) gather_instances_v4(
    const uint32_t* __restrict__ vid, int32_t rows, int F, int d4, const float4* __restrict__ G,
    float4* __restrict__ X, float4* __restrict__ fm_s, float* __restrict__ fm_sqp,
    const uint32_t* __restrict__ slot_of, int g4) {
  pdl_wait();
  // g4: row stride of G in float4 (d/4 for a common table, 3d/4 for the cache rows)
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t p = i >> 1;
  const int h = static_cast<int>(i & 1);
  const bool valid = p < static_cast<int64_t>(rows) * d4;
  const int64_t r = valid ? idiv(p, d4) : 0;
  const int c = static_cast<int>(p - r * d4);
  const int Fh = (F + 1) >> 1;
  const int f0 = h ? Fh : 0, f1 = h ? F : Fh;
  const uint32_t* vr = vid + r * F;
  float4* xr = X + r * F * d4 + c;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  float sq = 0.f;
  if (valid) {
    int f = f0;
    for (; f + 8 <= f1; f += 8) {  // 8 independent row loads in flight
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(vr + f + u);
      if (slot_of) {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(slot_of + v[u]);
      }
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldg(G + static_cast<int64_t>(v[u]) * g4 + c);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xr[(f + u) * d4] = a[u];
        s.x += a[u].x; s.y += a[u].y; s.z += a[u].z; s.w += a[u].w;
        sq += a[u].x * a[u].x + a[u].y * a[u].y + a[u].z * a[u].z + a[u].w * a[u].w;
      }
    }
    for (; f < f1; ++f) {
      uint32_t v = __ldg(vr + f);
      if (slot_of) v = __ldg(slot_of + v);
      const float4 a = __ldg(G + static_cast<int64_t>(v) * g4 + c);
      xr[f * d4] = a;
      s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
      sq += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
    }
  }
  s.x += __shfl_xor_sync(0xFFFFFFFFu, s.x, 1);
  s.y += __shfl_xor_sync(0xFFFFFFFFu, s.y, 1);
  s.z += __shfl_xor_sync(0xFFFFFFFFu, s.z, 1);
  s.w += __shfl_xor_sync(0xFFFFFFFFu, s.w, 1);
  sq += __shfl_xor_sync(0xFFFFFFFFu, sq, 1);
  if (valid && h == 0) {
    fm_s[r * d4 + c] = s;
    fm_sqp[r * d4 + c] = sq;
  }
}

__global__ void gather_instances_s(const uint32_t* __restrict__ vid, int32_t rows, int F, int d,
                                   int ldx, const float* __restrict__ G, float* __restrict__ X,
                                   float* __restrict__ fm_s, float* __restrict__ fm_sqp) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * d) return;
  const int64_t r = idiv(i, d);
  const int c = static_cast<int>(i - r * d);
  float s = 0.f, sq = 0.f;
  for (int f = 0; f < F; ++f) {
    const float a = G[static_cast<int64_t>(vid[r * F + f]) * d + c];
    X[r * ldx + f * d + c] = a;
    s += a;
    sq += a * a;
  }
  fm_s[r * d + c] = s;
  fm_sqp[r * d + c] = sq;
}

__global__ void fm_sums_kernel(const float* __restrict__ X, int32_t rows, int F, int d, int ldx,
                               float* __restrict__ fm_s, float* __restrict__ fm_sqp, int parts) {
  // thread per (row, column c); one partial per column (parts == d here)
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * d) return;
  const int64_t r = idiv(i, d);
  const int c = static_cast<int>(i - r * d);
  float s = 0.f, sq = 0.f;
  for (int f = 0; f < F; ++f) {
    const float a = X[r * ldx + f * d + c];
    s += a;
    sq += a * a;
  }
  fm_s[r * d + c] = s;
  // fold columns onto `parts` partial slots (parts divides d handling below)
  if (parts == d) fm_sqp[r * d + c] = sq;
  else atomicAdd(fm_sqp + r * parts + (c / 4), sq);
}

// The embedding gradient of position p = (row r, field f) is
//   dX_mlp[p] + scale * gz[r] * (S_r - v_p)          (FM: d/dv_f sum_{i<j}<v_i,v_j>)
// The tower writes the MLP part; the FM part is added here, where v_p = G[vid[p]]
// is an L2-resident re-read of the row being scattered to.
// Bsum != nullptr (deferred FM correction): the -scale*gz[r]*v_p part is linear in the
// row v_p = G[vid[p]], so it is summed per unique row as Bsum[u] = sum_p gz[r] and applied
// once by the optimizer (g -= scale * Bsum[u] * G[u], G[u] being the row it updates);
// this pass then reads only dX, not a gathered G row per position.
__global__ void segment_sum_v4(const uint32_t* __restrict__ vid, int32_t n, int F, int d4,
                               const float4* __restrict__ dX, const float4* __restrict__ G,
                               const float4* __restrict__ fm_s, const float* __restrict__ gz,
                               float scale, float* __restrict__ dG, float* __restrict__ Bsum) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(n) * d4) return;
  const int64_t p = idiv(i, d4);
  const int c = static_cast<int>(i - p * d4);
  const int64_t r = idiv(p, F);
  const uint32_t v = __ldg(vid + p);
  const float4 a = __ldcs(dX + i);
  const float4 s = __ldg(fm_s + r * d4 + c);
  const float gr = __ldg(gz + r);
  const float k = scale * gr;
  float* dst = dG + (static_cast<int64_t>(v) * d4 + c) * 4;
  if (Bsum) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a.x + k * s.x),
                 "f"(a.y + k * s.y), "f"(a.z + k * s.z), "f"(a.w + k * s.w)
                 : "memory");
    if (c == 0) atomicAdd(Bsum + v, gr);
    return;
  }
  const float4 e = __ldg(G + static_cast<int64_t>(v) * d4 + c);
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst),
               "f"(a.x + k * (s.x - e.x)), "f"(a.y + k * (s.y - e.y)), "f"(a.z + k * (s.z - e.z)),
               "f"(a.w + k * (s.w - e.w))
               : "memory");
}

__global__ void segment_sum_s(const uint32_t* __restrict__ vid, int32_t n, int F, int d, int ldx,
                              const float* __restrict__ dX, const float* __restrict__ G,
                              const float* __restrict__ fm_s, const float* __restrict__ gz,
                              float scale, float* __restrict__ dG) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(n) * d) return;
  const int64_t p = idiv(i, d);  // position = row * F + field
  const int c = static_cast<int>(i - p * d);
  const int64_t r = idiv(p, F);
  const int f = static_cast<int>(p - r * F);
  const int64_t v = vid[p];
  const float g = dX[r * ldx + f * d + c] + scale * gz[r] * (fm_s[r * d + c] - G[v * d + c]);
  atomicAdd(dG + v * d + c, g);
}

// dx[r, k] += scale * gz[r] * (fm_s[r, k % d] - x[r, k])  (standalone model op)
__global__ void fm_grad_add_kernel(const float* __restrict__ X, int32_t rows, int K, int d, int ldx,
                                   const float* __restrict__ fm_s, const float* __restrict__ gz,
                                   float scale, float* __restrict__ dX) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * K) return;
  const int64_t r = i / K;
  const int k = static_cast<int>(i - r * K);
  const int64_t o = r * ldx + k;
  dX[o] += scale * gz[r] * (fm_s[r * d + (k % d)] - X[o]);
}

// Lazy Adam: t = adam_steps + 1 per row; bias
// corrections 1 - beta^t from host-built fp64 tables.
__global__ void sparse_adam_kernel(const uint32_t* __restrict__ own_k,
                                   const uint32_t* __restrict__ own_slot, const int32_t* __restrict__ n_ptr, int32_t n_bound, int d,
                                   const float* __restrict__ dG, float* __restrict__ emb,
                                   float* __restrict__ mom, float* __restrict__ vel,
                                   const int32_t* __restrict__ steps, const float* __restrict__ bc1,
                                   const float* __restrict__ bc2, float lr, float b1, float b2,
                                   float omb1, float omb2, float eps) {
  const int32_t n_own = n_ptr ? *n_ptr : n_bound;
  const int64_t n = static_cast<int64_t>(n_own) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = idiv(i, d);
    const int c = static_cast<int>(i - j * d);
    const uint32_t s = own_slot[j];
    const int t = steps[s] + 1;
    const float g = dG[static_cast<int64_t>(own_k ? own_k[j] : j) * d + c];
    const int64_t o = static_cast<int64_t>(s) * 3 * d + c;  // cache rows: [emb | m | v]
    const float m = b1 * mom[o] + omb1 * g;
    const float v = b2 * vel[o] + omb2 * g * g;
    mom[o] = m;
    vel[o] = v;
    const float mh = m / bc1[t], vh = v / bc2[t];
    emb[o] -= lr * mh / (sqrtf(vh) + eps);
  }
}

__global__ void sparse_adam_v4(const uint32_t* __restrict__ own_k,
                               const uint32_t* __restrict__ own_slot, const int32_t* __restrict__ n_ptr, int32_t n_bound, int d4,
                               const float4* __restrict__ dG, float4* __restrict__ emb,
                               float4* __restrict__ mom, float4* __restrict__ vel,
                               const int32_t* __restrict__ steps, const float* __restrict__ bc1,
                               const float* __restrict__ bc2, float lr, float b1, float b2,
                               float omb1, float omb2, float eps, const float* __restrict__ Bsum,
                               float fm_scale) {
  pdl_wait();
  const int32_t n_own = n_ptr ? *n_ptr : n_bound;
  const int64_t n = static_cast<int64_t>(n_own) * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = idiv(i, d4);
    const int c = static_cast<int>(i - j * d4);
    const uint32_t s = __ldg(own_slot + j);
    const int t = __ldg(steps + s) + 1;
    const float c1 = __ldg(bc1 + t), c2 = __ldg(bc2 + t);
    const int64_t gr = own_k ? __ldg(own_k + j) : j;
    float4 g = __ldg(dG + gr * d4 + c);
    const int64_t o = static_cast<int64_t>(s) * 3 * d4 + c;  // cache rows: [emb | m | v]
    float4 m = mom[o], v = vel[o], e = emb[o];
    if (Bsum) {  // deferred FM term of segment_sum: e is the G row of the forward pass
      const float kb = fm_scale * __ldg(Bsum + gr);
      g.x -= kb * e.x;
      g.y -= kb * e.y;
      g.z -= kb * e.z;
      g.w -= kb * e.w;
    }
#define SFB_ADAM(X)                    \
  m.X = b1 * m.X + omb1 * g.X;         \
  v.X = b2 * v.X + omb2 * g.X * g.X;   \
  e.X -= lr * (m.X / c1) / (sqrtf(v.X / c2) + eps);
    SFB_ADAM(x) SFB_ADAM(y) SFB_ADAM(z) SFB_ADAM(w)
#undef SFB_ADAM
    mom[o] = m;
    vel[o] = v;
    emb[o] = e;
  }
}

__global__ void steps_inc_kernel(const uint32_t* __restrict__ own_slot, const int32_t* __restrict__ n_ptr, int32_t n_bound,
                                 int32_t* __restrict__ steps) {
  const int32_t n_own = n_ptr ? *n_ptr : n_bound;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_own; j += gridDim.x * blockDim.x)
    steps[own_slot[j]] += 1;
}

}  // namespace

int fm_sq_parts(int d) { return (d & 3) == 0 ? d / 4 : d; }

// grid for the count-bounded grid-stride kernels: one resident wave of 256-thread CTAs
// (148 SMs x 8), fewer when the bound is small; the device count ends the loops
static int wave_grid(int64_t n_bound) { return std::max(1, std::min(ceil_div(n_bound, 256), num_sms() * 8)); }

void gather_cache(const uint32_t* own_k, const uint32_t* own_slot, int32_t n_own,
                  const int32_t* d_n_own, const float* emb, int d, float* G, float* dG_zero,
                  cudaStream_t s, float* B_zero) {
  SFB_CHECK(!dG_zero || (d & 3) == 0, "gather_cache: fused dG zeroing needs d % 4 == 0");
  if (n_own <= 0) return;
  if ((d & 3) == 0) {
    const int64_t n = static_cast<int64_t>(n_own) * (d / 4);
    launch_pdl(gather_cache_v4, dim3(wave_grid(n)), dim3(256), 0, s, own_k, own_slot, d_n_own, n_own, d / 4,
                                                     reinterpret_cast<const float4*>(emb),
                                                     reinterpret_cast<float4*>(G),
                                                     reinterpret_cast<float4*>(dG_zero), B_zero);
  } else {
    const int64_t n = static_cast<int64_t>(n_own) * d;
    gather_cache_s<<<wave_grid(n), 256, 0, s>>>(own_k, own_slot, d_n_own, n_own, d, emb, G);
  }
  CUDA_LAUNCH_CHECK();
}

void zero_rows_b(const int32_t* d_n, int32_t n_bound, int d, float* dG, float* B, cudaStream_t s) {
  SFB_CHECK((d & 3) == 0, "zero_rows_b needs d % 4 == 0");
  if (n_bound <= 0) return;
  // manager stage: a capped grid (mgr_grid), not a full wave of resident CTAs
  launch_pdl(zero_rows_b_kernel, dim3(mgr_grid(wave_grid(static_cast<int64_t>(n_bound) * (d / 4)))),
             dim3(256), 0, s, d_n, d / 4, reinterpret_cast<float4*>(dG), B);
  CUDA_LAUNCH_CHECK();
}

void gather_instances(const uint32_t* vid, int32_t rows, int F, int d, int ldx, const float* G,
                      float* X, float* fm_s, float* fm_sqp, cudaStream_t s,
                      const uint32_t* slot_of, int g_ld) {
  if (rows <= 0) return;
  SFB_CHECK(!slot_of || (d & 3) == 0, "gather_instances: slot indirection needs d % 4 == 0");
  if ((d & 3) == 0) {
    const int64_t n = static_cast<int64_t>(rows) * (d / 4) * 2;  // two threads per chunk
    launch_pdl(gather_instances_v4, dim3(ceil_div(n, 256)), dim3(256), 0, s, vid, rows, F, d / 4, reinterpret_cast<const float4*>(G), reinterpret_cast<float4*>(X),
        reinterpret_cast<float4*>(fm_s), fm_sqp, slot_of, (g_ld ? g_ld : d) / 4);
  } else {
    const int64_t n = static_cast<int64_t>(rows) * d;
    gather_instances_s<<<ceil_div(n, 256), 256, 0, s>>>(vid, rows, F, d, ldx, G, X, fm_s, fm_sqp);
  }
  CUDA_LAUNCH_CHECK();
}

void fm_sums(const float* X, int32_t rows, int F, int d, int ldx, float* fm_s, float* fm_sqp,
             cudaStream_t s) {
  const int parts = fm_sq_parts(d);
  if (parts != d) CUDA_CHECK(cudaMemsetAsync(fm_sqp, 0, sizeof(float) * rows * parts, s));
  const int64_t n = static_cast<int64_t>(rows) * d;
  fm_sums_kernel<<<ceil_div(n, 256), 256, 0, s>>>(X, rows, F, d, ldx, fm_s, fm_sqp, parts);
  CUDA_LAUNCH_CHECK();
}

void fm_grad_add(const float* X, int32_t rows, int F, int d, int ldx, const float* fm_s,
                 const float* gz, float scale, float* dX, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(rows) * F * d;
  if (n <= 0) return;
  fm_grad_add_kernel<<<ceil_div(n, 256), 256, 0, s>>>(X, rows, F * d, d, ldx, fm_s, gz, scale, dX);
  CUDA_LAUNCH_CHECK();
}

void segment_sum(const uint32_t* vid, int32_t n, int F, int d, int ldx, const float* dX,
                 const float* G, const float* fm_s, const float* gz, float scale, float* dG,
                 cudaStream_t s, float* Bsum) {
  if (n <= 0) return;
  if ((d & 3) == 0 && ldx == F * d) {
    const int64_t m = static_cast<int64_t>(n) * (d / 4);
    segment_sum_v4<<<ceil_div(m, 256), 256, 0, s>>>(
        vid, n, F, d / 4, reinterpret_cast<const float4*>(dX), reinterpret_cast<const float4*>(G),
        reinterpret_cast<const float4*>(fm_s), gz, scale, dG, Bsum);
  } else {
    const int64_t m = static_cast<int64_t>(n) * d;
    SFB_CHECK(!Bsum, "segment_sum: deferred FM term needs d % 4 == 0");
    segment_sum_s<<<ceil_div(m, 256), 256, 0, s>>>(vid, n, F, d, ldx, dX, G, fm_s, gz, scale, dG);
  }
  CUDA_LAUNCH_CHECK();
}

namespace {
__global__ void iota_u32_kernel(uint32_t* p, int32_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = static_cast<uint32_t>(i);
}
struct SegStartFlag {
  const uint32_t* v;
  __device__ uint32_t operator()(int64_t i) const { return i == 0 || v[i] != v[i - 1] ? 1u : 0u; }
};
struct SegStartEmit {
  uint32_t* starts;
  __device__ void operator()(int64_t i, uint32_t flag, uint32_t rank) const {
    if (flag) starts[rank] = static_cast<uint32_t>(i);
  }
};
// one warp per segment (unique row v), positions in ascending order, columns over lanes
__global__ void segment_sum_csr_kernel(const uint32_t* __restrict__ vid_sorted,
                                       const uint32_t* __restrict__ pos_sorted,
                                       const uint32_t* __restrict__ starts,
                                       const int32_t* __restrict__ count, int32_t n, int F, int d,
                                       int ldx, const float* __restrict__ dX,
                                       const float* __restrict__ G, const float* __restrict__ fm_s,
                                       const float* __restrict__ gz, float scale,
                                       float* __restrict__ dG) {
  const int lane = threadIdx.x & 31;
  const int64_t nseg = *count;
  const int64_t wstride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sg = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; sg < nseg;
       sg += wstride) {
    const uint32_t q0 = starts[sg];
    const uint32_t q1 = sg + 1 < nseg ? starts[sg + 1] : static_cast<uint32_t>(n);
    const int64_t v = vid_sorted[q0];
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      if (c >= d) break;
      const float gv = G[v * d + c];
      float acc = 0.f;
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t p = pos_sorted[q];
        const uint32_t r = p / static_cast<uint32_t>(F), f = p - r * static_cast<uint32_t>(F);
        acc += dX[static_cast<int64_t>(r) * ldx + static_cast<int64_t>(f) * d + c] +
               scale * gz[r] * (fm_s[static_cast<int64_t>(r) * d + c] - gv);
      }
      dG[v * d + c] += acc;
    }
  }
}
}  // namespace

void SegCsr::init(int64_t n) {
  release();
  cap = std::max<int64_t>(n, 1);
  CUDA_CHECK(cudaMalloc(&pos_in, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&vid_out, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&pos_out, sizeof(uint32_t) * cap));
  CUDA_CHECK(cudaMalloc(&starts, sizeof(uint32_t) * (cap + 1)));
  CUDA_CHECK(cudaMalloc(&count, sizeof(int32_t)));
  CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, static_cast<const uint32_t*>(nullptr),
                                             static_cast<uint32_t*>(nullptr),
                                             static_cast<const uint32_t*>(nullptr),
                                             static_cast<uint32_t*>(nullptr), static_cast<int>(cap)));
  CUDA_CHECK(cudaMalloc(&temp, temp_bytes));
  tiles.init(cap);
}

void SegCsr::release() {
  for (void* p : {static_cast<void*>(pos_in), static_cast<void*>(vid_out),
                  static_cast<void*>(pos_out), static_cast<void*>(starts),
                  static_cast<void*>(count), temp})
    if (p) cudaFree(p);
  tiles.release();
  *this = SegCsr();
}

void segment_sum_csr(SegCsr& cs, const uint32_t* vid, int32_t n, int F, int d, int ldx,
                     const float* dX, const float* G, const float* fm_s, const float* gz,
                     float scale, float* dG, int vid_bits, cudaStream_t s) {
  if (n <= 0) return;
  SFB_CHECK(n <= cs.cap, "segment_sum_csr: batch exceeds scratch");
  iota_u32_kernel<<<ceil_div(n, 256), 256, 0, s>>>(cs.pos_in, n);
  CUDA_LAUNCH_CHECK();
  size_t tb = cs.temp_bytes;
  // LSD radix sort is stable: each unique's positions stay in ascending order
  CUDA_CHECK(cub::DeviceRadixSort::SortPairs(cs.temp, tb, vid, cs.vid_out, cs.pos_in, cs.pos_out, n,
                                             0, std::max(1, std::min(32, vid_bits)), s));
  g_launches += 1 + (vid_bits + 7) / 8;
  lookback_scan<8>(cs.tiles, n, SegStartFlag{cs.vid_out}, SegStartEmit{cs.starts}, cs.count, s);
  segment_sum_csr_kernel<<<num_sms() * 8, 256, 0, s>>>(cs.vid_out, cs.pos_out, cs.starts, cs.count,
                                                       n, F, d, ldx, dX, G, fm_s, gz, scale, dG);
  CUDA_LAUNCH_CHECK();
}

void sparse_adam(const uint32_t* own_k /* gradient row index, or null = j */,
                 const uint32_t* own_slot, int32_t n_own, const int32_t* d_n_own, const float* dG,
                 int d, float* emb, float* mom, float* vel, int32_t* steps, const float* bc1,
                 const float* bc2, float lr, double beta1, double beta2, float eps, cudaStream_t s,
                 bool inc_steps, const float* Bsum, float fm_scale) {
  if (n_own <= 0) return;
  const float omb1 = static_cast<float>(1.0 - beta1);
  const float omb2 = static_cast<float>(1.0 - beta2);
  if ((d & 3) == 0) {
    const int64_t n = static_cast<int64_t>(n_own) * (d / 4);
    // one wave of resident CTAs: a grid of 148 x 8 with 5 resident per SM (43 registers) ran
    // the grid-stride loop in 1.6 waves, the last one at 60 % occupancy
    static const int per_sm = [] {
      int b = 0;
      if (const char* e = std::getenv("SFCTR_ADAM_CTAS_PER_SM")) b = atoi(e);  // experiment switch
      if (b <= 0) CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sparse_adam_v4, 256, 0));
      return std::max(1, b);
    }();
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), num_sms() * per_sm)));
    launch_pdl(sparse_adam_v4, dim3(grid), dim3(256), 0, s, own_k, own_slot, d_n_own, n_own, d / 4, reinterpret_cast<const float4*>(dG),
        reinterpret_cast<float4*>(emb), reinterpret_cast<float4*>(mom),
        reinterpret_cast<float4*>(vel), steps, bc1, bc2, lr, beta1, beta2, omb1, omb2, eps, Bsum,
        fm_scale);
  } else {
    SFB_CHECK(!Bsum, "sparse_adam: deferred FM term needs d % 4 == 0");
    const int64_t n = static_cast<int64_t>(n_own) * d;
    sparse_adam_kernel<<<wave_grid(n), 256, 0, s>>>(own_k, own_slot, d_n_own, n_own, d, dG, emb, mom,
                                                        vel, steps, bc1, bc2, lr, beta1, beta2,
                                                        omb1, omb2, eps);
  }
  CUDA_LAUNCH_CHECK();
  if (inc_steps) {
    steps_inc_kernel<<<wave_grid(n_own), 256, 0, s>>>(own_slot, d_n_own, n_own, steps);
    CUDA_LAUNCH_CHECK();
  }
}

}  // namespace sfb
