// DeepFM-lite tower (model.cpp is missing from
// the reference): output z = FM2 + MLP, FM2 = sum_{i<j} <v_i, v_j>
// = 0.5 (|sum_f v_f|^2 - sum_f |v_f|^2), MLP = relu(x W1 + b1) . w2 + b2,
// p = sigmoid(z), mean BCE with p clamped to [1e-7, 1-1e-7].
//
// fp32 SIMT tiles: x [rows, K=F*d] row-major, W1 [K, H] row-major.
//   fwd   : hpre = x W1 + b1                      (64x64 output tile / CTA)
//   head  : per row z, p, loss, gz, dh, relu       (warp per row)
//   dx    : dX = s*(dh W1^T + gz (S_fm - x))       (64x64 tile over (rows, k))
//   dw1   : dW1 = x^T dh                          (k-tile x row-split partials,
//                                                   reduced in a fixed order)
//   small : db1, dw2, db2, loss                    (fixed-order block reductions)
// All reductions are in a fixed order, so a run is deterministic.
#include "kernels.h"

namespace sfb {

namespace {

constexpr int TB = 64;   // tile edge
constexpr int BK = 32;   // inner-dim chunk
constexpr float kClamp = 1e-7f;

// hpre[r, j] = b1[j] + sum_k x[r, k] w1[k, j]
__global__ void __launch_bounds__(256) fwd_gemm_kernel(const float* __restrict__ x,
                                                       const float* __restrict__ w1,
                                                       const float* __restrict__ b1, int rows,
                                                       int K, int H, float* __restrict__ hpre) {
  __shared__ __align__(16) float xs[BK][TB + 4];  // x^T tile
  __shared__ __align__(16) float ws[BK][TB];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int r0 = blockIdx.x * TB, j0 = blockIdx.y * TB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 256 * i;
      const int rr = e >> 5, kk = e & 31;  // 64 rows x 32 k
      const int r = r0 + rr, k = k0 + kk;
      xs[kk][rr] = (r < rows && k < K) ? __ldg(x + static_cast<int64_t>(r) * K + k) : 0.f;
      const int kk2 = e >> 6, jj = e & 63;  // 32 k x 64 j
      const int k2 = k0 + kk2, j = j0 + jj;
      ws[kk2][jj] = (k2 < K && j < H) ? __ldg(w1 + static_cast<int64_t>(k2) * H + j) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&xs[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&ws[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + ty * 4 + u;
    if (r >= rows) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tx * 4 + v;
      if (j < H) hpre[static_cast<int64_t>(r) * H + j] = acc[u][v] + b1[j];
    }
  }
}

// Warp per row: MLP head, FM term, sigmoid/BCE, dz, dh.
__global__ void head_kernel(int rows, int H, int d, int sq_parts, const float* __restrict__ hpre,
                            const float* __restrict__ w2, const float* __restrict__ b2p,
                            const float* __restrict__ fm_s,
                            const float* __restrict__ fm_sqp, const uint8_t* __restrict__ labels,
                            float inv_rows, float* __restrict__ logits, float* __restrict__ act,
                            float* __restrict__ dh, float* __restrict__ gz,
                            float* __restrict__ lossr) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* hr = hpre + static_cast<int64_t>(r) * H;
  float mlp = 0.f;
  for (int j = lane; j < H; j += 32) mlp += fmaxf(hr[j], 0.f) * w2[j];
  float ss = 0.f, sq = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = fm_s[static_cast<int64_t>(r) * d + c];
    ss += v * v;
  }
  for (int c = lane; c < sq_parts; c += 32) sq += fm_sqp[static_cast<int64_t>(r) * sq_parts + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mlp += __shfl_xor_sync(0xFFFFFFFFu, mlp, o);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
    sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
  }
  const float z = 0.5f * (ss - sq) + (mlp + __ldg(b2p));
  const float p = 1.f / (1.f + expf(-z));
  const float y = labels[r] ? 1.f : 0.f;
  const bool clamped = (p < kClamp) || (p > 1.f - kClamp);
  const float pc = fminf(fmaxf(p, kClamp), 1.f - kClamp);
  const float g = clamped ? 0.f : (p - y) * inv_rows;
  for (int j = lane; j < H; j += 32) {
    const float hv = hr[j];
    act[static_cast<int64_t>(r) * H + j] = fmaxf(hv, 0.f);
    dh[static_cast<int64_t>(r) * H + j] = hv > 0.f ? g * w2[j] : 0.f;
  }
  if (lane == 0) {
    logits[r] = z;
    gz[r] = g;
    lossr[r] = -(y * logf(pc) + (1.f - y) * log1pf(-pc));
  }
}

// dX[r, k] = scale * (sum_j dh[r, j] w1[k, j] + gz[r] * (fm_s[r, k % d] - x[r, k]))
__global__ void __launch_bounds__(256) dx_kernel(const float* __restrict__ x,
                                                 const float* __restrict__ w1,
                                                 const float* __restrict__ dh,
                                                 const float* __restrict__ gz,
                                                 const float* __restrict__ fm_s, int rows, int K,
                                                 int H, int d, float scale, float* __restrict__ dX) {
  __shared__ __align__(16) float ds[BK][TB + 4];  // dh^T tile [j][r]
  __shared__ __align__(16) float ws[BK][TB + 4];  // w1^T tile [j][k]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int r0 = blockIdx.x * TB, k0 = blockIdx.y * TB;
  float acc[4][4] = {};
  for (int j0 = 0; j0 < H; j0 += BK) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 256 * i;
      const int rr = e >> 5, jj = e & 31;
      const int r = r0 + rr, j = j0 + jj;
      ds[jj][rr] = (r < rows && j < H) ? __ldg(dh + static_cast<int64_t>(r) * H + j) : 0.f;
      const int k = k0 + rr;
      ws[jj][rr] = (k < K && j < H) ? __ldg(w1 + static_cast<int64_t>(k) * H + j) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int jj = 0; jj < BK; ++jj) {
      const float4 a = *reinterpret_cast<const float4*>(&ds[jj][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&ws[jj][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + ty * 4 + u;
    if (r >= rows) continue;
    const float g = gz[r];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int k = k0 + tx * 4 + v;
      if (k >= K) continue;
      const int64_t o = static_cast<int64_t>(r) * K + k;
      (void)g;  // the FM part is added by segment_sum / fm_grad_add
      dX[o] = scale * acc[u][v];
    }
  }
}

// part[split, k, j] = sum_{r in split} x[r, k] dh[r, j]
__global__ void __launch_bounds__(256) dw1_kernel(const float* __restrict__ x,
                                                  const float* __restrict__ dh, int rows, int K,
                                                  int H, int rows_per_split,
                                                  float* __restrict__ part) {
  __shared__ __align__(16) float xs[BK][TB + 4];  // [r][k]
  __shared__ __align__(16) float hs[BK][TB + 4];  // [r][j]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int k0 = blockIdx.x * TB, j0 = blockIdx.y * TB, split = blockIdx.z;
  const int rb = split * rows_per_split, re = min(rows, rb + rows_per_split);
  float acc[4][4] = {};
  for (int q0 = rb; q0 < re; q0 += BK) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 256 * i;
      const int rr = e >> 6, cc = e & 63;  // 32 rows x 64 cols
      const int r = q0 + rr;
      const int k = k0 + cc, j = j0 + cc;
      xs[rr][cc] = (r < re && k < K) ? __ldg(x + static_cast<int64_t>(r) * K + k) : 0.f;
      hs[rr][cc] = (r < re && j < H) ? __ldg(dh + static_cast<int64_t>(r) * H + j) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < BK; ++rr) {
      const float4 a = *reinterpret_cast<const float4*>(&xs[rr][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&hs[rr][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
  float* out = part + static_cast<int64_t>(split) * K * H;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = k0 + ty * 4 + u;
    if (k >= K) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tx * 4 + v;
      if (j < H) out[static_cast<int64_t>(k) * H + j] = acc[u][v];
    }
  }
}

__global__ void dw1_reduce_kernel(const float* __restrict__ part, int splits, int64_t n,
                                  float* __restrict__ out, int accumulate) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int q = 0; q < splits; ++q) s += part[q * n + i];
  out[i] = accumulate ? out[i] + s : s;
}

// Block b < H: db1[b] = sum_r dh[r,b], dw2[b] = sum_r gz[r] act[r,b];
// block H: db2 = sum gz; block H+1: loss_sum += sum lossr / rows. Fixed order.
__global__ void small_grads_kernel(const float* __restrict__ dh, const float* __restrict__ act,
                                   const float* __restrict__ gz, const float* __restrict__ lossr,
                                   int rows, int H, float inv_rows, float* __restrict__ g_db1,
                                   float* __restrict__ g_dw2, float* __restrict__ g_db2,
                                   float* __restrict__ g_loss, int accumulate) {
  __shared__ float red[2][256];
  const int b = blockIdx.x, tid = threadIdx.x;
  float s0 = 0.f, s1 = 0.f;
  for (int r = tid; r < rows; r += 256) {
    if (b < H) {
      s0 += dh[static_cast<int64_t>(r) * H + b];
      s1 += gz[r] * act[static_cast<int64_t>(r) * H + b];
    } else if (b == H) {
      s0 += gz[r];
    } else {
      s0 += lossr[r];
    }
  }
  red[0][tid] = s0;
  red[1][tid] = s1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      red[0][tid] += red[0][tid + o];
      red[1][tid] += red[1][tid + o];
    }
    __syncthreads();
  }
  if (tid) return;
  if (b < H) {
    g_db1[b] = accumulate ? g_db1[b] + red[0][0] : red[0][0];
    g_dw2[b] = accumulate ? g_dw2[b] + red[1][0] : red[1][0];
  } else if (b == H) {
    *g_db2 = accumulate ? *g_db2 + red[0][0] : red[0][0];
  } else {
    const float l = red[0][0] * inv_rows;
    *g_loss = accumulate ? *g_loss + l : l;
  }
}

__global__ void dense_adam_kernel(float* __restrict__ p, float* __restrict__ m,
                                  float* __restrict__ v, const float* __restrict__ g, int64_t n,
                                  float gs, float lr, float b1, float b2, float omb1, float omb2,
                                  float eps, float bc1, float bc2) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i] * gs;
  const float mi = b1 * m[i] + omb1 * gi;
  const float vi = b2 * v[i] + omb2 * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
}

__global__ void scale_add_kernel(float* __restrict__ y, const float* __restrict__ x, int64_t n,
                                 float a) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}

}  // namespace

void TowerBufs::init(int rc, int k, int h, int dim) {
  release();
  rows_cap = rc;
  K = k;
  H = h;
  d = dim;
  const size_t rh = static_cast<size_t>(rc) * h;
  CUDA_CHECK(cudaMalloc(&hpre, sizeof(float) * rh));
  CUDA_CHECK(cudaMalloc(&act, sizeof(float) * rh));
  CUDA_CHECK(cudaMalloc(&dh, sizeof(float) * rh));
  CUDA_CHECK(cudaMalloc(&gz, sizeof(float) * rc));
  CUDA_CHECK(cudaMalloc(&lossr, sizeof(float) * rc));
  // row splits so that (K tiles x H tiles x splits) fills ~2 waves of 148 SMs
  const int kt = ceil_div(K, TB), ht = ceil_div(H, TB);
  splits = std::max(1, std::min(ceil_div(rc, BK), (2 * num_sms() + kt * ht - 1) / (kt * ht)));
  CUDA_CHECK(cudaMalloc(&part, sizeof(float) * static_cast<size_t>(splits) * K * H));
  // kSgChunks chunks, or one per 8 rows when the tensor-core head writes them
  CUDA_CHECK(cudaMalloc(&sg_part, sizeof(float) * std::max(256, (rows_cap + 7) / 8) * (2 * h + 2)));
}

void TowerBufs::release() {
  for (float* p : {hpre, act, dh, gz, lossr, part, sg_part})
    if (p) cudaFree(p);
  sg_part = nullptr;
  hpre = act = dh = gz = lossr = part = nullptr;
}

void dw1_reduce(const float* part, int splits, int64_t n, float* out, bool accumulate,
                cudaStream_t s) {
  dw1_reduce_kernel<<<ceil_div(n, 256), 256, 0, s>>>(part, splits, n, out, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
}

namespace {
// Phase 1: block c reduces rows [c*R, (c+1)*R) with column-coalesced reads of
// dh/act (thread j <-> column j), writing partials [c][2H+2] =
// (db1[0..H) | dw2[0..H) | db2 | loss). Phase 2 sums the chunks in order.
constexpr int kSgChunks = 256;
__global__ void small_grads_p1(const float* __restrict__ dh, const float* __restrict__ act,
                               const float* __restrict__ gz, const float* __restrict__ lossr,
                               int rows, int H, float* __restrict__ part) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const int R = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = c * R, r1 = min(rows, r0 + R);
  float* out = part + static_cast<int64_t>(c) * (2 * H + 2);
  for (int j = tid; j < H; j += blockDim.x) {
    float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
    int r = r0;
    for (; r + 4 <= r1; r += 4) {  // 4 independent row streams in flight
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t o = static_cast<int64_t>(r + u) * H + j;
        a[u] += dh[o];
        b[u] += gz[r + u] * act[o];
      }
    }
    for (; r < r1; ++r) {
      const int64_t o = static_cast<int64_t>(r) * H + j;
      a[0] += dh[o];
      b[0] += gz[r] * act[o];
    }
    out[j] = (a[0] + a[1]) + (a[2] + a[3]);
    out[H + j] = (b[0] + b[1]) + (b[2] + b[3]);
  }
  __shared__ float red[2][256];
  float s0 = 0.f, s1 = 0.f;
  for (int r = r0 + tid; r < r1; r += blockDim.x) {
    s0 += gz[r];
    s1 += lossr[r];
  }
  red[0][tid] = s0;
  red[1][tid] = s1;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) {
      red[0][tid] += red[0][tid + o];
      red[1][tid] += red[1][tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    out[2 * H] = red[0][0];
    out[2 * H + 1] = red[1][0];
  }
}
// out_major: part is [2H+2][chunks] (the tensor-core head's layout, coalesced here), else
// [chunks][2H+2] (small_grads_p1)
__global__ void small_grads_p2(const float* __restrict__ part, int chunks, int H, float inv_rows,
                               float* __restrict__ g_db1, float* __restrict__ g_dw2,
                               float* __restrict__ g_db2, float* __restrict__ g_loss,
                               int accumulate, int out_major = 0) {
  // warp per output; lanes take chunks lane, lane+32, ...; fixed shuffle tree (deterministic)
  const int n = 2 * H + 2;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  float s = 0.f;
  for (int c = lane; c < chunks; c += 32)
    s += out_major ? part[static_cast<int64_t>(i) * chunks + c] : part[static_cast<int64_t>(c) * n + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if (lane) return;
  float* dst = i < H ? g_db1 + i : (i < 2 * H ? g_dw2 + (i - H) : (i == 2 * H ? g_db2 : g_loss));
  if (i == 2 * H + 1) s *= inv_rows;
  *dst = accumulate ? *dst + s : s;
}
}  // namespace

// block per output over output-major partials [2H+2][chunks]: 256 threads, a fixed-order
// strided sum then a fixed shuffle / shared-memory tree (deterministic)
__global__ void small_grads_final_kernel(const float* __restrict__ part, int chunks, int H,
                                         float inv_rows, float* __restrict__ g_db1,
                                         float* __restrict__ g_dw2, float* __restrict__ g_db2,
                                         float* __restrict__ g_loss, int accumulate) {
  __shared__ float red[8];
  const int i = blockIdx.x, tid = threadIdx.x;
  const float* row = part + static_cast<int64_t>(i) * chunks;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  int c = tid;
  for (; c + 3 * 256 < chunks; c += 4 * 256) {
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] += __ldg(row + c + u * 256);
  }
  for (; c < chunks; c += 256) a[0] += __ldg(row + c);
  float v = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid != 0) return;
  float sum = 0.f;
  for (int w = 0; w < 8; ++w) sum += red[w];
  float* dst = i < H ? g_db1 + i : (i < 2 * H ? g_dw2 + (i - H) : (i == 2 * H ? g_db2 : g_loss));
  if (i == 2 * H + 1) sum *= inv_rows;
  *dst = accumulate ? *dst + sum : sum;
}

// dW1 split-K sum (blocks [0, nb)) and the small-gradient final pass (blocks nb ..) in one
// launch; the split partials are loaded before they are summed (in split order)
__global__ void tower_reduce_kernel(const float* __restrict__ part3, int splits, int64_t kh,
                                    float* __restrict__ g_w1, int nb, const float* __restrict__ sg,
                                    int chunks, int H, float inv_rows, float* __restrict__ g_db1,
                                    float* __restrict__ g_dw2, float* __restrict__ g_db2,
                                    float* __restrict__ g_loss, int accumulate) {
  pdl_wait();  // GEMM3 partials
  if (static_cast<int>(blockIdx.x) < nb) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= kh) return;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = q < splits ? __ldg(part3 + q * kh + i) : 0.f;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < splits) s += v[q];
    for (int q = 8; q < splits; ++q) s += __ldg(part3 + q * kh + i);
    g_w1[i] = accumulate ? g_w1[i] + s : s;
    return;
  }
  __shared__ float red[8];
  const int i = blockIdx.x - nb, tid = threadIdx.x;
  const float* row = sg + static_cast<int64_t>(i) * chunks;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  int c = tid;
  for (; c + 3 * 256 < chunks; c += 4 * 256) {
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] += __ldg(row + c + u * 256);
  }
  for (; c < chunks; c += 256) a[0] += __ldg(row + c);
  float v = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid != 0) return;
  float sum = 0.f;
  for (int w = 0; w < 8; ++w) sum += red[w];
  float* dst = i < H ? g_db1 + i : (i < 2 * H ? g_dw2 + (i - H) : (i == 2 * H ? g_db2 : g_loss));
  if (i == 2 * H + 1) sum *= inv_rows;
  *dst = accumulate ? *dst + sum : sum;
}

void tower_reduce(const float* part3, int splits, int64_t kh, float* g_w1, TowerBufs& t,
                  int chunks, int rows, int H, float* g_b1, float* g_w2, float* g_b2,
                  float* g_loss, bool accumulate, cudaStream_t s) {
  const int nb = ceil_div(kh, 256);
  launch_pdl(tower_reduce_kernel, dim3(nb + 2 * H + 2), dim3(256), 0, s, part3, splits, kh, g_w1,
             nb, static_cast<const float*>(t.sg_part), chunks, H, 1.f / rows, g_b1, g_w2, g_b2,
             g_loss, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
}

void small_grads_final(TowerBufs& t, int chunks, int rows, int H, float* g_b1, float* g_w2,
                       float* g_b2, float* g_loss, bool accumulate, cudaStream_t s) {
  small_grads_final_kernel<<<2 * H + 2, 256, 0, s>>>(t.sg_part, chunks, H, 1.f / rows, g_b1, g_w2,
                                                     g_b2, g_loss, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
}

void small_grads(TowerBufs& t, int rows, int H, float* g_b1, float* g_w2, float* g_b2,
                 float* g_loss, bool accumulate, cudaStream_t s) {
  const int chunks = std::max(1, std::min(kSgChunks, rows));
  small_grads_p1<<<chunks, 256, 0, s>>>(t.dh, t.act, t.gz, t.lossr, rows, H, t.sg_part);
  CUDA_LAUNCH_CHECK();
  small_grads_p2<<<ceil_div(2 * H + 2, 8), 256, 0, s>>>(t.sg_part, chunks, H, 1.f / rows, g_b1,
                                                         g_w2, g_b2, g_loss, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
}

void tower_forward_backward_simt(TowerBufs& t, const float* X, const float* fm_s,
                                 const float* fm_sqp, const uint8_t* labels, int32_t rows, int F,
                                 int d, const float* dense, float* logits, float* dX,
                                 float emb_scale, float* grads, bool accumulate, cudaStream_t s) {
  const int K = F * d, H = t.H;
  SFB_CHECK(rows <= t.rows_cap && K == t.K, "tower buffers too small");
  const float* w1 = dense;
  const float* b1 = dense + static_cast<size_t>(K) * H;
  const float* w2 = b1 + H;
  const float* b2p = w2 + H;
  float* g_w1 = grads;
  float* g_b1 = grads + static_cast<size_t>(K) * H;
  float* g_w2 = g_b1 + H;
  float* g_b2 = g_w2 + H;
  float* g_loss = g_b2 + 1;
  dim3 gf(ceil_div(rows, TB), ceil_div(H, TB));
  fwd_gemm_kernel<<<gf, 256, 0, s>>>(X, w1, b1, rows, K, H, t.hpre);
  CUDA_LAUNCH_CHECK();
  head_kernel<<<ceil_div(static_cast<int64_t>(rows) * 32, 256), 256, 0, s>>>(
      rows, H, d, fm_sq_parts(d), t.hpre, w2, b2p, fm_s, fm_sqp, labels, 1.f / rows, logits,
      t.act, t.dh, t.gz, t.lossr);
  CUDA_LAUNCH_CHECK();
  dim3 gx(ceil_div(rows, TB), ceil_div(K, TB));
  dx_kernel<<<gx, 256, 0, s>>>(X, w1, t.dh, t.gz, fm_s, rows, K, H, d, emb_scale, dX);
  CUDA_LAUNCH_CHECK();
  const int rps = ceil_div(ceil_div(rows, t.splits), BK) * BK;
  const int splits = ceil_div(rows, rps);
  dim3 gw(ceil_div(K, TB), ceil_div(H, TB), splits);
  dw1_kernel<<<gw, 256, 0, s>>>(X, t.dh, rows, K, H, rps, t.part);
  CUDA_LAUNCH_CHECK();
  const int64_t kh = static_cast<int64_t>(K) * H;
  dw1_reduce_kernel<<<ceil_div(kh, 256), 256, 0, s>>>(t.part, splits, kh, g_w1, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
  small_grads_kernel<<<H + 2, 256, 0, s>>>(t.dh, t.act, t.gz, t.lossr, rows, H, 1.f / rows, g_b1,
                                           g_w2, g_b2, g_loss, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
}

void dense_adam(float* p, float* m, float* v, const float* g, int64_t n, float grad_scale, float lr,
                double beta1, double beta2, float eps, float bc1, float bc2, cudaStream_t s) {
  const float omb1 = static_cast<float>(1.0 - beta1);
  const float omb2 = static_cast<float>(1.0 - beta2);
  dense_adam_kernel<<<ceil_div(n, 256), 256, 0, s>>>(p, m, v, g, n, grad_scale, lr, beta1, beta2,
                                                     omb1, omb2, eps, bc1, bc2);
  CUDA_LAUNCH_CHECK();
}

void scale_add(float* y, const float* x, int64_t n, float a, cudaStream_t s) {
  scale_add_kernel<<<ceil_div(n, 256), 256, 0, s>>>(y, x, n, a);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
