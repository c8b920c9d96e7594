// Launchers for the worker-op kernels (embed.cu) and the DeepFM-lite tower
// (tower.cu).
#pragma once

#include "ops.h"

namespace sfb {

// ---------------- embed.cu — worker ops ----------------
// gather_cache: G[own_k[j]] = emb[own_slot[j]] for j < n_own
void gather_cache(const uint32_t* own_k, const uint32_t* own_slot, int32_t n_own,
                  const float* emb, int d, float* G, cudaStream_t s);
// gather_instances + FM sums: X[i] = G[vid[i]] for the lane's rows; s[r] = sum_f X[r,f];
// sqp[r, c4] = partial sum of squares
void gather_instances(const uint32_t* vid, int32_t rows, int F, int d, const float* G, float* X,
                      float* fm_s, float* fm_sqp, cudaStream_t s);
int fm_sq_parts(int d);  // columns of fm_sqp per row
// FM sums of a materialised X (standalone model op)
void fm_sums(const float* X, int32_t rows, int F, int d, float* fm_s, float* fm_sqp,
             cudaStream_t s);
// segment_sum: dG[vid[i]] += dX[i] (vector red.global.add.v4.f32)
void segment_sum(const uint32_t* vid, int32_t n, int d, const float* dX, float* dG,
                 cudaStream_t s);
// update_sparse: lazy Adam on the lane's owned rows, per-row step count
void sparse_adam(const uint32_t* own_k, const uint32_t* own_slot, int32_t n_own, const float* dG,
                 int d, float* emb, float* mom, float* vel, int32_t* steps, const float* bc1,
                 const float* bc2, float lr, double beta1, double beta2, float eps, cudaStream_t s);

// ---------------- tower.cu — DeepFM-lite ----------------
struct TowerBufs {
  int rows_cap = 0, K = 0, H = 0, d = 0;
  float* hpre = nullptr;   // [rows, H] pre-activation (b1 included)
  float* act = nullptr;    // [rows, H] relu
  float* dh = nullptr;     // [rows, H] d(mean loss)/d(hpre)
  float* gz = nullptr;     // [rows]    d(mean loss)/dz
  float* lossr = nullptr;  // [rows]    per-row BCE
  float* part = nullptr;   // [splits, K, H] dW1 partials
  int splits = 0;
  void init(int rows_cap, int K, int H, int d);
  void release();
};
// forward GEMM + head + backward (dX scaled by emb_scale, dense grads accumulated into
// grads = [dW1 | db1 | dw2 | db2 | loss_sum] when accumulate, else overwritten).
void tower_forward_backward(TowerBufs& t, const float* X, const float* fm_s, const float* fm_sqp,
                            const uint8_t* labels, int32_t rows, int F, int d, const float* dense,
                            float* logits, float* dX, float emb_scale, float* grads, bool accumulate,
                            cudaStream_t s);
// Adam over the dense parameter vector; bias corrections precomputed on the host in fp64.
void dense_adam(float* p, float* m, float* v, const float* g, int64_t n, float grad_scale,
                float lr, double beta1, double beta2, float eps, float bc1, float bc2,
                cudaStream_t s);
void scale_add(float* y, const float* x, int64_t n, float a, cudaStream_t s);

}  // namespace sfb
