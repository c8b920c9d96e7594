// Launchers for the worker-op kernels (embed.cu) and the DeepFM-lite tower
// (tower.cu).
#pragma once

#include "ops.h"

namespace sfb {

// ---------------- embed.cu — worker ops ----------------
// gather_cache: G[own_k[j]] = emb[own_slot[j]] for j < n_own
// n_own bounds the grid; d_n_own (nullable) is the device count the kernels honour
// dG_zero (nullable, d % 4 == 0): also zero the gradient rows G's rows map to
void gather_cache(const uint32_t* own_k, const uint32_t* own_slot, int32_t n_own,
                  const int32_t* d_n_own, const float* emb, int d, float* G, float* dG_zero,
                  cudaStream_t s, float* B_zero = nullptr);
// gather_instances + FM sums: X[i] = G[vid[i]] for the lane's rows; s[r] = sum_f X[r,f];
// sqp[r, c4] = partial sum of squares
// slot_of (nullable, d % 4 == 0): read unique k's row from G = the cache table at slot
// slot_of[k] (one worker: no separate G copy)
void gather_instances(const uint32_t* vid, int32_t rows, int F, int d, int ldx, const float* G,
                      float* X, float* fm_s, float* fm_sqp, cudaStream_t s,
                      const uint32_t* slot_of = nullptr, int g_ld = 0);  // g_ld: G row stride (0 = d)
// dG[0 : n*d) = 0 and B[0 : n) = 0 with n = *d_n (bounded by n_bound)
void zero_rows_b(const int32_t* d_n, int32_t n_bound, int d, float* dG, float* B, cudaStream_t s);
int fm_sq_parts(int d);  // columns of fm_sqp per row
// FM sums of a materialised X (standalone model op)
void fm_sums(const float* X, int32_t rows, int F, int d, int ldx, float* fm_s, float* fm_sqp,
             cudaStream_t s);
// segment_sum: dG[vid[p]] += dX_mlp[p] + scale*gz[r]*(fm_s[r] - G[vid[p]]) for the lane's
// positions p = (r, f) (vector red.global.add.v4.f32)
// Bsum != nullptr: the -scale*gz*G term is deferred: Bsum[vid[p]] += gz[r], and
// sparse_adam(..., Bsum, scale) subtracts scale * Bsum[u] * G[u] from the row's gradient
void segment_sum(const uint32_t* vid, int32_t n, int F, int d, int ldx, const float* dX,
                 const float* G, const float* fm_s, const float* gz, float scale, float* dG,
                 cudaStream_t s, float* Bsum = nullptr);
// Deterministic segment sum (config key deterministic): the lane's positions are sorted
// stably by vid, then one warp per unique sums its positions' gradients in ascending
// position order and adds the sum to dG[v] (no atomics: lanes run in stream order), so
// every run of the same inputs produces bit-identical gradients.
struct SegCsr {
  int64_t cap = 0;
  uint32_t *pos_in = nullptr, *vid_out = nullptr, *pos_out = nullptr, *starts = nullptr;
  int32_t* count = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  ScanTiles tiles;
  void init(int64_t n);
  void release();
};
void segment_sum_csr(SegCsr& cs, const uint32_t* vid, int32_t n, int F, int d, int ldx,
                     const float* dX, const float* G, const float* fm_s, const float* gz,
                     float scale, float* dG, int vid_bits, cudaStream_t s);
// dX[r, k] += scale * gz[r] * (fm_s[r, k % d] - X[r, k]) (FM part, standalone model op)
void fm_grad_add(const float* X, int32_t rows, int F, int d, int ldx, const float* fm_s,
                 const float* gz, float scale, float* dX, cudaStream_t s);
// update_sparse: lazy Adam on the lane's owned rows, per-row step count.
// The gradient of owned row j is dG[grad_idx[j]] (grad_idx == nullptr: dG[j]).
void sparse_adam(const uint32_t* grad_idx, const uint32_t* own_slot, int32_t n_own,
                 const int32_t* d_n_own, const float* dG,
                 int d, float* emb, float* mom, float* vel, int32_t* steps, const float* bc1,
                 const float* bc2, float lr, double beta1, double beta2, float eps, cudaStream_t s,
                 bool inc_steps = true,  // false: the caller bumps the per-row step counts
                 const float* Bsum = nullptr, float fm_scale = 0.f);  // deferred FM term

// Fused segment sum for the tower's dX GEMM (one worker, deferred FM term): the epilogue
// scatter-adds into dG / Bsum instead of writing dX (see tc_dx.cuh, embed.cu segment_sum).
struct DxScatter {
  const uint32_t* vid;
  const uint32_t* remap;  // nullable: the table row of position i is remap[vid[i]]
  const float* fm_s;
  const float* gz;
  float* dG;
  float* Bsum;
  int F, d;
};

// Optional callback between the tower's stages (the trainer records a phase event there).

// ---------------- tower.cu — DeepFM-lite ----------------
struct TowerBufs {
  int rows_cap = 0, K = 0, H = 0, d = 0;
  float* hpre = nullptr;   // [rows, H] pre-activation (b1 included)
  float* act = nullptr;    // [rows, H] relu
  float* dh = nullptr;     // [rows, H] d(mean loss)/d(hpre)
  float* gz = nullptr;     // [rows]    d(mean loss)/dz
  float* lossr = nullptr;  // [rows]    per-row BCE
  float* part = nullptr;   // [splits, K, H] dW1 partials
  float* sg_part = nullptr;  // [128, 2H+2] small-gradient chunk partials
  int splits = 0;
  void init(int rows_cap, int K, int H, int d);
  void release();
};
// Operand buffers of the tensor-core tower (tc_tower.cu): 3xTF32 hi/lo parts of
// W1 (both layouts) and dh (both layouts), split-K partials. Leading dims are
// padded to 16 B for TMA.
struct TowerTC {
  int rows_cap = 0, K = 0, H = 0, d = 0;
  int ldk = 0, ldh = 0, ldr = 0;  // padded K, H, rows
  int dp = 0, Kp = 0;             // fused path: padded field width, F * dp
  int s1_max = 1, s3_max = 1;     // split-K factors of GEMM1 / GEMM3
  float *w_hi = nullptr, *w_lo = nullptr;    // [K x ldh]
  float *wt_hi = nullptr, *wt_lo = nullptr;  // [H x ldk]
  float *dh_hi = nullptr, *dh_lo = nullptr;  // [rows x ldh]
  float* part1 = nullptr;  // [s1, rows, H]
  float* part3 = nullptr;  // [s3, K, H]
  void init(int rows_cap, int K, int H, int d);
  void release();
};
int tower_ldx(int K);  // row stride of X / dX (K rounded up to 4 floats)

// Forward + head + backward of one lane's rows on the tensor cores. w1_split_ready: the
// caller already holds W1's tf32 hi/lo parts in tc (the trainer's tail kernel writes them
// when it updates W1), so the per-call prep pass is skipped. X and dX
// have row stride ldx = tower_ldx(K); dX is scaled by emb_scale; dense grads go
// to grads = [dW1 | db1 | dw2 | db2 | loss_sum] (accumulated when accumulate).
void tower_forward_backward_tc(TowerBufs& t, TowerTC& tc, const float* X, int ldx,
                               const float* fm_s, const float* fm_sqp, const uint8_t* labels,
                               int32_t rows, int F, int d, const float* dense, float* logits,
                               float* dX, float emb_scale, float* grads, bool accumulate,
                               cudaStream_t s,
                               bool w1_split_ready = false, const PhaseHook& hook = {},
                               const DxScatter* scatter = nullptr,
                               const PhaseHook& after_dx = {});  // called once GEMM2 is queued
// whether the fused dX scatter (tc_dx.cuh) fits: d % 4 == 0 and its smem tables
bool dx_scatter_fits(int F, int d);
// Fused path (tc_fused.cuh): X = G[vid] is gathered straight into the GEMM
// operands and dX is scatter-added into dG (with the FM term) by the dX GEMM's
// epilogue; neither touches HBM. Writes fm_s [rows x d]. Needs d % 4 == 0, d <= 128.
bool tower_fused_supported(int d);
void tower_forward_backward_fused(TowerBufs& t, TowerTC& tc, const float* G, int64_t g_rows,
                                  const uint32_t* vid, const uint8_t* labels, int32_t rows, int F,
                                  int d, const float* dense, float* logits, float* fm_s,
                                  float emb_scale, float* dG, float* grads, bool accumulate,
                                  cudaStream_t s);
// fp32 SIMT reference tiles of the same tower (validation only; needs ldx == K)
void tower_forward_backward_simt(TowerBufs& t, const float* X, const float* fm_s,
                                 const float* fm_sqp, const uint8_t* labels, int32_t rows, int F,
                                 int d, const float* dense, float* logits, float* dX,
                                 float emb_scale, float* grads, bool accumulate, cudaStream_t s);
void dw1_reduce(const float* part, int splits, int64_t n, float* out, bool accumulate,
                cudaStream_t s);
// dW1's split-K sum and the small-gradient final pass over t.sg_part in one launch
void tower_reduce(const float* part3, int splits, int64_t kh, float* g_w1, TowerBufs& t,
                  int chunks, int rows, int H, float* g_b1, float* g_w2, float* g_b2,
                  float* g_loss, bool accumulate, cudaStream_t s);
// the final pass alone, over `chunks` partials already in t.sg_part (the head wrote them)
void small_grads_final(TowerBufs& t, int chunks, int rows, int H, float* g_b1, float* g_w2,
                       float* g_b2, float* g_loss, bool accumulate, cudaStream_t s);
void small_grads(TowerBufs& t, int rows, int H, float* g_b1, float* g_w2, float* g_b2,
                 float* g_loss, bool accumulate, cudaStream_t s);
// Adam over the dense parameter vector; bias corrections precomputed on the host in fp64.
void dense_adam(float* p, float* m, float* v, const float* g, int64_t n, float grad_scale,
                float lr, double beta1, double beta2, float eps, float bc1, float bc2,
                cudaStream_t s);
void scale_add(float* y, const float* x, int64_t n, float a, cudaStream_t s);

}  // namespace sfb
