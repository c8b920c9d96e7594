// Tensor-core path of the DeepFM-lite tower (tcgen05 3xTF32, see tc_gemm.cuh).
//
//   prep   : W1 -> (hi, lo) tf32 parts in both layouts (W1 [K x H] for dX,
//            W1^T [H x K] for the forward), once per step
//   GEMM1  : hpre_part[z] = X W1          A = X (K-major, split into TMEM), split-K z
//   head   : hpre = b1 + sum_z part; z, p, BCE, gz; dh (+ its hi/lo parts in
//            row-major and transposed layouts)
//   GEMM2  : dX = s * dh W1^T    persistent tile walker, TMA-store epilogue (tc_dx.cuh)
//   GEMM3  : dW1_part[z] = X^T dh         A = X^T (split into TMEM), split-K z
//   reduce : dW1 = sum_z part (fixed order); db1, dw2, db2, loss (fixed order)
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.h"
#include "tc_fused.cuh"
#include "tc_gemm.cuh"
#include "tc_ts.cuh"
#include "tc_dx.cuh"

namespace sfb {

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) fail(kCuda, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D fp32 tensor [outer][inner] with row stride ld (elements). SWIZZLE_128B
// boxes for K-major operands; SWIZZLE_128B_ATOM_32B (32 B chunks) for the
// MN-major tf32 operand (tcgen05's SWIZZLE_128B_BASE32B smem layout).
CUtensorMap tmap(const float* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_in,
                 uint32_t box_out,
                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * sizeof(float)};
  const cuuint32_t box[2] = {box_in, box_out};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base),
                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

__device__ __forceinline__ float rna(float x) { return tc::tf32_rna(x); }

// W1 [K x H] packed -> hi/lo of W1 [K x ldh] and W1^T [H x ldk]
__global__ void prep_w1_kernel(const float* __restrict__ w1, int K, int H, int ldh, int ldk,
                               float* __restrict__ w_hi, float* __restrict__ w_lo,
                               float* __restrict__ wt_hi, float* __restrict__ wt_lo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(K) * H) return;
  const int k = static_cast<int>(i / H), j = static_cast<int>(i % H);
  const float v = w1[i];
  const float h = rna(v), l = rna(v - h);
  w_hi[static_cast<int64_t>(k) * ldh + j] = h;
  w_lo[static_cast<int64_t>(k) * ldh + j] = l;
  wt_hi[static_cast<int64_t>(j) * ldk + k] = h;
  wt_lo[static_cast<int64_t>(j) * ldk + k] = l;
}

// Warp per row: sums the split-K partials of GEMM1, then the DeepFM-lite head. sg_part
// (nullable): each block's 8 rows reduced to (db1 | dw2 | db2 | loss) partials, [block][2H+2]
// (the first pass of small_grads, fused; H <= 64)
__global__ void head_tc_kernel(int rows, int H, int d, int sq_parts, const float* __restrict__ part,
                               int splits, long long split_stride, const float* __restrict__ b1,
                               const float* __restrict__ w2, const float* __restrict__ b2p,
                               const float* __restrict__ fm_s, const float* __restrict__ fm_sqp,
                               const uint8_t* __restrict__ labels, float inv_rows,
                               float* __restrict__ logits, float* __restrict__ act,
                               float* __restrict__ dh, float* __restrict__ gz,
                               float* __restrict__ lossr, float* __restrict__ dh_hi,
                               float* __restrict__ dh_lo, int ldh, float* __restrict__ sg_part) {
  __shared__ float sg[8][2 * 64 + 2];
  pdl_wait();  // GEMM1's partials
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (r >= rows) {  // (rows % 8 != 0) this warp's row contributes nothing
    if (sg_part) {
      for (int j = lane; j < 2 * H + 2; j += 32) sg[wib][j] = 0.f;
      __syncthreads();
      for (int j = threadIdx.x; j < 2 * H + 2; j += blockDim.x) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += sg[w][j];
        sg_part[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = t;  // output-major
      }
    }
    return;
  }
  float mlp = 0.f, ss = 0.f, sq = 0.f;
  float hreg[2] = {0.f, 0.f};
  // H = 64 (the DeepFM-lite width), <= 4 split-K partials, d <= 128: every load of the row is
  // issued up front (the generic loops chain one L2 round trip per load); same sums, same order
  const bool fast = H == 64 && splits <= 4 && d <= 128 && sq_parts <= 32;
  if (fast) {
    float pv[4][2];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const float* pz = part + z * split_stride + static_cast<long long>(r) * 64;
      pv[z][0] = z < splits ? __ldg(pz + lane) : 0.f;
      pv[z][1] = z < splits ? __ldg(pz + lane + 32) : 0.f;
    }
    float fs[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = lane + 32 * q;
      fs[q] = c < d ? __ldg(fm_s + static_cast<int64_t>(r) * d + c) : 0.f;
    }
    sq = lane < sq_parts ? __ldg(fm_sqp + static_cast<int64_t>(r) * sq_parts + lane) : 0.f;
    float h0 = __ldg(b1 + lane), h1 = __ldg(b1 + lane + 32);
#pragma unroll
    for (int z = 0; z < 4; ++z)
      if (z < splits) {
        h0 += pv[z][0];
        h1 += pv[z][1];
      }
    hreg[0] = h0;
    hreg[1] = h1;
    mlp = fmaxf(h0, 0.f) * __ldg(w2 + lane);
    mlp += fmaxf(h1, 0.f) * __ldg(w2 + lane + 32);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (lane + 32 * q < d) ss += fs[q] * fs[q];
  } else {
    for (int j = lane; j < H; j += 32) {
      float h = b1[j];
      for (int z = 0; z < splits; ++z) h += part[z * split_stride + static_cast<long long>(r) * H + j];
      act[static_cast<int64_t>(r) * H + j] = h;  // pre-activation for now
      mlp += fmaxf(h, 0.f) * w2[j];
    }
    for (int c = lane; c < d; c += 32) {
      const float v = fm_s[static_cast<int64_t>(r) * d + c];
      ss += v * v;
    }
    for (int c = lane; c < sq_parts; c += 32) sq += fm_sqp[static_cast<int64_t>(r) * sq_parts + c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mlp += __shfl_xor_sync(0xFFFFFFFFu, mlp, o);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
    sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
  }
  const float z = 0.5f * (ss - sq) + (mlp + __ldg(b2p));
  const float p = 1.f / (1.f + expf(-z));
  const float y = labels[r] ? 1.f : 0.f;
  constexpr float kClamp = 1e-7f;
  const bool clamped = (p < kClamp) || (p > 1.f - kClamp);
  const float pc = fminf(fmaxf(p, kClamp), 1.f - kClamp);
  const float g = clamped ? 0.f : (p - y) * inv_rows;
  for (int j = lane; j < H; j += 32) {
    const int64_t o = static_cast<int64_t>(r) * H + j;
    const float hv = fast ? hreg[j >> 5] : act[o];
    act[o] = fmaxf(hv, 0.f);
    const float dv = hv > 0.f ? g * w2[j] : 0.f;
    dh[o] = dv;
    const float h = rna(dv), l = rna(dv - h);
    dh_hi[static_cast<int64_t>(r) * ldh + j] = h;
    dh_lo[static_cast<int64_t>(r) * ldh + j] = l;
    if (sg_part) {
      sg[wib][j] = dv;                    // db1
      sg[wib][H + j] = g * fmaxf(hv, 0.f);  // dw2
    }
  }
  const float lr_ = -(y * logf(pc) + (1.f - y) * log1pf(-pc));
  if (lane == 0) {
    logits[r] = z;
    gz[r] = g;
    lossr[r] = lr_;
    if (sg_part) {
      sg[wib][2 * H] = g;
      sg[wib][2 * H + 1] = lr_;
    }
  }
  if (sg_part) {
    __syncthreads();
    for (int j = threadIdx.x; j < 2 * H + 2; j += blockDim.x) {  // rows in order
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t += sg[w][j];
      sg_part[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = t;  // output-major
    }
  }
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int BN, bool A_MN, bool SPLIT_A, int EPI, bool B_MN = false, int MAXST = 6>
void launch_gemm(dim3 grid, const CUtensorMap& a, const CUtensorMap& alo, const CUtensorMap& bhi,
                 const CUtensorMap& blo, const tc::Params& p, cudaStream_t s) {
  auto kern = tc::gemm_tf32x3_kernel<BN, A_MN, SPLIT_A, EPI, B_MN, MAXST>;
  constexpr int smem = tc::Layout<BN, MAXST>::SMEM;
  static bool configured = false;  // per instantiation
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, 192, smem, s>>>(a, alo, bhi, blo, p);
  CUDA_LAUNCH_CHECK();
}

// SFCTR_CTA_TRACE=n: launch n of a call site records every CTA's [start, end] globaltimer
// (ns); launch n + 20 prints the spread (first start .. last start, first end .. last end),
// synchronising once (diagnostics: how late persistent CTAs start next to the manager stage)
struct CtaTrace {
  const char* name;
  int launches = 0;
  unsigned long long* buf = nullptr;
  int grid = 0;
  unsigned long long* arm(int g) {
    static const int at = [] {
      const char* e = std::getenv("SFCTR_CTA_TRACE");
      return e ? atoi(e) : -1;
    }();
    const int i = launches++;
    if (at < 0) return nullptr;
    if (i == 0) CUDA_CHECK(cudaMalloc(&buf, sizeof(unsigned long long) * 2 * 1024));
    if (i == at) {
      grid = g;
      return buf;
    }
    if (i == at + 20 && grid) {
      std::vector<unsigned long long> h(2 * grid);
      CUDA_CHECK(cudaDeviceSynchronize());  // the host runs steps ahead of the device
      CUDA_CHECK(cudaMemcpy(h.data(), buf, sizeof(unsigned long long) * 2 * grid,
                            cudaMemcpyDeviceToHost));
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
      for (int c = 0; c < grid; ++c) {
        s0 = std::min(s0, h[2 * c]);
        s1 = std::max(s1, h[2 * c]);
        e0 = std::min(e0, h[2 * c + 1]);
        e1 = std::max(e1, h[2 * c + 1]);
      }
      fprintf(stderr, "cta trace %s grid %d: start spread %.2f us, end spread %.2f us, span %.2f us\n",
              name, grid, (s1 - s0) * 1e-3, (e1 - e0) * 1e-3, (e1 - s0) * 1e-3);
      std::vector<double> st(grid);
      for (int c = 0; c < grid; ++c) st[c] = (h[2 * c] - s0) * 1e-3;
      std::vector<double> so = st;
      std::sort(so.begin(), so.end());
      fprintf(stderr, "  start pct (us) p10 %.2f p50 %.2f p75 %.2f p90 %.2f p95 %.2f max %.2f; late (>5us) CTAs:",
              so[grid / 10], so[grid / 2], so[3 * grid / 4], so[9 * grid / 10], so[19 * grid / 20],
              so[grid - 1]);
      for (int c = 0; c < grid; ++c)
        if (st[c] > 5) fprintf(stderr, " %d(%.1f,dur %.1f)", c, st[c], (h[2 * c + 1] - h[2 * c]) * 1e-3);
      fprintf(stderr, "\n");
    }
    return nullptr;
  }
};

template <bool A_MN, bool B_MN>
void launch_ts_gemm(dim3 grid, const CUtensorMap& a, const CUtensorMap& bhi,
                    const CUtensorMap& blo, const tc::Params& p, cudaStream_t s) {
  auto kern = tc::gemm_ts_kernel<A_MN, B_MN>;
  constexpr int smem = tc::TsLayout::SMEM;
  static bool configured = false;  // per instantiation
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  static const int dbg = [] {  // experiment switch: SFCTR_TS_DBG (tc_ts.cuh p.dbg bits)
    const char* e = std::getenv("SFCTR_TS_DBG");
    return e ? atoi(e) : 0;
  }();
  tc::Params q = p;
  q.dbg = dbg;
  // SFCTR_TS_TRACE=n: the n-th launch of this instantiation records CTA 0's per-k-block
  // clock64 stamps and prints them (diagnostics; synchronises the stream)
  static const int trace_at = [] {
    const char* e = std::getenv("SFCTR_TS_TRACE");
    return e ? atoi(e) : -1;
  }();
  static int launches = 0;
  long long* tr = nullptr;
  if (launches++ == trace_at) {
    CUDA_CHECK(cudaMalloc(&tr, sizeof(long long) * 320));
    CUDA_CHECK(cudaMemsetAsync(tr, 0, sizeof(long long) * 320, s));
    q.trace = tr;
  }
  const int items = static_cast<int>(grid.x * grid.y * grid.z);
  static CtaTrace ct{A_MN ? "gemm3" : "gemm1"};
  q.cta_trace = ct.arm(items);
  launch_pdl(kern, grid, dim3(tc::kTsThreads), smem, s, a, bhi, blo, q);
  CUDA_LAUNCH_CHECK();
  if (tr) {
    long long h[320];
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(tr);
    const long long t0 = h[0];
    fprintf(stderr, "ts trace A_MN=%d (clk rel. to the first A issue): i a_issue split_start split_done mma_bfull mma_tready\n",
            A_MN ? 1 : 0);
    for (int i = 0; i < 64; ++i)
      fprintf(stderr, "%2d %8lld %8lld %8lld %8lld %8lld\n", i, h[i] ? h[i] - t0 : -1,
              h[64 + i] ? h[64 + i] - t0 : -1, h[128 + i] ? h[128 + i] - t0 : -1,
              h[192 + i] ? h[192 + i] - t0 : -1, h[256 + i] ? h[256 + i] - t0 : -1);
  }
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// GEMM2 as a persistent tile walker (tc_dx.cuh); needs H <= 64. With `sc`, the segment
// sum is fused into the epilogue (dX is never written).
void launch_dx_gemm(const TowerTC& tc_, const float* dh_hi, const float* dh_lo, int rows, int K,
                    int H, float* dX, int ldx, float scale, const DxScatter* sc, cudaStream_t s) {
  const CUtensorMap ah = tmap(dh_hi, H, rows, tc_.ldh, 32, 128);
  const CUtensorMap al = tmap(dh_lo, H, rows, tc_.ldh, 32, 128);
  const CUtensorMap bh = tmap(tc_.w_hi, H, K, tc_.ldh, 32, 64);
  const CUtensorMap bl = tmap(tc_.w_lo, H, K, tc_.ldh, 32, 64);
  tc::DxParams p{};
  p.M = rows;
  p.N = K;
  p.n_tiles = (K + 63) / 64;
  p.tiles = ((rows + 127) / 128) * p.n_tiles;
  p.scale = scale;
  static const int dx_grid = [] {  // experiment switch: SFCTR_DX_GRID (CTAs of GEMM2)
    const char* e = std::getenv("SFCTR_DX_GRID");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const int grid = std::min(p.tiles, dx_grid ? dx_grid : sm_count());
  if (sc) {
    p.a_hi = dh_hi;
    p.a_lo = dh_lo;
    p.lda = tc_.ldh;
    p.H = H;
    p.vid = sc->vid;
    p.remap = sc->remap;
    p.fm_s = sc->fm_s;
    p.gz = sc->gz;
    p.dG = sc->dG;
    p.Bsum = sc->Bsum;
    p.F = sc->F;
    p.d = sc->d;
    static const int dx_exp = [] {
      const char* e = std::getenv("SFCTR_DX_EXP");
      return e ? atoi(e) : 0;
    }();
    p.exp = dx_exp;
    // SFCTR_DX_EPI=0|1 (tc_dx.cuh DxParams::epi). 0 (default): the value-tile epilogue; 1,
    // the register transpose, measured level on the step (+1 % e2e, within noise on value)
    // but 2-3 us slower as a kernel alone
    static const int dx_epi = [] {
      const char* e = std::getenv("SFCTR_DX_EPI");
      return e ? atoi(e) : 0;
    }();
    p.epi = dx_epi;
    auto kern = tc::gemm_dx_persistent_kernel<true>;
    const int smem = 1024 + tc::DxLayout::B_STAGES * tc::DxLayout::B_STAGE +  // (A in TMEM)
                     ((tc::dx_scatter_bytes(p.F, p.d) + 15) & ~15) + 256;
    static int configured = 0;
    if (smem > configured) {
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured = smem;
    }
    static CtaTrace ct{"gemm2"};
    p.cta_trace = ct.arm(grid);
    // SFCTR_DX_TRACE=n: launch n records CTA 0's per-tile clock64 stamps and prints them
    static const int dx_trace_at = [] {
      const char* e = std::getenv("SFCTR_DX_TRACE");
      return e ? atoi(e) : -1;
    }();
    static int dx_launches = 0;
    long long* trbuf = nullptr;
    if (dx_launches++ == dx_trace_at) {
      CUDA_CHECK(cudaMalloc(&trbuf, sizeof(long long) * 192));
      CUDA_CHECK(cudaMemsetAsync(trbuf, 0, sizeof(long long) * 192, s));
      p.trace = trbuf;
    }
    launch_pdl(kern, dim3(grid), dim3(tc::dx_threads<true>()), smem, s, ah, al, bh, bl, bh, p);
    CUDA_LAUNCH_CHECK();
    if (trbuf) {
      long long h[192];
      CUDA_CHECK(cudaStreamSynchronize(s));
      CUDA_CHECK(cudaMemcpy(h, trbuf, sizeof(h), cudaMemcpyDeviceToHost));
      cudaFree(trbuf);
      const long long t0 = h[0];
      fprintf(stderr, "dx trace (clk rel. to the first MMA acc wait): i mma_acc_ok mma_b_ok epi_acc_full epi_drained epi_scattered epi_done\n");
      for (int i = 0; i < 32; ++i)
        fprintf(stderr, "%2d %8lld %8lld %8lld %8lld %8lld %8lld\n", i, h[i] ? h[i] - t0 : -1,
                h[32 + i] ? h[32 + i] - t0 : -1, h[64 + i] ? h[64 + i] - t0 : -1,
                h[96 + i] ? h[96 + i] - t0 : -1, h[128 + i] ? h[128 + i] - t0 : -1,
                h[160 + i] ? h[160 + i] - t0 : -1);
    }
    return;
  }
  const CUtensorMap out = tmap(dX, K, rows, ldx, 32, 128);
  auto kern = tc::gemm_dx_persistent_kernel<false>;
  constexpr int smem = tc::DxLayout::SMEM;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  launch_pdl(kern, dim3(grid), dim3(192), smem, s, ah, al, bh, bl, out, p);
  CUDA_LAUNCH_CHECK();
}

// split-K factor so that tiles * splits ~ one wave of 148 SMs, no empty split
void split_k(int tiles, int nkb, int* splits, int* kps) {
  int s = std::max(1, std::min(nkb, num_sms() / std::max(1, tiles)));
  *kps = (nkb + s - 1) / s;
  *splits = (nkb + *kps - 1) / *kps;
}

// ---------------- fused path (tc_fused.cuh) ----------------

// W1 [K x H] packed -> hi/lo of the padded-field layouts: W1p [Kp x ldh], W1p^T [H x Kp]
__global__ void prep_w1_padded_kernel(const float* __restrict__ w1, int F, int d, int dp, int H,
                                      int ldh, int Kp, float* __restrict__ w_hi,
                                      float* __restrict__ w_lo, float* __restrict__ wt_hi,
                                      float* __restrict__ wt_lo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(F) * d * H) return;
  const int k = static_cast<int>(i / H), j = static_cast<int>(i % H);
  const int kp = (k / d) * dp + (k % d);
  const float v = w1[i];
  const float h = rna(v), l = rna(v - h);
  w_hi[static_cast<int64_t>(kp) * ldh + j] = h;
  w_lo[static_cast<int64_t>(kp) * ldh + j] = l;
  wt_hi[static_cast<int64_t>(j) * Kp + kp] = h;
  wt_lo[static_cast<int64_t>(j) * Kp + kp] = l;
}

// dW1 [K x H] (packed) = sum_z part[z][kp(k)][:] in a fixed order (+= when accumulating)
__global__ void dw1_reduce_padded_kernel(const float* __restrict__ part, int splits, int F, int d,
                                         int dp, int H, float* __restrict__ out, int accumulate) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t n = static_cast<int64_t>(F) * d * H;
  if (i >= n) return;
  const int k = static_cast<int>(i / H), j = static_cast<int>(i % H);
  const int64_t kp = (k / d) * dp + (k % d);
  const int64_t ps = static_cast<int64_t>(F) * dp * H;
  float s = 0.f;
  for (int q = 0; q < splits; ++q) s += part[q * ps + kp * H + j];
  out[i] = accumulate ? out[i] + s : s;
}

// Warp per row: sums the split-K partials of the gathered forward GEMM, gathers
// the row's F embeddings through vid for the FM term (sum and sum of squares,
// fm_s written for the scatter epilogue), then the DeepFM-lite head as in head_tc.
__global__ void head_fused_kernel(int rows, int F, int d, int H, const float* __restrict__ part,
                                  int splits, long long split_stride,
                                  const uint32_t* __restrict__ vid, const float* __restrict__ G,
                                  const float* __restrict__ b1, const float* __restrict__ w2,
                                  const float* __restrict__ b2p,
                                  const uint8_t* __restrict__ labels, float inv_rows,
                                  float* __restrict__ logits, float* __restrict__ act,
                                  float* __restrict__ dh, float* __restrict__ gz,
                                  float* __restrict__ lossr, float* __restrict__ fm_s,
                                  float* __restrict__ dh_hi, float* __restrict__ dh_lo, int ldh) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int d4 = d >> 2;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  float sq = 0.f;
  const uint32_t* vr = vid + static_cast<int64_t>(r) * F;
  // lane f < F fetches vid[r, f] once; rows then go 4 at a time (d <= 128: lane c
  // owns the fixed 16 B column c of every row), all 4 gathers in flight
  const uint32_t my_v = lane < F ? __ldg(vr + lane) : 0u;
  for (int f0 = 0; f0 < F; f0 += 4) {
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = f0 + u;
      const uint32_t v = f < 32 ? __shfl_sync(0xFFFFFFFFu, my_v, f & 31)
                                : (f < F ? __ldg(vr + f) : 0u);
      a[u] = (f < F && lane < d4)
                 ? __ldg(reinterpret_cast<const float4*>(G + static_cast<int64_t>(v) * d) + lane)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s.x += a[u].x; s.y += a[u].y; s.z += a[u].z; s.w += a[u].w;
      sq += a[u].x * a[u].x + a[u].y * a[u].y + a[u].z * a[u].z + a[u].w * a[u].w;
    }
  }
  float ss = s.x * s.x + s.y * s.y + s.z * s.z + s.w * s.w;
  if (lane < d4) reinterpret_cast<float4*>(fm_s + static_cast<int64_t>(r) * d)[lane] = s;
  float mlp = 0.f;
  for (int j = lane; j < H; j += 32) {
    float h = b1[j];
    for (int z = 0; z < splits; ++z) h += part[z * split_stride + static_cast<long long>(r) * H + j];
    act[static_cast<int64_t>(r) * H + j] = h;
    mlp += fmaxf(h, 0.f) * w2[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mlp += __shfl_xor_sync(0xFFFFFFFFu, mlp, o);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
    sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
  }
  const float z = 0.5f * (ss - sq) + (mlp + __ldg(b2p));
  const float p = 1.f / (1.f + expf(-z));
  const float y = labels[r] ? 1.f : 0.f;
  constexpr float kClamp = 1e-7f;
  const bool clamped = (p < kClamp) || (p > 1.f - kClamp);
  const float pc = fminf(fmaxf(p, kClamp), 1.f - kClamp);
  const float g = clamped ? 0.f : (p - y) * inv_rows;
  for (int j = lane; j < H; j += 32) {
    const int64_t o = static_cast<int64_t>(r) * H + j;
    const float hv = act[o];
    act[o] = fmaxf(hv, 0.f);
    const float dv = hv > 0.f ? g * w2[j] : 0.f;
    dh[o] = dv;
    const float h = rna(dv), l = rna(dv - h);
    dh_hi[static_cast<int64_t>(r) * ldh + j] = h;
    dh_lo[static_cast<int64_t>(r) * ldh + j] = l;
  }
  if (lane == 0) {
    logits[r] = z;
    gz[r] = g;
    lossr[r] = -(y * logf(pc) + (1.f - y) * log1pf(-pc));
  }
}

template <int BN, bool A_MN, bool B_MN>
void launch_dec_gemm(dim3 grid, const CUtensorMap& a, const CUtensorMap& bhi,
                     const CUtensorMap& blo, const tc::Params& p, cudaStream_t s) {
  auto kern = tc::gemm_tf32x3_dec_kernel<BN, A_MN, B_MN>;
  constexpr int smem = tc::DecLayout<BN>::SMEM;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, tc::kTsThreads, smem, s>>>(a, bhi, blo, p);
  CUDA_LAUNCH_CHECK();
}

template <bool A_MN>
void launch_gather4_gemm(dim3 grid, const CUtensorMap& g, const CUtensorMap& bhi,
                         const CUtensorMap& blo, const tc::FusedParams& p, cudaStream_t s) {
  auto kern = tc::gather4_gemm_kernel<A_MN>;
  constexpr int smem = tc::Layout<64>::SMEM;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, 192, smem, s>>>(g, bhi, blo, p);
  CUDA_LAUNCH_CHECK();
}

template <bool A_MN>
void launch_gather_gemm(dim3 grid, const CUtensorMap& bhi, const CUtensorMap& blo,
                        const tc::FusedParams& p, cudaStream_t s) {
  auto kern = tc::gather_gemm_kernel<A_MN>;
  constexpr int smem = tc::Layout<64>::SMEM;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, tc::kFusedThreads, smem, s>>>(bhi, blo, p);
  CUDA_LAUNCH_CHECK();
}

template <int BN>
void launch_scatter_gemm(dim3 grid, const CUtensorMap& ah, const CUtensorMap& al,
                         const CUtensorMap& bh, const CUtensorMap& bl, const tc::FusedParams& p,
                         cudaStream_t s) {
  auto kern = tc::scatter_gemm_kernel<BN>;
  constexpr int smem = tc::Layout<BN, 2>::SMEM;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<grid, 192, smem, s>>>(ah, al, bh, bl, p);
  CUDA_LAUNCH_CHECK();
}

}  // namespace

bool dx_scatter_fits(int F, int d) {
  return d % 4 == 0 &&
         1024 + tc::DxLayout::A_BYTES + tc::DxLayout::B_STAGES * tc::DxLayout::B_STAGE +
                 ((tc::dx_scatter_bytes(F, d) + 15) & ~15) + 256 <=
             227 * 1024;
}


bool tower_fused_supported(int d) { return d % 4 == 0 && d <= 128; }

void TowerTC::init(int rc, int k, int h, int d_) {
  release();
  rows_cap = rc;
  K = k;
  H = h;
  d = d_;
  ldk = round_up(K, 4);
  ldh = round_up(H, 4);
  ldr = round_up(rc, 4);
  // padded-field layout of the fused path: field f at [f*dp, f*dp + d), dp = round_up(d, 32)
  dp = round_up(d, 32);
  Kp = (K / d) * dp;
  const int kmax = std::max(ldk, Kp);
  int kps, s_a, s_b;
  split_k(((rc + 127) / 128) * ((H + 63) / 64), (K + tc::BKE - 1) / tc::BKE, &s_a, &kps);
  split_k(((rc + 127) / 128) * ((H + 63) / 64), (Kp + tc::BKE - 1) / tc::BKE, &s_b, &kps);
  s1_max = std::max(s_a, s_b);
  const int nkb3 = (rc + tc::BKE - 1) / tc::BKE;
  split_k(((K + 127) / 128) * ((H + 63) / 64), nkb3, &s_a, &kps);
  split_k(((Kp + 127) / 128) * ((H + 63) / 64), nkb3, &s_b, &kps);
  s3_max = std::max(s_a, s_b);
  auto alloc = [](float** p, size_t n) { CUDA_CHECK(cudaMalloc(p, sizeof(float) * std::max<size_t>(n, 1))); };
  alloc(&w_hi, static_cast<size_t>(kmax) * ldh);
  alloc(&w_lo, static_cast<size_t>(kmax) * ldh);
  alloc(&wt_hi, static_cast<size_t>(H) * kmax);
  alloc(&wt_lo, static_cast<size_t>(H) * kmax);
  alloc(&dh_hi, static_cast<size_t>(rc) * ldh);
  alloc(&dh_lo, static_cast<size_t>(rc) * ldh);
  alloc(&part1, static_cast<size_t>(s1_max) * rc * H);
  alloc(&part3, static_cast<size_t>(s3_max) * kmax * H);
  // zero once: padding rows / columns of the W1 parts are never written
  for (float* p : {w_hi, w_lo})
    CUDA_CHECK(cudaMemset(p, 0, sizeof(float) * static_cast<size_t>(kmax) * ldh));
  for (float* p : {wt_hi, wt_lo})
    CUDA_CHECK(cudaMemset(p, 0, sizeof(float) * static_cast<size_t>(H) * kmax));
}

void TowerTC::release() {
  for (float* p : {w_hi, w_lo, wt_hi, wt_lo, dh_hi, dh_lo, part1, part3})
    if (p) cudaFree(p);
  w_hi = w_lo = wt_hi = wt_lo = dh_hi = dh_lo = part1 = part3 = nullptr;
}

int tower_ldx(int K) { return round_up(K, 4); }

void tower_forward_backward_tc(TowerBufs& t, TowerTC& tc_, const float* X, int ldx,
                               const float* fm_s, const float* fm_sqp, const uint8_t* labels,
                               int32_t rows, int F, int d, const float* dense, float* logits,
                               float* dX, float emb_scale, float* grads, bool accumulate,
                               cudaStream_t s, bool w1_split_ready,
                               const PhaseHook& hook,
                               const DxScatter* scatter, const PhaseHook& after_dx) {
  const int K = F * d, H = t.H;
  SFB_CHECK(rows <= t.rows_cap && rows <= tc_.rows_cap && K == tc_.K && ldx == tc_.ldk,
            "tower buffers too small");
  const float* w1 = dense;
  const float* b1 = dense + static_cast<size_t>(K) * H;
  const float* w2 = b1 + H;
  const float* b2p = w2 + H;
  float* g_w1 = grads;
  float* g_b1 = grads + static_cast<size_t>(K) * H;
  float* g_w2 = g_b1 + H;
  float* g_b2 = g_w2 + H;
  float* g_loss = g_b2 + 1;

  // W1 hi/lo in both layouts
  if (!w1_split_ready) {
    prep_w1_kernel<<<ceil_div(static_cast<int64_t>(K) * H, 256), 256, 0, s>>>(
        w1, K, H, tc_.ldh, tc_.ldk, tc_.w_hi, tc_.w_lo, tc_.wt_hi, tc_.wt_lo);
    CUDA_LAUNCH_CHECK();
  }

  // ---- GEMM1: hpre partials = X W1 (A = X K-major, B = W1^T)
  const int nkb1 = (K + tc::BKE - 1) / tc::BKE;
  const int mt = (rows + 127) / 128, nt = (H + 63) / 64;
  int s1, kps1;
  split_k(mt * nt, nkb1, &s1, &kps1);
  {
    const CUtensorMap a = tmap(X, K, rows, ldx, 32, 128);
    const CUtensorMap bh = tmap(tc_.wt_hi, K, H, tc_.ldk, 32, 64);
    const CUtensorMap bl = tmap(tc_.wt_lo, K, H, tc_.ldk, 32, 64);
    tc::Params p{};
    p.M = rows;
    p.N = H;
    p.K = K;
    p.num_k_blocks = nkb1;
    p.k_blocks_per_split = kps1;
    p.out = tc_.part1;
    p.ldo = H;
    p.split_stride = static_cast<long long>(rows) * H;
    launch_ts_gemm<false, false>(dim3(mt, nt, s1), a, bh, bl, p, s);
  }
  hook("tower_gemm1");
  // ---- head
  launch_pdl(head_tc_kernel, dim3(ceil_div(static_cast<int64_t>(rows) * 32, 256)), dim3(256), 0, s,
             rows, H, d, fm_sq_parts(d), static_cast<const float*>(tc_.part1), s1,
             static_cast<long long>(rows) * H, b1, w2, b2p, static_cast<const float*>(fm_s),
             static_cast<const float*>(fm_sqp), labels, 1.f / rows, logits, t.act, t.dh, t.gz,
             t.lossr, tc_.dh_hi, tc_.dh_lo, tc_.ldh, H <= 64 ? t.sg_part : nullptr);
  CUDA_LAUNCH_CHECK();
  hook("tower_head");
  // ---- GEMM2: dX = scale dh W1^T (A = dh hi/lo, B = W1 hi/lo, both K-major; the FM
  //      term is added by segment_sum)
  SFB_CHECK(!scatter || (H <= 64 && dx_scatter_fits(scatter->F, scatter->d)),
            "fused dX scatter needs H <= 64 and the staging tables to fit in smem");
  if (H <= 64) {
    launch_dx_gemm(tc_, tc_.dh_hi, tc_.dh_lo, rows, K, H, dX, ldx, emb_scale, scatter, s);
  } else {
    const CUtensorMap ah = tmap(tc_.dh_hi, H, rows, tc_.ldh, 32, 128);
    const CUtensorMap al = tmap(tc_.dh_lo, H, rows, tc_.ldh, 32, 128);
    const CUtensorMap bh = tmap(tc_.w_hi, H, K, tc_.ldh, 32, 64);
    const CUtensorMap bl = tmap(tc_.w_lo, H, K, tc_.ldh, 32, 64);
    tc::Params p{};
    p.M = rows;
    p.N = K;
    p.K = H;
    p.num_k_blocks = (H + tc::BKE - 1) / tc::BKE;
    p.k_blocks_per_split = p.num_k_blocks;
    p.out = dX;
    p.ldo = ldx;
    p.gz = t.gz;
    p.fm_s = fm_s;
    p.X = X;
    p.ldx = ldx;
    p.d = d;
    p.scale = emb_scale;
    // K = H is short (2 k-blocks at H = 64): a 2-stage, BN = 64 footprint (~97 KB)
    // puts two CTAs on every SM so one's epilogue overlaps the other's loads
    launch_gemm<64, false, false, tc::kEpiDx, false, 2>(dim3(mt, (K + 63) / 64, 1), ah, al, bh, bl,
                                                       p, s);
  }
  hook("tower_gemm2");
  after_dx("dx");  // the caller may start what needs only dX / the scattered gradients
  // ---- GEMM3: dW1 partials = X^T dh (A = X MN-major, B = dh hi/lo MN-major)
  const int nkb3 = (rows + tc::BKE - 1) / tc::BKE;
  const int mt3 = (K + 127) / 128;
  int s3, kps3;
  split_k(mt3 * nt, nkb3, &s3, &kps3);
  {
    const CUtensorMap a = tmap(X, K, rows, ldx, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap bh = tmap(tc_.dh_hi, H, rows, tc_.ldh, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const CUtensorMap bl = tmap(tc_.dh_lo, H, rows, tc_.ldh, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    tc::Params p{};
    p.M = K;
    p.N = H;
    p.K = rows;
    p.num_k_blocks = nkb3;
    p.k_blocks_per_split = kps3;
    p.out = tc_.part3;
    p.ldo = H;
    p.split_stride = static_cast<long long>(K) * H;
    launch_ts_gemm<true, true>(dim3(mt3, nt, s3), a, bh, bl, p, s);
  }
  hook("tower_gemm3");
  const int64_t kh = static_cast<int64_t>(K) * H;
  if (H <= 64) {  // the head left per-block partials: one launch finishes every dense gradient
    tower_reduce(tc_.part3, s3, kh, g_w1, t, ceil_div(rows, 8), rows, H, g_b1, g_w2, g_b2, g_loss,
                 accumulate, s);
  } else {
    dw1_reduce(tc_.part3, s3, kh, g_w1, accumulate, s);
    small_grads(t, rows, H, g_b1, g_w2, g_b2, g_loss, accumulate, s);
  }
}

void tower_forward_backward_fused(TowerBufs& t, TowerTC& tc_, const float* G, int64_t g_rows,
                                  const uint32_t* vid, const uint8_t* labels, int32_t rows, int F,
                                  int d, const float* dense, float* logits, float* fm_s,
                                  float emb_scale, float* dG, float* grads, bool accumulate,
                                  cudaStream_t s) {
  // A operand gathers: TMA tile::gather4 (default) or the SM producer warps
  static const bool gather_tma_ = [] {
    const char* e = std::getenv("SFCTR_GATHER_SM");
    return !(e && e[0] == '1');
  }();
  const int K = F * d, H = t.H;
  const int dp = tc_.dp, Kp = tc_.Kp;
  SFB_CHECK(tower_fused_supported(d) && rows <= tc_.rows_cap && K == tc_.K,
            "fused tower: unsupported shape");
  const float* w1 = dense;
  const float* b1 = dense + static_cast<size_t>(K) * H;
  const float* w2 = b1 + H;
  const float* b2p = w2 + H;
  float* g_w1 = grads;
  float* g_b1 = grads + static_cast<size_t>(K) * H;
  float* g_w2 = g_b1 + H;
  float* g_b2 = g_w2 + H;
  float* g_loss = g_b2 + 1;

  prep_w1_padded_kernel<<<ceil_div(static_cast<int64_t>(K) * H, 256), 256, 0, s>>>(
      w1, F, d, dp, H, tc_.ldh, Kp, tc_.w_hi, tc_.w_lo, tc_.wt_hi, tc_.wt_lo);
  CUDA_LAUNCH_CHECK();

  tc::FusedParams p{};
  p.rows = rows;
  p.F = F;
  p.d = d;
  p.dp = dp;
  p.H = H;
  p.vid = vid;
  p.G = G;
  p.fm_s = fm_s;
  p.gz = t.gz;
  p.scale = emb_scale;
  p.dG = dG;

  // ---- gathered forward GEMM: hpre partials = G[vid] W1 (split-K over fields)
  const int mt = (rows + 127) / 128, nt = (H + 63) / 64;
  const int nkb1 = Kp / tc::BKE;
  int s1, kps1;
  split_k(mt * nt, nkb1, &s1, &kps1);
  {
    const CUtensorMap bh = tmap(tc_.wt_hi, Kp, H, Kp, 32, 64);
    const CUtensorMap bl = tmap(tc_.wt_lo, Kp, H, Kp, 32, 64);
    tc::FusedParams q = p;
    q.num_k_blocks = nkb1;
    q.k_blocks_per_split = kps1;
    q.out = tc_.part1;
    q.ldo = H;
    q.split_stride = static_cast<long long>(rows) * H;
    if (gather_tma_) {
      const CUtensorMap g = tmap(G, d, std::max<int64_t>(g_rows, 1), d, 32, 1);
      launch_gather4_gemm<false>(dim3(mt, nt, s1), g, bh, bl, q, s);
    } else {
      launch_gather_gemm<false>(dim3(mt, nt, s1), bh, bl, q, s);
    }
  }
  // ---- head: DeepFM-lite with the FM sums gathered through vid
  head_fused_kernel<<<ceil_div(static_cast<int64_t>(rows) * 32, 256), 256, 0, s>>>(
      rows, F, d, H, tc_.part1, s1, static_cast<long long>(rows) * H, vid, G, b1, w2, b2p, labels,
      1.f / rows, logits, t.act, t.dh, t.gz, t.lossr, fm_s, tc_.dh_hi, tc_.dh_lo, tc_.ldh);
  CUDA_LAUNCH_CHECK();
  // ---- dX GEMM with the FM term + segment sum in the epilogue (one field per N tile)
  {
    const CUtensorMap ah = tmap(tc_.dh_hi, H, rows, tc_.ldh, 32, 128);
    const CUtensorMap al = tmap(tc_.dh_lo, H, rows, tc_.ldh, 32, 128);
    tc::FusedParams q = p;
    q.num_k_blocks = (H + tc::BKE - 1) / tc::BKE;
    const dim3 grid(mt, F);
    switch (dp) {
      case 32: {
        const CUtensorMap bh = tmap(tc_.w_hi, H, Kp, tc_.ldh, 32, 32);
        const CUtensorMap bl = tmap(tc_.w_lo, H, Kp, tc_.ldh, 32, 32);
        launch_scatter_gemm<32>(grid, ah, al, bh, bl, q, s);
        break;
      }
      case 64: {
        const CUtensorMap bh = tmap(tc_.w_hi, H, Kp, tc_.ldh, 32, 64);
        const CUtensorMap bl = tmap(tc_.w_lo, H, Kp, tc_.ldh, 32, 64);
        launch_scatter_gemm<64>(grid, ah, al, bh, bl, q, s);
        break;
      }
      case 96: {
        const CUtensorMap bh = tmap(tc_.w_hi, H, Kp, tc_.ldh, 32, 96);
        const CUtensorMap bl = tmap(tc_.w_lo, H, Kp, tc_.ldh, 32, 96);
        launch_scatter_gemm<96>(grid, ah, al, bh, bl, q, s);
        break;
      }
      default: {
        const CUtensorMap bh = tmap(tc_.w_hi, H, Kp, tc_.ldh, 32, 128);
        const CUtensorMap bl = tmap(tc_.w_lo, H, Kp, tc_.ldh, 32, 128);
        launch_scatter_gemm<128>(grid, ah, al, bh, bl, q, s);
        break;
      }
    }
  }
  // ---- gathered dW1 GEMM: partials = G[vid]^T dh (MN-major A and B), split-K over rows
  const int nkb3 = (rows + tc::BKE - 1) / tc::BKE;
  const int mt3 = (Kp + 127) / 128;
  int s3, kps3;
  split_k(mt3 * nt, nkb3, &s3, &kps3);
  {
    const CUtensorMap bh = tmap(tc_.dh_hi, H, rows, tc_.ldh, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const CUtensorMap bl = tmap(tc_.dh_lo, H, rows, tc_.ldh, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    tc::FusedParams q = p;
    q.num_k_blocks = nkb3;
    q.k_blocks_per_split = kps3;
    q.out = tc_.part3;
    q.ldo = H;
    q.split_stride = static_cast<long long>(Kp) * H;
    if (gather_tma_) {
      const CUtensorMap g = tmap(G, d, std::max<int64_t>(g_rows, 1), d, 32, 1,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      launch_gather4_gemm<true>(dim3(mt3, nt, s3), g, bh, bl, q, s);
    } else {
      launch_gather_gemm<true>(dim3(mt3, nt, s3), bh, bl, q, s);
    }
  }
  dw1_reduce_padded_kernel<<<ceil_div(static_cast<int64_t>(K) * H, 256), 256, 0, s>>>(
      tc_.part3, s3, F, d, dp, H, g_w1, accumulate ? 1 : 0);
  CUDA_LAUNCH_CHECK();
  small_grads(t, rows, H, g_b1, g_w2, g_b2, g_loss, accumulate, s);
}

}  // namespace sfb
