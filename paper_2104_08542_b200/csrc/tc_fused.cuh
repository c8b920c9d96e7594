// Fused embedding-gather / tensor-core / scatter-add kernels of the tower
// (SURVEY §8f rank 4): the minibatch embedding matrix X = G[vid] and its
// gradient dX never touch HBM.
//
//   gather GEMM (fwd, hpre = X W1)      : A tiles are gathered row by row from
//       the L2-resident table G through vid by 8 producer warps that also do
//       the 3xTF32 split, writing the canonical K-major SWIZZLE_128B layout;
//       B = W1^T (hi/lo) by TMA.
//   gather GEMM (dW1 = X^T dh)          : same producers writing the MN-major
//       SWIZZLE_128B_BASE32B layout; B = dh (hi/lo, MN-major) by TMA.
//   scatter GEMM (dX = dh W1^T)         : one N tile = one field; the epilogue
//       adds the FM term and red.global.add.v4.f32's each row straight into dG.
//
// Columns use a padded field layout: field f occupies [f*dp, f*dp + d) of
// K_pad = F*dp with dp = round_up(d, 32), so every 32-wide K block (and every
// 32-wide MN atom) lies inside one field; padded W1 rows are zero.
#pragma once

#include "tc_gemm.cuh"

namespace sfb {
namespace tc {

struct FusedParams {
  int rows;            // minibatch rows (M of the forward / scatter GEMMs)
  int F, d, dp;        // fields, embedding dim, padded field width
  int H;               // hidden
  int num_k_blocks;    // gather GEMMs: k-blocks of the reduction
  int k_blocks_per_split;
  const uint32_t* vid;  // [rows x F] rows of G
  const float* G;       // [* x d] embedding table (L2-resident)
  float* out;           // kEpiStore partials [z][M][ldo]
  int ldo;
  long long split_stride;
  // scatter epilogue
  const float* fm_s;   // [rows x d]
  const float* gz;     // [rows]
  float scale;         // 1/W
  float* dG;           // [* x d]
};

constexpr int kGatherWarps = 8;  // producers of the gathered A operand
constexpr int kFusedThreads = 64 + 32 * kGatherWarps;

// K-major SW128 byte offset of (row, 16 B chunk) in a 128-row x 128 B tile
__device__ __forceinline__ uint32_t kmajor_off(int row, int chunk) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4);
}
// MN-major SWIZZLE_128B_BASE32B byte offset of (m in 0..127, k-row kk in 0..31)
// for a float4 starting at m (m % 4 == 0): 4 KB per 32-wide m atom, 128 B per
// k-row, 32 B chunks XOR-swizzled by kk % 4.
__device__ __forceinline__ uint32_t mnmajor_off(int m, int kk) {
  const int a = m >> 5, e = m & 31;
  return a * 4096 + kk * 128 + ((((e >> 3) ^ (kk & 3))) << 5) + ((e & 7) << 2);
}

__device__ __forceinline__ float4 split_hi(float4 v, float4& lo) {
  float4 h;
  h.x = tf32_rna(v.x); lo.x = tf32_rna(v.x - h.x);
  h.y = tf32_rna(v.y); lo.y = tf32_rna(v.y - h.y);
  h.z = tf32_rna(v.z); lo.z = tf32_rna(v.z - h.z);
  h.w = tf32_rna(v.w); lo.w = tf32_rna(v.w - h.w);
  return h;
}

// Gathered 16-float segment: columns [c0, c0+16) of G row `v` (zeros past d or for
// an invalid row). d % 4 == 0, so a float4 is either fully valid or fully padding.
__device__ __forceinline__ void load_seg16(const float* __restrict__ G, int d, bool valid,
                                           uint32_t v, int c0, float4 (&x)[4]) {
  const float4* src = reinterpret_cast<const float4*>(G + static_cast<int64_t>(v) * d);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + 4 * q;
    x[q] = (valid && c < d) ? __ldg(src + (c >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// A_MN = false: forward GEMM (rows x K_pad) . (K_pad x H); A_MN = true: dW1 GEMM
// (K_pad x rows) . (rows x H). BN = 64 (H tile).
template <bool A_MN>
__global__ void __launch_bounds__(kFusedThreads, 1)
    gather_gemm_kernel(const __grid_constant__ CUtensorMap tmBhi,
                       const __grid_constant__ CUtensorMap tmBlo, const FusedParams p) {
  constexpr int BN = 64;
  using L = Layout<BN>;
  constexpr int ST = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint64_t* fullB = reinterpret_cast<uint64_t*>(smem + ST * L::STAGE_BYTES);
  uint64_t* readyA = fullB + ST;
  uint64_t* empty = readyA + ST;
  uint64_t* tmem_full = empty + ST;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_hi = [&](int s) { return smem + s * L::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * L::STAGE_BYTES + A_BYTES; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES + L::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.k_blocks_per_split;
  const int kb1 = min(p.num_k_blocks, kb0 + p.k_blocks_per_split);
  const int nkb = kb1 - kb0;
  const int M = A_MN ? p.F * p.dp : p.rows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(fullB + s, 1);
      mbar_init(readyA + s, 32 * kGatherWarps);
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer of B
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(empty + s, ((i / ST) & 1) ^ 1);
        mbar_expect_tx(fullB + s, 2 * L::B_BYTES);
        const int kc = (kb0 + i) * BKE;
        if constexpr (A_MN) {  // B = dh, MN-major: two 32-column atoms
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            tma_load_2d(&tmBhi, fullB + s, b_hi(s) + b * 4096, n0 + b * 32, kc);
            tma_load_2d(&tmBlo, fullB + s, b_lo(s) + b * 4096, n0 + b * 32, kc);
          }
        } else {  // B = W1^T, K-major
          tma_load_2d(&tmBhi, fullB + s, b_hi(s), kc, n0);
          tma_load_2d(&tmBlo, fullB + s, b_lo(s), kc, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN ? 1 : 0, A_MN ? 1 : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        mbar_wait(readyA + s, ph);
        mbar_wait(fullB + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t ah, al, bh, bl;
          if constexpr (A_MN) {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 1024, 4096, 512, 1);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 1024, 4096, 512, 1);
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 1024, 4096, 512, 1);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 1024, 4096, 512, 1);
          } else {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 32, 16, 1024);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 32, 16, 1024);
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 32, 16, 1024);
          }
          mma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, ah, bl, idesc, 1u);
          mma_tf32(tmem, al, bh, idesc, 1u);
        }
        mma_commit(empty + s);
      }
      mma_commit(tmem_full);
    }
  } else {
    // ---------------- gather + split producers (8 warps), then epilogue (warps 2..5)
    const int t = threadIdx.x - 64;  // 0..255
    // thread geometry. K-major (forward): tile row t%128, 16 of the block's 32
    // columns (half t/128). MN-major (dW1): k-row t/8 (a batch row), 16 m-columns
    // of atom (t%8)/2 (half t%2).
    const int g_rr = t & 127, g_half_k = t >> 7;
    const int g_kk = t >> 3, g_a = (t & 7) >> 1, g_half_m = t & 1;
    auto fetch = [&](int i, float4 (&x)[4]) {
      const int kb = kb0 + i;
      int r, f, c0;
      if constexpr (!A_MN) {
        r = m0 + g_rr;
        const int kcol = kb * BKE;  // padded column
        f = kcol / p.dp;
        c0 = kcol - f * p.dp + 16 * g_half_k;
      } else {
        r = kb * BKE + g_kk;
        const int mcol = m0 + g_a * 32 + 16 * g_half_m;  // padded column
        f = mcol / p.dp;
        c0 = mcol - f * p.dp;
      }
      const bool valid = r < p.rows && f < p.F;
      const uint32_t v = valid ? __ldg(p.vid + static_cast<int64_t>(r) * p.F + f) : 0u;
      load_seg16(p.G, p.d, valid, v, c0, x);
    };
    float4 xa[4], xb[4];
    if (nkb > 0) fetch(0, xa);
    for (int i = 0; i < nkb; ++i) {
      if (i + 1 < nkb) fetch(i + 1, xb);  // next block's gathers in flight during this one
      const int s = i % ST;
      mbar_wait(empty + s, ((i / ST) & 1) ^ 1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 lo;
        const float4 h = split_hi(xa[q], lo);
        const uint32_t off = A_MN ? mnmajor_off(g_a * 32 + 16 * g_half_m + 4 * q, g_kk)
                                  : kmajor_off(g_rr, 4 * g_half_k + q);
        *reinterpret_cast<float4*>(a_hi(s) + off) = h;
        *reinterpret_cast<float4*>(a_lo(s) + off) = lo;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(readyA + s);
#pragma unroll
      for (int q = 0; q < 4; ++q) xa[q] = xb[q];
    }
    if (warp < 6) {  // ---------------- epilogue (TMEM lane quarter = warp % 4)
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int q = warp & 3;
      const int row = q * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
      float* tile = reinterpret_cast<float*>(smem);  // ring is free: all MMAs completed
      constexpr int TS = BN + 1;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 8) {
        float v[8];
        tmem_ld8(trow + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) tile[row * TS + c0 + j] = v[j];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int w2 = warp - 2;
      if (nkb > 0)
        for (int rr = w2; rr < BM; rr += 4) {
          const int m = m0 + rr;
          if (m >= M) break;
          float* o = p.out + blockIdx.z * p.split_stride + static_cast<long long>(m) * p.ldo;
#pragma unroll
          for (int c = lane; c < BN; c += 32)
            if (n0 + c < p.H) o[n0 + c] = tile[rr * TS + c];
        }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(L::TMEM_COLS));
  }
}

// dX = dh W1^T for one field per N tile (BN = dp <= 128, padded W1 rows are
// zero), with the FM gradient and the segment sum fused into the epilogue:
//   dG[vid[r,f]] += scale * (acc + gz[r] * (S_r - G[vid[r,f]]))
template <int BN>
__global__ void __launch_bounds__(192, 1)
    scatter_gemm_kernel(const __grid_constant__ CUtensorMap tmAhi,
                        const __grid_constant__ CUtensorMap tmAlo,
                        const __grid_constant__ CUtensorMap tmBhi,
                        const __grid_constant__ CUtensorMap tmBlo, const FusedParams p) {
  using L = Layout<BN, 2>;
  constexpr int ST = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * L::STAGE_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tmem_full = empty + ST;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_hi = [&](int s) { return smem + s * L::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * L::STAGE_BYTES + A_BYTES; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES + L::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int f = blockIdx.y;  // field
  const int n0 = f * p.dp;
  const int nkb = p.num_k_blocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(empty + s, ((i / ST) & 1) ^ 1);
        mbar_expect_tx(full + s, 2 * A_BYTES + 2 * L::B_BYTES);
        const int kc = i * BKE;
        tma_load_2d(&tmAhi, full + s, a_hi(s), kc, m0);
        tma_load_2d(&tmAlo, full + s, a_lo(s), kc, m0);
        tma_load_2d(&tmBhi, full + s, b_hi(s), kc, n0);
        tma_load_2d(&tmBlo, full + s, b_lo(s), kc, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(BM, BN, 0, 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(full + s, (i / ST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          const uint64_t ah = smem_desc(smem_u32(a_hi(s)) + kk * 32, 16, 1024);
          const uint64_t al = smem_desc(smem_u32(a_lo(s)) + kk * 32, 16, 1024);
          const uint64_t bh = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
          const uint64_t bl = smem_desc(smem_u32(b_lo(s)) + kk * 32, 16, 1024);
          mma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, ah, bl, idesc, 1u);
          mma_tf32(tmem, al, bh, idesc, 1u);
        }
        mma_commit(empty + s);
      }
      mma_commit(tmem_full);
    }
  } else {
    // ---------------- epilogue: TMEM -> smem tile, then row by row (lanes on
    // consecutive 16 B of one row, as in segment_sum) FM term + scatter-add into dG
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* tile = reinterpret_cast<float*>(smem);  // ring is free: all MMAs completed
    constexpr int TS = BN + 1;
    {
      const int rr = q * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float a[16];
        tmem_ld16(trow + c0, a);
#pragma unroll
        for (int j = 0; j < 16; ++j) tile[rr * TS + c0 + j] = a[j];
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int d4 = p.d >> 2;
    const int w2 = warp - 2;
    if (nkb > 0) {
      // warp w2 owns tile rows w2 + 4 i (i < 32): lane i fetches row i's vid / gz once,
      // then rows go 4 at a time with their G / fm_s loads all in flight
      const int my_r = m0 + w2 + 4 * lane;
      const bool my_live = my_r < p.rows;
      const uint32_t my_v = my_live ? __ldg(p.vid + static_cast<int64_t>(my_r) * p.F + f) : 0u;
      const float my_k = my_live ? p.scale * __ldg(p.gz + my_r) : 0.f;
#pragma unroll 1
      for (int i0 = 0; i0 < 32; i0 += 4) {
        uint32_t vv[4];
        float kk[4];
        float4 s4[4], g4[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u;
          vv[u] = __shfl_sync(0xFFFFFFFFu, my_v, i);
          kk[u] = __shfl_sync(0xFFFFFFFFu, my_k, i);
          const int r = m0 + w2 + 4 * i;
          ok[u] = r < p.rows && lane < d4;
          if (ok[u]) {
            s4[u] = __ldg(reinterpret_cast<const float4*>(p.fm_s + static_cast<int64_t>(r) * p.d) + lane);
            g4[u] = __ldg(reinterpret_cast<const float4*>(p.G + static_cast<int64_t>(vv[u]) * p.d) + lane);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!ok[u]) continue;
          const float* a = tile + (w2 + 4 * (i0 + u)) * TS + 4 * lane;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                           p.dG + static_cast<int64_t>(vv[u]) * p.d + 4 * lane),
                       "f"(p.scale * a[0] + kk[u] * (s4[u].x - g4[u].x)),
                       "f"(p.scale * a[1] + kk[u] * (s4[u].y - g4[u].y)),
                       "f"(p.scale * a[2] + kk[u] * (s4[u].z - g4[u].z)),
                       "f"(p.scale * a[3] + kk[u] * (s4[u].w - g4[u].w))
                       : "memory");
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(L::TMEM_COLS));
  }
}

// TMA row gather: 4 rows (by index) x one 32-float box of the 2D table G into
// 4 consecutive 128 B smem rows (the tensor map's swizzle applies).
__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int col, uint32_t r0, uint32_t r1, uint32_t r2,
                                            uint32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}

// Gathered-A GEMM with the gather done by TMA (tile::gather4 on the table G):
// the producer warp issues 32 gather4 per k-block (one per lane, 4 rows each)
// plus the B tiles; 4 split warps turn the raw tile into tf32 hi/lo parts in
// place; one elected lane issues tcgen05.mma; the split warps then run the
// epilogue (split-K partials). A_MN = false: forward (rows x K_pad) . W1p;
// A_MN = true: dW1 (K_pad x rows) . dh.
template <bool A_MN>
__global__ void __launch_bounds__(192, 1)
    gather4_gemm_kernel(const __grid_constant__ CUtensorMap tmG,
                        const __grid_constant__ CUtensorMap tmBhi,
                        const __grid_constant__ CUtensorMap tmBlo, const FusedParams p) {
  constexpr int BN = 64;
  using L = Layout<BN>;
  constexpr int ST = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * L::STAGE_BYTES);
  uint64_t* ready = full + ST;
  uint64_t* empty = ready + ST;
  uint64_t* tmem_full = empty + ST;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_hi = [&](int s) { return smem + s * L::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * L::STAGE_BYTES + A_BYTES; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * L::STAGE_BYTES + 2 * A_BYTES + L::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.k_blocks_per_split;
  const int kb1 = min(p.num_k_blocks, kb0 + p.k_blocks_per_split);
  const int nkb = kb1 - kb0;
  const int M = A_MN ? p.F * p.dp : p.rows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(ready + s, 128);
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "n"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- producer warp: 32 x gather4 (A) + B tiles per k-block
    // lane geometry: forward: rows m0 + 4 lane .. +3 (one field per k-block);
    // dW1: atom a = lane / 8 (32 m-columns), batch rows 4 (lane % 8) .. +3 of the block
    auto rows_for = [&](int i, uint32_t (&v)[4], int& col) {
      const int kb = kb0 + i;
      int f, r0;
      if constexpr (!A_MN) {
        const int kcol = kb * BKE;
        f = kcol / p.dp;
        col = kcol - f * p.dp;
        r0 = m0 + 4 * lane;
      } else {
        const int mcol = m0 + (lane >> 3) * 32;
        f = mcol / p.dp;
        col = mcol - f * p.dp;
        r0 = kb * BKE + 4 * (lane & 7);
      }
      const bool fok = f < p.F;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + j;
        // rows past the batch gather row 0: forward -> masked output rows; dW1 ->
        // multiplied by the zero-filled dh rows
        v[j] = (fok && r < p.rows) ? __ldg(p.vid + static_cast<int64_t>(r) * p.F + f) : 0u;
      }
    };
    uint32_t va[4], vb[4];
    int ca = 0, cb = 0;
    if (nkb > 0) rows_for(0, va, ca);
    for (int i = 0; i < nkb; ++i) {
      if (i + 1 < nkb) rows_for(i + 1, vb, cb);  // next block's row ids in flight
      const int s = i % ST;
      if (lane == 0) {
        mbar_wait(empty + s, ((i / ST) & 1) ^ 1);
        mbar_expect_tx(full + s, A_BYTES + 2 * L::B_BYTES);
      }
      __syncwarp();
      const uint32_t dst = A_MN ? (lane >> 3) * 4096 + (lane & 7) * 512 : lane * 512;
      tma_gather4(&tmG, full + s, a_hi(s) + dst, ca, va[0], va[1], va[2], va[3]);
      if (lane == 0) {
        const int kc = (kb0 + i) * BKE;
        if constexpr (A_MN) {
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            tma_load_2d(&tmBhi, full + s, b_hi(s) + b * 4096, n0 + b * 32, kc);
            tma_load_2d(&tmBlo, full + s, b_lo(s) + b * 4096, n0 + b * 32, kc);
          }
        } else {
          tma_load_2d(&tmBhi, full + s, b_hi(s), kc, n0);
          tma_load_2d(&tmBlo, full + s, b_lo(s), kc, n0);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) va[j] = vb[j];
      ca = cb;
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN ? 1 : 0, A_MN ? 1 : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        mbar_wait(ready + s, (i / ST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t ah, al, bh, bl;
          if constexpr (A_MN) {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 1024, 4096, 512, 1);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 1024, 4096, 512, 1);
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 1024, 4096, 512, 1);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 1024, 4096, 512, 1);
          } else {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 32, 16, 1024);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 32, 16, 1024);
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 32, 16, 1024);
          }
          mma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, ah, bl, idesc, 1u);
          mma_tf32(tmem, al, bh, idesc, 1u);
        }
        mma_commit(empty + s);
      }
      mma_commit(tmem_full);
    }
  } else {
    const int t = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < nkb; ++i) {  // ---------------- in-place 3xTF32 split
      const int s = i % ST;
      mbar_wait(full + s, (i / ST) & 1);
      float4* hi = reinterpret_cast<float4*>(a_hi(s));
      float4* lo = reinterpret_cast<float4*>(a_lo(s));
#pragma unroll 4
      for (int e = t; e < A_BYTES / 16; e += 128) {
        float4 l;
        const float4 h = split_hi(hi[e], l);
        hi[e] = h;
        lo[e] = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(ready + s);
    }
    // ---------------- epilogue (split-K partials), staged for coalesced stores
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* tile = reinterpret_cast<float*>(smem);
    constexpr int TS = BN + 1;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 8) {
      float v[8];
      tmem_ld8(trow + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) tile[row * TS + c0 + j] = v[j];
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int w2 = t >> 5;
    if (nkb > 0)
      for (int rr = w2; rr < BM; rr += 4) {
        const int m = m0 + rr;
        if (m >= M) break;
        float* o = p.out + blockIdx.z * p.split_stride + static_cast<long long>(m) * p.ldo;
#pragma unroll
        for (int c = lane; c < BN; c += 32)
          if (n0 + c < p.H) o[n0 + c] = tile[rr * TS + c];
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(L::TMEM_COLS));
  }
}

}  // namespace tc
}  // namespace sfb
