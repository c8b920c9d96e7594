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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
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
    for (int i = 0; i < nkb; ++i) {
      const int s = i % ST;
      mbar_wait(empty + s, ((i / ST) & 1) ^ 1);
      const int kb = kb0 + i;
      float4 x[4], lo[4];
      if constexpr (!A_MN) {
        // row t%128 of the tile, 16 columns: half t/128 of the 32-wide block
        const int rr = t & 127, half = t >> 7;
        const int r = m0 + rr;
        const int kcol = kb * BKE;  // padded column
        const int f = kcol / p.dp, c0 = kcol - f * p.dp + 16 * half;
        const bool valid = r < p.rows && f < p.F;
        const uint32_t v = valid ? __ldg(p.vid + static_cast<int64_t>(r) * p.F + f) : 0u;
        load_seg16(p.G, p.d, valid, v, c0, x);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 h = split_hi(x[q], lo[q]);
          const uint32_t off = kmajor_off(rr, 4 * half + q);
          *reinterpret_cast<float4*>(a_hi(s) + off) = h;
          *reinterpret_cast<float4*>(a_lo(s) + off) = lo[q];
        }
      } else {
        // k-row kk = t/8 (a batch row), 16 m-columns: atom (t%8)/2, half t%2
        const int kk = t >> 3, a = (t & 7) >> 1, half = t & 1;
        const int r = kb * BKE + kk;
        const int mcol = m0 + a * 32 + 16 * half;  // padded column
        const int f = mcol / p.dp, c0 = mcol - f * p.dp;
        const bool valid = r < p.rows && f < p.F;
        const uint32_t v = valid ? __ldg(p.vid + static_cast<int64_t>(r) * p.F + f) : 0u;
        load_seg16(p.G, p.d, valid, v, c0, x);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 h = split_hi(x[q], lo[q]);
          const uint32_t off = mnmajor_off(a * 32 + 16 * half + 4 * q, kk);
          *reinterpret_cast<float4*>(a_hi(s) + off) = h;
          *reinterpret_cast<float4*>(a_lo(s) + off) = lo[q];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(readyA + s);
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
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
    // ---------------- epilogue: row per thread, FM term + scatter-add into dG
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int rr = q * 32 + lane;
    const int r = m0 + rr;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const bool live = r < p.rows && nkb > 0;
    const uint32_t v = live ? __ldg(p.vid + static_cast<int64_t>(r) * p.F + f) : 0u;
    const float k = live ? p.scale * __ldg(p.gz + r) : 0.f;
    const float4* S = reinterpret_cast<const float4*>(p.fm_s + static_cast<int64_t>(r) * p.d);
    const float4* Gv = reinterpret_cast<const float4*>(p.G + static_cast<int64_t>(v) * p.d);
    float* dst = p.dG + static_cast<int64_t>(v) * p.d;
#pragma unroll 1
    for (int c0 = 0; c0 < p.d; c0 += 16) {
      float a[16];
      tmem_ld16(trow + c0, a);  // columns past d exist in TMEM (BN >= d) and are ignored
      if (!live) continue;
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const int c = c0 + j;
        if (c >= p.d) break;
        const float4 s4 = __ldg(S + (c >> 2));
        const float4 g4 = __ldg(Gv + (c >> 2));
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + c),
                     "f"(p.scale * a[j] + k * (s4.x - g4.x)),
                     "f"(p.scale * a[j + 1] + k * (s4.y - g4.y)),
                     "f"(p.scale * a[j + 2] + k * (s4.z - g4.z)),
                     "f"(p.scale * a[j + 3] + k * (s4.w - g4.w))
                     : "memory");
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

}  // namespace tc
}  // namespace sfb
