// Streamed 3xTF32 GEMM with the A operand in TMEM (tcgen05.mma ... [d], [a_tmem], b_desc).
//
// The SS kernel (tc_gemm.cuh) is shared-memory-bandwidth bound for the tower's
// skinny GEMMs (N = H = 64): every k-block the tensor core re-reads the A tile
// from smem once per product (ah*bh, ah*bl, al*bh) and the split warps read the
// raw tile and write back two parts, ~150 KB of smem traffic per 16 KB of A.
// Here:
//   * the split warps (thread = TMEM lane = A row) read the raw A row once from
//     smem and write its tf32 hi/lo parts straight into TMEM (tcgen05.st);
//   * B hi and lo sit back to back in smem, so [B_hi; B_lo] is ONE N = 128
//     operand: ah x [bh | bl] lands in accumulator columns [0, 64) / [64, 128)
//     with a single MMA, al x bh (N = 64) accumulates into [0, 64);
//   * the epilogue sums the two accumulator halves.
// Per k-block smem traffic: TMA 32 KB in, 16 KB split reads, 24 KB B reads.
//
// A_MN = false: A = X tile [128 rows x 32 k], K-major, SWIZZLE_128B (GEMM1).
// A_MN = true : A = X^T: TMA box {128 X-columns, 32 X-rows}, no swizzle; thread m
//               reads column m (conflict-free, 32 consecutive floats per warp) (GEMM3).
// B_MN = false: B K-major SWIZZLE_128B boxes {32 k, 64 n}; true: MN-major
//               BASE32B boxes {32 n, 32 k} x 2 per part.
// Output: split-K partial [z][M][N] (store epilogue).
#pragma once

#include "tc_gemm.cuh"

namespace sfb {
namespace tc {

constexpr int kTsStages = 6;  // TMEM: 128 accumulator columns + 6 x 64 A columns = 512

struct TsLayout {
  static constexpr int A_RAW = BM * BKE * 4;          // 16 KB raw fp32 A tile
  static constexpr int B_PART = 64 * BKE * 4;         // 8 KB per (hi | lo) part
  static constexpr int STAGE_BYTES = A_RAW + 2 * B_PART;
  static constexpr int SMEM = 1024 + kTsStages * STAGE_BYTES + 256;
  static_assert(kTsStages * STAGE_BYTES >= BM * 65 * 4, "epilogue tile must fit the ring");
};

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]),
      "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]),
      "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(192, 1)
    gemm_ts_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmBhi,
                   const __grid_constant__ CUtensorMap tmBlo, const Params p) {
  using L = TsLayout;
  constexpr int ST = kTsStages;
  constexpr int BN = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * L::STAGE_BYTES);
  uint64_t* ready = full + ST;
  uint64_t* empty = ready + ST;
  uint64_t* tmem_full = empty + ST;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_raw = [&](int s) { return smem + s * L::STAGE_BYTES; };
  auto b_hi = [&](int s) { return smem + s * L::STAGE_BYTES + L::A_RAW; };
  auto b_lo = [&](int s) { return smem + s * L::STAGE_BYTES + L::A_RAW + L::B_PART; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.k_blocks_per_split;
  const int kb1 = min(p.num_k_blocks, kb0 + p.k_blocks_per_split);
  const int nkb = kb1 - kb0;
  // CTAs sharing a B tile start at different k-blocks so they do not all read
  // the same L2 lines at the same moment
  const int rot = nkb > 0 ? static_cast<int>((blockIdx.x * 5u) % static_cast<unsigned>(nkb)) : 0;
  auto kblk = [&](int i) { const int j = i + rot; return kb0 + (j >= nkb ? j - nkb : j); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(ready + s, 128);
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;  // accumulator: columns [0, 128)
  auto a_col = [&](int s) { return tmem + 128u + static_cast<uint32_t>(s) * 64u; };  // hi | lo

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      constexpr uint32_t bytes = L::A_RAW + 2 * L::B_PART;
      constexpr int PD = 2 * ST;  // L2 prefetch distance (k-blocks) for the streamed A
      auto prefetch_a = [&](int i) {
        const int kc = kblk(i) * BKE;
        if constexpr (A_MN) tma_prefetch_2d(&tmA, m0, kc);
        else tma_prefetch_2d(&tmA, kc, m0);
      };
      for (int i = 0; i < PD && i < nkb; ++i) prefetch_a(i);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        if (i + PD < nkb) prefetch_a(i + PD);
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect_tx(full + s, bytes - ((p.dbg & 4) ? L::A_RAW : 0) - ((p.dbg & 8) ? 2 * L::B_PART : 0));
        const int kc = kblk(i) * BKE;
        if (p.dbg & 4) {
        } else if constexpr (A_MN) tma_load_2d(&tmA, full + s, a_raw(s), m0, kc);
        else tma_load_2d(&tmA, full + s, a_raw(s), kc, m0);
        if (p.dbg & 8) {
        } else if constexpr (B_MN) {
#pragma unroll
          for (int b = 0; b < BN / 32; ++b) {
            tma_load_2d(&tmBhi, full + s, b_hi(s) + b * 4096, n0 + b * 32, kc);
            tma_load_2d(&tmBlo, full + s, b_lo(s) + b * 4096, n0 + b * 32, kc);
          }
        } else {
          tma_load_2d(&tmBhi, full + s, b_hi(s), kc, n0);
          tma_load_2d(&tmBlo, full + s, b_lo(s), kc, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t id128 = idesc_tf32(BM, 2 * BN, 0, B_MN ? 1 : 0);
      constexpr uint32_t id64 = idesc_tf32(BM, BN, 0, B_MN ? 1 : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        mbar_wait(ready + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t bd;
          if constexpr (B_MN) bd = smem_desc(smem_u32(b_hi(s)) + kk * 1024, 4096, 512, 1);
          else bd = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
          const uint32_t ah = a_col(s) + kk * 8, al = a_col(s) + 32 + kk * 8;
          if (p.dbg & 2) continue;
          mma_tf32_ts(tmem, ah, bd, id128, (i > 0 || kk > 0) ? 1u : 0u);  // [hh | hl]
          mma_tf32_ts(tmem, al, bd, id64, 1u);                              // += lh
        }
        mma_commit(empty + s);  // frees the smem stage and the TMEM A stage
      }
      mma_commit(tmem_full);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    // ---------------- split: raw A row -> tf32 hi / lo columns in TMEM
    for (int i = 0; i < nkb; ++i) {
      const int s = i % ST;
      const uint32_t ph = (i / ST) & 1;
      mbar_wait(empty + s, ph ^ 1);  // the MMAs of k-block i - ST have left this TMEM stage
      mbar_wait(full + s, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float hi[32], lo[32];
      if (p.dbg & 1) {
        mbar_arrive(ready + s);
        continue;
      }
      if constexpr (A_MN) {
        const float* src = reinterpret_cast<const float*>(a_raw(s)) + row;
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = src[k * BM];
      } else {
        const float4* src = reinterpret_cast<const float4*>(a_raw(s) + row * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = src[j ^ (row & 7)];
          hi[4 * j] = v.x;
          hi[4 * j + 1] = v.y;
          hi[4 * j + 2] = v.z;
          hi[4 * j + 3] = v.w;
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float v = hi[k];
        hi[k] = tf32_rna(v);
        lo[k] = tf32_rna(v - hi[k]);
      }
      tmem_st32(a_col(s) + lane_off, hi);
      tmem_st32(a_col(s) + 32 + lane_off, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(ready + s);
    }
    // ---------------- epilogue: acc[:, c] + acc[:, 64 + c] -> smem tile -> coalesced store
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t trow = tmem + lane_off;
    float* tile = reinterpret_cast<float*>(smem);
    constexpr int TS = BN + 1;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16], w[16];
      tmem_ld16(trow + c0, v);
      tmem_ld16(trow + BN + c0, w);
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[row * TS + c0 + j] = v[j] + w[j];
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int w2 = (threadIdx.x - 64) >> 5;
    if (nkb > 0) {
#pragma unroll 1
      for (int r = w2; r < BM; r += 4) {
        const int m = m0 + r;
        if (m >= p.M) break;
        float* o = p.out + blockIdx.z * p.split_stride + static_cast<long long>(m) * p.ldo;
#pragma unroll
        for (int c = lane; c < BN; c += 32) {
          const int n = n0 + c;
          if (n < p.N) o[n] = tile[r * TS + c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc
}  // namespace sfb
