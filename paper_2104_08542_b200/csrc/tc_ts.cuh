// Streamed 3xTF32 GEMM with the A operand in TMEM (tcgen05.mma ... [d], [a_tmem], b_desc).
//
// Used for the tower's two X-streaming GEMMs (N = H = 64, K or M = the 3120-wide
// activation): they are HBM streams of X with a skinny MMA, so the design goal is
// bytes in flight, not MMA shape.
//   * raw A tiles land by TMA in a smem ring (kTsARing x 16 KB) that is released as
//     soon as the split warps have read a tile — not when the MMA is done — so ~5 tiles
//     of X are always in flight per SM (Little's law at ~1.5 us loaded DRAM latency);
//   * the split warps (thread = TMEM lane = A row; two warp groups taking alternate
//     k-blocks) round the row to tf32 hi/lo in registers and write both parts
//     straight into a TMEM stage (tcgen05.st);
//   * B hi and lo come from L2 through their own ring (separate producer warp); they
//     sit back to back in smem, so [B_hi; B_lo] is ONE N = 128 operand:
//     ah x [bh | bl] lands in accumulator columns [0, 64) / [64, 128) with a single
//     MMA and al x bh (N = 64) accumulates into [0, 64); the epilogue sums the halves.
// Measured issue rate of that pair: 96 clk per 8-deep k step (tf32 TS, B200), i.e.
// 384 clk per 32-wide k-block.
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

// 6 raw A tiles: 161 KB of shared memory per CTA instead of 193 KB with 8, which leaves room
// for the manager stage's CTAs beside the GEMM (+1.5 % at cfg2 N = 1; 6 tiles = ~2 us of
// X in flight at ~700 clk per k-block still covers the loaded DRAM latency)
#ifndef SFB_TS_ARING
#define SFB_TS_ARING 6
#endif
#ifndef SFB_TS_BRING
#define SFB_TS_BRING 4
#endif
constexpr int kTsARing = SFB_TS_ARING;  // raw A tiles (smem)
constexpr int kTsBRing = SFB_TS_BRING;  // B hi/lo tiles (smem)
// (odd ring depths crashed when tried: the two split groups take alternate k-blocks)
static_assert(kTsARing % 2 == 0 && kTsBRing % 2 == 0, "ring depths must be even");
constexpr int kTsStages = 6;  // TMEM A stages: 128 accumulator columns + 6 x 64 = 512
constexpr int kTsThreads = 352;  // 11 warps: A producer, MMA, 8 split/epilogue, B producer

struct TsLayout {
  static constexpr int A_RAW = BM * BKE * 4;   // 16 KB raw fp32 A tile
  static constexpr int B_PART = 64 * BKE * 4;  // 8 KB per (hi | lo) part
  static constexpr int B_STAGE = 2 * B_PART;
  static constexpr int SMEM = 1024 + kTsARing * A_RAW + kTsBRing * B_STAGE + 512;
  static_assert(kTsARing * A_RAW >= BM * 65 * 4, "epilogue tile must fit the A ring");
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kTsThreads, 1)
    gemm_ts_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmBhi,
                   const __grid_constant__ CUtensorMap tmBlo, const Params p) {
  using L = TsLayout;
  constexpr int RA = kTsARing, RB = kTsBRing, TS = kTsStages;
  constexpr int BN = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint8_t* a_ring = smem;
  uint8_t* b_ring = smem + RA * L::A_RAW;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(b_ring + RB * L::B_STAGE);
  uint64_t* a_empty = a_full + RA;
  uint64_t* b_full = a_empty + RA;
  uint64_t* b_empty = b_full + RB;
  uint64_t* t_ready = b_empty + RB;
  uint64_t* t_empty = t_ready + TS;
  uint64_t* tmem_full = t_empty + TS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_raw = [&](int s) { return a_ring + s * L::A_RAW; };
  auto b_hi = [&](int s) { return b_ring + s * L::B_STAGE; };
  auto b_lo = [&](int s) { return b_ring + s * L::B_STAGE + L::B_PART; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int m0 = bx * BM, n0 = by * BN;
  const int kb0 = bz * p.k_blocks_per_split;
  const int kb1 = min(p.num_k_blocks, kb0 + p.k_blocks_per_split);
  const int nkb = kb1 - kb0;
  // CTAs sharing a B tile start at different k-blocks so they do not all read
  // the same L2 lines at the same moment
  const int rot = nkb > 0 ? static_cast<int>((bx * 5u) % static_cast<unsigned>(nkb)) : 0;
  auto kblk = [&](int i) { const int j = i + rot; return kb0 + (j >= nkb ? j - nkb : j); };
  const bool tr = p.trace && bx == 0 && by == 0 && bz == 0;
  const int cta = (bz * gridDim.y + by) * gridDim.x + bx;
  if (p.cta_trace && threadIdx.x == 0) p.cta_trace[2 * cta] = global_ns();

  if (threadIdx.x == 0) {
    for (int s = 0; s < RA; ++s) {
      mbar_init(a_full + s, 1);
      mbar_init(a_empty + s, 4);
    }
    for (int s = 0; s < RB; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < TS; ++s) {
      mbar_init(t_ready + s, 4);
      mbar_init(t_empty + s, 1);
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
  // PDL: the predecessor's outputs (X / dh) are read only after it has completed. No early
  // trigger: successors launched early sit on SM slots the concurrent row update needs
  // (measured: -8 % at cfg2 N = 1 with a trigger here and in the dX GEMM)
  pdl_wait();
  const uint32_t tmem = *tmem_holder;  // accumulator: columns [0, 128)
  auto a_col = [&](int s) { return tmem + 128u + static_cast<uint32_t>(s) * 64u; };  // hi | lo

  if (warp == 0) {
    if (lane == 0) {  // ---------------- A producer: raw X tiles, RA deep
      for (int i = 0; i < nkb; ++i) {
        const int s = i % RA;
        mbar_wait(a_empty + s, ((i / RA) & 1) ^ 1);
        if (tr && i < 64) p.trace[i] = clock64();
        if (p.dbg & 4) {
          mbar_arrive(a_full + s);
          continue;
        }
        mbar_expect_tx(a_full + s, L::A_RAW);
        const int kc = kblk(i) * BKE;
        if constexpr (A_MN) tma_load_2d(&tmA, a_full + s, a_raw(s), m0, kc);
        else tma_load_2d(&tmA, a_full + s, a_raw(s), kc, m0);
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- B producer: W / dh hi+lo tiles from L2
      for (int i = 0; i < nkb; ++i) {
        const int s = i % RB;
        if (p.dbg & 128) mbar_wait_sleep(b_empty + s, ((i / RB) & 1) ^ 1, 256);
        else mbar_wait(b_empty + s, ((i / RB) & 1) ^ 1);
        if (p.dbg & 8) {
          mbar_arrive(b_full + s);
          continue;
        }
        mbar_expect_tx(b_full + s, L::B_STAGE);
        const int kc = kblk(i) * BKE;
        if constexpr (B_MN) {
#pragma unroll
          for (int b = 0; b < BN / 32; ++b) {
            tma_load_2d(&tmBhi, b_full + s, b_hi(s) + b * 4096, n0 + b * 32, kc);
            tma_load_2d(&tmBlo, b_full + s, b_lo(s) + b * 4096, n0 + b * 32, kc);
          }
        } else {
          tma_load_2d(&tmBhi, b_full + s, b_hi(s), kc, n0);
          tma_load_2d(&tmBlo, b_full + s, b_lo(s), kc, n0);
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (warp-wide loop, elected issue)
    constexpr uint32_t id128 = idesc_tf32(BM, 2 * BN, 0, B_MN ? 1 : 0);
    constexpr uint32_t id64 = idesc_tf32(BM, BN, 0, B_MN ? 1 : 0);
    const uint32_t b0 = smem_u32(b_ring);
    for (int i = 0; i < nkb; ++i) {
      const int t = i % TS, s = i % RB;
      mbar_wait(t_ready + t, (i / TS) & 1);
      if (tr && lane == 0 && i < 64) p.trace[256 + i] = clock64();
      mbar_wait(b_full + s, (i / RB) & 1);
      if (tr && lane == 0 && i < 64) p.trace[192 + i] = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (elect_one()) {
        const uint32_t bs = b0 + static_cast<uint32_t>(s) * L::B_STAGE;
        const uint32_t at = tmem + 128u + static_cast<uint32_t>(t) * 64u;
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t bd;
          if constexpr (B_MN) bd = smem_desc(bs + kk * 1024, 4096, 512, 1);
          else bd = smem_desc(bs + kk * 32, 16, 1024);
          if (p.dbg & 2) continue;
          mma_tf32_ts(tmem, at + kk * 8, bd, id128, (i > 0 || kk > 0) ? 1u : 0u);  // [hh | hl]
          mma_tf32_ts(tmem, at + 32 + kk * 8, bd, id64, 1u);                         // += lh
        }
        mma_commit(b_empty + s);
        mma_commit(t_empty + t);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(tmem_full);
    __syncwarp();
  } else {
    // ---------------- split: raw A row -> tf32 hi / lo columns in TMEM. The two warp
    // groups take alternate k-blocks so one group's TMEM-store latency overlaps the
    // other's loads and rounding.
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;   // warp group: k-blocks i = h (mod 2)
    const int row = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const bool tl = tr && threadIdx.x == 64;
    for (int i = h; i < nkb; i += 2) {
      const int s = i % RA, t = i % TS;
      mbar_wait(a_full + s, (i / RA) & 1);
      if (tl && i < 64) p.trace[64 + i] = clock64();
      float hi[32], lo[32];
      if (p.dbg & 1) {
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = 0.f;
      } else if constexpr (A_MN) {
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
      __syncwarp();
      if (lane == 0) mbar_arrive(a_empty + s);  // raw tile consumed: the TMA may refill it
      if (p.dbg & 128) mbar_wait_sleep(t_empty + t, ((i / TS) & 1) ^ 1, 256);
      else mbar_wait(t_empty + t, ((i / TS) & 1) ^ 1);  // MMAs of k-block i - TS left this stage
      if (!(p.dbg & 64)) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (!(p.dbg & 16)) {
          tmem_st32(a_col(t) + lane_off, hi);
          tmem_st32(a_col(t) + 32 + lane_off, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else if (p.dbg & 1) {
        hi[0] += lo[5];  // keep the registers live
        if (hi[0] == 12345.f) p.out[0] = hi[0];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(t_ready + t);
      if (tl && i < 64) p.trace[128 + i] = clock64();
    }
    // ---------------- epilogue: acc[:, c] + acc[:, 64 + c] -> smem tile -> coalesced store
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t trow = tmem + lane_off;
    float* tile = reinterpret_cast<float*>(smem);  // A ring: every raw tile has been consumed
    constexpr int TSW = BN + 1;
#pragma unroll 1
    for (int c0 = 32 * h; c0 < 32 * h + 32; c0 += 16) {
      float v[16], w[16];
      tmem_ld16(trow + c0, v);
      tmem_ld16(trow + BN + c0, w);
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[row * TSW + c0 + j] = v[j] + w[j];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int w2 = warp - 2;  // 0..7
    if (nkb > 0) {
#pragma unroll 1
      for (int r = w2; r < BM; r += 8) {
        const int m = m0 + r;
        if (m >= p.M) break;
        float* o = p.out + bz * p.split_stride + static_cast<long long>(m) * p.ldo;
#pragma unroll
        for (int c = lane; c < BN; c += 32) {
          const int n = n0 + c;
          if (n < p.N) o[n] = tile[r * TSW + c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (p.cta_trace && threadIdx.x == 0) p.cta_trace[2 * cta + 1] = global_ns();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc
}  // namespace sfb
