// Persistent dX GEMM of the tower backward (GEMM2):  dX = scale * dh W1^T
//   dh [rows x H], W1 [K x H] (both pre-split into tf32 hi/lo, K-major), H <= 64.
//
// The contraction is only H = 64 deep while the output is the full [rows x K]
// activation gradient (102 MB at cfg2), so the kernel is an HBM write stream
// with a short MMA per tile. The one-tile-per-CTA version paid CTA setup, TMEM
// allocation and an unoverlapped epilogue for each of the ~3100 tiles. Here one
// CTA per SM walks a contiguous range of (m, n) tiles in m-major order:
//   warp 0     : TMA producer — dh hi/lo tile of the current m (64 KB, reloaded only
//                when m changes) and a 3-deep ring of W1 hi/lo n-tiles (32 KB each)
//   warp 1     : MMA issuer — per tile 2 k-blocks x 4 x (ah x [bh | bl] N = 128,
//                al x bh N = 64) into one of two TMEM accumulators (2 x 128 columns)
//   warps 2..5 : epilogue — tcgen05.ld both accumulator halves, sum, scale, write the
//                128 x 64 tile into a SWIZZLE_128B staging buffer and TMA-store it
//                (cp.async.bulk.tensor shared -> global), overlapping the next tile's MMA
//
// SCATTER = true fuses the segment sum into the epilogue (one worker, deferred FM term):
// dX is never written; every 16 B chunk of a tile row goes straight to
//   dG[vid[r, f]][c..c+3] += scale * (acc + gz[r] * fm_s[r][c..c+3])   (red.global.add.v4.f32)
// with (f, c) = divmod(column, d), and Bsum[vid[r, f]] += gz[r] once per position (the
// column c == 0 chunk). vid / gz of the CTA's current 128 rows are staged in smem when m
// changes (once per ~21 tiles). The accumulator is drained to an smem value tile first
// (thread = row), then each half-warp scatters one row's 16 chunks: consecutive lanes hit
// consecutive 16 B of the same dG row, so a red instruction is 2 coalesced 256 B segments
// instead of 32 scattered 16 B ones.
#pragma once

#include "tc_gemm.cuh"

namespace sfb {
namespace tc {

struct DxLayout {
  static constexpr int A_PART = BM * BKE * 4;     // 16 KB: 128 rows x 32 k
  static constexpr int A_BYTES = 4 * A_PART;      // hi kb0, hi kb1, lo kb0, lo kb1
  static constexpr int B_PART = 64 * BKE * 4;     // 8 KB: 64 n x 32 k
  static constexpr int B_STAGE = 4 * B_PART;      // kb0 [hi; lo], kb1 [hi; lo]
#ifndef SFB_DX_BSTAGES
#define SFB_DX_BSTAGES 3
#endif
  static constexpr int B_STAGES = SFB_DX_BSTAGES;
  static constexpr int OUT_BYTES = BM * 64 * 4;   // 32 KB staging (2 boxes of 32 columns)
  static constexpr int SMEM = 1024 + A_BYTES + B_STAGES * B_STAGE + OUT_BYTES + 256;
};

struct DxParams {
  int M, N;       // rows, K (columns of dX)
  int n_tiles;    // ceil(N / 64)
  int tiles;      // ceil(M / 128) * n_tiles
  float scale;
  // SCATTER only
  const uint32_t* vid;  // [M x F] table rows of the positions
  const uint32_t* remap;  // nullable: row = remap[vid] (owner-routed: global unique -> local row)
  const float* fm_s;    // [M x d] FM field sums
  const float* gz;      // [M]
  float* dG;            // [rows x d] gradient table (red.add)
  float* Bsum;          // [rows] deferred FM coefficients (red.add)
  int F, d;
  int exp;              // experiment: 1 = no global reductions, 2 = no FM-sum loads,
                        // 3 = drain the accumulator only (no tile, no scatter)
  unsigned long long* cta_trace;  // profiling (nullable): per-CTA [start, end] globaltimer
  long long* trace;               // profiling (nullable): CTA 0 per-tile clock64 stamps
  // SCATTER: the A operand (dh hi / lo, [rows x lda], pre-split) is written into TMEM by
  // four A-writer warps once per 128-row tile and the MMAs read it from there (TS form)
  const float* a_hi;
  const float* a_lo;
  int lda;
  int H;    // contraction length (<= 64): A columns >= H are written as zeros
  int epi;  // SCATTER epilogue: 0 = through a shared-memory value tile (half-warp per row),
            // 1 = warp-local register transpose (no tile, no per-tile block barriers)
};

// smem for the scatter epilogue: value tile [128 x 68] f32, vid [128 x F] u32, gz [128]
constexpr int kDxTileStride = 68;  // 64 columns + 4 pad (16 B aligned rows, fewer conflicts)
__host__ __device__ constexpr int dx_scatter_bytes(int F, int d) {
  return BM * kDxTileStride * 4 + BM * F * 4 + BM * 4 + 0 * d;
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}

// SCATTER runs kDxScatterWarps epilogue warps (several per TMEM lane quarter): the scatter is bound by how
// many red.global.add instructions are in flight per SM
#ifndef SFB_DX_EW
#define SFB_DX_EW 16
#endif
constexpr int kDxScatterWarps = SFB_DX_EW;  // 4 per TMEM lane quarter
template <bool SCATTER>
constexpr int dx_threads() { return SCATTER ? 64 + 32 * kDxScatterWarps + 128 : 192; }
constexpr int kDxAWriter0 = 2 + kDxScatterWarps;  // first of the 4 A-writer warps (SCATTER)
constexpr uint32_t kDxTmemA = 256;                 // TMEM column of A (SCATTER): hi [0,64), lo [64,128)

template <bool SCATTER>
__global__ void __launch_bounds__(dx_threads<SCATTER>(), 1)
    gemm_dx_persistent_kernel(const __grid_constant__ CUtensorMap tmAhi,
                              const __grid_constant__ CUtensorMap tmAlo,
                              const __grid_constant__ CUtensorMap tmBhi,
                              const __grid_constant__ CUtensorMap tmBlo,
                              const __grid_constant__ CUtensorMap tmOut, const DxParams p) {
  using L = DxLayout;
  constexpr int BS = L::B_STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint8_t* a_s = smem;  // SCATTER: A lives in TMEM, no shared-memory A region
  uint8_t* b_s = smem + (SCATTER ? 0 : L::A_BYTES);
  uint8_t* out_s = b_s + BS * L::B_STAGE;  // TMA-store staging, or the scatter tables
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      out_s + (SCATTER ? ((dx_scatter_bytes(p.F, p.d) + 15) & ~15) : L::OUT_BYTES));
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 1;
  uint64_t* b_full = bars + 2;
  uint64_t* b_empty = b_full + BS;
  uint64_t* acc_full = b_empty + BS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.cta_trace && threadIdx.x == 0) p.cta_trace[2 * blockIdx.x] = global_ns();
  const int t0 = static_cast<int>(static_cast<long long>(blockIdx.x) * p.tiles / gridDim.x);
  const int t1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * p.tiles / gridDim.x);

  if (threadIdx.x == 0) {
    mbar_init(a_full, SCATTER ? 4 : 1);  // SCATTER: the four A-writer warps
    mbar_init(a_empty, 1);
    for (int s = 0; s < BS; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, SCATTER ? kDxScatterWarps : 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmOut)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(tmem_holder)), "n"(SCATTER ? 512 : 256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  pdl_wait();  // dh (head) / vid, gz, fm_s are read below
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int cur_m = -1, gen = 0;
      for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int m = t / p.n_tiles, n = t - m * p.n_tiles;
        if (m != cur_m) {
          if constexpr (!SCATTER) {  // (SCATTER: A goes to TMEM through the A-writer warps)
            if (gen > 0) mbar_wait(a_empty, (gen - 1) & 1);
            mbar_expect_tx(a_full, L::A_BYTES);
#pragma unroll
            for (int kb = 0; kb < 2; ++kb) {
              tma_load_2d(&tmAhi, a_full, a_s + kb * L::A_PART, kb * BKE, m * BM);
              tma_load_2d(&tmAlo, a_full, a_s + (2 + kb) * L::A_PART, kb * BKE, m * BM);
            }
          }
          cur_m = m;
          ++gen;
        }
        const int s = i % BS;
        mbar_wait(b_empty + s, ((i / BS) & 1) ^ 1);
        mbar_expect_tx(b_full + s, L::B_STAGE);
        uint8_t* bs = b_s + s * L::B_STAGE;
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          tma_load_2d(&tmBhi, b_full + s, bs + (2 * kb) * L::B_PART, kb * BKE, n * 64);
          tma_load_2d(&tmBlo, b_full + s, bs + (2 * kb + 1) * L::B_PART, kb * BKE, n * 64);
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (warp-wide loop, elected issue)
    constexpr uint32_t id128 = idesc_tf32(BM, 128, 0, 0);
    constexpr uint32_t id64 = idesc_tf32(BM, 64, 0, 0);
    const uint32_t as = smem_u32(a_s);
    const uint32_t bs0 = smem_u32(b_s);
    int cur_m = -1, gen = 0;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int m = t / p.n_tiles;
      if (m != cur_m) {
        mbar_wait(a_full, gen & 1);
        cur_m = m;
        ++gen;
      }
      const int s = i % BS, buf = i & 1;
      mbar_wait(acc_empty + buf, ((i >> 1) & 1) ^ 1);
      if (p.trace && blockIdx.x == 0 && lane == 0 && i < 32) p.trace[i] = clock64();
      mbar_wait(b_full + s, (i / BS) & 1);
      if (p.trace && blockIdx.x == 0 && lane == 0 && i < 32) p.trace[32 + i] = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (elect_one()) {
        const uint32_t d = tmem + static_cast<uint32_t>(buf) * 128u;
        const uint32_t bs = bs0 + static_cast<uint32_t>(s) * L::B_STAGE;
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
          for (int kk = 0; kk < BKE / 8; ++kk) {
            const uint64_t bd = smem_desc(bs + 2 * kb * L::B_PART + kk * 32, 16, 1024);  // [hi; lo]
            if constexpr (SCATTER) {  // A from TMEM: no shared-memory A reads per tile
              const uint32_t at = tmem + kDxTmemA + static_cast<uint32_t>(kb * 32 + kk * 8);
              mma_tf32_ts(d, at, bd, id128, (kb > 0 || kk > 0) ? 1u : 0u);
              mma_tf32_ts(d, at + 64u, bd, id64, 1u);
            } else {
              const uint64_t ah = smem_desc(as + kb * L::A_PART + kk * 32, 16, 1024);
              const uint64_t al = smem_desc(as + (2 + kb) * L::A_PART + kk * 32, 16, 1024);
              mma_tf32(d, ah, bd, id128, (kb > 0 || kk > 0) ? 1u : 0u);
              mma_tf32(d, al, bd, id64, 1u);
            }
          }
        }
        mma_commit(b_empty + s);
        mma_commit(acc_full + buf);
        const int mn = (t + 1) / p.n_tiles;
        if (t + 1 >= t1 || mn != m) mma_commit(a_empty);
      }
      __syncwarp();
    }
  } else if (SCATTER && warp >= kDxAWriter0) {  // ---------------- A writer (SCATTER)
    // dh hi / lo rows of the current 128-row tile into TMEM columns [kDxTmemA, +128): warp
    // (lane quarter q) writes rows 32 q .. 32 q + 31, thread = row; once per tile row, after
    // the MMAs of the previous one have completed (a_empty)
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int cur_m = -1, gen = 0;
    for (int t = t0; t < t1; ++t) {
      const int m = t / p.n_tiles;
      if (m == cur_m) continue;
      if (gen > 0) mbar_wait(a_empty, (gen - 1) & 1);
      const int row = m * BM + q * 32 + lane;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int part = 0; part < 4; ++part) {  // hi k 0-31, hi k 32-63, lo k 0-31, lo k 32-63
        const float* src = (part < 2 ? p.a_hi : p.a_lo) + static_cast<int64_t>(row) * p.lda +
                           (part & 1) * 32;
        float v[32];
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          const int k = (part & 1) * 32 + 4 * k4;  // column of dh (contraction index)
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < p.M) {
            if (k + 4 <= p.H) {
              x = __ldg(reinterpret_cast<const float4*>(src) + k4);
            } else if (k < p.H) {  // the row's last partial group (H % 4 != 0)
              x.x = __ldg(src + 4 * k4);
              if (k + 1 < p.H) x.y = __ldg(src + 4 * k4 + 1);
              if (k + 2 < p.H) x.z = __ldg(src + 4 * k4 + 2);
            }
          }
          v[4 * k4] = x.x;
          v[4 * k4 + 1] = x.y;
          v[4 * k4 + 2] = x.z;
          v[4 * k4 + 3] = x.w;
        }
        tmem_st32(tmem + kDxTmemA + static_cast<uint32_t>(part * 32) + lane_off, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full);
      cur_m = m;
      ++gen;
    }
  } else if constexpr (SCATTER) {  // ---------------- scatter epilogue (segment sum)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    constexpr int EW = kDxScatterWarps, CW = 64 / (EW / 4);  // columns each warp drains
    const int et = threadIdx.x - 64;  // 0 .. 32 EW - 1
    const int ew = et >> 5;           // epilogue warp
    const int h = ew >> 2;            // column slice [CW h, CW h + CW) this warp drains
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const int F = p.F, d = p.d;
    float* tile = reinterpret_cast<float*>(out_s);
    uint32_t* vid_s = reinterpret_cast<uint32_t*>(out_s + BM * kDxTileStride * 4);
    float* gz_s = reinterpret_cast<float*>(vid_s + BM * F);
    int cur_m = -1;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int m = t / p.n_tiles, n = t - m * p.n_tiles;
      const int buf = i & 1;
      const int r0 = m * BM;
      // epi 1 has no per-tile barrier: every warp must be past the previous tile row's
      // scatter before its tables are restaged, and the staging done before they are read
      if (p.epi == 1 && m != cur_m && cur_m >= 0)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (m != cur_m) {  // stage this m-tile's vid / gz (the previous tile's scatter is done)
        // 8 independent loads in flight per thread (a plain loop is a chain of dependent
        // L2 round trips: ~10 per thread per m-tile, twice that with the remap)
        const int nst = BM * F;
        for (int base = 0; base < nst; base += 32 * EW * 8) {
          uint32_t v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int idx = base + u * 32 * EW + et;
            const bool in = idx < nst && r0 + idx / F < p.M;
            v[u] = in ? __ldg(p.vid + static_cast<int64_t>(r0) * F + idx) : 0u;
          }
          if (p.remap) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int idx = base + u * 32 * EW + et;
              if (idx < nst && r0 + idx / F < p.M) v[u] = __ldg(p.remap + v[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int idx = base + u * 32 * EW + et;
            if (idx < nst) vid_s[idx] = v[u];
          }
        }
        if (et < BM) gz_s[et] = r0 + et < p.M ? __ldg(p.gz + r0 + et) : 0.f;
        cur_m = m;
        if (p.epi == 1) asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      }
      if (p.epi == 1) {
        // warp (q, h) owns rows 32 q .. 32 q + 31 and columns 16 h .. 16 h + 15 of the tile.
        // After the TMEM drain (thread = row) a register transpose gives, for k = 0..3, lane l
        // the 16 B chunk (l & 3) of row 8 k + (l >> 2): each red covers 8 rows x 64 B
        const int cl = lane & 3;
        const int col = n * 64 + 16 * h + 4 * cl;
        const int f = col / d, cc = col - f * d;
        float4 fmk[4];
        bool okk[4];
        int rrk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          rrk[k] = q * 32 + 8 * k + (lane >> 2);
          okk[k] = r0 + rrk[k] < p.M && col < p.N;
          fmk[k] = okk[k] && p.exp != 2 ? __ldg(reinterpret_cast<const float4*>(
                                             p.fm_s + static_cast<int64_t>(r0 + rrk[k]) * d + cc))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        mbar_wait(acc_full + buf, (i >> 1) & 1);
        const bool trc = p.trace && blockIdx.x == 0 && et == 0 && i < 32;
        if (trc) p.trace[64 + i] = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t trow = tmem + static_cast<uint32_t>(buf) * 128u + lane_off;
        float v[16], w[16];
        tmem_ld16(trow + 16 * h, v);
        tmem_ld16(trow + 64 + 16 * h, w);
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] += w[c];
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + buf);  // the MMA of the next tile may start
        if (trc) p.trace[96 + i] = clock64();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int src = 8 * k + (lane >> 2);
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 4; ++c) {  // the source row's chunk c; lane keeps c == cl
            const float x0 = __shfl_sync(0xFFFFFFFFu, v[4 * c], src);
            const float x1 = __shfl_sync(0xFFFFFFFFu, v[4 * c + 1], src);
            const float x2 = __shfl_sync(0xFFFFFFFFu, v[4 * c + 2], src);
            const float x3 = __shfl_sync(0xFFFFFFFFu, v[4 * c + 3], src);
            if (c == cl) a = make_float4(x0, x1, x2, x3);
          }
          if (!okk[k] || p.exp == 1 || p.exp == 3) continue;
          const int rr = rrk[k];
          const float g = gz_s[rr];
          const float kf = p.scale * g;
          const uint32_t u = vid_s[rr * F + f];
          float* dstg = p.dG + static_cast<int64_t>(u) * d + cc;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dstg),
                       "f"(p.scale * a.x + kf * fmk[k].x), "f"(p.scale * a.y + kf * fmk[k].y),
                       "f"(p.scale * a.z + kf * fmk[k].z), "f"(p.scale * a.w + kf * fmk[k].w));
          if (cc == 0) atomicAdd(p.Bsum + u, g);
        }
        if (trc) p.trace[128 + i] = clock64();
        if (trc) p.trace[160 + i] = clock64();
        continue;
      }
      // (0) this tile's FM sums (they do not depend on the accumulator): loads issued
      // before the wait, so their L2 latency overlaps the MMA / TMEM drain
      const int j = lane & 15;
      const int col = n * 64 + 4 * j;
      const int f = col / d, cc = col - f * d;
      constexpr int NB = BM / (2 * EW);  // rows per half-warp per tile
      static_assert(NB >= 1 && NB <= 8, "scatter epilogue row split");
      float4 fm[NB];
      bool ok[NB];
#pragma unroll
      for (int u8 = 0; u8 < NB; ++u8) {
        const int rr = 2 * EW * u8 + 2 * ew + (lane >> 4);
        ok[u8] = r0 + rr < p.M && col < p.N;
        fm[u8] = ok[u8] && p.exp != 2 ? __ldg(reinterpret_cast<const float4*>(
                              p.fm_s + static_cast<int64_t>(r0 + rr) * d + cc))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      mbar_wait(acc_full + buf, (i >> 1) & 1);
      const bool trc = p.trace && blockIdx.x == 0 && et == 0 && i < 32;
      if (trc) p.trace[64 + i] = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // (1) accumulator -> value tile, thread = row
      const uint32_t trow = tmem + static_cast<uint32_t>(buf) * 128u + lane_off;
#pragma unroll
      for (int c0 = CW * h; c0 < CW * h + CW; c0 += 16) {
        float v[16], w[16];
        tmem_ld16(trow + c0, v);
        tmem_ld16(trow + 64 + c0, w);
        float4* dst = reinterpret_cast<float4*>(tile + row * kDxTileStride + c0);
        if (p.exp == 3) {  // experiment: drain only (no shared-memory tile, no scatter)
          if (v[0] + w[0] == 12345.f) p.dG[0] = v[1];
          continue;
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          dst[jj] = make_float4(v[4 * jj] + w[4 * jj], v[4 * jj + 1] + w[4 * jj + 1],
                                v[4 * jj + 2] + w[4 * jj + 2], v[4 * jj + 3] + w[4 * jj + 3]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + buf);  // the MMA of the next tile may start
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
      if (trc) p.trace[96 + i] = clock64();
      // (2) half-warp per row: lane & 15 = 16 B chunk of the tile's 64 columns
#pragma unroll
      for (int u8 = 0; u8 < NB && p.exp != 3; ++u8) {
        const int rr = 2 * EW * u8 + 2 * ew + (lane >> 4);
        if (!ok[u8]) continue;
        const float4 a = *reinterpret_cast<const float4*>(tile + rr * kDxTileStride + 4 * j);
        const float g = gz_s[rr];
        const float k = p.scale * g;
        const uint32_t u = vid_s[rr * F + f];
        float* dstg = p.dG + static_cast<int64_t>(u) * d + cc;
        if (p.exp == 1) continue;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dstg),
                     "f"(p.scale * a.x + k * fm[u8].x), "f"(p.scale * a.y + k * fm[u8].y),
                     "f"(p.scale * a.z + k * fm[u8].z), "f"(p.scale * a.w + k * fm[u8].w));
        if (cc == 0) atomicAdd(p.Bsum + u, g);
      }
      if (trc) p.trace[128 + i] = clock64();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // value tile / tables free
      if (trc) p.trace[160 + i] = clock64();
    }
  } else {  // ---------------- epilogue
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const bool leader = threadIdx.x == 64;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int m = t / p.n_tiles, n = t - m * p.n_tiles;
      const int buf = i & 1;
      mbar_wait(acc_full + buf, (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // the previous tile's TMA store must have finished reading the staging buffer
      if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const uint32_t trow = tmem + static_cast<uint32_t>(buf) * 128u + lane_off;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16], w[16];
        tmem_ld16(trow + c0, v);
        tmem_ld16(trow + 64 + c0, w);
        float4* box = reinterpret_cast<float4*>(out_s + (c0 >> 5) * (BM * 128) + row * 128);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int chunk = ((c0 & 31) >> 2) + j;
          box[chunk ^ (row & 7)] =
              make_float4(p.scale * (v[4 * j] + w[4 * j]), p.scale * (v[4 * j + 1] + w[4 * j + 1]),
                          p.scale * (v[4 * j + 2] + w[4 * j + 2]),
                          p.scale * (v[4 * j + 3] + w[4 * j + 3]));
        }
      }
      // accumulator drained: hand it back to the MMA warp (one arrival per warp)
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + buf);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (leader) {
        tma_store_2d(&tmOut, out_s, n * 64, m * BM);
        tma_store_2d(&tmOut, out_s + BM * 128, n * 64 + 32, m * BM);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (p.cta_trace && threadIdx.x == 0) p.cta_trace[2 * blockIdx.x + 1] = global_ns();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(SCATTER ? 512 : 256));
  }
}

}  // namespace tc
}  // namespace sfb
