// Blackwell (sm_100a) tensor-core GEMM for the DeepFM-lite tower:
// tcgen05.mma kind::tf32 with TMEM accumulators, TMA-fed shared-memory
// stages, and the 3xTF32 split (a*b ~= ah*bh + ah*bl + al*bh, each part
// rounded to tf32) so that fp32-level accuracy is kept against the fp64
// oracle.
//
// One CTA = 6 warps:
//   warp 0     : TMA producer (one elected lane) into a ring of smem stages
//   warp 1     : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5 : split the A tile in place into (hi, lo) tf32 parts when A is
//                not pre-split, then run the epilogue (tcgen05.ld TMEM ->
//                registers -> global)
// M tile = 128 rows (TMEM lane = row), N tile = BN columns, K block = 32 fp32
// (one 128 B swizzle span). Operands use the canonical SWIZZLE_128B layouts
// that TMA writes: K-major (8-row x 128 B atoms) or MN-major (32-element x
// 8-row atoms, A only).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace sfb {
namespace tc {

// The dynamic shared memory rounded up to 1024 B (SWIZZLE_128B operands need it) by pointer
// arithmetic on the shared array itself: an integer round trip through uintptr_t loses the
// address space, and every access through the result becomes a generic LD.E / ST.E instead
// of LDS / STS.
__device__ __forceinline__ uint8_t* smem_1024(uint8_t* raw) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
  return raw + ((1024u - (a & 1023u)) & 1023u);
}


constexpr int BM = 128;
constexpr int BKE = 32;                  // K elements per block (128 B)
constexpr int A_BYTES = BM * BKE * 4;    // 16 KB

enum Epi : int { kEpiStore = 0, kEpiDx = 1 };

struct Params {
  int M, N, K;            // logical GEMM sizes
  int num_k_blocks;       // ceil(K / 32)
  int k_blocks_per_split; // blockIdx.z covers [z*kps, (z+1)*kps)
  // kEpiStore: out[z][m][n] with leading dim ldo, split stride split_stride
  float* out;
  int ldo;
  long long split_stride;
  // kEpiDx: dX[m][n] = scale * (acc + gz[m] * (fm_s[m][n % d] - X[m][n])), ld = ldx
  const float* gz;
  const float* fm_s;
  const float* X;
  int ldx;
  int d;
  float scale;
  // MN-major A descriptor strides (bytes): between 32-element MN atoms, between
  // 4-row K groups of the SWIZZLE_128B_BASE32B layout
  uint32_t mn_lbo = 4096;
  uint32_t mn_sbo = 512;
  // profiling knobs (0 in production): bit0 skip the split arithmetic, bit1 skip
  // the MMAs, bit2 skip the A loads, bit3 skip the B loads
  int dbg = 0;
  long long* trace = nullptr;  // profiling: per-k-block clock64 stamps of CTA 0 (scratch only)
  unsigned long long* cta_trace = nullptr;  // profiling: per-CTA [start, end] globaltimer
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait with a back-off between polls: for barriers the tensor core arrives on
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, int ns) {
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}

// TMA prefetch of a box into L2 (no smem, no barrier): lets the producer run
// far ahead of the smem ring so DRAM latency overlaps the stages in flight.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// sm_100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48),
// base offset 0, layout type [61,64): 2 = SWIZZLE_128B (16 B chunks, 8-row
// atoms; K-major operands), 1 = SWIZZLE_128B_BASE32B (32 B chunks, 4-row
// atoms; the only layout tcgen05 accepts for MN-major tf32 operands).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout = 2) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// Instruction descriptor for kind::tf32 (cute::UMMA::InstrDescriptor):
// c_format F32 (1) at [4,6), a/b format TF32 (2) at [7,10)/[10,13),
// a_major [15], b_major [16], N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand in TMEM (tcgen05.mma ... [d], [a_tmem], b_desc): the streamed GEMMs (tc_ts.cuh)
// and the dX GEMM (tc_dx.cuh)
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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// one lane of a converged warp; the MMA issuer runs its loop warp-wide and issues under
// elect_one() so the descriptors stay in uniform registers (a lane-0-only loop makes the
// compiler move every operand with R2UR in front of each tcgen05.mma, a serial chain)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Round to the nearest tf32 (ties away from zero) = cvt.rna.tf32.f32 for finite x, in two
// integer ops: ptxas expands cvt.rna.tf32 on sm_100a into an inf/nan-guarded sequence
// (FSETP + SEL + ...), and the split warps of the X-streaming GEMMs (tc_ts.cuh) run 64 of
// these per row per k-block, which made the split the pacing stage of GEMM1 / GEMM3.
// (Non-finite inputs are never split: a non-finite activation already fails the step.)
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// MAXST caps the ring depth: a short-K GEMM needs few stages, and a smaller
// footprint lets several CTAs share an SM to overlap each other's latencies.
template <int BN, int MAXST = 6>
struct Layout {
  static constexpr int B_BYTES = BN * BKE * 4;  // K-major B tile, 128 B per row
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES_FIT = STAGES_RAW > 6 ? 6 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int STAGES = STAGES_FIT < MAXST ? STAGES_FIT : MAXST;
  static_assert(STAGES * STAGE_BYTES >= BM * (BN + 1) * 4, "epilogue tile must fit the ring");
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  // dynamic smem: 1 KB alignment slack + stages + barriers
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

// A_MN: A is MN-major (4 TMA boxes of 32 m x 32 k); otherwise K-major (box 32 k x 128 m).
// SPLIT_A: A arrives as raw fp32 and is split in smem; otherwise tmAlo supplies the lo part.
// B_MN: B is MN-major (BN/32 TMA boxes of 32 n x 32 k, BASE32B layout); otherwise K-major.
template <int BN, bool A_MN, bool SPLIT_A, int EPI, bool B_MN = false, int MAXST = 6>
__global__ void __launch_bounds__(192, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmAlo,
                       const __grid_constant__ CUtensorMap tmBhi,
                       const __grid_constant__ CUtensorMap tmBlo, const Params p) {
  using L = Layout<BN, MAXST>;
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
  // CTAs sharing a B tile start at different k-blocks so that they do not all
  // hit the same L2 lines at the same moment (every M tile reads all of B)
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
    if (lane == 0) {  // ---------------- TMA producer
      constexpr uint32_t bytes = (SPLIT_A ? A_BYTES : 2 * A_BYTES) + 2 * L::B_BYTES;
      constexpr int PD = 2 * ST;  // L2 prefetch distance (k-blocks) for the streamed A operand
      auto prefetch_a = [&](int i) {
        const int kc = kblk(i) * BKE;
        if constexpr (A_MN) {
#pragma unroll
          for (int a = 0; a < 4; ++a) tma_prefetch_2d(&tmA, m0 + a * 32, kc);
        } else {
          tma_prefetch_2d(&tmA, kc, m0);
        }
      };
      if constexpr (SPLIT_A)
        for (int i = 0; i < PD && i < nkb; ++i) prefetch_a(i);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        if constexpr (SPLIT_A)
          if (i + PD < nkb) prefetch_a(i + PD);
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect_tx(full + s, bytes - ((p.dbg & 4) ? A_BYTES : 0) - ((p.dbg & 8) ? 2 * L::B_BYTES : 0));
        const int kc = kblk(i) * BKE;
        if (p.dbg & 4) {
        } else if constexpr (A_MN) {
#pragma unroll
          for (int a = 0; a < 4; ++a) tma_load_2d(&tmA, full + s, a_hi(s) + a * 4096, m0 + a * 32, kc);
        } else {
          tma_load_2d(&tmA, full + s, a_hi(s), kc, m0);
          if constexpr (!SPLIT_A) tma_load_2d(&tmAlo, full + s, a_lo(s), kc, m0);
        }
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
      static_assert(!B_MN || BN % 32 == 0, "MN-major B needs whole 32-column atoms");
      constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        if constexpr (SPLIT_A) mbar_wait(ready + s, ph);
        else mbar_wait(full + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t ah, al;
          if constexpr (A_MN) {  // 8 k-rows = two 512 B K-groups; MN atoms 4 KB apart
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 1024, p.mn_lbo, p.mn_sbo, 1);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 1024, p.mn_lbo, p.mn_sbo, 1);
          } else {  // K-major: advance 32 B inside the 128 B swizzle row
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 32, 16, 1024);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 32, 16, 1024);
          }
          uint64_t bh, bl;
          if constexpr (B_MN) {
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 1024, 4096, 512, 1);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 1024, 4096, 512, 1);
          } else {
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 32, 16, 1024);
          }
          if (p.dbg & 2) continue;
          mma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, ah, bl, idesc, 1u);
          mma_tf32(tmem, al, bh, idesc, 1u);
        }
        mma_commit(empty + s);  // frees the stage once these MMAs have read it
      }
      mma_commit(tmem_full);
    }
  } else {
    const int t = threadIdx.x - 64;  // 0..127
    if constexpr (SPLIT_A) {         // ---------------- in-place 3xTF32 split of A
      for (int i = 0; i < nkb; ++i) {
        const int s = i % ST;
        const uint32_t ph = (i / ST) & 1;
        mbar_wait(full + s, ph);
        float4* hi = reinterpret_cast<float4*>(a_hi(s));
        float4* lo = reinterpret_cast<float4*>(a_lo(s));
#pragma unroll 4
        for (int e = t; e < A_BYTES / 16; e += 128) {
          if (p.dbg & 1) break;
          const float4 v = hi[e];
          float4 h, l;
          h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
          h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
          h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
          h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
          hi[e] = h;
          lo[e] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(ready + s);
      }
    }
    // ---------------- epilogue: TMEM lane quarter = warp % 4
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // (1) TMEM -> smem tile [128][BN+1] (one row per thread; the +1 pad makes
    //     the row-per-thread stores bank-conflict free). All MMAs have
    //     completed, so the stage ring is free to reuse.
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
    // (2) coalesced write-out: warp w2 takes rows w2, w2+4, ...; lanes sweep columns
    const int w2 = t >> 5;
    if (nkb > 0) {
#pragma unroll 1
      for (int r = w2; r < BM; r += 4) {
        const int m = m0 + r;
        if (m >= p.M) break;
        // store-only epilogue: no global loads, so nothing serialises on DRAM latency
        float* o = p.out + blockIdx.z * p.split_stride + static_cast<long long>(m) * p.ldo;
        const float sc = EPI == kEpiStore ? 1.f : p.scale;
#pragma unroll
        for (int c = lane; c < BN; c += 32) {
          const int n = n0 + c;
          if (n < p.N) o[n] = sc * tile[r * TS + c];
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

// Streaming-A variant with DECOUPLED rings (split A, store epilogue):
//   raw ring (RS x 16 KB)  : TMA lands raw fp32 A tiles; a slot is released as soon
//                            as the split warps have read it (not when the MMA is done)
//   operand ring (OS)      : tf32 hi/lo A parts + B hi/lo (B loaded by TMA when the
//                            split warps claim the stage), released by tcgen05.commit
// so DRAM latency is covered by RS raw stages while the split -> MMA hand-off runs
// on a short ring of its own.
constexpr int kRawStages = 6;
constexpr int kOpStages = 2;

template <int BN>
struct DecLayout {
  static constexpr int B_BYTES = BN * BKE * 4;
  static constexpr int OP_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int RAW_BYTES = kRawStages * A_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static_assert(RAW_BYTES >= BM * (BN + 1) * 4, "epilogue tile must fit the raw ring");
  static constexpr int SMEM = 1024 + RAW_BYTES + kOpStages * OP_BYTES + 512;
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(192, 1)
    gemm_tf32x3_dec_kernel(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmBhi,
                           const __grid_constant__ CUtensorMap tmBlo, const Params p) {
  using L = DecLayout<BN>;
  constexpr int RS = kRawStages, OS = kOpStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_1024(smem_raw);
  uint8_t* raw = smem;
  uint8_t* ops = smem + L::RAW_BYTES;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(ops + OS * L::OP_BYTES);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* op_bfull = raw_empty + RS;
  uint64_t* op_ready = op_bfull + OS;
  uint64_t* op_empty = op_ready + OS;
  uint64_t* tmem_full = op_empty + OS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto a_raw = [&](int s) { return raw + s * A_BYTES; };
  auto a_hi = [&](int s) { return ops + s * L::OP_BYTES; };
  auto a_lo = [&](int s) { return ops + s * L::OP_BYTES + A_BYTES; };
  auto b_hi = [&](int s) { return ops + s * L::OP_BYTES + 2 * A_BYTES; };
  auto b_lo = [&](int s) { return ops + s * L::OP_BYTES + 2 * A_BYTES + L::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.k_blocks_per_split;
  const int kb1 = min(p.num_k_blocks, kb0 + p.k_blocks_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(raw_full + s, 1);
      mbar_init(raw_empty + s, 128);
    }
    for (int s = 0; s < OS; ++s) {
      mbar_init(op_bfull + s, 1);
      mbar_init(op_ready + s, 128);
      mbar_init(op_empty + s, 1);
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
    if (lane == 0) {  // ---------------- raw A producer, RS stages ahead
      for (int i = 0; i < nkb; ++i) {
        const int s = i % RS;
        mbar_wait(raw_empty + s, ((i / RS) & 1) ^ 1);
        mbar_expect_tx(raw_full + s, A_BYTES);
        const int kc = (kb0 + i) * BKE;
        if constexpr (A_MN) {
#pragma unroll
          for (int a = 0; a < 4; ++a) tma_load_2d(&tmA, raw_full + s, a_raw(s) + a * 4096, m0 + a * 32, kc);
        } else {
          tma_load_2d(&tmA, raw_full + s, a_raw(s), kc, m0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_tf32(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % OS;
        const uint32_t ph = (i / OS) & 1;
        mbar_wait(op_ready + s, ph);
        mbar_wait(op_bfull + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BKE / 8; ++kk) {
          uint64_t ah, al, bh, bl;
          if constexpr (A_MN) {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 1024, 4096, 512, 1);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 1024, 4096, 512, 1);
          } else {
            ah = smem_desc(smem_u32(a_hi(s)) + kk * 32, 16, 1024);
            al = smem_desc(smem_u32(a_lo(s)) + kk * 32, 16, 1024);
          }
          if constexpr (B_MN) {
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 1024, 4096, 512, 1);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 1024, 4096, 512, 1);
          } else {
            bh = smem_desc(smem_u32(b_hi(s)) + kk * 32, 16, 1024);
            bl = smem_desc(smem_u32(b_lo(s)) + kk * 32, 16, 1024);
          }
          mma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, ah, bl, idesc, 1u);
          mma_tf32(tmem, al, bh, idesc, 1u);
        }
        mma_commit(op_empty + s);
      }
      mma_commit(tmem_full);
    }
  } else {
    const int t = threadIdx.x - 64;
    for (int i = 0; i < nkb; ++i) {  // ---------------- split raw -> operand stage
      const int s = i % OS;
      const int r = i % RS;
      mbar_wait(op_empty + s, ((i / OS) & 1) ^ 1);
      if (t == 0) {  // claim the operand stage: its B tiles
        mbar_expect_tx(op_bfull + s, 2 * L::B_BYTES);
        const int kc = (kb0 + i) * BKE;
        if constexpr (B_MN) {
#pragma unroll
          for (int b = 0; b < BN / 32; ++b) {
            tma_load_2d(&tmBhi, op_bfull + s, b_hi(s) + b * 4096, n0 + b * 32, kc);
            tma_load_2d(&tmBlo, op_bfull + s, b_lo(s) + b * 4096, n0 + b * 32, kc);
          }
        } else {
          tma_load_2d(&tmBhi, op_bfull + s, b_hi(s), kc, n0);
          tma_load_2d(&tmBlo, op_bfull + s, b_lo(s), kc, n0);
        }
      }
      mbar_wait(raw_full + r, (i / RS) & 1);
      const float4* src = reinterpret_cast<const float4*>(a_raw(r));
      float4* hi = reinterpret_cast<float4*>(a_hi(s));
      float4* lo = reinterpret_cast<float4*>(a_lo(s));
#pragma unroll 4
      for (int e = t; e < A_BYTES / 16; e += 128) {
        const float4 v = src[e];
        float4 h, l;
        h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
        h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
        h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
        h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
        hi[e] = h;
        lo[e] = l;
      }
      mbar_arrive(raw_empty + r);  // raw slot free for the next TMA
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(op_ready + s);
    }
    // ---------------- epilogue (split-K partials) staged through the raw ring
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float* tile = reinterpret_cast<float*>(raw);
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
        if (m >= p.M) break;
        float* o = p.out + blockIdx.z * p.split_stride + static_cast<long long>(m) * p.ldo;
#pragma unroll
        for (int c = lane; c < BN; c += 32) {
          const int n = n0 + c;
          if (n < p.N) o[n] = tile[rr * TS + c];
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
