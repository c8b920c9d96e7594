// Owner-routed embedding exchange (sync = alltoall; SURVEY §8f rank 2,
// PAPER.md:535 "All2All"): instead of all-reducing the zero-padded U x d
// common embedding and common gradients, every rank moves
// only the rows its own minibatch touches, straight from / to the row's owner.
//
// All ranks run the same VSI, so every rank can derive, without any request
// round, the touched mask tm[k] (bit w <=> worker w's rows contain unique k):
//   receive plan (me)  : R_o = [k : owner(k) = o, bit me]      -> local row lpos[k]
//   send plan (me = o) : S_w = [k owned by me : bit w]        -> send slot spos[j][w]
// Forward: owner packs S_w rows, grouped ncclSend/ncclRecv, rows land in the
// local table E (owner-major blocks). Backward: the local gradient table dE is
// sent back block by block; the owner sums the contributions of workers
// 0..W-1 in that fixed order (the reference's ordered sum).
#include "exchange.h"

#include <cstdlib>

namespace sfb {

namespace {

// tm[vid[i]] |= 1 << worker(i); warp peers with the same vid pre-combine
// Touched-by-worker masks without atomics: position i of worker w = i / per_worker stores a
// plain 1 into byte w of unique vid[i]'s 8-byte row (idempotent, no read-modify-write), and
// touch_pack turns the live rows into bit masks tm[k] and clears them for the next step.
// (The atomicOr formulation ran at ~20 G positions/s, bound by L2 atomics.)
__global__ void touch_mark_kernel(const uint32_t* __restrict__ vid, int64_t n, int64_t per_worker,
                                  uint8_t* __restrict__ tb8) {
  pdl_wait();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  tb8[static_cast<int64_t>(__ldg(vid + i)) * 8 + idiv(i, static_cast<int>(per_worker))] = 1;
}

__global__ void touch_pack_kernel(const int32_t* __restrict__ U, uint8_t* __restrict__ tb8,
                                  uint32_t* __restrict__ tm) {
  pdl_wait();
  const int32_t n = *U;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    uint64_t* row = reinterpret_cast<uint64_t*>(tb8) + k;
    const uint64_t x = *row;
    uint32_t m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m |= ((x >> (8 * w)) & 0xFFu) ? (1u << w) : 0u;
    tm[k] = m;
    *row = 0;
  }
}

__global__ void lvid_kernel(const uint32_t* __restrict__ vid, int64_t n,
                            const uint32_t* __restrict__ lpos, uint32_t* __restrict__ lvid) {
  pdl_wait();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) lvid[i] = lpos[vid[i]];
}

// Forward pack: owned row j goes to sendbuf[soff[w] + spos[j][w]] for every
// remote worker w that touches it, and to E[lpos] when I touch it myself.
// One warp per owned row, 16 B lanes.
__global__ void pack_rows_kernel(const uint32_t* __restrict__ own_k,
                                 const uint32_t* __restrict__ own_slot, int32_t n_own,
                                 const uint32_t* __restrict__ tm, const Cnt8* __restrict__ sscan,
                                 const int32_t* __restrict__ totals, uint32_t W, uint32_t me,
                                 const uint32_t* __restrict__ lpos, const float4* __restrict__ emb,
                                 int d4, float4* __restrict__ sendbuf, float4* __restrict__ E) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n_own) return;
  const uint32_t k = own_k[j];
  const uint32_t m = tm[k];
  const float4* src = emb + static_cast<int64_t>(own_slot[j]) * 3 * d4;  // [emb | m | v] rows
  uint32_t soff = 0;
  for (uint32_t w = 0; w < W; ++w) {
    if ((m >> w) & 1u) {
      float4* dst = (w == me) ? E + static_cast<int64_t>(lpos[k]) * d4
                              : sendbuf + static_cast<int64_t>(soff + sscan[j].c[w]) * d4;
      for (int c = lane; c < d4; c += 32) dst[c] = src[c];
    }
    if (w != me) soff += static_cast<uint32_t>(totals[8 + w]);
  }
}

// Backward: g[j] = sum over w = 0..W-1 (fixed order) of worker w's partial
// gradient of owned row j (mine from dE, the others from recvbuf).
__global__ void owner_reduce_kernel(const uint32_t* __restrict__ own_k, int32_t n_own,
                                    const uint32_t* __restrict__ tm, const Cnt8* __restrict__ sscan,
                                    const int32_t* __restrict__ totals, uint32_t W, uint32_t me,
                                    const uint32_t* __restrict__ lpos, const float4* __restrict__ dE,
                                    const float4* __restrict__ recvbuf, int d4,
                                    float4* __restrict__ g) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(n_own) * d4) return;
  const int64_t j = idiv(i, d4);
  const int c = static_cast<int>(i - j * d4);
  const uint32_t k = own_k[j];
  const uint32_t m = tm[k];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t soff = 0;
  for (uint32_t w = 0; w < W; ++w) {
    if ((m >> w) & 1u) {
      const float4 v = (w == me) ? dE[static_cast<int64_t>(lpos[k]) * d4 + c]
                                 : recvbuf[static_cast<int64_t>(soff + sscan[j].c[w]) * d4 + c];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (w != me) soff += static_cast<uint32_t>(totals[8 + w]);
  }
  g[i] = acc;
}

__global__ void offsets_kernel(const int32_t* __restrict__ totals, int me,
                               int32_t* __restrict__ offs);

}  // namespace

void Exchange::init(int W_, int me_, int64_t cap_, int d_) {
  release();
  W = W_;
  me = me_;
  cap = cap_;
  d = d_;
  SFB_CHECK(W <= 8, "alltoall sync supports at most 8 workers");
  SFB_CHECK((d & 3) == 0, "alltoall sync needs embedding_dim % 4 == 0");
  const int ntiles = ceil_div(cap, 1024);
  CUDA_CHECK(cudaMalloc(&tb8, 8 * static_cast<size_t>(cap)));
  CUDA_CHECK(cudaMemset(tb8, 0, 8 * static_cast<size_t>(cap)));
  for (PlanSet& p : sets) {
    CUDA_CHECK(cudaMalloc(&p.tm, sizeof(uint32_t) * cap));
    CUDA_CHECK(cudaMalloc(&p.lpos, sizeof(uint32_t) * cap));
    CUDA_CHECK(cudaMalloc(&p.sscan, sizeof(Cnt8) * cap));
    CUDA_CHECK(cudaMalloc(&p.tile_cnt, sizeof(uint32_t) * 2 * 8 * ntiles));  // recv | send tables
    CUDA_CHECK(cudaMalloc(&p.tile_off, sizeof(uint32_t) * 2 * 8 * ntiles));
    CUDA_CHECK(cudaMalloc(&p.totals, sizeof(int32_t) * kTotals));
    CUDA_CHECK(cudaMalloc(&p.offs, sizeof(int32_t) * 160));
    CUDA_CHECK(cudaMemset(p.offs, 0, sizeof(int32_t) * 160));
  }
  use(0);
  CUDA_CHECK(cudaMalloc(&buf, sizeof(float) * cap * d));
  CUDA_CHECK(cudaMalloc(&gown, sizeof(float) * cap * d));
}

void Exchange::release() {
  if (p2p)
    for (int w = 0; w < W; ++w) {
      if (w == me) continue;
      if (peer_E[w]) cudaIpcCloseMemHandle(peer_E[w]);
      if (peer_buf[w]) cudaIpcCloseMemHandle(peer_buf[w]);
      if (peer_flags[w]) cudaIpcCloseMemHandle(peer_flags[w]);
    }
  if (bar) cudaFree(bar);
  if (flags) cudaFree(flags);
  for (const PlanSet& q : sets)
    for (void* p : {static_cast<void*>(q.tm), static_cast<void*>(q.lpos),
                    static_cast<void*>(q.sscan), static_cast<void*>(q.tile_cnt),
                    static_cast<void*>(q.tile_off), static_cast<void*>(q.totals),
                    static_cast<void*>(q.offs)})
      if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(buf), static_cast<void*>(gown), static_cast<void*>(tb8)})
    if (p) cudaFree(p);
  *this = Exchange();
}

namespace {

__global__ void count_matrix_kernel(const uint32_t* __restrict__ uniq,
                                    const int32_t* __restrict__ U, int cap,
                                    const uint32_t* __restrict__ tm, uint32_t W,
                                    int32_t* __restrict__ cnt);

// ---- multi-plane ranking: for every element with mask bits p, its rank among
// the earlier elements that have bit p (8 planes at once, ballot + popc). A
// tile is 4 rounds x 256 threads = 1024 elements.
constexpr int kTile = 1024;

// element mask: receive plan = bit(owner) if I touch unique k; send plan = touched mask
template <bool SEND>
__device__ __forceinline__ uint32_t plan_mask(int i, const uint32_t* __restrict__ keys,
                                              const int32_t* __restrict__ live,
                                              const uint32_t* __restrict__ tm, uint32_t W,
                                              uint32_t me) {
  if (i >= *live) return 0u;
  if (SEND) return tm[keys[i]] & ((1u << W) - 1u);  // keys = own_k
  return ((tm[i] >> me) & 1u) ? (1u << (keys[i] % W)) : 0u;  // keys = uniq
}

template <bool SEND>
__device__ __forceinline__ void plan_count_tile(int tile, const uint32_t* __restrict__ keys,
                                                const int32_t* __restrict__ live, int cap,
                                                const uint32_t* __restrict__ tm, uint32_t W,
                                                uint32_t me, uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t wc[8][8];  // [warp][plane]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = 0; r < 4; ++r) {
    const int i = tile * kTile + r * 256 + threadIdx.x;
    const uint32_t m = i < cap ? plan_mask<SEND>(i, keys, live, tm, W, me) : 0u;
#pragma unroll
    for (int p = 0; p < 8; ++p) acc[p] += __popc(__ballot_sync(0xFFFFFFFFu, (m >> p) & 1u));
  }
  if (lane == 0)
#pragma unroll
    for (int p = 0; p < 8; ++p) wc[warp][p] = acc[p];
  __syncthreads();
  if (threadIdx.x < 8) {
    uint32_t s = 0;
    for (int w = 0; w < 8; ++w) s += wc[w][threadIdx.x];
    tile_cnt[tile * 8 + threadIdx.x] = s;
  }
  __syncthreads();  // wc is reused by the CTA's next tile
}

// warp p scans plane p over the tiles (exclusive), totals[p] = plane total
// two tables at once (receive plan, send plan): warp q < 16 scans plane q % 8 of table q / 8.
// Only the tiles holding live elements (live0 / live1: the tables' element counts) are
// scanned (the others rank nothing), four 32-tile chunks' loads in flight at a time.
__global__ void plan_scan_tiles_kernel(const uint32_t* __restrict__ tile_cnt_all, int ntiles,
                                       uint32_t* __restrict__ tile_off_all,
                                       int32_t* __restrict__ totals_all,
                                       const int32_t* __restrict__ live0,
                                       const int32_t* __restrict__ live1) {
  pdl_wait();
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q >= 16) return;
  const int p = q & 7;
  const uint32_t* tile_cnt = tile_cnt_all + (q >> 3) * ntiles * 8;
  uint32_t* tile_off = tile_off_all + (q >> 3) * ntiles * 8;
  int32_t* totals = totals_all + (q >> 3) * 8;
  const int32_t live = max(0, *((q >> 3) ? live1 : live0));
  const int nt = min(ntiles, (live + kTile - 1) / kTile);
  uint32_t carry = 0;
  for (int t0 = 0; t0 < nt; t0 += 128) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * 32 + lane;
      v[u] = t < nt ? tile_cnt[t * 8 + p] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * 32 + lane;
      uint32_t x = v[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      if (t < nt) tile_off[t * 8 + p] = carry + x - v[u];
      carry += __shfl_sync(0xFFFFFFFFu, x, 31);
    }
  }
  if (lane == 0) totals[p] = static_cast<int32_t>(carry);
}

template <bool SEND>
__device__ __forceinline__ void plan_rank_tile(int tile, const uint32_t* __restrict__ keys,
                                                        const int32_t* __restrict__ live, int cap,
                                                        const uint32_t* __restrict__ tm,
                                                        uint32_t W, uint32_t me,
                                                        const uint32_t* __restrict__ tile_off,
                                                        const int32_t* __restrict__ totals,
                                                        Cnt8* __restrict__ ranks,
                                                        uint32_t* __restrict__ lpos) {
  __shared__ uint32_t wc[4][8][8];  // [round][warp][plane] -> exclusive offsets in tile order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t m[4], pre[4][8];
  for (int r = 0; r < 4; ++r) {
    const int i = tile * kTile + r * 256 + threadIdx.x;
    m[r] = i < cap ? plan_mask<SEND>(i, keys, live, tm, W, me) : 0u;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const unsigned b = __ballot_sync(0xFFFFFFFFu, (m[r] >> p) & 1u);
      pre[r][p] = __popc(b & lt);
      if (lane == 0) wc[r][warp][p] = __popc(b);
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) {  // plane p: exclusive prefix over (round, warp) in tile order
    const int p = threadIdx.x;
    uint32_t run = tile_off[tile * 8 + p];
    for (int rr = 0; rr < 4; ++rr)
      for (int w = 0; w < 8; ++w) {
        const uint32_t c = wc[rr][w][p];
        wc[rr][w][p] = run;
        run += c;
      }
  }
  __syncthreads();
  for (int r = 0; r < 4; ++r) {
    const int i = tile * kTile + r * 256 + threadIdx.x;
    if (i >= cap) continue;
    Cnt8 out{};
#pragma unroll
    for (int p = 0; p < 8; ++p) out.c[p] = wc[r][warp][p] + pre[r][p];
    if (SEND) {
      ranks[i] = out;
    } else if (m[r]) {  // lpos = owner block offset + rank within the owner's block
      const uint32_t o = __ffs(m[r]) - 1;
      uint32_t base = 0;
      for (uint32_t q = 0; q < o; ++q) base += static_cast<uint32_t>(totals[q]);
      lpos[i] = base + out.c[o];
    } else {
      lpos[i] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();  // wc is reused by the CTA's next tile
}


// blockIdx.y = 0: receive plan over the uniques; 1: send plan over my owned uniques
// (send_only: blockIdx.y = 0 is the send plan). Persistent over the table's tiles; tiles past
// the live count are neither counted nor ranked (the tile scan stops at the last live one)
__global__ void __launch_bounds__(256) plan_count_kernel(
    const uint32_t* __restrict__ uniq, const int32_t* __restrict__ U,
    const uint32_t* __restrict__ own_k, const int32_t* __restrict__ n_own, int cap,
    const uint32_t* __restrict__ tm, uint32_t W, uint32_t me, int ntiles,
    uint32_t* __restrict__ tile_cnt, int send_only) {
  pdl_wait();
  const bool send = send_only || blockIdx.y == 1;
  const int32_t live = send ? *n_own : *U;
  for (int tile = blockIdx.x; tile < ntiles && tile * kTile < live; tile += gridDim.x) {
    if (send) plan_count_tile<true>(tile, own_k, n_own, cap, tm, W, me, tile_cnt + ntiles * 8);
    else plan_count_tile<false>(tile, uniq, U, cap, tm, W, me, tile_cnt);
  }
}

__global__ void __launch_bounds__(256) plan_rank_kernel(
    const uint32_t* __restrict__ uniq, const int32_t* __restrict__ U,
    const uint32_t* __restrict__ own_k, const int32_t* __restrict__ n_own, int cap,
    const uint32_t* __restrict__ tm, uint32_t W, uint32_t me, int ntiles,
    const uint32_t* __restrict__ tile_off, const int32_t* __restrict__ totals,
    Cnt8* __restrict__ sscan, uint32_t* __restrict__ lpos, int send_only) {
  pdl_wait();
  const bool send = send_only || blockIdx.y == 1;
  const int32_t live = send ? *n_own : *U;
  for (int tile = blockIdx.x; tile < ntiles && tile * kTile < live; tile += gridDim.x) {
    if (send)
      plan_rank_tile<true>(tile, own_k, n_own, cap, tm, W, me, tile_off + ntiles * 8, totals,
                           sscan, nullptr);
    else
      plan_rank_tile<false>(tile, uniq, U, cap, tm, W, me, tile_off, totals, nullptr, lpos);
  }
}

// The send plan of the owner-sharded manager in one kernel: its producer (shardplan.cu's
// first-position emit) already counted the owned uniques per (1024-row tile, destination) in
// tile_cnt, and own_k is the identity. Each CTA sums the counts of the tiles before its own
// (at most a few hundred) instead of a separate tile scan; block 0 also writes the totals.
__global__ void __launch_bounds__(256) send_rank_counted_kernel(
    const int32_t* __restrict__ n_own_p, const uint32_t* __restrict__ tm, uint32_t W, int cap,
    const uint32_t* __restrict__ tile_cnt, Cnt8* __restrict__ sscan, int32_t* __restrict__ totals) {
  pdl_wait();
  __shared__ uint32_t red[8][8];  // [warp][plane]
  __shared__ uint32_t off[8];
  __shared__ uint32_t wc[4][8][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t wm = W >= 32 ? 0xFFFFFFFFu : (1u << W) - 1u;
  const int32_t n_own = *n_own_p;
  const int nt = (n_own + kTile - 1) / kTile;
  auto sum_tiles = [&](int limit) {  // off[p] = sum of tile_cnt[q][p] over q < limit
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = threadIdx.x; q < limit; q += blockDim.x) {
      const uint4 a = reinterpret_cast<const uint4*>(tile_cnt)[2 * q];
      const uint4 b = reinterpret_cast<const uint4*>(tile_cnt)[2 * q + 1];
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      uint32_t v = acc[p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      if (lane == 0) red[warp][p] = v;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
      uint32_t v = 0;
      for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
      off[threadIdx.x] = v;
    }
    __syncthreads();
  };
  if (blockIdx.x == 0) {
    sum_tiles(nt);
    if (threadIdx.x < 8) totals[8 + threadIdx.x] = static_cast<int32_t>(off[threadIdx.x]);
    __syncthreads();
  }
  for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
    sum_tiles(tile);
    uint32_t m[4], pre[4][8];
    for (int r = 0; r < 4; ++r) {
      const int i = tile * kTile + r * 256 + threadIdx.x;
      m[r] = i < n_own ? (tm[i] & wm) : 0u;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const unsigned b = __ballot_sync(0xFFFFFFFFu, (m[r] >> p) & 1u);
        pre[r][p] = __popc(b & lt);
        if (lane == 0) wc[r][warp][p] = __popc(b);
      }
    }
    __syncthreads();
    if (threadIdx.x < 8) {  // plane p: exclusive prefix over (round, warp) in tile order
      const int p = threadIdx.x;
      uint32_t run = off[p];
      for (int rr = 0; rr < 4; ++rr)
        for (int w = 0; w < 8; ++w) {
          const uint32_t c = wc[rr][w][p];
          wc[rr][w][p] = run;
          run += c;
        }
    }
    __syncthreads();
    for (int r = 0; r < 4; ++r) {
      const int i = tile * kTile + r * 256 + threadIdx.x;
      if (i >= n_own || i >= cap) continue;
      Cnt8 out{};
#pragma unroll
      for (int p = 0; p < 8; ++p) out.c[p] = wc[r][warp][p] + pre[r][p];
      sscan[i] = out;
    }
    __syncthreads();  // wc / off are reused by the CTA's next tile
  }
}

}  // namespace

void Exchange::plan(const uint32_t* d_vid, int64_t n_global, int64_t per_worker,
                    const uint32_t* d_uniq, const int32_t* d_U, const uint32_t* d_own_k,
                    const int32_t* d_n_own, cudaStream_t s, const PhaseHook& hook) {
  const int c = static_cast<int>(cap);
  const int ntiles = ceil_div(c, kTile);
  launch_pdl(touch_mark_kernel, dim3(ceil_div(n_global, 256)), dim3(256), 0, s, d_vid, n_global, per_worker, tb8);
  CUDA_LAUNCH_CHECK();
  hook("plan_mark");
  launch_pdl(touch_pack_kernel, dim3(std::max(1, std::min(ceil_div(c, 256), num_sms() * 8))), dim3(256), 0, s, d_U, tb8, tm);
  CUDA_LAUNCH_CHECK();
  hook("plan_touch");
  // receive plan (y = 0, over the uniques) and send plan (y = 1, over my owned uniques)
  const int gx = std::max(1, std::min(ntiles, num_sms() * 4));  // persistent over the tiles
  launch_pdl(plan_count_kernel, dim3(gx, 2), dim3(256), 0, s, d_uniq, d_U, d_own_k, d_n_own, c,
             tm, W, me, ntiles, tile_cnt, 0);
  CUDA_LAUNCH_CHECK();
  launch_pdl(plan_scan_tiles_kernel, dim3(1), dim3(512), 0, s, tile_cnt, ntiles, tile_off, totals, d_U, d_n_own);
  CUDA_LAUNCH_CHECK();
  launch_pdl(plan_rank_kernel, dim3(gx, 2), dim3(256), 0, s, d_uniq, d_U, d_own_k, d_n_own, c, tm,
             W, me, ntiles, tile_off, totals, sscan, lpos, 0);
  CUDA_LAUNCH_CHECK();
  hook("plan_rank");
  // every peer's layout (peer-store transport)
  CUDA_CHECK(cudaMemsetAsync(totals + 16, 0, sizeof(int32_t) * 64, s));
  launch_pdl(count_matrix_kernel, dim3(std::min(ceil_div(c, 256), num_sms() * 4)), dim3(256), 0, s, d_uniq, d_U, c, tm, W,
                                                                           totals + 16);
  CUDA_LAUNCH_CHECK();
  launch_pdl(offsets_kernel, dim3(1), dim3(32), 0, s, totals, me, offs);
  CUDA_LAUNCH_CHECK();
}

void Exchange::send_plan_counted(const int32_t* d_n_own, cudaStream_t s) {
  const int c = static_cast<int>(cap);
  const int ntiles = ceil_div(c, kTile);
  launch_pdl(send_rank_counted_kernel, dim3(std::max(1, std::min(ntiles, num_sms() * 4))),
             dim3(256), 0, s, d_n_own, static_cast<const uint32_t*>(tm), static_cast<uint32_t>(W),
             c, static_cast<const uint32_t*>(tile_cnt), sscan, totals);
  CUDA_LAUNCH_CHECK();
}

void Exchange::plan_offsets(cudaStream_t s) {
  launch_pdl(offsets_kernel, dim3(1), dim3(32), 0, s, totals, me, offs);
  CUDA_LAUNCH_CHECK();
}

void Exchange::local_vids(const uint32_t* d_vid_mine, int64_t n, uint32_t* d_lvid, cudaStream_t s,
                          const uint32_t* table) {
  launch_pdl(lvid_kernel, dim3(ceil_div(n, 256)), dim3(256), 0, s, d_vid_mine, n, table ? table : lpos, d_lvid);
  CUDA_LAUNCH_CHECK();
}

void Exchange::set_counts(const int32_t* h_totals) {
  recv_rows.assign(h_totals, h_totals + 8);
  send_rows.assign(h_totals + 8, h_totals + 16);
  recv_off.assign(9, 0);
  for (int o = 0; o < 8; ++o) recv_off[o + 1] = recv_off[o] + recv_rows[o];
  send_off.assign(9, 0);
  for (int w = 0; w < 8; ++w) send_off[w + 1] = send_off[w] + (w == me ? 0 : send_rows[w]);
  // cnt[w][o] = h_totals[16 + w*8 + o]
  roff_all.assign(64, 0);
  boff_all.assign(64, 0);
  for (int w = 0; w < 8; ++w)
    for (int o = 1; o < 8; ++o)
      roff_all[w * 8 + o] = roff_all[w * 8 + o - 1] + h_totals[16 + w * 8 + o - 1];
  for (int o = 0; o < 8; ++o)
    for (int w = 1; w < 8; ++w)
      boff_all[o * 8 + w] =
          boff_all[o * 8 + w - 1] + (w - 1 == o ? 0 : h_totals[16 + (w - 1) * 8 + o]);
}

namespace {

// count matrix cnt[w][o] = #uniques owned by o that worker w touches (every
// rank computes all of it, so each knows every peer's receive layout)
__global__ void count_matrix_kernel(const uint32_t* __restrict__ uniq,
                                    const int32_t* __restrict__ U, int cap,
                                    const uint32_t* __restrict__ tm, uint32_t W,
                                    int32_t* __restrict__ cnt) {
  pdl_wait();
  __shared__ int32_t c[64];
  if (threadIdx.x < 64) c[threadIdx.x] = 0;
  __syncthreads();
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cap; k += gridDim.x * blockDim.x) {
    if (k >= *U) break;
    const uint32_t o = uniq[k] % W;
    uint32_t m = tm[k];
    while (m) {
      const uint32_t w = __ffs(m) - 1;
      m &= m - 1;
      atomicAdd(c + w * 8 + o, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < 64 && c[threadIdx.x]) atomicAdd(cnt + threadIdx.x, c[threadIdx.x]);
}

struct PeerRows {
  float4* E[8];        // every rank's local table E (mine included)
  float4* buf[8];      // every rank's gradient receive buffer
  uint32_t e_off[8];   // row where my owner block starts in rank w's E
  uint32_t b_off[8];   // row where my block starts in owner o's receive buffer
};

// Forward over NVLink: owned row j is stored straight into the E of every
// worker that touches it (one warp per row, 16 B lanes, peer stores).
__global__ void push_rows_p2p_kernel(const uint32_t* __restrict__ own_k,
                                     const uint32_t* __restrict__ own_slot, int32_t n_own,
                                     const uint32_t* __restrict__ tm,
                                     const Cnt8* __restrict__ sscan, uint32_t W,
                                     const float4* __restrict__ emb, int d4, PeerRows pr) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  // persistent warps (grid-stride) so the per-CTA fence below is paid once
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_own; j += nwarps) {
    const uint32_t m = tm[own_k[j]];
    const float4* src = emb + static_cast<int64_t>(own_slot[j]) * 3 * d4;  // [emb | m | v] rows
    for (uint32_t w = 0; w < W; ++w) {
      if (!((m >> w) & 1u)) continue;
      float4* dst = pr.E[w] + static_cast<int64_t>(pr.e_off[w] + sscan[j].c[w]) * d4;
      for (int c = lane; c < d4; c += 32) dst[c] = src[c];
    }
  }
  // one cumulative system-scope fence per CTA (after the CTA barrier) orders
  // all of this CTA's peer stores before the barrier collective that follows
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

struct PeerBlocks {
  float4* dst[8];      // owner o's receive buffer at my block
  int64_t src_row[8];  // my dE rows of owner o start here
  int64_t rows[8];     // 0 for myself
};

// Backward over NVLink, all owners in one launch (blockIdx.y = owner o): my
// contiguous partial-gradient block for o is stored into o's receive buffer.
__global__ void push_blocks_p2p_kernel(const float4* __restrict__ dE, int d4, PeerBlocks pb) {
  const int o = blockIdx.y;
  const int64_t n = pb.rows[o] * d4;
  const float4* src = dE + pb.src_row[o] * d4;
  float4* dst = pb.dst[o];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

// Backward over NVLink: my partial-gradient block for owner o (rows
// [src_row, src_row + n)) goes to o's receive buffer at dst_row.
__global__ void push_block_p2p_kernel(const float4* __restrict__ dE, int64_t src_row, int64_t n,
                                      int d4, float4* __restrict__ dst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * d4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = dE[src_row * d4 + i];
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

}  // namespace

namespace {

// the host's set_counts, on the device: every rank's receive layout (the totals staged in
// shared memory, then thread w builds row w of roff, thread 8 + o column o of boff)
__global__ void offsets_kernel(const int32_t* __restrict__ totals, int me, int32_t* __restrict__ offs) {
  pdl_wait();
  __shared__ int32_t t[Exchange::kTotals];
  for (int i = threadIdx.x; i < Exchange::kTotals; i += blockDim.x) t[i] = totals[i];
  __syncthreads();
  const int32_t* cnt = t + 16;  // cnt[w][o]
  const int x = threadIdx.x;
  if (x < 8) {
    int32_t* roff = offs + Exchange::kOffRoff + x * 8;
    int32_t run = 0;
    for (int o = 0; o < 8; ++o) {
      roff[o] = run;
      run += cnt[x * 8 + o];
    }
  } else if (x < 16) {
    const int o = x - 8;
    int32_t* boff = offs + Exchange::kOffBoff + o * 8;
    int32_t run = 0;
    for (int w = 0; w < 8; ++w) {
      boff[w] = run;
      if (w != o) run += cnt[w * 8 + o];
    }
  } else if (x == 16) {
    int32_t* recv_off = offs + Exchange::kOffRecv;
    int32_t* send_off = offs + Exchange::kOffSend;
    recv_off[0] = 0;
    send_off[0] = 0;
    for (int o = 0; o < 8; ++o) {
      recv_off[o + 1] = recv_off[o] + t[o];
      send_off[o + 1] = send_off[o] + (o == me ? 0 : t[8 + o]);
    }
  }
}

// forward over NVLink, offsets from the device plan (see push_rows_p2p_kernel). Flat
// (owned row, 16 B chunk) items, two per thread per round with independent load chains,
// so many rows' index loads and row reads are in flight at once; each chunk is stored to
// every rank that touches the row (my own E included).
__global__ void __launch_bounds__(256) push_rows_p2p_dev_kernel(
    const uint32_t* __restrict__ own_k, const uint32_t* __restrict__ own_slot,
    const int32_t* __restrict__ n_ptr, const uint32_t* __restrict__ tm,
    const Cnt8* __restrict__ sscan, uint32_t W, uint32_t me, const int32_t* __restrict__ offs,
    const float4* __restrict__ emb, int d4, PeerRows pr) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(*n_ptr) * d4;
  uint32_t e_off[8];
#pragma unroll
  for (int w = 0; w < 8; ++w)
    e_off[w] = w < static_cast<int>(W) ? offs[Exchange::kOffRoff + w * 8 + me] : 0u;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n;
       i0 += 2 * stride) {
    int64_t j[2];
    int c[2];
    bool ok[2];
    uint32_t m[2];
    float4 v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + u * stride;
      ok[u] = i < n;
      j[u] = ok[u] ? idiv(i, d4) : 0;
      c[u] = static_cast<int>(i - j[u] * d4);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      m[u] = ok[u] ? __ldg(tm + __ldg(own_k + j[u])) : 0u;
      v[u] = ok[u] ? __ldg(emb + static_cast<int64_t>(__ldg(own_slot + j[u])) * 3 * d4 + c[u])
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t mm = m[u] & ((1u << W) - 1u);
#pragma unroll
      for (int w = 0; w < 8; ++w) {  // unrolled over the 8 possible destinations: e_off[] and
        // pr.E[] are indexed statically (no local-memory copy of either)
        if (!((mm >> w) & 1u)) continue;
        const uint32_t pos = e_off[w] + __ldg(&sscan[j[u]].c[w]);
        pr.E[w][static_cast<int64_t>(pos) * d4 + c[u]] = v[u];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

// Forward in two phases (SFCTR_FWD_STAGED=1; the fused push_rows kernel is the default):
// pack_fwd gathers every owned row a peer touches into that
// peer's contiguous block of the staging buffer (HBM only, many threads for the random slot
// reads) and writes my own touched rows straight into my E; push_fwd then copies each block
// to its destination's E with one wave of writer CTAs per peer (the backward's pattern,
// which sustains ~0.7 of the peer-copy peak where the fused gather+push reached ~0.6).
__global__ void __launch_bounds__(256) pack_fwd_kernel(
    const uint32_t* __restrict__ own_k, const uint32_t* __restrict__ own_slot,
    const int32_t* __restrict__ n_ptr, const uint32_t* __restrict__ tm,
    const Cnt8* __restrict__ sscan, uint32_t W, uint32_t me, const int32_t* __restrict__ offs,
    const float4* __restrict__ emb, int d4, float4* __restrict__ E_mine,
    float4* __restrict__ stage) {
  const int64_t n = static_cast<int64_t>(*n_ptr) * d4;
  const uint32_t e_me = offs[Exchange::kOffRoff + me * 8 + me];
  uint32_t soff[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) soff[w] = w < static_cast<int>(W) ? offs[Exchange::kOffSend + w] : 0u;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int64_t j = idiv(i, d4);
    const int c = static_cast<int>(i - j * d4);
    uint32_t m = __ldg(tm + __ldg(own_k + j)) & ((1u << W) - 1u);
    const float4 v = __ldg(emb + static_cast<int64_t>(__ldg(own_slot + j)) * 3 * d4 + c);
    while (m) {
      const int w = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t r = __ldg(&sscan[j].c[w]);
      if (w == static_cast<int>(me)) E_mine[static_cast<int64_t>(e_me + r) * d4 + c] = v;
      else stage[static_cast<int64_t>(soff[w] + r) * d4 + c] = v;
    }
  }
}

// blockIdx.y = destination w: my staged block for w -> rank w's E at my owner offset
__global__ void push_fwd_kernel(const float4* __restrict__ stage, int d4, uint32_t me,
                                const int32_t* __restrict__ totals,
                                const int32_t* __restrict__ offs, PeerRows pr) {
  const int w = blockIdx.y;
  if (w != static_cast<int>(me)) {
    const int64_t n = static_cast<int64_t>(totals[8 + w]) * d4;
    const float4* src = stage + static_cast<int64_t>(offs[Exchange::kOffSend + w]) * d4;
    float4* dst = pr.E[w] + static_cast<int64_t>(offs[Exchange::kOffRoff + w * 8 + me]) * d4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n;
         i0 += 2 * stride) {
      const float4 a = src[i0];
      const bool two = i0 + stride < n;
      const float4 b = two ? src[i0 + stride] : a;
      dst[i0] = a;
      if (two) dst[i0 + stride] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

struct OwnerAdam {
  float4 *emb, *mom, *vel;
  const uint32_t* own_slot;
  const int32_t* steps;
  const float *bc1, *bc2;
  float lr, b1, b2, omb1, omb2, eps;
};

// Deferred FM term (fm != nullptr): the segment sum left -scale * B[r] * E[r] out of the
// local gradient row r (B[r] = sum of gz over the positions that hit r); it is added here,
// as the row leaves for its owner, and in owner_reduce for the owner's own rows.
struct FmDefer {
  const float4* E;  // local table rows (the forward's G)
  const float* B;
  float scale;
};
__device__ __forceinline__ float4 with_fm(float4 v, const FmDefer& fm, int64_t row, int c, int d4) {
  const float k = fm.scale * __ldg(fm.B + row);
  const float4 e = __ldg(fm.E + row * d4 + c);
  v.x -= k * e.x;
  v.y -= k * e.y;
  v.z -= k * e.z;
  v.w -= k * e.w;
  return v;
}

__global__ void push_blocks_p2p_dev_kernel(const float4* __restrict__ dE, int d4, uint32_t me,
                                           const int32_t* __restrict__ totals,
                                           const int32_t* __restrict__ offs, PeerRows pr,
                                           FmDefer fm) {
  pdl_wait();
  const int o = blockIdx.y;
  if (o != static_cast<int>(me)) {
    const int64_t n = static_cast<int64_t>(totals[o]) * d4;
    const int64_t r0 = offs[Exchange::kOffRecv + o];
    const float4* src = dE + r0 * d4;
    float4* dst = pr.buf[o] + static_cast<int64_t>(offs[Exchange::kOffBoff + o * 8 + me]) * d4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n;
         i0 += 2 * stride) {  // two independent rows' chunks in flight per thread
      float4 v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= n) continue;
        v[u] = src[i];
        if (fm.B) {
          const int64_t q = idiv(i, d4);
          v[u] = with_fm(v[u], fm, r0 + q, static_cast<int>(i - q * d4), d4);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (i0 + u * stride < n) dst[i0 + u * stride] = v[u];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

__global__ void zero_rows_dev_kernel(float4* __restrict__ p, const int32_t* __restrict__ offs,
                                     int d4, float* __restrict__ B) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(offs[Exchange::kOffRecv + 8]) * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (B) {
      const int64_t q = idiv(i, d4);
      if (i == q * d4) B[q] = 0.f;
    }
  }
}

// The owner's sum goes straight into the lazy Adam update of its cache slot (same math as
// sparse_adam_v4, embed.cu) instead of being written to gown and read back.
//
// Deferred FM term of the owner's OWN rows: -scale * B[r] * E[r] with E[r] the row this rank
// pushed into its own receive table in the forward, i.e. emb[own_slot[j]] before this
// update. It is taken from the cache row loaded here, never from E: after the gradient
// barrier a faster peer may already be storing its step t+1 forward rows into E (the
// owner-major block offsets move between steps), so E is not read past that barrier.
__global__ void __launch_bounds__(256, 5) owner_reduce_adam_dev_kernel(
    const uint32_t* __restrict__ own_k, const int32_t* __restrict__ n_ptr,
    const uint32_t* __restrict__ tm, const Cnt8* __restrict__ sscan,
    const int32_t* __restrict__ totals, uint32_t W, uint32_t me, const uint32_t* __restrict__ lpos,
    const float4* __restrict__ dE, const float4* __restrict__ recvbuf, int d4,
    const float* __restrict__ fmB, float fm_scale, OwnerAdam a) {
  pdl_wait();
  const int64_t n = static_cast<int64_t>(*n_ptr) * d4;
  uint32_t soff[8];  // start of source w's block in my receive buffer
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    soff[w] = run;
    if (w < static_cast<int>(W) && w != static_cast<int>(me)) run += static_cast<uint32_t>(totals[8 + w]);
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // One (row, chunk) item per thread per round. The loads are issued in three dependent
  // levels instead of a chain: (own_k, own_slot) by row; then the source mask, the local
  // row, the step count and the [emb | m | v] state by key / slot; then the gradient rows
  // and the bias corrections. The Adam state does not depend on the gradient sum, so it
  // is in flight while the sources are read.
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const int64_t j = idiv(i, d4);
    const int c = static_cast<int>(i - j * d4);
    const uint32_t k = __ldg(own_k + j);
    const uint32_t s = __ldg(a.own_slot + j);
    const uint32_t m = __ldg(tm + k);
    const int64_t lr = ((m >> me) & 1u) ? static_cast<int64_t>(__ldg(lpos + k)) : 0;
    const int t = __ldg(a.steps + s) + 1;
    const int64_t o = static_cast<int64_t>(s) * 3 * d4 + c;  // [emb | m | v] rows
    float4 mm = a.mom[o];
    float4 vv = a.vel[o];
    float4 e = a.emb[o];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 8; ++w) {  // fixed source order (same as owner_reduce_kernel);
      // unrolled over the 8 possible sources so soff[] stays in registers
      if (w >= static_cast<int>(W) || !((m >> w) & 1u)) continue;
      float4 v;
      if (w == static_cast<int>(me)) {
        v = dE[lr * d4 + c];
        if (fmB) {
          const float kk = fm_scale * __ldg(fmB + lr);
          v.x -= kk * e.x;
          v.y -= kk * e.y;
          v.z -= kk * e.z;
          v.w -= kk * e.w;
        }
      } else {
        v = __ldg(recvbuf + static_cast<int64_t>(soff[w] + __ldg(&sscan[j].c[w])) * d4 + c);
      }
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    // update_sparse, lazy per-row step count
    const float c1 = __ldg(a.bc1 + t), c2 = __ldg(a.bc2 + t);
#define SFB_ADAM(X)                                   \
  mm.X = a.b1 * mm.X + a.omb1 * acc.X;                \
  vv.X = a.b2 * vv.X + a.omb2 * acc.X * acc.X;        \
  e.X -= a.lr * (mm.X / c1) / (sqrtf(vv.X / c2) + a.eps);
    SFB_ADAM(x) SFB_ADAM(y) SFB_ADAM(z) SFB_ADAM(w)
#undef SFB_ADAM
    a.mom[o] = mm;
    a.vel[o] = vv;
    a.emb[o] = e;
  }
}

}  // namespace

void Exchange::forward_dev(const uint32_t* d_own_k, const uint32_t* d_own_slot, int32_t n_bound,
                           const int32_t* d_n_own, const float* emb, cudaStream_t s) {
  PeerRows pr{};
  for (int w = 0; w < W; ++w) pr.E[w] = reinterpret_cast<float4*>(peer_E[w]);
  static const int fwd_blocks = [] {  // experiment switch: SFCTR_FWD_PUSH_BLOCKS
    const char* e = std::getenv("SFCTR_FWD_PUSH_BLOCKS");
    return e ? std::max(1, atoi(e)) : num_sms() * 2;
  }();
  // SFCTR_FWD_STAGED=1: pack per destination, then block pushes (measured slower at cfg2:
  // 93.5 vs 80 us at N = 4, the pack's HBM pass costs more than the pushes gain)
  static const bool fused = [] {
    const char* e = std::getenv("SFCTR_FWD_STAGED");
    return !(e && e[0] == '1');
  }();
  if (fused) {
    launch_pdl(push_rows_p2p_dev_kernel, dim3(std::max(1, std::min(ceil_div(static_cast<int64_t>(n_bound) * (d / 4), 512),
                                                    fwd_blocks))), dim3(256), 0, s, d_own_k, d_own_slot, d_n_own, tm, sscan, W, me, offs,
                                            reinterpret_cast<const float4*>(emb), d / 4, pr);
    CUDA_LAUNCH_CHECK();
    return;
  }
  // the staging rows live in buf: it is free until the backward, which peers only start
  // after this step's forward barrier
  pack_fwd_kernel<<<std::max(1, std::min(ceil_div(static_cast<int64_t>(n_bound) * (d / 4), 256),
                                         num_sms() * 16)),
                    256, 0, s>>>(d_own_k, d_own_slot, d_n_own, tm, sscan, W, me, offs,
                                 reinterpret_cast<const float4*>(emb), d / 4,
                                 reinterpret_cast<float4*>(peer_E[me]),
                                 reinterpret_cast<float4*>(buf));
  CUDA_LAUNCH_CHECK();
  push_fwd_kernel<<<dim3(num_sms(), W), 256, 0, s>>>(reinterpret_cast<const float4*>(buf), d / 4, me,
                                                totals, offs, pr);
  CUDA_LAUNCH_CHECK();
}

void Exchange::backward_send_dev(const float* dE, cudaStream_t s, const float* E, const float* B,
                                 float fm_scale) {
  PeerRows pr{};
  for (int o = 0; o < W; ++o) pr.buf[o] = reinterpret_cast<float4*>(peer_buf[o]);
  // one wave of writers per destination: more concurrent NVLink writers congest the switch
  // (microbench/nvlink_push.cu: 569 GB/s out per GPU with 148 CTAs per peer at W = 4,
  // 444 GB/s with 592, 406 GB/s with 1184)
  launch_pdl(push_blocks_p2p_dev_kernel, dim3(dim3(num_sms(), W)), dim3(256), 0, s, reinterpret_cast<const float4*>(dE), d / 4, me, totals, offs, pr,
      FmDefer{reinterpret_cast<const float4*>(E), B, fm_scale});
  CUDA_LAUNCH_CHECK();
}

void Exchange::backward_reduce_adam_dev(const uint32_t* d_own_k, int32_t n_bound,
                                        const int32_t* d_n_own, const float* dE, cudaStream_t s,
                                        const float* B, float fm_scale, const AdamRows& ar) {
  const int d4 = d / 4;
  OwnerAdam a{reinterpret_cast<float4*>(ar.emb), reinterpret_cast<float4*>(ar.mom),
              reinterpret_cast<float4*>(ar.vel), ar.own_slot, ar.steps, ar.bc1, ar.bc2, ar.lr,
              ar.b1, ar.b2, ar.omb1, ar.omb2, ar.eps};
  launch_pdl(owner_reduce_adam_dev_kernel, dim3(std::max(1, std::min(ceil_div(static_cast<int64_t>(n_bound) * d4, 256),
                                                      num_sms() * 15))), dim3(256), 0, s, d_own_k, d_n_own, tm, sscan, totals, W, me, lpos,
                                              reinterpret_cast<const float4*>(dE),
                                              reinterpret_cast<const float4*>(buf), d4, B,
                                              fm_scale, a);
  CUDA_LAUNCH_CHECK();
}

void Exchange::zero_local_dev(float* dE, cudaStream_t s, float* B) {
  launch_pdl(zero_rows_dev_kernel, dim3(mgr_grid(num_sms() * 8)), dim3(256), 0, s, reinterpret_cast<float4*>(dE), offs,
                                                                d / 4, B);
  CUDA_LAUNCH_CHECK();
}

void Exchange::setup_p2p(float* E, ncclComm_t comm, cudaStream_t s) {
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  // every rank must reach every peer over NVLink; otherwise keep NCCL send/recv
  std::vector<int> devs(W, -1);
  int* d_dev = nullptr;
  CUDA_CHECK(cudaMalloc(&d_dev, sizeof(int) * W));
  CUDA_CHECK(cudaMemcpyAsync(d_dev + me, &dev, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_dev + me, d_dev, 1, ncclInt32, comm, s));
  CUDA_CHECK(cudaMemcpyAsync(devs.data(), d_dev, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_dev);
  int ok = 1;
  for (int w = 0; w < W; ++w) {
    if (w == me) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, devs[w]) != cudaSuccess || !can) ok = 0;
  }
  cudaGetLastError();
  // agree on the transport (min over ranks)
  int* d_ok = nullptr;
  CUDA_CHECK(cudaMalloc(&d_ok, sizeof(int)));
  CUDA_CHECK(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, comm, s));
  CUDA_CHECK(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_ok);
  if (!ok) return;
  // exchange IPC handles of E, buf and the barrier flags
  CUDA_CHECK(cudaMalloc(&flags, sizeof(uint64_t) * 8));
  CUDA_CHECK(cudaMemset(flags, 0, sizeof(uint64_t) * 8));
  cudaIpcMemHandle_t mine[3];
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[0], E));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[1], buf));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[2], flags));
  const size_t hb = sizeof(mine);
  uint8_t* d_h = nullptr;
  CUDA_CHECK(cudaMalloc(&d_h, hb * W));
  CUDA_CHECK(cudaMemcpyAsync(d_h + hb * me, mine, hb, cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_h + hb * me, d_h, hb, ncclUint8, comm, s));
  std::vector<cudaIpcMemHandle_t> all(3 * W);
  CUDA_CHECK(cudaMemcpyAsync(all.data(), d_h, hb * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_h);
  for (int w = 0; w < W; ++w) {
    if (w == me) {
      peer_E[w] = E;
      peer_buf[w] = buf;
      peer_flags[w] = flags;
      continue;
    }
    void* pe = nullptr;
    void* pb = nullptr;
    void* pf = nullptr;
    CUDA_CHECK(cudaIpcOpenMemHandle(&pe, all[3 * w], cudaIpcMemLazyEnablePeerAccess));
    CUDA_CHECK(cudaIpcOpenMemHandle(&pb, all[3 * w + 1], cudaIpcMemLazyEnablePeerAccess));
    CUDA_CHECK(cudaIpcOpenMemHandle(&pf, all[3 * w + 2], cudaIpcMemLazyEnablePeerAccess));
    peer_E[w] = static_cast<float*>(pe);
    peer_buf[w] = static_cast<float*>(pb);
    peer_flags[w] = static_cast<uint64_t*>(pf);
  }
  CUDA_CHECK(cudaMalloc(&bar, sizeof(float)));
  CUDA_CHECK(cudaMemset(bar, 0, sizeof(float)));
  p2p = true;
}

namespace {
struct PeerFlags {
  uint64_t* peer[8];  // every rank's flag words (mine included)
};
// NVLink flag barrier (flag_barrier_wait, common.cuh). The peer stores being published were
// made by the previous kernel on this stream, which ended every block with
// __threadfence_system().
__global__ void flag_barrier_kernel(PeerFlags pf, int W, int me, uint64_t epoch,
                                    uint64_t timeout_ns, int32_t* abort_flag) {
  pdl_wait();
  flag_barrier_wait(pf.peer, W, me, epoch, timeout_ns, abort_flag);
}
}  // namespace

void Exchange::barrier(ncclComm_t comm, cudaStream_t s) {
  // stream-ordered rendezvous: every rank's peer stores (kernel complete +
  // system fence) precede its arrival, so after this all are visible
  if (flags && !nccl_barrier) {
    PeerFlags pf{};
    for (int w = 0; w < W; ++w) pf.peer[w] = peer_flags[w];
    launch_pdl(flag_barrier_kernel, dim3(1), dim3(32), 0, s, pf, W, me, ++epoch, barrier_timeout_ns(), abort_flag);
    CUDA_LAUNCH_CHECK();
    return;
  }
  NCCL_CHECK(ncclAllReduce(bar, bar, 1, ncclFloat32, ncclSum, comm, s));
}

int64_t Exchange::forward(const uint32_t* d_own_k, const uint32_t* d_own_slot, int32_t n_own,
                          const float* emb, float* E, ncclComm_t comm, cudaStream_t s,
                          bool do_barrier) {
  const int d4 = d / 4;
  if (p2p) {
    PeerRows pr{};
    int64_t bytes = 0;
    for (int w = 0; w < W; ++w) {
      pr.E[w] = reinterpret_cast<float4*>(peer_E[w]);
      pr.e_off[w] = static_cast<uint32_t>(roff_all[w * 8 + me]);
      if (w != me) bytes += static_cast<int64_t>(send_rows[w]) * d * 4;
    }
    if (copy_engine) {
      // pack locally (HBM), then one DMA copy per peer over NVLink
      if (n_own > 0) {
        pack_rows_kernel<<<ceil_div(static_cast<int64_t>(n_own) * 32, 256), 256, 0, s>>>(
            d_own_k, d_own_slot, n_own, tm, sscan, totals, W, me, lpos,
            reinterpret_cast<const float4*>(emb), d4, reinterpret_cast<float4*>(buf),
            reinterpret_cast<float4*>(E));
        CUDA_LAUNCH_CHECK();
      }
      for (int w = 0; w < W; ++w) {
        if (w == me || send_rows[w] == 0) continue;
        CUDA_CHECK(cudaMemcpyAsync(peer_E[w] + static_cast<size_t>(roff_all[w * 8 + me]) * d,
                                   buf + static_cast<size_t>(send_off[w]) * d,
                                   sizeof(float) * static_cast<size_t>(send_rows[w]) * d,
                                   cudaMemcpyDeviceToDevice, s));
      }
    } else if (n_own > 0) {
      push_rows_p2p_kernel<<<std::min(ceil_div(static_cast<int64_t>(n_own) * 32, 256), num_sms() * 8),
                             256, 0, s>>>(
          d_own_k, d_own_slot, n_own, tm, sscan, W, reinterpret_cast<const float4*>(emb), d4, pr);
      CUDA_LAUNCH_CHECK();
    }
    if (do_barrier) barrier(comm, s);
    return bytes;
  }
  if (n_own > 0) {
    pack_rows_kernel<<<ceil_div(static_cast<int64_t>(n_own) * 32, 256), 256, 0, s>>>(
        d_own_k, d_own_slot, n_own, tm, sscan, totals, W, me, lpos,
        reinterpret_cast<const float4*>(emb), d4, reinterpret_cast<float4*>(buf),
        reinterpret_cast<float4*>(E));
    CUDA_LAUNCH_CHECK();
  }
  int64_t bytes = 0;
  NCCL_CHECK(ncclGroupStart());
  for (int w = 0; w < W; ++w) {
    if (w == me) continue;
    if (send_rows[w] > 0) {
      NCCL_CHECK(ncclSend(buf + static_cast<size_t>(send_off[w]) * d,
                          static_cast<size_t>(send_rows[w]) * d, ncclFloat32, w, comm, s));
      bytes += static_cast<int64_t>(send_rows[w]) * d * 4;
    }
    if (recv_rows[w] > 0)
      NCCL_CHECK(ncclRecv(E + static_cast<size_t>(recv_off[w]) * d,
                          static_cast<size_t>(recv_rows[w]) * d, ncclFloat32, w, comm, s));
  }
  NCCL_CHECK(ncclGroupEnd());
  return bytes;
}

int64_t Exchange::backward(const uint32_t* d_own_k, int32_t n_own, const float* dE, ncclComm_t comm,
                           cudaStream_t s) {
  const int64_t bytes = backward_send(dE, comm, s);
  if (p2p) barrier(comm, s);
  backward_reduce(d_own_k, n_own, dE, s);
  return bytes;
}

int64_t Exchange::backward_send(const float* dE, ncclComm_t comm, cudaStream_t s) {
  int64_t bytes = 0;
  if (p2p) {
    const int d4 = d / 4;
    if (copy_engine) {
      for (int o = 0; o < W; ++o) {
        if (o == me || recv_rows[o] == 0) continue;
        CUDA_CHECK(cudaMemcpyAsync(peer_buf[o] + static_cast<size_t>(boff_all[o * 8 + me]) * d,
                                   dE + static_cast<size_t>(recv_off[o]) * d,
                                   sizeof(float) * static_cast<size_t>(recv_rows[o]) * d,
                                   cudaMemcpyDeviceToDevice, s));
        bytes += recv_rows[o] * d * 4;
      }
    } else {  // every peer block in one launch: blockIdx.y = owner
      PeerBlocks pb{};
      int64_t most = 0;
      for (int o = 0; o < W; ++o) {
        pb.dst[o] = reinterpret_cast<float4*>(peer_buf[o]) + boff_all[o * 8 + me] * d4;
        pb.src_row[o] = recv_off[o];
        pb.rows[o] = (o == me) ? 0 : recv_rows[o];
        most = std::max<int64_t>(most, pb.rows[o]);
        bytes += pb.rows[o] * d * 4;
      }
      if (most > 0) {
        push_blocks_p2p_kernel<<<dim3(std::min(ceil_div(most * d4, 256), num_sms() * 2), W), 256, 0,
                                 s>>>(reinterpret_cast<const float4*>(dE), d4, pb);
        CUDA_LAUNCH_CHECK();
      }
    }
    return bytes;
  }
  {
  NCCL_CHECK(ncclGroupStart());
  for (int w = 0; w < W; ++w) {
    if (w == me) continue;
    if (recv_rows[w] > 0) {  // my partial gradients of rows owned by w
      NCCL_CHECK(ncclSend(dE + static_cast<size_t>(recv_off[w]) * d,
                          static_cast<size_t>(recv_rows[w]) * d, ncclFloat32, w, comm, s));
      bytes += static_cast<int64_t>(recv_rows[w]) * d * 4;
    }
    if (send_rows[w] > 0)  // worker w's partial gradients of rows I own
      NCCL_CHECK(ncclRecv(buf + static_cast<size_t>(send_off[w]) * d,
                          static_cast<size_t>(send_rows[w]) * d, ncclFloat32, w, comm, s));
  }
  NCCL_CHECK(ncclGroupEnd());
  }
  return bytes;
}

void Exchange::backward_reduce(const uint32_t* d_own_k, int32_t n_own, const float* dE,
                               cudaStream_t s) {
  const int d4 = d / 4;
  if (n_own > 0) {
    owner_reduce_kernel<<<ceil_div(static_cast<int64_t>(n_own) * d4, 256), 256, 0, s>>>(
        d_own_k, n_own, tm, sscan, totals, W, me, lpos, reinterpret_cast<const float4*>(dE),
        reinterpret_cast<const float4*>(buf), d4, reinterpret_cast<float4*>(gown));
    CUDA_LAUNCH_CHECK();
  }
}

}  // namespace sfb
