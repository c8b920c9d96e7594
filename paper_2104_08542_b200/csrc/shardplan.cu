// Owner-sharded manager stage (see shardplan.h). Per step, on the manager stream:
//   1. route: every local position i (global position me*n + i) sends (f, position) to owner
//      f mod W by peer stores into the owner's region for this source (one cursor atomic per
//      owner per block); rix[i] records where the owner's reply for i will land. Flag
//      barrier B1 delivers the pair counts (and the bad-id bit)
//   2. dedup: the owner inserts the pairs it received into a hashed table (match_any merges
//      a warp's equal ids first): min global position and touched-by-rank mask per feature
//   3. order: a bit at every owned unique's first global position, one fused look-back scan
//      over the bitmap words, then each unique's rank among the set bits -> owned uniques in
//      global first-appearance order (= the global_ids order of vsi.cpp:41-46 filtered by
//      owner, as the replicated VSI produces it), the touched masks by owned index,
//      own_k = identity, and the send plan's per-(tile, destination) counts
//   4. plan: ranks of each owned unique among those each rank touches (one kernel,
//      Exchange::send_plan_counted, over per-tile counts the emit of step 3 accumulated), my
//      column of the count matrix published to every rank with my unique count; barrier B2
//   5. layout: the full matrix, my receive totals, U, my own rows' local-table rows (lpos)
//   6. reply: for every pair it received the owner stores the local-table row of that
//      position into its source's reply buffer, contiguously (pair i of region r -> r's
//      reply[me * n + i]); the source reads its row for position i as reply[rix[i]]. No
//      third barrier: a source reads its replies only in its training stage, after the
//      forward exchange barrier, which every owner reaches after its reply stores; pairs /
//      inbox / reply / rix are parity sets, so a fast rank can route step t+1 while a slow
//      owner still reads step t
// The result is bit-for-bit the replicated manager's plan: the same owners, the same
// first-appearance order per owner, the same block layout of every rank's local table.
#include "shardplan.h"

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace sfb {

namespace {

constexpr uint32_t kUnseenPos = 0xFFFFFFFFu;
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kTagOwned = 0x80000000u;
constexpr uint64_t kBadBit = 1ull << 63;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

struct PeerPairs {
  uint64_t* dst[8];  // every rank's pair buffer
};

// 1. route (f, p) to owner f mod W into region `me` of the owner's pair buffer. A block takes
// 256 x kRouteItems consecutive positions: per-owner ranks by warp ballots, one cursor
// atomic per owner per block, then the peer stores (a block's pairs for one owner land
// contiguously, in position order). rix[i] = o * n + (index of position i's pair in region
// me of owner o): where owner o's reply for position i lands.
constexpr int kRouteItems = 4;
__global__ void __launch_bounds__(256) route_pairs_kernel(const uint64_t* __restrict__ ids,
                                                          int64_t n, uint64_t vocab, int W, int me,
                                                          int32_t* __restrict__ bad,
                                                          int32_t* __restrict__ cursor,
                                                          PeerPairs pp, uint32_t* __restrict__ rix) {
  pdl_wait();
  __shared__ uint32_t wc[kRouteItems][8][8];  // [item][warp][owner]: counts -> offsets
  __shared__ uint32_t bbase[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * 256 * kRouteItems;
  uint32_t f[kRouteItems], rk[kRouteItems];
  int o[kRouteItems];
  bool saw_bad = false;
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    const int64_t i = base + u * 256 + threadIdx.x;
    const bool live = i < n;
    uint64_t a = live ? ids[i] : 0;
    if (live && a >= vocab) {  // gated step: the position still routes (as feature 0)
      saw_bad = true;
      a = 0;
    }
    f[u] = static_cast<uint32_t>(a);
    o[u] = live ? static_cast<int>(f[u] % static_cast<uint32_t>(W)) : -1;
    rk[u] = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      if (w >= W) break;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, o[u] == w);
      if (o[u] == w) rk[u] = __popc(m & lt);
      if (lane == 0) wc[u][warp][w] = __popc(m);
    }
  }
  __syncthreads();
  if (threadIdx.x < W) {
    const int w = threadIdx.x;
    uint32_t run = 0;
    for (int u = 0; u < kRouteItems; ++u)
      for (int q = 0; q < 8; ++q) {
        const uint32_t c = wc[u][q][w];
        wc[u][q][w] = run;
        run += c;
      }
    bbase[w] = run ? static_cast<uint32_t>(atomicAdd(cursor + w, static_cast<int32_t>(run))) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kRouteItems; ++u) {
    if (o[u] < 0) continue;
    const int64_t i = base + u * 256 + threadIdx.x;
    const uint32_t idx = bbase[o[u]] + wc[u][warp][o[u]] + rk[u];
    uint64_t* dst = nullptr;
#pragma unroll
    for (int w = 0; w < 8; ++w)  // static index: pp stays in the param space
      if (w == o[u]) dst = pp.dst[w];
    dst[static_cast<int64_t>(me) * n + idx] =
        (static_cast<uint64_t>(f[u]) << 32) |
        static_cast<uint32_t>(static_cast<int64_t>(me) * n + i);
    rix[i] = static_cast<uint32_t>(o[u]) * static_cast<uint32_t>(n) + idx;
  }
  if (saw_bad) *bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

struct PeerInts {
  int32_t* p[8];
};
struct PeerFlagsS {
  uint64_t* p[8];
};

// The step's two small publications, then the flag barrier (common.cuh's protocol; bit 63 of
// the published word carries the bad-id flag to every rank). Thread x writes rank x's inbox:
//   kind 0 (B1): inbox[72 + me] = pairs I routed to owner x (cursor[x])
//   kind 1 (B2): inbox[w * 8 + me] = rows of mine rank w touches (send totals[8 + w]) for
//                every w, inbox[64 + me] = my owned unique count
__global__ void publish_barrier_kernel(int kind, PeerInts inbox, const int32_t* __restrict__ cursor,
                                       const int32_t* __restrict__ totals,
                                       const int32_t* __restrict__ n_own, PeerFlagsS pf, int W,
                                       int me, uint64_t epoch, uint64_t timeout_ns,
                                       int32_t* abort_flag, int32_t* bad) {
  pdl_wait();
  const int x = threadIdx.x;
  if (x < W) {
    int32_t* dst = inbox.p[x];
    if (kind == 0) {
      dst[72 + me] = cursor[x];
    } else if (kind == 1) {
      for (int w = 0; w < W; ++w) dst[w * 8 + me] = totals[8 + w];
      dst[64 + me] = *n_own;
    }
  }
  __threadfence_system();
  __syncwarp();
  if (x >= W || x == me) return;
  const uint64_t word = epoch | (bad && *bad ? kBadBit : 0ull);
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pf.p[x] + me), "l"(word) : "memory");
  const uint64_t* mine = pf.p[me] + x;
  uint64_t v = 0, t0 = 0, now = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if ((v & ~kBadBit) >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      if (abort_flag) atomicExch(abort_flag, 1);
      return;
    }
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
  if ((v & kBadBit) && bad) atomicExch(bad, 1);
}

// 2. dedup the received pairs; blockIdx.y = source region r (inbox[72 + r] pairs)
__global__ void __launch_bounds__(256) dedup_pairs_kernel(const uint64_t* __restrict__ pairs,
                                                          int64_t n,
                                                          const int32_t* __restrict__ inbox,
                                                          uint32_t* __restrict__ keys,
                                                          uint32_t* __restrict__ pos,
                                                          uint32_t* __restrict__ tmask,
                                                          uint64_t mask,
                                                          uint32_t* __restrict__ hslot) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.y;
  const int64_t cnt = inbox[72 + r];
  const uint64_t* src = pairs + static_cast<int64_t>(r) * n;
  uint32_t* hs = hslot + static_cast<int64_t>(r) * n;
  const uint32_t bit = 1u << r;
  for (int64_t i0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) & ~31ll;
       i0 < cnt; i0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = i0 + lane;
    const bool live = i < cnt;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, live);
    if (live) {
      const uint64_t pr = src[i];
      const uint32_t f = static_cast<uint32_t>(pr >> 32), p = static_cast<uint32_t>(pr);
      const unsigned peers = __match_any_sync(act, f);
      const int leader = __ffs(peers) - 1;
      // the group's smallest position (a region's pairs are not in position order)
      uint32_t pmin = p;
      for (unsigned m = peers; m; m &= m - 1) {
        const uint32_t o = __shfl_sync(peers, p, __ffs(m) - 1);
        pmin = o < pmin ? o : pmin;
      }
      uint32_t slot = 0;
      if (lane == leader) {
        uint64_t h = mix64(f) & mask;
        for (;;) {
          const uint32_t cur = __ldcg(keys + h);
          if (cur == f) break;
          if (cur == kEmptyKey) {
            const uint32_t prev = atomicCAS(keys + h, kEmptyKey, f);
            if (prev == kEmptyKey || prev == f) break;
          }
          h = (h + 1) & mask;
        }
        slot = static_cast<uint32_t>(h);
        if (__ldcg(pos + slot) > pmin) atomicMin(pos + slot, pmin);
        if (!(__ldcg(tmask + slot) & bit)) atomicOr(tmask + slot, bit);
      }
      hs[i] = __shfl_sync(peers, slot, leader);
    }
  }
}

// 3a. mark the first global position of every owned unique in the position bitmap
// (blockIdx.y = source region)
__global__ void __launch_bounds__(256) first_bits_kernel(const uint64_t* __restrict__ pairs,
                                                         int64_t n,
                                                         const int32_t* __restrict__ inbox,
                                                         const uint32_t* __restrict__ hslot,
                                                         const uint32_t* __restrict__ pos,
                                                         uint32_t* __restrict__ bits,
                                                         uint32_t* __restrict__ tile_cnt,
                                                         int tile_words) {
  pdl_wait();
  const int r = blockIdx.y;
  if (blockIdx.x == 0 && blockIdx.y == 0)  // the send plan's per-tile counts (3c adds to them)
    for (int q = threadIdx.x; q < tile_words; q += blockDim.x) tile_cnt[q] = 0;
  const int64_t cnt = inbox[72 + r];
  const int64_t off = static_cast<int64_t>(r) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = static_cast<uint32_t>(pairs[off + i]);
    if (pos[hslot[off + i]] == p) atomicOr(bits + (p >> 5), 1u << (p & 31));
  }
}

// 3b. exclusive prefix of the set bits over the bitmap words (fused look-back scan; the
// total is the owned count)
struct WordCount {
  const uint32_t* bits;
  __device__ uint32_t operator()(int64_t wi) const { return __popc(bits[wi]); }
};
struct WordPrefix {
  uint32_t* wpre;
  __device__ void operator()(int64_t wi, uint32_t, uint32_t rank) const { wpre[wi] = rank; }
};

// 3c. owned index of every owned unique = its first position's rank among the set bits:
// owned uniques in global first-appearance order (blockIdx.y = source region)
__global__ void __launch_bounds__(256) first_emit_kernel(
    const uint64_t* __restrict__ pairs, int64_t n, const int32_t* __restrict__ inbox,
    const uint32_t* __restrict__ hslot, uint32_t* __restrict__ pos,
    const uint32_t* __restrict__ bits, const uint32_t* __restrict__ wpre,
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ tmask,
    uint32_t* __restrict__ owned, uint32_t* __restrict__ own_k, uint32_t* __restrict__ tm,
    uint32_t* __restrict__ uslot, uint32_t* __restrict__ tile_cnt) {
  pdl_wait();
  const int r = blockIdx.y;
  const int64_t cnt = inbox[72 + r];
  const int64_t off = static_cast<int64_t>(r) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = static_cast<uint32_t>(pairs[off + i]);
    const uint32_t sl = hslot[off + i];
    // (a tagged slot never equals a position: positions stay below 2^31)
    if (pos[sl] != p) continue;
    const uint32_t rank = wpre[p >> 5] + __popc(bits[p >> 5] & ((1u << (p & 31)) - 1u));
    owned[rank] = keys[sl];
    own_k[rank] = rank;
    const uint32_t mk = tmask[sl];
    tm[rank] = mk;
    uslot[rank] = sl;
    pos[sl] = rank | kTagOwned;  // the slot now names its owned index
    // the send plan's count of owned uniques per (1024-row tile, destination rank)
    for (uint32_t m = mk; m; m &= m - 1) atomicAdd(tile_cnt + (rank >> 10) * 8 + (__ffs(m) - 1), 1u);
  }
}

struct PeerReply {
  uint32_t* p[8];  // every rank's reply buffer (this step's set)
};

// 5 + 6 after B2 (the inbox holds the whole count matrix cnt[w][o]):
//   blockIdx.y = r < W: the local-table row of every pair received from source r, stored
//     into r's reply buffer at [me * n + i] (pair i of region r: contiguous peer stores).
//     Rank r's block of my rows starts at roff[r][me] = sum_{o < me} cnt[r][o]; owned index
//     j is row sscan[j].c[r] of that block
//   blockIdx.y = W: my own rows' local-table rows by owned index (the owner reduction reads
//     its own partial gradients at lpos[own_k[j]], own_k = identity here); block 0 also
//     writes the matrix and my receive totals into totals, and U = sum of owned counts
__global__ void __launch_bounds__(256) reply_kernel(int64_t n, int W, int me,
                                                    const int32_t* __restrict__ inbox,
                                                    const uint32_t* __restrict__ hslot,
                                                    const uint32_t* __restrict__ pos,
                                                    const Cnt8* __restrict__ sscan,
                                                    const uint32_t* __restrict__ tm,
                                                    const int32_t* __restrict__ n_own,
                                                    uint32_t* __restrict__ lpos,
                                                    int32_t* __restrict__ totals,
                                                    int32_t* __restrict__ U_global,
                                                    PeerReply pr) {
  pdl_wait();
  const int r = blockIdx.y;
  if (r == W) {
    uint32_t base = 0;  // roff[me][me]
    for (int o = 0; o < me; ++o) base += static_cast<uint32_t>(inbox[me * 8 + o]);
    const int32_t cnt = *n_own;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x)
      lpos[j] = ((tm[j] >> me) & 1u) ? base + sscan[j].c[me] : 0xFFFFFFFFu;
    if (blockIdx.x == 0) {
      const int t = threadIdx.x;
      if (t < 64) totals[16 + t] = (t / 8 < W && t % 8 < W) ? inbox[t] : 0;  // cnt[w][o]
      if (t < 8) totals[t] = t < W ? inbox[me * 8 + t] : 0;                   // from owner t
      if (t == 0) {
        int32_t u = 0;
        for (int o = 0; o < W; ++o) u += inbox[64 + o];
        *U_global = u;
      }
    }
    return;
  }
  const int64_t cnt = inbox[72 + r];
  const int64_t off = static_cast<int64_t>(r) * n;
  uint32_t roff = 0;
  for (int o = 0; o < me; ++o) roff += static_cast<uint32_t>(inbox[r * 8 + o]);
  uint32_t* dst = nullptr;
#pragma unroll
  for (int w = 0; w < 8; ++w)
    if (w == r) dst = pr.p[w];
  dst += static_cast<int64_t>(me) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t j = pos[hslot[off + i]] & ~kTagOwned;
    dst[i] = roff + sscan[j].c[r];
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

// 7. clear the hashed table behind the batch, the routing cursors and the bitmap
__global__ void reset_table_kernel(const uint32_t* __restrict__ uslot,
                                   const int32_t* __restrict__ n_own, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ pos, uint32_t* __restrict__ tmask,
                                   int32_t* __restrict__ cursor, uint32_t* __restrict__ bits,
                                   int64_t nwords) {
  pdl_wait();
  const int32_t cnt = *n_own;
  if (blockIdx.x == 0 && threadIdx.x < 8) cursor[threadIdx.x] = 0;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nwords;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bits[q] = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x) {
    const uint32_t sl = uslot[j];
    keys[sl] = kEmptyKey;
    pos[sl] = kUnseenPos;
    tmask[sl] = 0;
  }
}

}  // namespace

void ShardPlan::init(int W_, int me_, int64_t n_, int64_t cap_) {
  release();
  W = W_;
  me = me_;
  n = n_;
  cap = cap_;
  SFB_CHECK(static_cast<int64_t>(W) * n < (1ll << 31), "sharded manager: global batch >= 2^31");
  const int64_t total = static_cast<int64_t>(W) * n;
  // pairs, inbox, reply and rix come in two sets (step parity, set k at offset k * size)
  CUDA_CHECK(cudaMalloc(&pairs, sizeof(uint64_t) * 2 * total));
  CUDA_CHECK(cudaMalloc(&inbox, sizeof(int32_t) * 2 * kInbox));
  CUDA_CHECK(cudaMemset(inbox, 0, sizeof(int32_t) * 2 * kInbox));
  CUDA_CHECK(cudaMalloc(&reply, sizeof(uint32_t) * 2 * total));
  CUDA_CHECK(cudaMalloc(&rix, sizeof(uint32_t) * 2 * n));
  CUDA_CHECK(cudaMalloc(&cursor, sizeof(int32_t) * 8));
  CUDA_CHECK(cudaMemset(cursor, 0, sizeof(int32_t) * 8));
  hmask = 1;
  while (hmask + 1 < static_cast<uint64_t>(2 * cap)) hmask = 2 * hmask + 1;
  CUDA_CHECK(cudaMalloc(&hkeys, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMemset(hkeys, 0xFF, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMalloc(&hpos, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMemset(hpos, 0xFF, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMalloc(&hmask_bits, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMemset(hmask_bits, 0, sizeof(uint32_t) * (hmask + 1)));
  CUDA_CHECK(cudaMalloc(&hslot, sizeof(uint32_t) * total));
  nwords = (total + 31) / 32;
  CUDA_CHECK(cudaMalloc(&wpre, sizeof(uint32_t) * nwords));
  CUDA_CHECK(cudaMalloc(&bits, sizeof(uint32_t) * nwords));
  CUDA_CHECK(cudaMemset(bits, 0, sizeof(uint32_t) * nwords));
  CUDA_CHECK(cudaMalloc(&uslot, sizeof(uint32_t) * cap));
  tiles.init(nwords);
}

void ShardPlan::release() {
  if (ready)
    for (int w = 0; w < W; ++w) {
      if (w == me) continue;
      for (void* p : {static_cast<void*>(peer_pairs[w]), static_cast<void*>(peer_inbox[w]),
                      static_cast<void*>(peer_reply[w]), static_cast<void*>(peer_flags[w])})
        if (p) cudaIpcCloseMemHandle(p);
    }
  for (void* p : {static_cast<void*>(pairs), static_cast<void*>(inbox),
                  static_cast<void*>(reply), static_cast<void*>(rix), static_cast<void*>(flags),
                  static_cast<void*>(cursor), static_cast<void*>(hkeys), static_cast<void*>(hpos),
                  static_cast<void*>(hmask_bits), static_cast<void*>(hslot),
                  static_cast<void*>(wpre), static_cast<void*>(bits),
                  static_cast<void*>(uslot)})
    if (p) cudaFree(p);
  tiles.release();
  *this = ShardPlan();
}

bool ShardPlan::setup_p2p(ncclComm_t comm, cudaStream_t s) {
  if (W > 8) return false;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  int* d_x = nullptr;
  CUDA_CHECK(cudaMalloc(&d_x, sizeof(int) * (W + 1)));
  CUDA_CHECK(cudaMemcpyAsync(d_x + me, &dev, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_x + me, d_x, 1, ncclInt32, comm, s));
  std::vector<int> devs(W);
  CUDA_CHECK(cudaMemcpyAsync(devs.data(), d_x, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  int ok = 1;
  for (int w = 0; w < W; ++w) {
    if (w == me) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, devs[w]) != cudaSuccess || !can) ok = 0;
  }
  cudaGetLastError();
  CUDA_CHECK(cudaMemcpyAsync(d_x + W, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllReduce(d_x + W, d_x + W, 1, ncclInt32, ncclMin, comm, s));
  CUDA_CHECK(cudaMemcpyAsync(&ok, d_x + W, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_x);
  if (!ok) return false;
  CUDA_CHECK(cudaMalloc(&flags, sizeof(uint64_t) * 8));
  CUDA_CHECK(cudaMemset(flags, 0, sizeof(uint64_t) * 8));
  constexpr int kH = 4;
  cudaIpcMemHandle_t mine[kH];
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[0], pairs));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[1], inbox));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[2], reply));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[3], flags));
  const size_t hb = sizeof(mine);
  uint8_t* d_h = nullptr;
  CUDA_CHECK(cudaMalloc(&d_h, hb * W));
  CUDA_CHECK(cudaMemcpyAsync(d_h + hb * me, mine, hb, cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_h + hb * me, d_h, hb, ncclUint8, comm, s));
  std::vector<cudaIpcMemHandle_t> all(kH * W);
  CUDA_CHECK(cudaMemcpyAsync(all.data(), d_h, hb * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_h);
  for (int w = 0; w < W; ++w) {
    if (w == me) {
      peer_pairs[w] = pairs;
      peer_inbox[w] = inbox;
      peer_reply[w] = reply;
      peer_flags[w] = flags;
      continue;
    }
    void* p[kH] = {};
    for (int q = 0; q < kH; ++q)
      CUDA_CHECK(cudaIpcOpenMemHandle(&p[q], all[kH * w + q], cudaIpcMemLazyEnablePeerAccess));
    peer_pairs[w] = static_cast<uint64_t*>(p[0]);
    peer_inbox[w] = static_cast<int32_t*>(p[1]);
    peer_reply[w] = static_cast<uint32_t*>(p[2]);
    peer_flags[w] = static_cast<uint64_t*>(p[3]);
  }
  ready = true;
  return true;
}

void ShardPlan::run(const uint64_t* d_ids, uint64_t vocab, int32_t* d_bad, int k, Exchange& xch,
                    uint32_t* owned_uniq, uint32_t* own_k, int32_t* d_n_own, int32_t* d_U_global,
                    cudaStream_t s, const PhaseHook& hook) {
  const int64_t total = static_cast<int64_t>(W) * n;
  PeerPairs pp{};
  PeerInts pi{};
  PeerFlagsS pf{};
  PeerReply pr{};
  for (int w = 0; w < W; ++w) {
    pp.dst[w] = peer_pairs[w] + k * total;
    pi.p[w] = peer_inbox[w] + k * kInbox;
    pf.p[w] = peer_flags[w];
    pr.p[w] = peer_reply[w] + k * total;
  }
  const uint64_t* prs = pairs + k * total;
  const int32_t* ibx = inbox + k * kInbox;
  const uint64_t tmo = barrier_timeout_ns();
  const int gx = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(n, 256), num_sms() * 8 / W)));  // per source region
  // 1. route + B1 (pair counts into every owner's inbox[72 + me], the bad-id bit)
  launch_pdl(route_pairs_kernel, dim3(static_cast<int>(std::max<int64_t>(1, ceil_div(n, 256 * kRouteItems)))), dim3(256), 0, s, d_ids, n, vocab, W, me, d_bad, cursor, pp, rix + k * n);
  CUDA_LAUNCH_CHECK();
  hook("shard_route");
  launch_pdl(publish_barrier_kernel, dim3(1), dim3(32), 0, s, 0, pi, cursor, nullptr, nullptr, pf, W, me, ++epoch,
                                          tmo, abort_flag, d_bad);
  CUDA_LAUNCH_CHECK();
  hook("shard_b1");
  // 2. dedup, 3. first positions -> owned uniques in global first-appearance order
  launch_pdl(dedup_pairs_kernel, dim3(dim3(gx, W)), dim3(256), 0, s, prs, n, ibx, hkeys, hpos, hmask_bits, hmask,
                                                 hslot);
  CUDA_LAUNCH_CHECK();
  hook("shard_dedup");
  launch_pdl(first_bits_kernel, dim3(dim3(gx, W)), dim3(256), 0, s, prs, n, ibx, hslot, hpos, bits,
             xch.tile_cnt, xch.tile_words());
  CUDA_LAUNCH_CHECK();
  hook("shard_first");
  lookback_scan<4>(tiles, nwords, WordCount{bits}, WordPrefix{wpre}, d_n_own, s);
  hook("shard_scan");
  launch_pdl(first_emit_kernel, dim3(dim3(gx, W)), dim3(256), 0, s, prs, n, ibx, hslot, hpos, bits, wpre, hkeys,
                                                hmask_bits, owned_uniq, own_k, xch.tm, uslot, xch.tile_cnt);
  CUDA_LAUNCH_CHECK();
  hook("shard_emit");
  // 4. send plan over my owned uniques, my column of the count matrix + my count; B2
  xch.send_plan_counted(d_n_own, s);
  hook("shard_plan");
  launch_pdl(publish_barrier_kernel, dim3(1), dim3(32), 0, s, 1, pi, nullptr, xch.totals, d_n_own, pf, W, me, ++epoch,
                                          tmo, abort_flag, nullptr);
  CUDA_LAUNCH_CHECK();
  hook("shard_b2");
  // 5 + 6. layout + replies, then the table reset (no barrier after the replies, see top)
  launch_pdl(reply_kernel, dim3(dim3(gx, W + 1)), dim3(256), 0, s, n, W, me, ibx, hslot, hpos, xch.sscan, xch.tm,
                                               d_n_own, xch.lpos, xch.totals, d_U_global, pr);
  CUDA_LAUNCH_CHECK();
  hook("shard_reply");
  xch.plan_offsets(s);
  launch_pdl(reset_table_kernel, dim3(std::max(1, std::min(ceil_div(cap, 256), num_sms() * 4))), dim3(256), 0, s, uslot, d_n_own, hkeys, hpos, hmask_bits, cursor, bits, nwords);
  CUDA_LAUNCH_CHECK();
  hook("shard_reset");
}

}  // namespace sfb
