// MixCache on the device: the HostStore (host_store.hpp:61-92) as a pinned,
// mapped host table indexed by owned row r = f / W, the CacheBuffer
// (cache_buffer.hpp:40-86) as an HBM slot pool per worker lane, and the
// manager policy (missing manager.cpp) reproduced exactly:
//
//   needed_soon  := owned resident features of the window batches       (mark[s] == t)
//   hits         := owned resident features of batch t, touched         (last_use[s] = t)
//   working      := owned non-resident features, in global_ids order    (scan-compacted)
//   evict        := max(0, |working| - free) eligible slots with the smallest
//                   (last_use, admit_seq), oldest first; each pushes its slot on the
//                   LIFO free stack (cache_buffer.cpp:64)
//   admit        := working[i] takes free_stack[top - 1 - i] (pop order of
//                   cache_buffer.cpp:41-42), admit_seq = seq0 + i, last_use = t
//
// Per-row state moves host <-> HBM by zero-copy loads/stores from the kernels
// (PCIe) into a lazily grown pool of pinned host slabs (HostPool, cache.h);
// never-touched rows are initialised on the device with the reference's
// initial_embedding stream (generator.cpp:110-115) instead of being read over
// PCIe, so only rows that were evicted at least once hold host memory. The
// LRU victims are selected exactly by a last_use histogram + a threshold step
// + a sort of the few candidates at or below it (never a sort over C slots).
#include "cache.h"

namespace sfb {

namespace {

// Counts live on the device (U, n_own): the scans cover the upper bound `cap` and items
// past the live count contribute 0, so no host round trip sizes the manage kernels.
// Both selections below are one fused look-back scan each (scan.cuh): the flag, the scan
// and the compaction in a single launch.

// owned uniques of worker w (f mod W == w), in global_ids order -> own_k;
// first != nullptr: also clears the VSI first-position table behind the batch (every unique
// passes here once)
struct OwnedFlag {
  const uint32_t* gids;
  const int32_t* U;
  uint32_t W, w;
  uint32_t* first;
  __device__ uint32_t operator()(int64_t i) const {
    if (i >= *U) return 0u;
    const uint32_t f = gids[i];
    if (first) first[f] = kEmpty;
    return f % W == w ? 1u : 0u;
  }
};
struct OwnedEmit {
  uint32_t* own_k;
  __device__ void operator()(int64_t i, uint32_t flag, uint32_t rank) const {
    if (flag) own_k[rank] = static_cast<uint32_t>(i);
  }
};

__global__ void own_all_kernel(const int32_t* __restrict__ U_ptr, uint32_t* __restrict__ own_k,
                               int32_t* __restrict__ count, const uint32_t* __restrict__ gids,
                               uint32_t* __restrict__ first) {
  pdl_wait();
  const int32_t U = *U_ptr;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < U; j += gridDim.x * blockDim.x) {
    own_k[j] = static_cast<uint32_t>(j);
    if (first) first[gids[j]] = kEmpty;  // VSI table reset (see OwnedFlag)
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = U;
}

// Probe the owned features of batch t: hits are touched and marked needed_soon, misses
// listed for admission in global_ids order with their probe-time feature and index entry
// (work_j / work_f / work_w), so admit reads them coalesced.
struct ProbeFlag {
  const uint32_t* own_k;
  const int32_t* n_own;
  const uint32_t* gids;
  uint32_t W;
  const uint32_t* index;
  uint32_t C;
  int32_t t;
  int32_t* last_use;
  int32_t* mark;
  uint32_t* own_slot;
  int32_t* marked;
  uint32_t* own_f;
  __device__ uint32_t operator()(int64_t j) const {
    if (j >= *n_own) return 0u;
    const uint32_t f = gids[own_k[j]];
    const uint32_t s = index[f / W];
    own_slot[j] = s;  // host slot / kNever until admit assigns the slot
    bool newly_marked = false;
    if (s < C) {
      if (t > last_use[s]) last_use[s] = t;  // CacheBuffer::touch (cache_buffer.cpp:69-72)
      newly_marked = atomicExch(mark + s, t) != t;
    } else {
      own_f[j] = f;
    }
    // one counter atomic per group of converged lanes, not per hit: ~100 k hits per step
    // on a single address were serialised at one L2 slice
    const unsigned am = __activemask();
    const unsigned bal = __ballot_sync(am, newly_marked);
    if (bal && (threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(marked, __popc(bal));
    return s < C ? 0u : 1u;
  }
};
struct ProbeEmit {
  const uint32_t* own_f;
  const uint32_t* own_slot;
  uint32_t* work_j;
  uint32_t* work_f;
  uint32_t* work_w;
  __device__ void operator()(int64_t j, uint32_t miss, uint32_t rank) const {
    if (!miss) return;
    work_j[rank] = static_cast<uint32_t>(j);
    work_f[rank] = own_f[j];
    work_w[rank] = own_slot[j];
  }
};

// needed_soon for resident owned features of a lookahead batch
__global__ void mark_window_kernel(const uint32_t* __restrict__ gids,
                                   const int32_t* __restrict__ U_ptr, int32_t cap, uint32_t W,
                                   uint32_t w, const uint32_t* __restrict__ index, uint32_t C,
                                   int32_t t, int32_t* __restrict__ mark,
                                   int32_t* __restrict__ marked) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool newly = false;
  if (i < cap && i < *U_ptr) {
    const uint32_t f = gids[i];
    if (f % W == w) {
      const uint32_t s = index[f / W];
      newly = s < C && atomicExch(mark + s, t) != t;
    }
  }
  const unsigned bal = __ballot_sync(0xFFFFFFFFu, newly);  // one counter atomic per warp
  if (bal && (threadIdx.x & 31) == 0) atomicAdd(marked, __popc(bal));
}

// LRU histogram over last_use of the eligible slots (occupied && !needed_soon; pins are
// implied by BSP stream order: batch t-1's update has completed before manage(t) runs, and
// the pipelined manager checks counters[kCntOld] before evicting), in two levels so the
// bins always fit shared memory: level 1 bins last_use >> shift over [0, t]; level 2 (when
// shift > 0) counts the 2^shift steps of the threshold's coarse bin exactly. Each block
// owns a contiguous chunk of slots and a shared-memory histogram (lanes of a warp with the
// same value merge through match_any: slots admitted together sit next to each other), and
// flushes its non-zero bins with one global atomic each: same-address global atomics from
// every warp were the bottleneck of a single global histogram.
// base_bin: level 2 restricts to [cnt[kCntSelB] << base_shift, + nbins); count_old also
// counts the eligible slots last used before step t-1 (pipelined eviction safety).
constexpr int kHistBins = 8192;  // shared-memory bins per level
__global__ void __launch_bounds__(1024) lru_hist_kernel(
    uint32_t C, const uint32_t* __restrict__ slot_feat, const int32_t* __restrict__ mark, int32_t t,
    const int32_t* __restrict__ last_use, uint32_t* __restrict__ hist, int nbins, int shift,
    int32_t* __restrict__ cnt, int base_shift, bool level2, const uint8_t* __restrict__ pin) {
  pdl_wait();
  __shared__ uint32_t sh[kHistBins];
  __shared__ uint32_t old_blk;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) old_blk = 0;
  __syncthreads();
  const int32_t base = level2 ? (cnt[kCntSelB] << base_shift) : 0;
  const int lane = threadIdx.x & 31;
  // 4 slots per thread per round (16 B loads of slot_feat / mark / last_use, issued before
  // any use): the pass streams 12 B per slot at HBM rate instead of one dependent chain
  const uint64_t C4 = (static_cast<uint64_t>(C) + 3) >> 2;
  const uint64_t chunk = (C4 + gridDim.x - 1) / gridDim.x;
  const uint64_t q0 = blockIdx.x * chunk, q1 = q0 + chunk < C4 ? q0 + chunk : C4;
  uint32_t old = 0;
  for (uint64_t qw = q0 + (threadIdx.x & ~31u); qw < q1; qw += blockDim.x) {
    const uint64_t q = qw + lane;
    uint4 f = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    int4 mk = make_int4(t, t, t, t), lu = make_int4(0, 0, 0, 0);
    if (q < q1) {
      if (4 * q + 3 < C) {
        f = __ldcs(reinterpret_cast<const uint4*>(slot_feat) + q);
        mk = __ldcs(reinterpret_cast<const int4*>(mark) + q);
        lu = __ldcs(reinterpret_cast<const int4*>(last_use) + q);
      } else {
        uint32_t* fp = &f.x;
        int* mp = &mk.x;
        int* lp = &lu.x;
        for (int e = 0; e < 4 && 4 * q + e < C; ++e) {
          fp[e] = slot_feat[4 * q + e];
          mp[e] = mark[4 * q + e];
          lp[e] = last_use[4 * q + e];
        }
      }
    }
    uint32_t fa[4] = {f.x, f.y, f.z, f.w};
    const int32_t ma[4] = {mk.x, mk.y, mk.z, mk.w}, la[4] = {lu.x, lu.y, lu.z, lu.w};
    if (pin && q < q1)  // standalone CacheBuffer: pinned slots are not evictable
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < C && pin[4 * q + e]) fa[e] = kEmpty;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int bin = -1;
      if (fa[e] != kEmpty && ma[e] != t) {
        old += la[e] < t - 1;
        const int32_t b = (la[e] - base) >> shift;
        if (la[e] >= base && b < nbins) bin = b;
      }
      const unsigned act = __ballot_sync(0xFFFFFFFFu, bin >= 0);
      if (bin >= 0) {
        const unsigned peers = __match_any_sync(act, bin);
        if (lane == __ffs(peers) - 1) atomicAdd(sh + bin, static_cast<uint32_t>(__popc(peers)));
      }
    }
  }
  if (!level2) {
    for (int off = 16; off > 0; off >>= 1) old += __shfl_xor_sync(0xFFFFFFFFu, old, off);
    if (lane == 0 && old) atomicAdd(&old_blk, old);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
  if (threadIdx.x == 0 && old_blk) atomicAdd(cnt + kCntOld, static_cast<int32_t>(old_blk));
}

// One block: the bin B = min{B : #(bins <= B) >= need} of a level's histogram, with need =
// n_evict (level 1) or n_evict - #(below the coarse bin) (level 2); the last bin when fewer
// eligible slots exist (the eviction kernel then flags the capacity deadlock). Level 1
// writes B and #(bins < B) (kCntSelB / kCntSelBelow) and, when it is final (shift 0), the
// threshold step kCntSelT; level 2 writes kCntSelT = (coarse bin << shift) + B.
__global__ void __launch_bounds__(1024) lru_select_kernel(const uint32_t* __restrict__ hist,
                                                          int32_t nbins, int32_t n_evict,
                                                          int32_t* __restrict__ cnt, int shift,
                                                          bool level2) {
  pdl_wait();
  __shared__ uint64_t part[1024];
  __shared__ int32_t found;
  __shared__ uint64_t found_below;
  const int tid = threadIdx.x;
  const uint64_t need =
      static_cast<uint64_t>(n_evict) - (level2 ? static_cast<uint64_t>(cnt[kCntSelBelow]) : 0);
  const int per = (nbins + 1023) / 1024;
  const int lo = min(nbins, tid * per), hi = min(nbins, lo + per);
  uint64_t sum = 0;
  for (int i = lo; i < hi; ++i) sum += hist[i];
  part[tid] = sum;
  if (tid == 0) {
    found = nbins - 1;
    found_below = 0;
  }
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan of the chunk sums
    const uint64_t v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  const uint64_t before = tid ? part[tid - 1] : 0;
  if (tid == 1023 && part[1023] < need) found_below = part[1023] - (nbins ? hist[nbins - 1] : 0);
  if (before < need && part[tid] >= need) {
    uint64_t run = before;
    for (int i = lo; i < hi; ++i) {
      if (run + hist[i] >= need) {
        found = i;
        found_below = run;
        break;
      }
      run += hist[i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (level2) {
      cnt[kCntSelT] = (cnt[kCntSelB] << shift) + found;
    } else {
      cnt[kCntSelB] = found;
      cnt[kCntSelBelow] = static_cast<int32_t>(found_below);
      cnt[kCntSelTotal] = static_cast<int32_t>(part[1023] < 0x7FFFFFFFull ? part[1023] : 0x7FFFFFFFull);
      if (shift == 0) cnt[kCntSelT] = found;
    }
    cnt[kCntSelN] = 0;
  }
}

// The victim candidates: eligible slots with last_use <= T, key (last_use, admit_seq).
// At most n_evict - 1 + #(last_use == T) <= n_evict + umax of them (the slots last used at
// step T were touched by that step's owned uniques). Unused entries keep the ~0 key.
__global__ void lru_collect_kernel(uint32_t C, const uint32_t* __restrict__ slot_feat,
                                   const int32_t* __restrict__ mark, int32_t t,
                                   const int32_t* __restrict__ last_use,
                                   const uint64_t* __restrict__ admit_seq,
                                   int32_t* __restrict__ cnt, int64_t cap,
                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                                   const uint8_t* __restrict__ pin) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int32_t T = cnt[kCntSelT];
  const uint64_t C4 = (static_cast<uint64_t>(C) + 3) >> 2;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // 4 slots per thread per round, as in lru_hist_kernel
  for (uint64_t qw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
       qw < C4; qw += nthreads) {
    const uint64_t q = qw + lane;
    uint4 f = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    int4 mk = make_int4(t, t, t, t), lu = make_int4(0, 0, 0, 0);
    if (q < C4) {
      if (4 * q + 3 < C) {
        f = __ldcs(reinterpret_cast<const uint4*>(slot_feat) + q);
        mk = __ldcs(reinterpret_cast<const int4*>(mark) + q);
        lu = __ldcs(reinterpret_cast<const int4*>(last_use) + q);
      } else {
        uint32_t* fp = &f.x;
        int* mp = &mk.x;
        int* lp = &lu.x;
        for (int e = 0; e < 4 && 4 * q + e < C; ++e) {
          fp[e] = slot_feat[4 * q + e];
          mp[e] = mark[4 * q + e];
          lp[e] = last_use[4 * q + e];
        }
      }
    }
    uint32_t fa[4] = {f.x, f.y, f.z, f.w};
    const int32_t ma[4] = {mk.x, mk.y, mk.z, mk.w}, la[4] = {lu.x, lu.y, lu.z, lu.w};
    if (pin && q < C4)
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < C && pin[4 * q + e]) fa[e] = kEmpty;
    uint32_t take = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (fa[e] != kEmpty && ma[e] != t && la[e] <= T) take |= 1u << e;
    const int mine = __popc(take);
    // warp-inclusive scan of the per-thread candidate counts
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, off);
      if (lane >= off) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (!total) continue;
    int32_t base = 0;
    if (lane == 31) base = atomicAdd(cnt + kCntSelN, total);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    int64_t pos = base + incl - mine;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!((take >> e) & 1u)) continue;
      const uint64_t sl = 4 * q + e;
      if (pos < cap) {
        keys[pos] = (static_cast<uint64_t>(la[e] + 1) << 40) | (admit_seq[sl] & ((1ull << 40) - 1));
        ids[pos] = static_cast<uint32_t>(sl);
      }
      ++pos;
    }
  }
}

// pull_parameters_to_host: one warp per victim, 16 B zero-copy stores into the victim's
// host slot (its old one, or a new one from the pool); the slot goes on top of the free
// stack.
__global__ void evict_kernel(int32_t n_evict, const uint64_t* __restrict__ sorted_keys,
                             const uint32_t* __restrict__ sorted_ids, uint32_t* __restrict__ slot_feat,
                             uint32_t W, int d, const float* __restrict__ emb,
                             const float* __restrict__ mom, const float* __restrict__ vel,
                             const int32_t* __restrict__ steps, HostTab host,
                             uint32_t* __restrict__ slot_host, int32_t* __restrict__ host_next,
                             uint32_t* __restrict__ index, uint32_t* __restrict__ free_stack,
                             const int32_t* __restrict__ free_top_ptr, int32_t* __restrict__ err) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_evict) return;
  if (sorted_keys[warp] == ~0ull) {  // fewer eligible slots than needed: capacity deadlock
    if (lane == 0) *err = 1;
    return;
  }
  const uint32_t s = sorted_ids[warp];
  const uint32_t f = slot_feat[s];
  const uint64_t r = f / W;
  uint32_t h = 0;
  if (lane == 0) {
    h = slot_host[s];
    if (h == kNoHost) h = static_cast<uint32_t>(atomicAdd(host_next, 1));
  }
  h = __shfl_sync(0xFFFFFFFFu, h, 0);
  float* dst = host.row(h, 3 * d);
  const size_t so = static_cast<size_t>(s) * 3 * d;  // slot rows: [emb | m | v]
  if ((d & 3) == 0) {
    const int d4 = d >> 2;
    for (int c = lane; c < 3 * d4; c += 32) {
      const int which = c / d4, cc = c - which * d4;
      const float* src = (which == 0 ? emb : which == 1 ? mom : vel) + so;
      reinterpret_cast<float4*>(dst)[c] = reinterpret_cast<const float4*>(src)[cc];
    }
  } else {
    for (int c = lane; c < 3 * d; c += 32) {
      const int which = c / d, cc = c - which * d;
      dst[c] = (which == 0 ? emb : which == 1 ? mom : vel)[so + cc];
    }
  }
  if (lane == 0) {
    *host.step(h) = steps[s];
    index[r] = kHostBit | h;
    slot_feat[s] = kEmpty;
    slot_host[s] = kNoHost;
    free_stack[*free_top_ptr + warp] = s;
  }
}

// push_parameters_to_cache: one warp per admitted feature.
// One warp per kAdmitRows admitted rows. The probe already recorded each miss's
// feature and index entry (work_f / work_w), so the per-row facts are coalesced loads:
// lane l < kAdmitRows takes row i0 + l (bookkeeping + its lazy-init seed), then all 32
// lanes fill the group's (row, 16 B chunk) items with 128-bit stores.
constexpr int kAdmitRows = 8;
__global__ void admit_kernel(const int32_t* __restrict__ counters, int32_t n_evict,
                             const uint32_t* __restrict__ work_j,
                             const uint32_t* __restrict__ work_f,
                             const uint32_t* __restrict__ work_w, uint32_t W, int d,
                             const uint32_t* __restrict__ free_stack,
                             uint32_t* __restrict__ index, HostTab host,
                             uint32_t* __restrict__ slot_host, uint64_t seed,
                             uint64_t embed_hash, float* __restrict__ emb, float* __restrict__ mom,
                             float* __restrict__ vel, int32_t* __restrict__ steps,
                             uint32_t* __restrict__ slot_feat, int32_t* __restrict__ last_use,
                             uint64_t* __restrict__ admit_seq,
                             int32_t* __restrict__ mark, int32_t t,
                             uint32_t* __restrict__ own_slot, int32_t* __restrict__ n_from_host) {
  pdl_wait();
  const int32_t n_work = counters[kCntWorking];
  const int32_t free_top = counters[kCntFreeTop] + n_evict;
  const uint64_t seq0 = *reinterpret_cast<const uint64_t*>(counters + kCntSeq);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // grid-stride over warps: the grid is capped (mgr_grid) so the manager stage never fills an
  // SM that a persistent training kernel is about to need
  for (int64_t wi = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       wi * kAdmitRows < n_work; wi += nwarps) {
  const int64_t i0 = wi * kAdmitRows;
  const int64_t mi = i0 + lane;
  const bool mine = lane < kAdmitRows && mi < n_work;
  uint32_t my_f = 0, my_s = 0, my_where = kNever;
  uint64_t my_se = 0;
  if (mine) {
    const uint32_t j = work_j[mi];
    my_f = work_f[mi];
    my_where = work_w[mi];
    my_s = free_stack[free_top - 1 - mi];
    slot_feat[my_s] = my_f;
    last_use[my_s] = t;
    admit_seq[my_s] = seq0 + static_cast<uint64_t>(mi);
    mark[my_s] = t;
    index[my_f / W] = my_s;
    own_slot[j] = my_s;
    if (on_host(my_where)) {
      steps[my_s] = *host.step(my_where & ~kHostBit);
      slot_host[my_s] = my_where & ~kHostBit;
    } else {
      steps[my_s] = 0;
      slot_host[my_s] = kNoHost;
      my_se = derive_seed_h(seed, embed_hash, my_f);  // HostStore::get_or_init (host_store.cpp:25-33)
    }
  }
  const unsigned from_host = __ballot_sync(0xFFFFFFFFu, mine && on_host(my_where));
  if (lane == 0 && from_host) atomicAdd(n_from_host, __popc(from_host));
  const int nrows = n_work - i0 < kAdmitRows ? static_cast<int>(n_work - i0) : kAdmitRows;
  const bool vec = (d & 3) == 0;
  const int per = vec ? d >> 2 : d;  // items per row: 16 B chunks (or scalars)
  const int items = nrows * per;
  for (int base = 0; base < items; base += 32) {  // uniform trip count: all lanes shuffle
    const int it = base + lane;
    const int k = it < items ? it / per : 0;
    const uint32_t sl = __shfl_sync(0xFFFFFFFFu, my_s, k);
    const uint32_t where = __shfl_sync(0xFFFFFFFFu, my_where, k);
    const uint64_t se = __shfl_sync(0xFFFFFFFFu, my_se, k);
    if (it >= items) continue;
    const int c = it - k * per;  // chunk (or column) within the row
    const size_t so = static_cast<size_t>(sl) * 3 * d;  // slot rows: [emb | m | v]
    if (on_host(where)) {
      const float* src = host.row(where & ~kHostBit, 3 * d);
      if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        reinterpret_cast<float4*>(emb + so)[c] = s4[c];
        reinterpret_cast<float4*>(mom + so)[c] = s4[per + c];
        reinterpret_cast<float4*>(vel + so)[c] = s4[2 * per + c];
      } else {
        emb[so + c] = src[c];
        mom[so + c] = src[d + c];
        vel[so + c] = src[2 * d + c];
      }
    } else {
      auto init = [&](int col) {
        return static_cast<float>(
            uniform_from(splitmix_mix(se + (col + 1) * kGolden), -0.01, 0.01));
      };
      if (vec) {
        const int c0 = 4 * c;
        reinterpret_cast<float4*>(emb + so)[c] =
            make_float4(init(c0), init(c0 + 1), init(c0 + 2), init(c0 + 3));
        reinterpret_cast<float4*>(mom + so)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(vel + so)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        emb[so + c] = init(c);
        mom[so + c] = 0.f;
        vel[so + c] = 0.f;
      }
    }
  }
  }
}

// Fused pull_parameters_to_host + push_parameters_to_cache for eviction steps: admission
// i < n_evict lands in the slot of victim n_evict-1-i (the LIFO pop order of evict's pushes,
// cache_buffer.cpp:41-42,64), so one warp writes that victim back to the pinned host table
// and then fills its slot, and admissions i >= n_evict pop the free stack below the victims.
// Every warp both stores to and loads from host memory, which keeps PCIe busy in both
// directions at once (the write-back alone runs at ~44 GB/s of SM stores; see
// microbench/pcie_rows.cu). The slot's victim state is staged in registers before the
// admitted row overwrites it: 3*d/4 <= 64 float4 chunks per row (d <= 84).
__global__ void __launch_bounds__(256) swap_kernel(
    const int32_t* __restrict__ counters, int32_t n_evict,
    const uint64_t* __restrict__ sorted_keys, const uint32_t* __restrict__ sorted_ids,
    const uint32_t* __restrict__ work_j, const uint32_t* __restrict__ work_f,
    const uint32_t* __restrict__ work_w, uint32_t W, int d4,
    const uint32_t* __restrict__ free_stack, uint32_t* __restrict__ index, HostTab host,
    uint32_t* __restrict__ slot_host, int32_t* __restrict__ host_next, uint64_t seed,
    uint64_t embed_hash, float4* __restrict__ emb, float4* __restrict__ mom,
    float4* __restrict__ vel, int32_t* __restrict__ steps, uint32_t* __restrict__ slot_feat,
    int32_t* __restrict__ last_use, uint64_t* __restrict__ admit_seq,
    int32_t* __restrict__ mark, int32_t t, uint32_t* __restrict__ own_slot,
    int32_t* __restrict__ n_from_host, int32_t* __restrict__ err) {
  pdl_wait();
  __shared__ __align__(128) float4 wb_stage[8][64];   // per warp: the victim row (<= 64 chunks)
  __shared__ __align__(128) float4 adm_stage[8][64];  // per warp: the refilled host row
  __shared__ __align__(8) uint64_t adm_bar[8];
  const int32_t n_work = counters[kCntWorking];
  const int32_t free_top = counters[kCntFreeTop];
  const uint64_t seq0 = *reinterpret_cast<const uint64_t*>(counters + kCntSeq);
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_work) return;
  const int per = 3 * d4;  // float4 chunks per row: emb | m | v
  auto src_of = [&](int c, float4* e, float4* m, float4* v, size_t so) -> float4* {
    const int which = c / d4;
    return (which == 0 ? e : which == 1 ? m : v) + so + (c - which * d4);
  };
  uint32_t s;
  float4 keep[2];
  if (i < n_evict) {
    const int64_t vi = n_evict - 1 - i;
    if (sorted_keys[vi] == ~0ull) {  // fewer eligible slots than needed: capacity deadlock
      if (lane == 0) *err = 1;
      return;
    }
    s = sorted_ids[vi];
    const uint32_t fo = slot_feat[s];
    const uint64_t ro = fo / W;
    uint32_t ho = 0;  // the victim's host slot: its old one, or a new one from the pool
    if (lane == 0) {
      ho = slot_host[s];
      if (ho == kNoHost) ho = static_cast<uint32_t>(atomicAdd(host_next, 1));
    }
    ho = __shfl_sync(0xFFFFFFFFu, ho, 0);
    const size_t so = static_cast<size_t>(s) * 3 * d4;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = lane + 32 * q;
      if (c < per) keep[q] = *src_of(c, emb, mom, vel, so);
    }
    // write-back by one TMA bulk store per row (smem -> pinned host row): larger PCIe
    // writes than 16 B SM stores (microbench/pcie_rows.cu: 48 vs 44.5 GB/s)
    float4* stage = wb_stage[threadIdx.x >> 5];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = lane + 32 * q;
      if (c < per) stage[c] = keep[q];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                       host.row(ho, 4 * per)),
                   "r"(sa), "r"(per * 16)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (lane == 0) {
      *host.step(ho) = steps[s];
      index[ro] = kHostBit | ho;
    }
  } else {
    s = free_stack[free_top - 1 - (i - n_evict)];
  }
  const uint32_t f = work_f[i];
  const uint32_t where = work_w[i];
  const uint64_t r = f / W;
  const size_t so = static_cast<size_t>(s) * 3 * d4;
  if (on_host(where)) {
    // refill by one TMA bulk load of the host row (one large PCIe read instead of 16 B SM
    // loads), completion tracked by the warp's mbarrier
    const int wid = threadIdx.x >> 5;
    float4* astage = adm_stage[wid];
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&adm_bar[wid]));
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(per * 16)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<uint32_t>(__cvta_generic_to_shared(astage))),
          "l"(host.row(where & ~kHostBit, 4 * per)), "r"(per * 16), "r"(bar)
          : "memory");
    }
    __syncwarp();
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W;\n\t}" ::"r"(bar)
        : "memory");
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = lane + 32 * q;
      if (c < per) *src_of(c, emb, mom, vel, so) = astage[c];
    }
  } else {
    const uint64_t se = derive_seed_h(seed, embed_hash, f);  // HostStore::get_or_init
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = lane + 32 * q;
      if (c >= per) continue;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < d4) {
        auto init = [&](int col) {
          return static_cast<float>(uniform_from(splitmix_mix(se + (col + 1) * kGolden), -0.01, 0.01));
        };
        x = make_float4(init(4 * c), init(4 * c + 1), init(4 * c + 2), init(4 * c + 3));
      }
      *src_of(c, emb, mom, vel, so) = x;
    }
  }
  if (lane == 0) {
    steps[s] = on_host(where) ? *host.step(where & ~kHostBit) : 0;
    slot_host[s] = on_host(where) ? (where & ~kHostBit) : kNoHost;
    slot_feat[s] = f;
    last_use[s] = t;
    admit_seq[s] = seq0 + static_cast<uint64_t>(i);
    mark[s] = t;
    index[r] = s;
    own_slot[work_j[i]] = s;
  }
  const unsigned fh = __ballot_sync(0xFFFFFFFFu, lane == 0 && on_host(where));
  if (lane == 0 && fh) atomicAdd(n_from_host, 1);
  // the staged row must be read (and written) before the warp's shared memory is released
  if (lane == 0 && i < n_evict) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void init_lane_kernel(uint32_t C, uint32_t* slot_feat, int32_t* last_use,
                                 int32_t* mark, uint32_t* free_stack) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < C; s += gridDim.x * blockDim.x) {
    slot_feat[s] = kEmpty;
    last_use[s] = -1;
    mark[s] = -1;
    free_stack[s] = C - 1 - s;  // lower slots at the top (cache_buffer.cpp:27-28)
  }
}

// device free-stack height and admit_seq after this step's evictions and admissions
__global__ void advance_kernel(int32_t* counters, int32_t n_evict) {
  pdl_wait();
  const int32_t n_work = counters[kCntWorking];
  counters[kCntFreeTop] += n_evict - n_work;
  *reinterpret_cast<uint64_t*>(counters + kCntSeq) += static_cast<uint64_t>(n_work);
}

__global__ void fill_u32(uint32_t* p, uint64_t n, uint32_t v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

}  // namespace

void HostPool::init(int dim, uint64_t owned_rows, uint64_t reserve_rows) {
  d = dim;
  CUDA_CHECK(cudaGetDevice(&dev));
  // slab_rows = 2^shift: the largest power of two with slab_rows * 12d <= 256 MB, but no
  // larger than the owned shard needs (small tables get small slabs)
  const uint64_t row_bytes = 12ull * static_cast<uint64_t>(dim);
  shift = 10;
  while (shift < 30 && (2ull << shift) * row_bytes <= (256ull << 20) &&
         (1ull << shift) < owned_rows)
    ++shift;
  CUDA_CHECK(cudaMalloc(&d_rows, sizeof(float*) * kMaxSlabs));
  CUDA_CHECK(cudaMalloc(&d_steps, sizeof(int32_t*) * kMaxSlabs));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_rows_tab), sizeof(float*) * kMaxSlabs, 0));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_steps_tab), sizeof(int32_t*) * kMaxSlabs, 0));
  cap = hi = 0;
  if (reserve_rows) ensure(reserve_rows, nullptr);
}

std::pair<float*, int32_t*> HostPool::alloc_slab() {
  const uint64_t slab_rows = 1ull << shift;
  float* r = nullptr;
  int32_t* st = nullptr;
  if (cudaHostAlloc(reinterpret_cast<void**>(&r), sizeof(float) * slab_rows * 3 * d,
                    cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&st), sizeof(int32_t) * slab_rows,
                    cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    if (r) cudaFreeHost(r);
    return {nullptr, nullptr};
  }
  return {r, st};
}

void HostPool::prefetch() {
  {
    std::lock_guard<std::mutex> g(mu);
    if (filler_failed || static_cast<int>(spares.size()) >= kAhead) return;
  }
  if (filler.joinable()) {  // a previous round finished (or is finishing): reap it
    filler.join();
  }
  filler = std::thread([this] {
    cudaSetDevice(dev);
    for (;;) {
      {
        std::lock_guard<std::mutex> g(mu);
        if (static_cast<int>(spares.size()) >= kAhead) return;
      }
      auto slab = alloc_slab();
      std::lock_guard<std::mutex> g(mu);
      if (!slab.first) {
        filler_failed = true;
        return;
      }
      spares.push_back(slab);
    }
  });
}

void HostPool::ensure(uint64_t slots, cudaStream_t s) {
  const uint64_t slab_rows = 1ull << shift;
  if (slots > cap) {
    const size_t first = rows_h.size();
    while (cap < slots) {
      if (rows_h.size() >= static_cast<size_t>(kMaxSlabs) || cap + slab_rows > (1ull << 31) - 1)
        fail(kRun, "host pool exhausted: " + std::to_string(cap) + " evicted rows per worker");
      std::pair<float*, int32_t*> slab{nullptr, nullptr};
      {
        std::lock_guard<std::mutex> g(mu);
        if (!spares.empty()) {
          slab = spares.back();
          spares.pop_back();
        }
      }
      if (!slab.first) slab = alloc_slab();
      if (!slab.first)
        fail(kRun, "cannot pin " + std::to_string((sizeof(float) * slab_rows * 3 * d) >> 20) +
                       " MiB more for the host pool (" + std::to_string(cap) +
                       " evicted rows held)");
      float* rd = nullptr;
      int32_t* sd = nullptr;
      CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&rd), slab.first, 0));
      CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&sd), slab.second, 0));
      h_rows_tab[rows_h.size()] = rd;
      h_steps_tab[rows_h.size()] = sd;
      rows_h.push_back(slab.first);
      steps_h.push_back(slab.second);
      cap += slab_rows;
    }
    const size_t n = rows_h.size() - first;
    CUDA_CHECK(cudaMemcpyAsync(d_rows + first, h_rows_tab + first, sizeof(float*) * n,
                               cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(d_steps + first, h_steps_tab + first, sizeof(int32_t*) * n,
                               cudaMemcpyHostToDevice, s));
    if (!s) CUDA_CHECK(cudaStreamSynchronize(nullptr));
  }
  if (cap - std::min(cap, slots) < static_cast<uint64_t>(kAhead) * slab_rows) prefetch();
}

void HostPool::release() {
  if (filler.joinable()) filler.join();
  for (auto& p : spares) {
    cudaFreeHost(p.first);
    cudaFreeHost(p.second);
  }
  spares.clear();
  for (float* p : rows_h) cudaFreeHost(p);
  for (int32_t* p : steps_h) cudaFreeHost(p);
  if (d_rows) cudaFree(d_rows);
  if (d_steps) cudaFree(d_steps);
  if (h_rows_tab) cudaFreeHost(h_rows_tab);
  if (h_steps_tab) cudaFreeHost(h_steps_tab);
  rows_h.clear();
  steps_h.clear();
  d = shift = dev = 0;
  cap = hi = 0;
  d_rows = nullptr;
  d_steps = nullptr;
  h_rows_tab = nullptr;
  h_steps_tab = nullptr;
  filler_failed = false;
}

void CacheLane::init(uint64_t capacity, int dim, uint64_t owned_rows, uint64_t host_reserve,
                     int64_t max_unique) {
  C = capacity;
  d = dim;
  rows = owned_rows;
  umax = max_unique > 0 ? max_unique : 1;
  const size_t cd = static_cast<size_t>(C) * d;
  // one [C x 3d] table: slot s holds [emb | m | v] contiguously (960 B at d = 80), so the
  // Adam update, admission and write-back touch one contiguous segment per slot instead of
  // three (microbench/adam_layout.cu: +12-17 % for the random-slot update)
  CUDA_CHECK(cudaMalloc(&emb, sizeof(float) * cd * 3));
  CUDA_CHECK(cudaMemset(emb, 0, sizeof(float) * cd * 3));
  mom = emb + d;
  vel = emb + 2 * d;
  CUDA_CHECK(cudaMalloc(&steps, sizeof(int32_t) * C));
  CUDA_CHECK(cudaMemset(steps, 0, sizeof(int32_t) * C));
  CUDA_CHECK(cudaMalloc(&slot_feat, sizeof(uint32_t) * C));
  CUDA_CHECK(cudaMalloc(&last_use, sizeof(int32_t) * C));
  CUDA_CHECK(cudaMalloc(&admit_seq, sizeof(uint64_t) * C));
  CUDA_CHECK(cudaMemset(admit_seq, 0, sizeof(uint64_t) * C));
  CUDA_CHECK(cudaMalloc(&mark, sizeof(int32_t) * C));
  CUDA_CHECK(cudaMalloc(&free_stack, sizeof(uint32_t) * C));
  CUDA_CHECK(cudaMalloc(&slot_host, sizeof(uint32_t) * C));
  CUDA_CHECK(cudaMemset(slot_host, 0xFF, sizeof(uint32_t) * C));
  CUDA_CHECK(cudaMalloc(&index, sizeof(uint32_t) * rows));
  init_lane_kernel<<<592, 256>>>(static_cast<uint32_t>(C), slot_feat, last_use, mark, free_stack);
  CUDA_LAUNCH_CHECK();
  fill_u32<<<1184, 256>>>(index, rows, kNever);
  CUDA_LAUNCH_CHECK();
  // host pool: a cache that holds the whole owned shard never evicts, so no row ever lives
  // on the host and nothing is pinned; otherwise `host_reserve` slots are pinned up front
  // and the pool grows on demand at eviction steps
  host.init(d, rows, C >= rows ? 0 : host_reserve);
  free_top = static_cast<int32_t>(C);
  next_seq = 0;
  // per-step scratch
  tiles.init(umax);
  for (int k = 0; k < 2; ++k) {
    CUDA_CHECK(cudaMalloc(&own_k_set[k], sizeof(uint32_t) * umax));
    CUDA_CHECK(cudaMalloc(&own_slot_set[k], sizeof(uint32_t) * umax));
  }
  use(0);
  CUDA_CHECK(cudaMalloc(&work_j, sizeof(uint32_t) * umax));
  CUDA_CHECK(cudaMalloc(&own_f, sizeof(uint32_t) * umax));
  CUDA_CHECK(cudaMalloc(&work_f, sizeof(uint32_t) * umax));
  CUDA_CHECK(cudaMalloc(&work_w, sizeof(uint32_t) * umax));
  sort_bytes = 0;
  {  // LRU candidate lists of n_evict + umax <= 2 umax (also the explicit eviction lists)
    cand_cap = 2 * umax;
    CUDA_CHECK(cudaMalloc(&keys, sizeof(uint64_t) * cand_cap));
    CUDA_CHECK(cudaMalloc(&keys_sorted, sizeof(uint64_t) * cand_cap));
    CUDA_CHECK(cudaMalloc(&ids, sizeof(uint32_t) * cand_cap));
    CUDA_CHECK(cudaMalloc(&ids_sorted, sizeof(uint32_t) * cand_cap));
    sort_bytes = sort_pairs_temp_bytes(cand_cap);
  }
  CUDA_CHECK(cudaMalloc(&temp, sort_bytes));
  CUDA_CHECK(cudaMalloc(&counters, sizeof(int32_t) * kCntWords));
  CUDA_CHECK(cudaMemset(counters, 0, sizeof(int32_t) * kCntWords));
  CUDA_CHECK(cudaMemcpy(counters + kCntFreeTop, &free_top, sizeof(int32_t), cudaMemcpyHostToDevice));
  CUDA_CHECK(cudaDeviceSynchronize());
}

void CacheLane::release() {
  for (void* p : {static_cast<void*>(emb),
                  static_cast<void*>(steps), static_cast<void*>(slot_feat),
                  static_cast<void*>(last_use), static_cast<void*>(admit_seq),
                  static_cast<void*>(mark), static_cast<void*>(free_stack),
                  static_cast<void*>(slot_host), static_cast<void*>(hist),
                  static_cast<void*>(index),
                  static_cast<void*>(own_k_set[0]), static_cast<void*>(own_slot_set[0]),
                  static_cast<void*>(own_k_set[1]), static_cast<void*>(own_slot_set[1]),
                  static_cast<void*>(work_j),
                  static_cast<void*>(own_f), static_cast<void*>(work_f), static_cast<void*>(work_w),
                  static_cast<void*>(keys), static_cast<void*>(keys_sorted),
                  static_cast<void*>(ids), static_cast<void*>(ids_sorted), temp,
                  static_cast<void*>(counters)})
    if (p) cudaFree(p);
  host.release();
  tiles.release();
  *this = CacheLane();
}

void CacheLane::select_owned(const uint32_t* d_gids, const int32_t* d_U, int32_t cap, uint32_t W,
                             uint32_t w, uint32_t* vsi_first, cudaStream_t s) {
  if (cap <= 0) return;
  if (W == 1) {  // a single worker owns every unique: own_k = identity, count = U
    launch_pdl(own_all_kernel, dim3(mgr_grid(std::min(ceil_div(cap, 256), num_sms() * 8))), dim3(256),
               0, s, d_U, own_k, counters + kCntOwned, d_gids, vsi_first);
    CUDA_LAUNCH_CHECK();
    return;
  }
  lookback_scan<2>(tiles, cap, OwnedFlag{d_gids, d_U, W, w, vsi_first}, OwnedEmit{own_k},
                   counters + kCntOwned, s, d_U);
}

void CacheLane::mark_window(const uint32_t* d_gids, const int32_t* d_U, int32_t cap, uint32_t W,
                            uint32_t w, int32_t t, cudaStream_t s) {
  if (cap <= 0) return;
  launch_pdl(mark_window_kernel, dim3(ceil_div(cap, 256)), dim3(256), 0, s, d_gids, d_U, cap, W, w, index,
                                                        static_cast<uint32_t>(C), t, mark,
                                                        counters + kCntMarked);
  CUDA_LAUNCH_CHECK();
}

void CacheLane::probe(const uint32_t* d_gids, int32_t cap, uint32_t W, int32_t t, cudaStream_t s) {
  if (cap <= 0) return;
  lookback_scan<1>(tiles, cap,
                ProbeFlag{own_k, counters + kCntOwned, d_gids, W, index, static_cast<uint32_t>(C), t,
                          last_use, mark, own_slot, counters + kCntMarked, own_f},
                ProbeEmit{own_f, own_slot, work_j, work_f, work_w}, counters + kCntWorking, s,
                counters + kCntOwned);
}

void CacheLane::victim_select(int32_t t, int32_t n_evict, cudaStream_t s, const uint8_t* pinned) {
  if (!hist) CUDA_CHECK(cudaMalloc(&hist, sizeof(uint32_t) * 2 * kHistBins));
  // level 1: last_use >> shift over [0, t] in at most kHistBins bins
  int shift = 0;
  while ((static_cast<int64_t>(t) >> shift) + 1 > kHistBins) ++shift;
  const int nb1 = static_cast<int>((static_cast<int64_t>(t) >> shift) + 1);
  CUDA_CHECK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2 * kHistBins, s));
  CUDA_CHECK(cudaMemsetAsync(counters + kCntOld, 0, sizeof(int32_t), s));
  const int grid = std::max(1, std::min<int>(ceil_div(static_cast<int64_t>(C), 16384), 2 * num_sms()));
  launch_pdl(lru_hist_kernel, dim3(grid), dim3(1024), 0, s, static_cast<uint32_t>(C), slot_feat, mark, t, last_use,
                                        hist, nb1, shift, counters, 0, false, pinned);
  CUDA_LAUNCH_CHECK();
  launch_pdl(lru_select_kernel, dim3(1), dim3(1024), 0, s, hist, nb1, n_evict, counters, shift, false);
  CUDA_LAUNCH_CHECK();
  if (shift > 0) {  // level 2: the 2^shift steps of the coarse bin, exactly
    launch_pdl(lru_hist_kernel, dim3(grid), dim3(1024), 0, s, static_cast<uint32_t>(C), slot_feat, mark, t, last_use,
                                          hist + kHistBins, 1 << shift, 0, counters, shift, true,
                                          pinned);
    CUDA_LAUNCH_CHECK();
    launch_pdl(lru_select_kernel, dim3(1), dim3(1024), 0, s, hist + kHistBins, 1 << shift, n_evict, counters, shift,
                                         true);
    CUDA_LAUNCH_CHECK();
  }
}

void CacheLane::victim_sort(int32_t t, int32_t n_evict, cudaStream_t s, const uint8_t* pinned) {
  const int64_t bound = std::min<int64_t>(cand_cap, static_cast<int64_t>(n_evict) + umax);
  CUDA_CHECK(cudaMemsetAsync(keys, 0xFF, sizeof(uint64_t) * bound, s));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(static_cast<int64_t>(C), 1024), num_sms() * 8));
  launch_pdl(lru_collect_kernel, dim3(grid), dim3(256), 0, s, static_cast<uint32_t>(C), slot_feat, mark, t, last_use,
                                          admit_seq, counters, bound, keys, ids, pinned);
  CUDA_LAUNCH_CHECK();
  sort_pairs_u64_u32(temp, sort_bytes, keys, keys_sorted, ids, ids_sorted, bound, 64, s);
}

void CacheLane::evict(int32_t n_evict, uint32_t W, int32_t t, cudaStream_t s, bool selected,
                      const uint8_t* pinned) {
  if (n_evict <= 0) return;
  if (!selected) victim_select(t, n_evict, s, pinned);
  victim_sort(t, n_evict, s, pinned);
  launch_pdl(evict_kernel, dim3(ceil_div(static_cast<int64_t>(n_evict) * 32, 256)), dim3(256), 0, s, n_evict, keys_sorted, ids_sorted, slot_feat, W, d, emb, mom, vel, steps, host.tab(),
      slot_host, counters + kCntHostNext, index, free_stack, counters + kCntFreeTop,
      counters + kCntError);
  CUDA_LAUNCH_CHECK();
}

bool CacheLane::swap_supported() const { return (d & 3) == 0 && 3 * (d / 4) <= 64; }

void CacheLane::evict_admit(int32_t n_evict, int32_t n_work, uint32_t W, uint64_t seed, int32_t t,
                            cudaStream_t s, bool selected, const PhaseHook& hook,
                            const uint8_t* pinned) {
  if (n_evict > 0) {  // every victim may need a new host slot (host.hi: exact as of the
    host.ensure(host.hi + static_cast<uint64_t>(n_evict), s);  // last host wait)
    host.hi += static_cast<uint64_t>(n_evict);
  }
  if (n_evict <= 0 || !swap_supported()) {
    evict(n_evict, W, t, s, selected, pinned);
    admit(n_work, n_evict, W, seed, t, s);
    return;
  }
  if (!selected) victim_select(t, n_evict, s, pinned);
  hook("evict_select");
  victim_sort(t, n_evict, s, pinned);
  hook("evict_sort");
  launch_pdl(swap_kernel, dim3(ceil_div(static_cast<int64_t>(n_work) * 32, 256)), dim3(256), 0, s, counters, n_evict, keys_sorted, ids_sorted, work_j, work_f, work_w, W, d / 4, free_stack,
      index, host.tab(), slot_host, counters + kCntHostNext, seed, fnv1a64("embed"),
      reinterpret_cast<float4*>(emb), reinterpret_cast<float4*>(mom),
      reinterpret_cast<float4*>(vel), steps, slot_feat, last_use, admit_seq, mark, t, own_slot,
      counters + kCntFromHost, counters + kCntError);
  CUDA_LAUNCH_CHECK();
  launch_pdl(advance_kernel, dim3(1), dim3(1), 0, s, counters, n_evict);
  CUDA_LAUNCH_CHECK();
}

void CacheLane::admit(int32_t n_bound, int32_t n_evict, uint32_t W, uint64_t seed, int32_t t,
                      cudaStream_t s) {
  if (n_bound > 0) {
    launch_pdl(admit_kernel, dim3(mgr_grid(ceil_div(ceil_div(static_cast<int64_t>(n_bound), kAdmitRows) * 32, 256))), dim3(256), 0, s, counters, n_evict, work_j, work_f, work_w, W, d, free_stack, index,
                        host.tab(), slot_host, seed, fnv1a64("embed"), emb, mom, vel, steps,
                        slot_feat, last_use, admit_seq, mark, t, own_slot,
                        counters + kCntFromHost);
    CUDA_LAUNCH_CHECK();
  }
  launch_pdl(advance_kernel, dim3(1), dim3(1), 0, s, counters, n_evict);
  CUDA_LAUNCH_CHECK();
}

// ---- explicit CacheBuffer operations (the standalone device CacheBuffer, cachebuf.cu) ----
namespace {
// err = min over offending positions of (i << 8 | code): 1 already resident, 2 not resident,
// 3 pinned, 4 inside the lookahead window (cache_buffer.cpp:39,57-61). mode 0: admit (must
// not be resident), 1: must be resident, 2: evict (resident, unpinned, not needed_soon)
__global__ void check_list_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                                  const uint32_t* __restrict__ index, uint32_t C,
                                  const uint8_t* __restrict__ pinned,
                                  const int32_t* __restrict__ mark, int32_t epoch, int mode,
                                  unsigned long long* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = index[static_cast<uint32_t>(feats[i]) / W];
  unsigned long long code = 0;
  if (mode == 0) {
    if (s < C) code = 1;
  } else if (s >= C) {
    code = 2;
  } else if (mode == 2) {
    if (pinned && pinned[s]) code = 3;
    else if (mark[s] == epoch) code = 4;
  }
  if (code) atomicMin(err, (static_cast<unsigned long long>(i) << 8) | code);
}
__global__ void admit_list_prep_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                                       const uint32_t* __restrict__ index,
                                       uint32_t* __restrict__ work_j, uint32_t* __restrict__ work_f,
                                       uint32_t* __restrict__ work_w, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) cnt[kCntWorking] = n;
  if (i >= n) return;
  const uint32_t f = static_cast<uint32_t>(feats[i]);
  work_j[i] = static_cast<uint32_t>(i);
  work_f[i] = f;
  work_w[i] = index[f / W];  // host slot / kNever (checked: not resident)
}
// the slots of `feats` in order as the "sorted" victims of evict_kernel
__global__ void evict_list_prep_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                                       const uint32_t* __restrict__ index,
                                       uint64_t* __restrict__ keys, uint32_t* __restrict__ ids,
                                       int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) cnt[kCntWorking] = 0;
  if (i >= n) return;
  keys[i] = 0;
  ids[i] = index[static_cast<uint32_t>(feats[i]) / W];
}
}  // namespace

void CacheLane::check_list(const uint64_t* d_feats, int32_t n, uint32_t W, const uint8_t* pinned,
                           int32_t epoch, int mode, unsigned long long* d_err, cudaStream_t s) {
  if (n <= 0) return;
  check_list_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_feats, n, W, index, static_cast<uint32_t>(C),
                                                     pinned, mark, epoch, mode, d_err);
  CUDA_LAUNCH_CHECK();
}

void CacheLane::admit_list(const uint64_t* d_feats, int32_t n, uint32_t W, uint64_t seed,
                           int32_t t, cudaStream_t s) {
  if (n <= 0) return;
  admit_list_prep_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_feats, n, W, index, work_j, work_f,
                                                          work_w, counters);
  CUDA_LAUNCH_CHECK();
  admit(n, 0, W, seed, t, s);
}

void CacheLane::evict_list(const uint64_t* d_feats, int32_t n, uint32_t W, cudaStream_t s) {
  if (n <= 0) return;
  host.ensure(host.hi + static_cast<uint64_t>(n), s);
  host.hi += static_cast<uint64_t>(n);
  evict_list_prep_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_feats, n, W, index, keys_sorted,
                                                          ids_sorted, counters);
  CUDA_LAUNCH_CHECK();
  launch_pdl(evict_kernel, dim3(ceil_div(static_cast<int64_t>(n) * 32, 256)), dim3(256), 0, s, n, keys_sorted, ids_sorted, slot_feat, W, d, emb, mom, vel, steps, host.tab(), slot_host,
      counters + kCntHostNext, index, free_stack, counters + kCntFreeTop, counters + kCntError);
  CUDA_LAUNCH_CHECK();
  launch_pdl(advance_kernel, dim3(1), dim3(1), 0, s, counters, n);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
