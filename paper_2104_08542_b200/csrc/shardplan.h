// Owner-sharded manager stage for the owner-routed exchange over NVLink peer stores
// (shardplan.cu). Instead of every rank all-gathering the W·b·F global batch and running the
// same VSI + exchange plan over all of it, each rank routes its own ids to their owners
// (f mod W); an owner deduplicates what it received, orders its uniques by
// first global position (= the global_ids order of vsi.cpp:41-46 filtered by owner), plans
// which rank needs which of its rows, and writes every rank's positions' local-table rows
// back to them. Per-rank work is O(b·F) plus one flag scan over the global positions,
// instead of O(W·b·F) random-access passes.
#pragma once

#include <nccl.h>

#include "exchange.h"
#include "scan.cuh"

namespace sfb {

struct ShardPlan {
  int W = 0, me = 0;
  int64_t n = 0;    // ids per rank and step
  int64_t cap = 0;  // bound on owned uniques per step
  bool ready = false;
  // two sets by step parity k (set k at offset k * size); pairs / inbox / reply peer-mapped
  uint64_t* pairs = nullptr;    // [2][W * n] received (feature << 32 | global position) pairs,
                                // region r = source r
  int32_t* inbox = nullptr;     // [2][kInbox]: cnt[w][o] at w*8+o (column o written by owner
                                // o), owners' unique counts at 64 + o, pair counts from
                                // source r at 72 + r
  uint32_t* reply = nullptr;    // [2][W * n]: owner o's replies at [o * n, ...): the
                                // local-table row of each pair this rank routed to o
  uint32_t* rix = nullptr;      // [2][n]: reply index of each of my positions
  uint64_t* flags = nullptr;    // [8] barrier words
  uint64_t* peer_pairs[8] = {};
  int32_t* peer_inbox[8] = {};
  uint32_t* peer_reply[8] = {};
  uint64_t* peer_flags[8] = {};
  uint64_t epoch = 0;
  int32_t* abort_flag = nullptr;
  // local scratch
  int32_t* cursor = nullptr;          // [8] pairs routed per owner this step
  uint32_t* hkeys = nullptr;          // hashed features [hmask + 1]
  uint32_t* hpos = nullptr;           // first global position, then the owned index | tag
  uint32_t* hmask_bits = nullptr;     // touched-by-rank mask per slot
  uint64_t hmask = 0;
  uint32_t* hslot = nullptr;          // [W * n] slot per received pair
  uint32_t* bits = nullptr;           // [nwords] first-position bitmap (kept zero)
  uint32_t* wpre = nullptr;           // [nwords] set bits before each word
  int64_t nwords = 0;
  uint32_t* uslot = nullptr;          // [cap] slot per owned unique
  ScanTiles tiles;
  static constexpr int kInbox = 80;

  // position i's local-table row of step parity k is rows(k)[index(k)[i]] (the training
  // stage's remap: vid = index(k), remap = rows(k))
  const uint32_t* index(int k) const { return rix + k * n; }
  const uint32_t* rows(int k) const { return reply + k * static_cast<int64_t>(W) * n; }

  void init(int W, int me, int64_t n, int64_t cap);
  void release();
  // CUDA IPC mappings of every rank's buffers (handles all-gathered over NCCL); false when
  // not every pair of ranks has peer access (the replicated manager stays in use)
  bool setup_p2p(ncclComm_t comm, cudaStream_t s);
  // The manager stage's ids + VSI + exchange plan for step parity k: d_ids (this rank's u64
  // features) -> owned_uniq [n_own] in first-appearance order, *d_n_own, *d_U_global, and
  // the exchange plan in xch (tm / sscan / lpos by owned index, totals, offs), index(k);
  // rows(k) is complete once the training stage has passed its forward exchange barrier
  // (every owner stores its replies before its own training stage starts). Ids >= vocab
  // set *d_bad on every rank.
  // own_k receives the identity (owned index j is its own key) for the per-owned-row kernels
  void run(const uint64_t* d_ids, uint64_t vocab, int32_t* d_bad, int k, Exchange& xch,
           uint32_t* owned_uniq, uint32_t* own_k, int32_t* d_n_own, int32_t* d_U_global,
           cudaStream_t s, const PhaseHook& hook = PhaseHook{});
};

}  // namespace sfb
