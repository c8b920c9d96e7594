// One worker lane's MixCache state in HBM + its partition of the pinned host
// table (see cache.cu for the policy and the reference lines it follows).
#pragma once

#include "ops.h"

namespace sfb {

// device counters per lane; kCntMarked = resident slots stamped needed_soon this step
// kCntFreeTop = free-stack height and kCntSeq (u64 over [6, 8)) = next admit_seq: both
// live on the device (admit / evict read and advance them), host copies are refreshed at
// every step that waits on the host
enum {
  kCntOwned = 0,
  kCntWorking = 1,
  kCntFromHost = 2,
  kCntError = 3,
  kCntMarked = 4,
  kCntFreeTop = 5,
  kCntSeq = 6,  // u64 over [6, 8)
  kCntOld = 8,  // pipelined manager: eligible victims older than the in-flight batch
  kCntWords = 16
};

struct CacheLane {
  uint64_t C = 0;       // slots (cache_capacity)
  int d = 0;
  uint64_t rows = 0;    // owned rows = ceil(vocab / W); row r holds feature r*W + w
  uint64_t host_cap = 0;
  int64_t umax = 0;     // max uniques per step (scratch sizing)

  // CacheBuffer slots (cache_buffer.hpp:42-50): the ParamEntry state of slot s is the
  // contiguous row [emb | m | v] at emb + 3d*s (mom = emb + d, vel = emb + 2d: same stride)
  float* emb = nullptr;        // [C x 3d] allocation
  float* mom = nullptr;        // = emb + d
  float* vel = nullptr;        // = emb + 2d
  int32_t* steps = nullptr;    // [C]  ParamEntry::adam_steps
  uint32_t* slot_feat = nullptr;  // [C] feature, kEmpty when free
  int32_t* last_use = nullptr;    // [C]
  uint64_t* admit_seq = nullptr;  // [C]
  int32_t* mark = nullptr;        // [C] step stamp: needed_soon <=> mark == t
  uint32_t* free_stack = nullptr; // [C] LIFO free list
  int32_t free_top = 0;           // host copy of counters[kCntFreeTop] (refreshed at host waits)
  uint64_t next_seq = 0;          // host copy of the device admit_seq counter
  uint32_t* index = nullptr;      // [rows] slot | kOnHost | kNever
  float* host_rows = nullptr;     // pinned mapped [host_cap * 3d]
  int32_t* host_steps = nullptr;  // pinned mapped [host_cap]

  // per-step scratch; own_k / own_slot are read by the training stage, so they come in
  // two sets (step parity) and the manager of step t+1 fills one while step t trains
  uint32_t *flag = nullptr, *rank = nullptr, *own_k = nullptr, *own_slot = nullptr;
  uint32_t *own_k_set[2] = {nullptr, nullptr}, *own_slot_set[2] = {nullptr, nullptr};
  uint32_t *miss = nullptr, *miss_rank = nullptr, *work_j = nullptr;
  // probe-time facts about the misses, so admit reads them coalesced instead of
  // chasing work_j -> own_k -> gids -> index: feature and index entry (kOnHost / kNever)
  uint32_t *own_f = nullptr, *work_f = nullptr, *work_w = nullptr;
  uint64_t *keys = nullptr, *keys_sorted = nullptr;
  uint32_t *ids = nullptr, *ids_sorted = nullptr;
  void* temp = nullptr;
  size_t scan_bytes = 0, sort_bytes = 0;
  int32_t* counters = nullptr;  // [kCntWords] device counters (kCnt*)

  void init(uint64_t capacity, int dim, uint64_t owned_rows, uint64_t host_rows_cap,
            int64_t max_unique);
  void release();
  void use(int set) {
    own_k = own_k_set[set];
    own_slot = own_slot_set[set];
  }

  // U / n_own are device counts; `cap` bounds the grids (the global batch size)
  // vsi_first (nullable): VSI first-position table to clear behind the batch
  void select_owned(const uint32_t* d_gids, const int32_t* d_U, int32_t cap, uint32_t W,
                    uint32_t w, uint32_t* vsi_first, cudaStream_t s);
  void mark_window(const uint32_t* d_gids, const int32_t* d_U, int32_t cap, uint32_t W, uint32_t w,
                   int32_t t, cudaStream_t s);
  void probe(const uint32_t* d_gids, int32_t cap, uint32_t W, int32_t t, cudaStream_t s);
  // LRU keys of every slot (eligible = occupied && !needed_soon); with count_old, also
  // counts the eligible slots whose last use precedes step t-1 into counters[kCntOld]
  void victim_keys(int32_t t, bool count_old, cudaStream_t s);
  // victims go on top of the device free stack; n_evict is host-known (sync steps only);
  // keys_ready: victim_keys already ran for this step
  void evict(int32_t n_evict, uint32_t W, int32_t t, cudaStream_t s, bool keys_ready = false);
  // admits counters[kCntWorking] rows (device count, <= n_bound) from the device free
  // stack, then advances the device free-stack height (+ n_evict - n_work) and admit_seq
  void admit(int32_t n_bound, int32_t n_evict, uint32_t W, uint64_t seed, int32_t t,
             cudaStream_t s);
  // eviction step (host-known n_evict / n_work): write-back and admission fused per slot
  // (swap_kernel) when the row fits the register staging, else evict() then admit()
  void evict_admit(int32_t n_evict, int32_t n_work, uint32_t W, uint64_t seed, int32_t t,
                   cudaStream_t s, bool keys_ready);
  bool swap_supported() const;
};

}  // namespace sfb
