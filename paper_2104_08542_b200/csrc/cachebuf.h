// The standalone device CacheBuffer + HostStore + MixCache manager of ONE worker
// (sfctr_cache_* in include/sfctr_b200.h): the reference's CacheBuffer operation surface
// (cache_buffer.hpp:52-78) and the manager step over the same device
// MixCache the trainer uses (CacheLane, cache.h).
#pragma once

#include <string>

#include "cache.h"

namespace sfb {

class DeviceCache {
 public:
  // capacity slots of [emb | m | v] rows of `dim`; the worker owns features f with
  // f % num_workers == worker, f < key_space (the vocabulary); max_batch bounds the ids of
  // one prepare() / one explicit batch call; host_reserve pins host-pool rows up front
  DeviceCache(uint64_t capacity, int dim, uint64_t seed, uint64_t key_space, int num_workers,
              int worker, int64_t max_batch, uint64_t host_reserve, int device);
  ~DeviceCache();

  // CacheBuffer::admit(f, host.take(f), step) for each feature in order (cache_buffer.cpp:38-53):
  // LogicError when one is resident or no free slot is left; slots_out (nullable) = SlotIds
  void admit(int64_t n, const uint64_t* features, int64_t step, uint64_t* slots_out);
  // host.put(f, CacheBuffer::evict(f)) in order (cache_buffer.cpp:55-67): LogicError for a
  // non-resident, pinned or needed_soon feature (nothing moves then)
  void evict(int64_t n, const uint64_t* features);
  void touch(int64_t n, const uint64_t* features, int64_t step);     // cache_buffer.cpp:69-72
  void pin(int64_t n, const uint64_t* features, bool on);             // pin / unpin
  void set_needed_soon(int64_t n, const uint64_t* features, bool on);
  // SlotId per feature, -1 when not resident (CacheBuffer::slot_of throws there; the
  // C++ facade does)
  void slot_of(int64_t n, const uint64_t* features, int64_t* out);
  uint64_t free_count();
  // CacheBuffer::slots(): feature (UINT64_MAX = free), last_use, admit_seq, pinned, needed_soon
  void slots(uint64_t* feature, int64_t* last_use, uint64_t* admit_seq, uint8_t* pinned,
             uint8_t* needed_soon);
  // capacity, occupied, free, pinned, needed_soon (occupancy_diagnostics, cache_buffer.cpp:81-92)
  void occupancy(uint64_t out[5]);
  std::string occupancy_diagnostics();
  // HostStore::peek / CacheBuffer::slot(s).entry: [emb | m | v] rows + adam_steps of
  // touched features, wherever they live (LogicError for a never-touched one)
  void peek(int64_t n, const uint64_t* features, float* rows, int64_t* steps);
  // One manager step (manager_get + pull_parameters_to_host + push_parameters_to_cache,
  // SPEC.md:189-217) for this worker: global_ids = the step's unique features (DedupBatch
  // order), window_ids = every feature of the lookahead batches t..t+L-1 (duplicates
  // allowed; empty = batch t only). needed_soon is recomputed (window), hits are touched,
  // misses admitted in global_ids order after evicting the LRU (last_use, admit_seq)
  // eligible slots (!pinned, !needed_soon). RunError (with the occupancy diagnostics) when
  // the working set cannot fit. out: owned, hits, admitted, evicted, refilled from host.
  void prepare(int64_t step, int64_t n_global, const uint64_t* global_ids, int64_t n_window,
               const uint64_t* window_ids, int64_t out[5]);

 private:
  void to_device(int64_t n, const uint64_t* features, bool owned_check);
  void check_err(const char* op);
  void refresh_counters();
  void restamp(int64_t n, bool admitted_only);

  CacheLane L_;
  int W_, w_, d_, dev_;
  uint64_t seed_, key_space_;
  int64_t max_batch_;
  cudaStream_t s_ = nullptr;
  int32_t epoch_ = -2;  // needed_soon <=> mark[s] == epoch_ (the last prepare's step)
  int64_t max_step_ = 0;
  uint8_t* pinned_ = nullptr;      // [C]
  uint64_t* d_feats_ = nullptr;    // [max_batch] staging
  uint32_t* d_ids32_ = nullptr;    // [max_batch]
  uint32_t* d_win32_ = nullptr;    // [max_batch]
  int32_t* d_scal_ = nullptr;      // [0] U, [1] bad, [2] window count
  unsigned long long* d_err_ = nullptr;
  int64_t* d_occ_ = nullptr;       // [4] occupancy reduction
  int32_t* h_cnt_ = nullptr;       // pinned copy of the lane counters
};

}  // namespace sfb
