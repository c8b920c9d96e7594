// One worker lane's MixCache state in HBM + its partition of the pinned host
// table (see cache.cu for the policy and the reference lines it follows).
#pragma once

#include <mutex>
#include <thread>
#include <utility>
#include <vector>

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
  kCntHostNext = 9,  // host slots handed out by the host pool (first evictions)
  kCntSelT = 10,     // LRU select: threshold step T (victims have last_use <= T)
  kCntSelN = 11,     // LRU select: candidates collected (last_use <= T)
  kCntSelB = 12,     // LRU select: coarse (level-1) bin of the threshold
  kCntSelBelow = 13, // LRU select: eligible slots below the coarse bin
  kCntSelTotal = 14, // LRU select: eligible slots in total
  kCntWords = 16
};

// Device view of the host pool: host slot h lives in slab h >> shift at row h & mask.
struct HostTab {
  float* const* rows;     // [HostPool::kMaxSlabs] slab tables, [slab_rows x 3d] fp32 each
  int32_t* const* steps;  // [HostPool::kMaxSlabs] slab adam_steps, [slab_rows] each
  int shift;
  uint32_t mask;
#ifdef __CUDACC__
  __device__ __forceinline__ float* row(uint32_t h, int d3) const {
    return rows[h >> shift] + static_cast<size_t>(h & mask) * d3;
  }
  __device__ __forceinline__ int32_t* step(uint32_t h) const { return steps[h >> shift] + (h & mask); }
#endif
};

// The HostStore (host_store.hpp:61-92, host_store.cpp:25-56) of one worker lane: a lazily
// grown pool of pinned, mapped host slabs (never a dense [vocab/W x 3d] table). Rows that
// were never evicted have no host state at all: HostStore::get_or_init's lazy
// initialisation happens on the device when the row is admitted. A row gets a host slot
// the first time it is evicted (pull_parameters_to_host) and keeps it: refills read it,
// later write-backs of the same feature reuse it. Only evicted rows cost host memory.
struct HostPool {
  HostPool() = default;
  HostPool(HostPool&& o) noexcept { *this = std::move(o); }
  HostPool& operator=(HostPool&& o) noexcept {  // moved only while idle (no filler running)
    d = o.d; shift = o.shift; dev = o.dev; cap = o.cap; hi = o.hi;
    rows_h = std::move(o.rows_h); steps_h = std::move(o.steps_h);
    d_rows = o.d_rows; d_steps = o.d_steps; h_rows_tab = o.h_rows_tab; h_steps_tab = o.h_steps_tab;
    spares = std::move(o.spares); filler_failed = o.filler_failed;
    o.d_rows = nullptr; o.d_steps = nullptr; o.h_rows_tab = nullptr; o.h_steps_tab = nullptr;
    return *this;
  }
  static constexpr int kMaxSlabs = 4096;
  int d = 0, shift = 0, dev = 0;
  uint64_t cap = 0;  // host slots allocated (slabs x slab_rows)
  uint64_t hi = 0;   // upper bound of the slots handed out (the device counter kCntHostNext)
  std::vector<float*> rows_h;
  std::vector<int32_t*> steps_h;
  float** d_rows = nullptr;  // device pointer tables [kMaxSlabs]
  int32_t** d_steps = nullptr;
  float** h_rows_tab = nullptr;  // pinned mirrors: append-only sources of the async uploads
  int32_t** h_steps_tab = nullptr;
  // Pinning a 256 MB slab takes ~100 ms (page pinning runs at a few GB/s): while the pool
  // is within kAhead slabs of its high-water mark, a background thread pins spare slabs
  // ahead so the step that needs one takes it ready instead of stalling the manager stage.
  // (At eviction rates above the pinning rate only the up-front reservation helps.)
  static constexpr int kAhead = 4;
  std::thread filler;
  std::mutex mu;
  std::vector<std::pair<float*, int32_t*>> spares;  // guarded by mu
  bool filler_failed = false;                        // guarded by mu
  std::pair<float*, int32_t*> alloc_slab();  // (rows, steps) pinned + mapped, or nulls
  void prefetch();
  // slab_rows = 2^shift: about 256 MB per slab, smaller for small tables
  void init(int dim, uint64_t owned_rows, uint64_t reserve_rows);
  // grows the pool to at least `slots` host slots; new slab pointers are uploaded on s
  void ensure(uint64_t slots, cudaStream_t s);
  void release();
  HostTab tab() const { return HostTab{d_rows, d_steps, shift, (1u << shift) - 1u}; }
  const float* row_host(uint32_t h) const {
    return rows_h[h >> shift] + static_cast<size_t>(h & ((1u << shift) - 1u)) * 3 * d;
  }
  int32_t step_host(uint32_t h) const { return steps_h[h >> shift][h & ((1u << shift) - 1u)]; }
};

struct CacheLane {
  uint64_t C = 0;       // slots (cache_capacity)
  int d = 0;
  uint64_t rows = 0;    // owned rows = ceil(vocab / W); row r holds feature r*W + w
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
  uint32_t* index = nullptr;      // [rows] slot | kHostBit | host slot | kNever
  uint32_t* slot_host = nullptr;  // [C] host slot of the slot's row (kNoHost: none yet)
  HostPool host;                  // evicted rows (pinned, mapped host slabs)
  uint32_t* hist = nullptr;       // LRU histograms (two levels of kHistBins)

  // per-step scratch; own_k / own_slot are read by the training stage, so they come in
  // two sets (step parity) and the manager of step t+1 fills one while step t trains
  uint32_t *own_k = nullptr, *own_slot = nullptr;
  uint32_t *own_k_set[2] = {nullptr, nullptr}, *own_slot_set[2] = {nullptr, nullptr};
  uint32_t* work_j = nullptr;
  // probe-time facts about the misses, so admit reads them coalesced instead of
  // chasing work_j -> own_k -> gids -> index: feature and index entry (host slot / kNever)
  uint32_t *own_f = nullptr, *work_f = nullptr, *work_w = nullptr;
  // LRU victim candidates (last_use <= the select threshold) and their sorted order:
  // at most n_evict + umax entries (cand_cap = 2 umax), never O(C)
  uint64_t *keys = nullptr, *keys_sorted = nullptr;
  uint32_t *ids = nullptr, *ids_sorted = nullptr;
  int64_t cand_cap = 0;
  void* temp = nullptr;     // victim sort scratch
  size_t sort_bytes = 0;
  ScanTiles tiles;           // fused look-back scans (owned selection, probe)
  int32_t* counters = nullptr;  // [kCntWords] device counters (kCnt*)

  // host_reserve: host-pool slots pinned up front (the pool grows on demand beyond it)
  void init(uint64_t capacity, int dim, uint64_t owned_rows, uint64_t host_reserve,
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
  // Exact LRU selection without sorting the C slots: a histogram of the eligible slots
  // (occupied && !needed_soon) over last_use, then the threshold step T with
  // #(last_use < T) < n_evict <= #(last_use <= T) (counters[kCntSelT]), and the count of
  // eligible slots last used before step t-1 (counters[kCntOld], pipelined eviction safety)
  // pinned (nullable): per-slot pin flags of a standalone CacheBuffer (cachebuf.cu); the
  // trainer's pins are implied by stream order
  void victim_select(int32_t t, int32_t n_evict, cudaStream_t s, const uint8_t* pinned = nullptr);
  // collects the candidates (last_use <= T) and sorts them by (last_use, admit_seq): the
  // first n_evict are the victims, oldest first
  void victim_sort(int32_t t, int32_t n_evict, cudaStream_t s, const uint8_t* pinned = nullptr);
  // victims go on top of the device free stack; n_evict is host-known (sync steps only);
  // selected: victim_select already ran for this step
  void evict(int32_t n_evict, uint32_t W, int32_t t, cudaStream_t s, bool selected = false,
             const uint8_t* pinned = nullptr);
  // admits counters[kCntWorking] rows (device count, <= n_bound) from the device free
  // stack, then advances the device free-stack height (+ n_evict - n_work) and admit_seq
  void admit(int32_t n_bound, int32_t n_evict, uint32_t W, uint64_t seed, int32_t t,
             cudaStream_t s);
  // eviction step (host-known n_evict / n_work): write-back and admission fused per slot
  // (swap_kernel) when the row fits the register staging, else evict() then admit()
  void evict_admit(int32_t n_evict, int32_t n_work, uint32_t W, uint64_t seed, int32_t t,
                   cudaStream_t s, bool selected, const PhaseHook& hook = {},
                   const uint8_t* pinned = nullptr);
  bool swap_supported() const;
  // Explicit CacheBuffer operations on a device list of n <= umax owned features (the
  // standalone DeviceCache, cachebuf.cu). check_list: *d_err = min (i << 8 | code) over the
  // offending positions (1 already resident, 2 not resident, 3 pinned, 4 needed_soon, i.e.
  // mark == epoch); mode 0 admit, 1 resident, 2 evict. admit_list / evict_list expect a
  // checked list: admissions pop the LIFO free list in list order, evictions push their
  // slots in list order (cache_buffer.cpp:41-42,64).
  void check_list(const uint64_t* d_feats, int32_t n, uint32_t W, const uint8_t* pinned,
                  int32_t epoch, int mode, unsigned long long* d_err, cudaStream_t s);
  void admit_list(const uint64_t* d_feats, int32_t n, uint32_t W, uint64_t seed, int32_t t,
                  cudaStream_t s);
  void evict_list(const uint64_t* d_feats, int32_t n, uint32_t W, cudaStream_t s);
};

}  // namespace sfb
