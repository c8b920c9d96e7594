// Host-side launchers of the sm_100a kernels (one .cu per subsystem).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace sfb {

// per-phase timing callback (Trainer::phase): records a named CUDA event on the stream
struct PhaseHook {
  void (*fn)(void* ctx, const char* name) = nullptr;
  void* ctx = nullptr;
  void operator()(const char* name) const {
    if (fn) fn(ctx, name);
  }
};

// ---------------- generator.cu — SyntheticGenerator (generator.cpp:32-115) ----------------
struct GenTables {
  int fields = 0;
  uint64_t vocab = 0, seed = 0, base = 0;
  double zipf = 0, truth_scale = 0;
  uint64_t* d_shard_starts = nullptr;  // [F+1]
  double* d_cdf_base = nullptr;        // [base]
  double* d_cdf_big = nullptr;         // [base+1] or null
  double* d_tw = nullptr;              // scratch truth weights [max_ids]
  int64_t tw_cap = 0;
  std::vector<uint64_t> shard_starts;  // host copy
  void build(int fields, uint64_t vocab, uint64_t seed, double zipf);  // host CDFs (std::pow)
  void release();
};
void generate_rows(GenTables& g, int64_t step, int32_t row0, int32_t nrows, uint64_t* d_features,
                   uint8_t* d_labels, cudaStream_t s);
void initial_embedding_device(uint64_t seed, uint64_t feature, int dim, double* d_out,
                              cudaStream_t s);

// ---------------- vsi.cu — virtual_sparse_id (vsi.cpp:23-54) ----------------
struct VsiScratch {
  uint64_t key_space = 0;          // 0: hashed table for arbitrary u64 ids
  int64_t cap = 0;                 // max ids per call
  // direct-mapped: [key_space] first position per feature (0xFFFFFFFF = unseen), re-tagged
  // with the unique's rank during the scan; hashed: the per-slot equivalent [hmask + 2]
  uint32_t* d_first = nullptr;
  unsigned long long* d_hkeys = nullptr;  // hashed: keys [hmask + 2] (last = the ~0 id)
  uint32_t* d_hkeys32 = nullptr;          // hashed32: u32 keys [hmask + 2]
  bool hashed32 = false;  // u32 ids through an L2-resident hashed table (no vocab-sized table)
  uint64_t hmask = 0;
  uint32_t* d_hslot = nullptr;     // hashed: table slot per position [cap]
  uint32_t* d_uslot = nullptr;     // hashed: table slot per unique [cap]
  ScanTiles tiles;                 // fused look-back scan state
  // hash32: u32 ids below key_space through the hashed table (always reset behind a batch)
  void init(uint64_t key_space, int64_t cap, bool hash32 = false);
  void release();
};
// arbitrary u64 ids [n] -> global_ids u64 [U], vids u32 [n], *d_unique (key_space 0 context)
void vsi_device_hashed(VsiScratch& v, const uint64_t* d_ids, int64_t n, uint64_t* d_gids,
                       uint32_t* d_vids, int32_t* d_unique, cudaStream_t s);
// ids u32 [n] -> global_ids u32 [U] (first-appearance order), vids u32 [n], *d_unique.
// reset = false leaves the first-position table dirty: the caller clears it (the
// trainer folds that into its owned-set kernel)
void vsi_device(VsiScratch& v, const uint32_t* d_ids, int64_t n, uint32_t* d_gids,
                uint32_t* d_vids, int32_t* d_unique, cudaStream_t s, bool reset = true);
// u64 -> u32 with range check; *d_bad set to 1 when any id >= limit
void ids_to_u32(const uint64_t* d_in, uint32_t* d_out, int64_t n, uint64_t limit, int32_t* d_bad,
                cudaStream_t s);
void u32_to_u64(const uint32_t* d_in, uint64_t* d_out, int64_t n, cudaStream_t s);

// ---------------- victim sort (CUB radix sort of the few LRU candidates) ----------------
size_t sort_pairs_temp_bytes(int64_t n);
void sort_pairs_u64_u32(void* temp, size_t temp_bytes, const uint64_t* keys_in, uint64_t* keys_out,
                        const uint32_t* vals_in, uint32_t* vals_out, int64_t n, int end_bit,
                        cudaStream_t s);

}  // namespace sfb
