// Global-batch id all-gather over NVLink peer stores (idgather.cu).
#pragma once

#include <nccl.h>

#include <vector>

#include "exchange.h"  // NCCL_CHECK

namespace sfb {

struct IdGather {
  int W = 0, me = 0;
  int64_t n = 0;                       // ids per rank and step
  bool p2p = false;
  uint32_t* gids[2] = {nullptr, nullptr};  // my global-batch buffers [W * n], by step parity
  uint32_t* peer_gids[2][8] = {};
  uint64_t* flags = nullptr;           // flag-barrier words, slot w = rank w's epoch
  uint64_t* peer_flags[8] = {};
  uint64_t epoch = 0;
  int32_t* abort_flag = nullptr;       // device word raised by a timed-out barrier (trainer's)

  void init(int W, int me, int64_t n);
  void release();
  // maps every rank's buffers (CUDA IPC, handles all-gathered over NCCL) when all pairs
  // have peer access; false (NCCL all-gather stays in use) otherwise
  bool setup_p2p(ncclComm_t comm, cudaStream_t s);
  // this rank's u64 ids -> u32 (ids >= limit set *d_bad) into every rank's buffer of
  // parity k, then a flag barrier; returns the global batch (gids[k]) for stream s
  const uint32_t* gather(const uint64_t* d_ids, uint64_t limit, int32_t* d_bad, int k,
                         cudaStream_t s);
};

}  // namespace sfb
