// Owner-routed all-to-all exchange of embedding rows / gradients (exchange.cu).
#pragma once

#include <nccl.h>

#include <string>
#include <vector>

#include "kernels.h"

namespace sfb {

#ifndef NCCL_CHECK
#define NCCL_CHECK(expr)                                                                  \
  do {                                                                                    \
    ncclResult_t r_ = (expr);                                                             \
    if (r_ != ncclSuccess)                                                                \
      ::sfb::fail(::sfb::kNccl, std::string(#expr) + ": " + ncclGetErrorString(r_));      \
  } while (0)
#endif

struct Cnt8 {  // per-worker counters (at most 8 workers on one NVSwitch box)
  uint32_t c[8];
};

struct Exchange {
  int W = 0, me = 0, d = 0;
  int64_t cap = 0;               // bound on uniques per step
  uint32_t* tm = nullptr;        // [cap] touched-by-worker bitmask per unique
  uint8_t* tb8 = nullptr;        // [cap x 8] touched bytes (planning scratch, kept zero)
  uint32_t* lpos = nullptr;      // [cap] row in the local table E (or ~0)
  Cnt8* sscan = nullptr;         // [cap] send slot of owned row j for each destination
  uint32_t* tile_cnt = nullptr;  // [tiles x 8] per-tile plane counts (planning scratch)
  uint32_t* tile_off = nullptr;  // [tiles x 8] exclusive tile offsets
  // [80]: recv rows per owner (8) | send rows per destination (8) | cnt[w][o] (64)
  int32_t* totals = nullptr;
  float* buf = nullptr;          // [cap x d] forward send / backward receive rows
  float* gown = nullptr;         // [cap x d] owner-summed gradients, owned order
  std::vector<int64_t> recv_rows, send_rows, recv_off, send_off;  // host copies
  // NVLink peer-store transport (all peers reachable): every rank's E and buf
  bool p2p = false;
  bool copy_engine = false;  // p2p rows move by SM peer stores (default) or DMA (pack + memcpy)
  float* peer_E[8] = {};
  float* peer_buf[8] = {};
  float* bar = nullptr;                    // 1-float all-reduce barrier (NCCL fallback)
  uint64_t* flags = nullptr;               // [8] NVLink flag barrier: slot w = rank w's epoch
  uint64_t* peer_flags[8] = {};
  uint64_t epoch = 0;
  int32_t* abort_flag = nullptr;           // device word raised by a timed-out barrier
  bool nccl_barrier = false;               // SFCTR_NCCL_BARRIER=1: all-reduce barrier instead
  std::vector<int64_t> roff_all, boff_all;  // [w*8+o]: rank w's E block of owner o;
                                            // [o*8+w]: owner o's buf block of source w
  static constexpr int kTotals = 80;
  // device copy of the layout set_counts derives on the host, written by plan():
  // [0, 64) roff_all, [64, 128) boff_all, [128, 137) recv_off, [137, 146) send_off
  int32_t* offs = nullptr;
  static constexpr int kOffRoff = 0, kOffBoff = 64, kOffRecv = 128, kOffSend = 137;
  // The plan (tm .. offs) is written by the manager stage and read by the training stage:
  // two sets (step parity), so the plan of step t+1 is built while step t trains.
  struct PlanSet {
    uint32_t *tm = nullptr, *lpos = nullptr, *tile_cnt = nullptr, *tile_off = nullptr;
    Cnt8* sscan = nullptr;
    int32_t *totals = nullptr, *offs = nullptr;
  };
  PlanSet sets[2];
  void use(int set) {
    tm = sets[set].tm;
    lpos = sets[set].lpos;
    sscan = sets[set].sscan;
    tile_cnt = sets[set].tile_cnt;
    tile_off = sets[set].tile_off;
    totals = sets[set].totals;
    offs = sets[set].offs;
  }

  void init(int W, int me, int64_t cap, int d);
  void release();
  // maps every peer's E / buf (CUDA IPC, handles all-gathered over NCCL) when
  // all pairs have peer access; otherwise the exchange uses NCCL send/recv
  void setup_p2p(float* E, ncclComm_t comm, cudaStream_t s);
  void barrier(ncclComm_t comm, cudaStream_t s);
  // device-only planning (no host wait); totals land in `totals`
  void plan(const uint32_t* d_vid, int64_t n_global, int64_t per_worker, const uint32_t* d_uniq,
            const int32_t* d_U, const uint32_t* d_own_k, const int32_t* d_n_own, cudaStream_t s,
            const PhaseHook& hook = PhaseHook{});
  // the send plan when the producer of the owned uniques already counted them per
  // (1024-row tile, destination) into tile_cnt (zeroed before) and own_k is the identity:
  // one kernel (shardplan.cu); writes sscan and totals[8..16)
  void send_plan_counted(const int32_t* d_n_own, cudaStream_t s);
  int tile_words() const { return 8 * ((static_cast<int>(cap) + 1023) / 1024); }
  // the layout offsets (offs) from totals
  void plan_offsets(cudaStream_t s);
  void set_counts(const int32_t* h_totals);  // after the step's host wait
  // d_lvid[i] = table[d_vid_mine[i]], table = lpos by default
  void local_vids(const uint32_t* d_vid_mine, int64_t n, uint32_t* d_lvid, cudaStream_t s,
                  const uint32_t* table = nullptr);
  int64_t local_rows() const { return recv_off.empty() ? 0 : recv_off[8]; }
  // returns the bytes this rank sent
  // with the peer-store transport the caller may defer the barrier (do_barrier = false)
  int64_t forward(const uint32_t* d_own_k, const uint32_t* d_own_slot, int32_t n_own,
                  const float* emb, float* E, ncclComm_t comm, cudaStream_t s,
                  bool do_barrier = true);
  // Peer-store transport driven by device counts only (no host copy of the plan):
  // n_bound bounds the grids, d_n_own is the owned count; nothing returns bytes
  void forward_dev(const uint32_t* d_own_k, const uint32_t* d_own_slot, int32_t n_bound,
                   const int32_t* d_n_own, const float* emb, cudaStream_t s);
  // B != nullptr: the segment sum deferred the FM term -fm_scale * B[r] * E[r] of local row
  // r; both the push to the owners and the owner's reduction add it
  void backward_send_dev(const float* dE, cudaStream_t s, const float* E = nullptr,
                         const float* B = nullptr, float fm_scale = 0.f);
  // the owner's reduction fused with the lazy Adam update of its rows (no gown round trip)
  struct AdamRows {
    float *emb, *mom, *vel;
    const uint32_t* own_slot;
    const int32_t* steps;
    const float *bc1, *bc2;
    float lr, b1, b2, omb1, omb2, eps;
  };
  // B != nullptr: add the deferred FM term of the owner's own rows, taken from the cache
  // row itself (E is not read: peers may already be filling it for the next step)
  void backward_reduce_adam_dev(const uint32_t* d_own_k, int32_t n_bound, const int32_t* d_n_own,
                                const float* dE, cudaStream_t s, const float* B, float fm_scale,
                                const AdamRows& ar);
  // dE[0 : local rows) = 0 (and B[0 : local rows) when given), row count read on the device
  void zero_local_dev(float* dE, cudaStream_t s, float* B = nullptr);
  bool device_driven() const { return p2p && !copy_engine; }
  int64_t backward(const uint32_t* d_own_k, int32_t n_own, const float* dE, ncclComm_t comm,
                   cudaStream_t s);
  // the same in parts: send my partial gradients (no barrier), then the owner-side sum
  int64_t backward_send(const float* dE, ncclComm_t comm, cudaStream_t s);
  void backward_reduce(const uint32_t* d_own_k, int32_t n_own, const float* dE, cudaStream_t s);
};

}  // namespace sfb
