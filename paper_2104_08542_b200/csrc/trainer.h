// The per-process training engine behind sfctr_trainer_* (include/sfctr_b200.h).
#pragma once

#include <nccl.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/sfctr_b200.h"
#include "cache.h"
#include "exchange.h"
#include "idgather.h"
#include "shardplan.h"
#include "kernels.h"

namespace sfb {

void validate_config(const sfctr_config& c);

class Trainer {
 public:
  Trainer(const sfctr_config& cfg, int rank, int world, const uint8_t* nccl_id, int device);
  ~Trainer();

  // one BSP step over this process's rows; inputs on the device
  void step_device(int64_t step, const uint64_t* d_features, const uint8_t* d_labels,
                   const uint64_t* d_window, float* d_loss);
  // the same in its two stages (prepare = Host-Manager, train = GPU-Worker); prepare(t)
  // must be followed by train(t) before prepare(t + 1)
  void prepare(int64_t step, const uint64_t* d_features, const uint64_t* d_window);
  void train(int64_t step, const uint8_t* d_labels, float* d_loss);
  // host-buffer variant: H2D copies, step, loss read back
  double step_host(int64_t step, const uint64_t* features, const uint8_t* labels,
                   const uint64_t* window);
  // the same split in two: submit_host enqueues the H2D copies, the step and the D2H copy
  // of its loss and returns; loss_of(step) waits for that loss. At most four submitted
  // steps are outstanding (the loss of step t must be read before step t+4 is submitted).
  void submit_host(int64_t step, const uint64_t* features, const uint8_t* labels,
                   const uint64_t* window);
  double loss_of(int64_t step);
  bool pipelined() const { return pipelined_; }
  void synchronize();
  int64_t free_steps() const { return free_steps_; }

  cudaStream_t stream() const { return stream_; }
  int lanes() const { return lanes_; }
  int rows() const { return lanes_ * cfg_.batch_size_per_worker; }

  void logits(float* out);
  // slots [first, first + count) of a lane (clamped to the capacity)
  void cache_slots(int lane, uint64_t* feature, int64_t* last_use, uint64_t* admit_seq,
                   uint64_t first = 0, uint64_t count = ~0ull);
  // HostStore::peek over this process's features: [emb | m | v] + adam step per feature
  void peek_rows(int64_t n, const uint64_t* features, float* rows, int64_t* steps);
  // dense parameters and their Adam moments [P] = W1 | b1 | w2 | b2, and the dense step
  void dense_state(float* p, float* m, float* v, int64_t* step);
  uint64_t free_count(int lane);
  int64_t snapshot(uint64_t* features, float* rows, int64_t* steps);
  void get_dense(float* w1, float* b1, float* w2, float* b2);
  void set_dense(const float* w1, const float* b1, const float* w2, const float* b2);
  void ledger(int64_t out[4]);
  sfctr_step_stats stats();
  // enabling (re)starts the per-phase accumulation; phase_times() returns the
  // per-phase device-time sums over the steps run since
  void set_timing(bool on) {
    timing_ = on;
    if (on) phase_ms_.clear();
  }
  const std::vector<std::pair<std::string, float>>& phase_times() {
    finish_phases();
    return phase_ms_;
  }

 private:
  void ensure_bias_tables(int64_t t_max);
  // rows of one lane by owned-row index (see peek_rows)
  void read_rows(int lane, const uint64_t* rows_idx, int64_t n, float* rows, int64_t* steps,
                 bool* never);
  void phase(const char* name, cudaStream_t s = nullptr);
  void sync_all();
  void finish_phases();
  void check_device_errors(int64_t step);
  // clears the sticky bad-id flag, rolls the host's dense step back over the gated steps
  // and raises the reference-style LogicError
  [[noreturn]] void raise_bad_id(int64_t step);
  // waits for the stream, folds the device-side totals of host-wait-free steps into the
  // host ledger / stats, refreshes the per-step counters and the free-stack copies
  void refresh();

  sfctr_config cfg_;
  int rank_, world_, lanes_, W_, lane0_, dev_;
  int d_, F_, b_, H_, K_;
  int64_t n_local_, n_global_;  // ids per step: this process / whole global batch
  size_t P_;                    // dense parameter count
  cudaStream_t stream_ = nullptr;   // training stage (GPU-Worker)
  ncclComm_t comm_ = nullptr;
  // Pipelined mode (RunMode::kPipelined, config.hpp:30): the manager stage
  // (ids, VSI, MixCache admission/eviction, exchange plan) of step t+1 runs on mstream_
  // while step t trains on stream_. Buffers the training stage reads come in two sets
  // (step parity); prep_done_/train_done_ order the stages. Sequential mode issues both
  // stages on stream_.
  struct Prepared {  // what the manager stage of a step hands to its training stage
    int64_t step = -1;
    int k = 0;
    cudaStream_t sm = nullptr;
    bool free_step = false, xdev = false;
    int32_t U = 0;
    std::vector<int32_t> n_own;
    int64_t launches0 = 0;
  } prep_;
  bool pipelined_ = false;
  bool no_free_steps_ = false;  // experiment switch: every step waits for the exact counts
  cudaStream_t mstream_ = nullptr;
  ncclComm_t mcomm_ = nullptr;       // manager-stage communicator (id all-gather)
  IdGather idg_;                     // NVLink peer-store id all-gather (world > 1)
  cudaStream_t dstream_ = nullptr;   // dense-gradient all-reduce, overlapping the row exchange
  // sparse update stream: once the dX GEMM has scattered the embedding gradients, the row
  // update (sparse Adam, or at W > 1 the gradient push + owner reduction + Adam) runs here
  // while the training stream computes dW1 (GEMM3) and its reduction
  cudaStream_t ustream_ = nullptr;
  cudaEvent_t dx_done_ = nullptr, upd_done_ = nullptr;
  void launch_row_update(cudaStream_t us, int k, bool a2a, bool defer_fm, float emb_scale,
                         const float* grad_rows);
  bool no_update_fork_ = false;  // SFCTR_NO_UPDATE_FORK=1: the update stays on the training stream
  int32_t prep_n_own0_ = 0;      // the training step's owned-count bound and parity set
  int prep_k_ = 0;
  cudaEvent_t dense_ready_ = nullptr, dense_done_ = nullptr;
  cudaEvent_t prep_done_[2] = {}, train_done_[2] = {};
  bool prep_recorded_[2] = {false, false};
  cudaStream_t cstream_ = nullptr;   // host-input copies (pipelined submit_host)
  cudaEvent_t in_ready_[2] = {};
  bool input_wait_ = false;          // the next prepare() waits for in_ready_
  bool train_pending_[2] = {false, false};
  int32_t* d_snap_[2] = {};          // [1 + kCntWords * lanes]: U, then every lane's counters
  uint32_t* d_uniq_set_[2] = {};
  float* d_dG_set_[2] = {};          // gradient tables (dG / the exchange's dE), per parity
  float* d_B_set_[2] = {};
  // one worker, fused FM deferral: dG / B are cleared by the manager stage (see train())
  bool early_clear_direct() const {
    return W_ == 1 && !a2a_ && d_ % 4 == 0 && !tower_fused_;
  }
  uint32_t* d_vid_set_[2] = {};
  uint64_t* d_in_feat_set_[2] = {};
  uint8_t* d_in_lab_set_[2] = {};
  uint64_t* d_in_win_set_[2] = {};
  float* d_loss_set_[2] = {};
  // losses of submitted steps (slot = step % kLossRing): the host may run up to kLossRing
  // steps ahead of the loss it reads; the device-side parity sets are ordered by events
  static constexpr int kLossRing = 4;
  float* h_loss_ring_ = nullptr;     // pinned, mapped [kLossRing]
  float* d_loss_ring_ = nullptr;     // its device alias
  cudaEvent_t loss_ev_[kLossRing] = {};
  int64_t loss_step_[kLossRing] = {-1, -1, -1, -1};

  VsiScratch vsi_;
  uint32_t* d_ids32_ = nullptr;     // local ids, u32
  uint32_t* d_gids_ = nullptr;      // global batch ids (all-gathered)
  uint32_t* d_uniq_ = nullptr;      // global_ids [U]        (current set, see d_uniq_set_)
  uint32_t* d_vid_ = nullptr;       // virtual ids [n_global] (current set)
  int32_t* d_scalars_ = nullptr;    // [0]=U, [1]=bad id flag, [2..]=window U
  uint32_t* d_wuniq_ = nullptr;     // window batch uniques (one batch at a time)
  uint32_t* d_wvid_ = nullptr;
  float* d_G_ = nullptr;            // global common embedding [U x d]
  float* d_dG_ = nullptr;           // global common gradients [U x d]
  float* d_B_ = nullptr;            // [U] deferred FM coefficient per unique (one worker)
  float* d_X_ = nullptr;            // minibatch embeddings [b x K]
  float* d_dX_ = nullptr;
  float* d_fm_s_ = nullptr;
  float* d_fm_sqp_ = nullptr;
  float* d_logits_ = nullptr;       // [rows]
  float* d_dense_ = nullptr;        // [P] = W1 | b1 | w2 | b2
  float* d_dense_m_ = nullptr;
  float* d_dense_v_ = nullptr;
  float* d_grads_ = nullptr;        // [P + 1] (+ loss sum)
  float* d_loss_ = nullptr;         // current set's loss (host-buffer steps)
  float* d_bc1_ = nullptr;          // sparse Adam bias-correction tables [t_cap + 1]
  float* d_bc2_ = nullptr;
  int64_t bc_cap_ = 0, bc_filled_ = 0;
  int32_t* h_scalars_ = nullptr;    // pinned mirrors
  int32_t* h_counts_ = nullptr;     // [lanes * kCntWords]

  std::vector<CacheLane> lane_;
  TowerBufs tower_;
  TowerTC towertc_;
  bool a2a_ = false;              // owner-routed all-to-all sync (world > 1)
  Exchange xch_;
  uint32_t* d_lvid_ = nullptr;    // [n_local] local-table rows of this process's positions
  // owner-sharded manager stage (shardplan.h): ids routed to their owners instead of the
  // all-gather + replicated VSI + replicated plan (alltoall over peer stores, lookahead 1;
  // SFCTR_SHARD_MANAGER=0 keeps the replicated stage)
  ShardPlan shard_;
  bool sharded_ = false;
  // SFCTR_STEP_TRACE diagnostics: stage-boundary stamps, printed at destruction
  unsigned long long* d_stamps_ = nullptr;
  int64_t last_stamped_ = -1;
  void stamp(int64_t step, int slot, cudaStream_t s);
  void dump_stamps();
  unsigned long long* d_pst_ = nullptr;  // SFCTR_PHASE_STAMPS ring
  int pst_cap_ = 0;
  int64_t pst_n_ = 0;
  std::vector<std::string> pst_names_;
  std::vector<cudaStream_t> pst_streams_;
  void phase_stamp(const char* name, cudaStream_t s);
  void dump_phase_stamps();
  int32_t* h_totals_ = nullptr;   // pinned [16] exchange plan totals
  int ldx_ = 0;
  bool tower_simt_ = false;
  bool det_ = false;              // deterministic: fixed-order segment sums (segment_sum_csr)
  SegCsr csr_;
  bool tower_fused_ = false;
  bool w1_split_ready_ = false;  // towertc_ holds the tf32 parts of the current W1
  int64_t dense_steps_ = 0;
  int64_t steps_done_ = 0;
  int64_t led_[4] = {0, 0, 0, 0};
  // Steps that need no host wait (world 1, no eviction possible) run the manager on
  // device counts alone: free_lb_[l] is a lower bound of lane l's device free-stack
  // height (exact after every waiting step, minus the per-step admission bound after
  // each free one); d_acc_ accumulates their totals: U, owned, working, interworker bytes
  std::vector<int64_t> free_lb_;
  int64_t* d_acc_ = nullptr;
  // [0] a flag barrier timed out (a peer never arrived), [1] steps gated by a bad id:
  // after an id >= vocab is seen (d_scalars_[1], sticky until the host reports it) every
  // step runs with no owned rows and skips the dense update, so no state moves
  int32_t* d_err_ = nullptr;
  int64_t* h_acc_ = nullptr;
  bool acc_pending_ = false;    // d_acc_ holds steps not folded into the host totals yet
  bool last_step_free_ = false; // the last step skipped the host wait
  int64_t free_steps_ = 0;      // steps run without a host wait (for the bench / tests)
  int64_t from_host_seen_ = 0;
  sfctr_step_stats stats_{};

  bool timing_ = false;
  std::vector<cudaEvent_t> ev_;
  std::vector<std::string> ev_names_;
  std::vector<cudaStream_t> ev_streams_;
  std::vector<std::pair<std::string, float>> phase_ms_;
};

}  // namespace sfb
