// One process = one GPU = `lanes` worker lanes of Algorithm 1.
// The step is the reference's BSP step in stream order:
//
//   ids u64->u32 | allgather ids (NCCL) | VSI | [host: U]
//   per lane: owned select, window marks, probe          | [host: n_own, n_work]
//   per lane: evict (LRU sort + write-back), admit (fill / lazy init)
//   gather_cache -> G | allreduce G (NCCL)
//   per lane: gather_instances(+FM sums) -> tower fwd/bwd -> segment_sum -> dG
//   allreduce dG + dense grads (NCCL) | per lane sparse Adam | dense Adam
//
// The two host waits ("[host: ...]") read the few counts that size the NCCL
// payloads and the eviction sort; everything else is asynchronous.
#include "trainer.h"

#include "tc_gemm.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

namespace sfb {

thread_local int64_t g_launches = 0;

namespace {
__global__ void finalize_loss_kernel(const float* sum, float inv_w, float* out) {
  if (threadIdx.x == 0) *out = *sum * inv_w;
}
__global__ void dense_init_kernel(float* p, int64_t n, uint64_t stream_seed, double a) {
  // W ~ U(-a, a) from the counter-based stream derive_seed(seed, label, 0)
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n)
    p[i] = static_cast<float>(
        uniform_from(splitmix_mix(stream_seed + static_cast<uint64_t>(i + 1) * kGolden), -a, a));
}
}  // namespace

// default VSI table: the hashed one (L2-resident at every shipped size)
bool vsi_hash_default() { return true; }

void validate_config(const sfctr_config& c) {  // config.cpp:55-78 + device limits
  auto require = [](bool ok, const char* msg) {
    if (!ok) fail(kConfig, msg);
  };
  require(c.num_workers > 0, "workers must be positive");
  require(c.embedding_dim > 0, "dim must be positive");
  require(c.num_fields > 0, "fields must be positive");
  require(c.batch_size_per_worker > 0, "batch-size must be positive");
  require(c.vocabulary_size > 0, "vocab must be positive");
  require(c.cache_capacity > 0, "cache-capacity must be positive");
  require(c.lookahead_depth > 0, "lookahead must be positive");
  require(c.hidden_dim > 0, "hidden must be positive");
  require(c.learning_rate > 0, "lr must be positive");
  require(c.adam_beta1 > 0 && c.adam_beta1 < 1, "beta1 must be in (0,1)");
  require(c.adam_beta2 > 0 && c.adam_beta2 < 1, "beta2 must be in (0,1)");
  require(c.adam_epsilon > 0, "epsilon must be positive");
  require(c.zipf_exponent >= 0, "zipf exponent must be non-negative");
  require(c.vocabulary_size >= static_cast<uint64_t>(c.num_fields),
          "vocab must be at least the number of fields (fields use disjoint vocabulary shards)");
  // device-path limits
  require(c.strategy == SFCTR_STRATEGY_CACHE,
          "the device path implements the cache strategy (host/prefetch are simulator-only)");
  require(c.vocabulary_size < 0xFFFFFFF0ull, "vocab must fit 32-bit device feature ids");
  require(c.cache_capacity < 0x7FFFFFF0ull, "cache-capacity must fit 31-bit slots");
  require(static_cast<int64_t>(c.num_workers) * c.batch_size_per_worker * c.num_fields <
              (1ll << 31),
          "global batch ids must fit 31 bits");
  require(c.sync_mode == SFCTR_SYNC_ALLREDUCE || c.sync_mode == SFCTR_SYNC_ALLTOALL,
          "sync must be allreduce or alltoall");
  require(c.run_mode == SFCTR_MODE_SEQUENTIAL || c.run_mode == SFCTR_MODE_PIPELINED,
          "mode must be pipelined or sequential");
  if (c.data_source == SFCTR_DATA_CRITEO) {  // config.cpp:74-77
    require(c.criteo_path[0] != 0, "criteo data source needs a file path");
    require(c.num_fields == 26, "criteo format has 26 categorical fields; set fields=26");
  } else {
    require(c.data_source == SFCTR_DATA_SYNTHETIC, "data must be synthetic or criteo:<path>");
  }
  require(c.deterministic == 0 || c.deterministic == 1, "deterministic must be 0 or 1");
}

Trainer::Trainer(const sfctr_config& cfg, int rank, int world, const uint8_t* nccl_id, int device)
    : cfg_(cfg), rank_(rank), world_(world), dev_(device) {
  validate_config(cfg_);
  if (world < 1 || rank < 0 || rank >= world) fail(kConfig, "bad rank/world");
  if (cfg_.num_workers % world != 0) fail(kConfig, "workers must be a multiple of the process count");
  W_ = cfg_.num_workers;
  lanes_ = W_ / world;
  lane0_ = rank * lanes_;
  d_ = cfg_.embedding_dim;
  F_ = cfg_.num_fields;
  b_ = cfg_.batch_size_per_worker;
  H_ = cfg_.hidden_dim;
  K_ = F_ * d_;
  n_local_ = static_cast<int64_t>(lanes_) * b_ * F_;
  n_global_ = static_cast<int64_t>(W_) * b_ * F_;
  P_ = static_cast<size_t>(K_) * H_ + 2 * H_ + 1;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(kCuda, "no CUDA device available (the device path has no CPU fallback)");
  }
  CUDA_CHECK(cudaSetDevice(device));
  pipelined_ = cfg_.run_mode == SFCTR_MODE_PIPELINED;
  int prio_lo = 0, prio_hi = 0;
  CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // the training stage is the step's critical path: in pipelined mode its CTAs are
  // scheduled ahead of the manager stage's (which only has to finish within the step)
  // Stream priorities (SFCTR_STREAM_PRIO): "same" (default) = both stages at one priority;
  // "train" = training high, manager low; "manager" = the reverse. Both stages run all the
  // time and the manager sets the step, so favouring the training stage does
  // not pay: same vs train measured 66.6 vs 65.0 M samples/s at N = 4, 28.4 vs 28.1 M at N = 1
  int prio_train = prio_lo, prio_mgr = prio_lo;
  if (const char* e = std::getenv("SFCTR_STREAM_PRIO")) {
    if (std::string(e) == "train" && pipelined_) prio_train = prio_hi;
    if (std::string(e) == "manager" && pipelined_) prio_mgr = prio_hi;
  }
  CUDA_CHECK(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, prio_train));
  if (const char* e = std::getenv("SFCTR_NO_FREE_STEPS")) no_free_steps_ = e[0] == '1';
  if (const char* e = std::getenv("SFCTR_NO_UPDATE_FORK")) no_update_fork_ = e[0] == '1';
  CUDA_CHECK(cudaStreamCreateWithPriority(&ustream_, cudaStreamNonBlocking, prio_train));
  CUDA_CHECK(cudaEventCreateWithFlags(&dx_done_, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&upd_done_, cudaEventDisableTiming));
  CUDA_CHECK(cudaMalloc(&d_err_, sizeof(int32_t) * 4));
  CUDA_CHECK(cudaMemset(d_err_, 0, sizeof(int32_t) * 4));
  mstream_ = stream_;
  if (pipelined_) {
    CUDA_CHECK(cudaStreamCreateWithPriority(&mstream_, cudaStreamNonBlocking, prio_mgr));
    CUDA_CHECK(cudaStreamCreateWithFlags(&cstream_, cudaStreamNonBlocking));
    for (auto& e : in_ready_) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (world_ > 1) {
    if (!nccl_id) fail(kConfig, "world > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    NCCL_CHECK(ncclCommInitRank(&comm_, world_, id, rank_));
    // collectives of the two stages overlap, so they run on separate communicators
    mcomm_ = comm_;
    if (pipelined_) NCCL_CHECK(ncclCommSplit(comm_, 0, rank_, &mcomm_, nullptr));
    CUDA_CHECK(cudaStreamCreateWithFlags(&dstream_, cudaStreamNonBlocking));
    const char* ni = std::getenv("SFCTR_NCCL_IDS");  // debugging: NCCL id all-gather
    if (!(ni && ni[0] == '1')) {
      idg_.init(world_, rank_, n_local_);
      if (!idg_.setup_p2p(comm_, stream_)) idg_.release();
      idg_.abort_flag = d_err_;
    }
    CUDA_CHECK(cudaEventCreateWithFlags(&dense_ready_, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&dense_done_, cudaEventDisableTiming));
  }

  // VSI first-position table: hashed (2 x the global batch, L2-resident) or direct-mapped
  // over the vocabulary (SFCTR_VSI_HASH=0|1 overrides the default)
  {
    bool hash = vsi_hash_default();
    if (const char* e = std::getenv("SFCTR_VSI_HASH")) hash = e[0] == '1';
    vsi_.init(cfg_.vocabulary_size, n_global_, hash);
  }
  if (lanes_ > 8) fail(kConfig, "at most 8 worker lanes per process");
  for (int k = 0; k < 2; ++k) {  // per-step-parity sets (see trainer.h)
    CUDA_CHECK(cudaMalloc(&d_in_feat_set_[k], sizeof(uint64_t) * n_local_));
    CUDA_CHECK(cudaMalloc(&d_in_lab_set_[k], static_cast<size_t>(lanes_) * b_));
    if (cfg_.lookahead_depth > 1)
      CUDA_CHECK(cudaMalloc(&d_in_win_set_[k],
                            sizeof(uint64_t) * n_local_ * (cfg_.lookahead_depth - 1)));
    CUDA_CHECK(cudaMalloc(&d_uniq_set_[k], sizeof(uint32_t) * n_global_));
    CUDA_CHECK(cudaMalloc(&d_vid_set_[k], sizeof(uint32_t) * n_global_));
    CUDA_CHECK(cudaMalloc(&d_snap_[k], sizeof(int32_t) * (1 + kCntWords * lanes_)));
    CUDA_CHECK(cudaMemset(d_snap_[k], 0, sizeof(int32_t) * (1 + kCntWords * lanes_)));
    CUDA_CHECK(cudaMalloc(&d_loss_set_[k], sizeof(float)));
    CUDA_CHECK(cudaEventCreateWithFlags(&prep_done_[k], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&train_done_[k], cudaEventDisableTiming));

  }
  d_uniq_ = d_uniq_set_[0];
  d_vid_ = d_vid_set_[0];
  CUDA_CHECK(cudaMalloc(&d_ids32_, sizeof(uint32_t) * n_local_));
  CUDA_CHECK(cudaMalloc(&d_gids_, sizeof(uint32_t) * n_global_));
  CUDA_CHECK(cudaMalloc(&d_scalars_, sizeof(int32_t) * 8));
  CUDA_CHECK(cudaMemset(d_scalars_, 0, sizeof(int32_t) * 8));
  if (cfg_.lookahead_depth > 1) {
    CUDA_CHECK(cudaMalloc(&d_wuniq_, sizeof(uint32_t) * n_global_));
    CUDA_CHECK(cudaMalloc(&d_wvid_, sizeof(uint32_t) * n_global_));
  }
  const size_t gd = static_cast<size_t>(n_global_) * d_;
  CUDA_CHECK(cudaMalloc(&d_G_, sizeof(float) * gd));
  for (int k = 0; k < 2; ++k) {  // per step parity: the manager stage clears the next step's
    CUDA_CHECK(cudaMalloc(&d_dG_set_[k], sizeof(float) * gd));  // set while this one trains
    CUDA_CHECK(cudaMalloc(&d_B_set_[k], sizeof(float) * n_global_));
  }
  d_dG_ = d_dG_set_[0];
  d_B_ = d_B_set_[0];
  ldx_ = tower_ldx(K_);
  const size_t bk = static_cast<size_t>(b_) * ldx_;
  CUDA_CHECK(cudaMalloc(&d_X_, sizeof(float) * bk));
  CUDA_CHECK(cudaMalloc(&d_dX_, sizeof(float) * bk));
  CUDA_CHECK(cudaMalloc(&d_fm_s_, sizeof(float) * b_ * d_));
  CUDA_CHECK(cudaMalloc(&d_fm_sqp_, sizeof(float) * b_ * d_));
  CUDA_CHECK(cudaMalloc(&d_logits_, sizeof(float) * lanes_ * b_));
  CUDA_CHECK(cudaMalloc(&d_dense_, sizeof(float) * P_));
  CUDA_CHECK(cudaMalloc(&d_dense_m_, sizeof(float) * P_));
  CUDA_CHECK(cudaMalloc(&d_dense_v_, sizeof(float) * P_));
  CUDA_CHECK(cudaMalloc(&d_grads_, sizeof(float) * (P_ + 1)));
  d_loss_ = d_loss_set_[0];
  CUDA_CHECK(cudaMemset(d_dense_, 0, sizeof(float) * P_));
  CUDA_CHECK(cudaMemset(d_dense_m_, 0, sizeof(float) * P_));
  CUDA_CHECK(cudaMemset(d_dense_v_, 0, sizeof(float) * P_));
  // dense init (identical on every process: pure function of the seed)
  const int64_t kh = static_cast<int64_t>(K_) * H_;
  dense_init_kernel<<<ceil_div(kh, 256), 256, 0, stream_>>>(
      d_dense_, kh, derive_seed_h(cfg_.seed, fnv1a64("dense_w1"), 0),
      std::sqrt(6.0 / static_cast<double>(K_ + H_)));
  CUDA_LAUNCH_CHECK();
  dense_init_kernel<<<ceil_div(H_, 256), 256, 0, stream_>>>(
      d_dense_ + kh + H_, H_, derive_seed_h(cfg_.seed, fnv1a64("dense_w2"), 0),
      std::sqrt(6.0 / static_cast<double>(H_ + 1)));
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_scalars_), sizeof(int32_t) * 8, 0));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_counts_),
                           sizeof(int32_t) * kCntWords * lanes_, 0));
  // mapped: the step's last kernel stores the loss straight into the host slot (no D2H copy
  // between one step's training stage and the next on the worker stream)
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_loss_ring_), sizeof(float) * kLossRing,
                           cudaHostAllocMapped));
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_loss_ring_), h_loss_ring_, 0));
  for (int q = 0; q < kLossRing; ++q)
    CUDA_CHECK(cudaEventCreateWithFlags(&loss_ev_[q], cudaEventDisableTiming));
  CUDA_CHECK(cudaMalloc(&d_acc_, sizeof(int64_t) * 8));
  CUDA_CHECK(cudaMemset(d_acc_, 0, sizeof(int64_t) * 8));

  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_acc_), sizeof(int64_t) * 8, 0));
  tower_.init(b_, K_, H_, d_);
  towertc_.init(b_, K_, H_, d_);
  // validation switch: the fp32 SIMT tiles instead of tcgen05 (only when rows are unpadded)
  const char* ts = std::getenv("SFCTR_TOWER_SIMT");
  tower_simt_ = ts && ts[0] == '1' && ldx_ == K_;
  // fused gather/GEMM/scatter tower (SFCTR_TOWER_FUSED=1): X / dX never touch HBM,
  // but on B200 the streamed path below is faster today (profiles/), so it is opt-in
  const char* tf = std::getenv("SFCTR_TOWER_FUSED");
  det_ = cfg_.deterministic != 0;
  tower_fused_ = !tower_simt_ && !det_ && tower_fused_supported(d_) && tf && tf[0] == '1';
  if (det_) csr_.init(static_cast<int64_t>(b_) * F_);

  const uint64_t owned_rows = (cfg_.vocabulary_size + W_ - 1) / W_;
  lane_.resize(lanes_);
  const int64_t umax = std::min<int64_t>(n_global_, static_cast<int64_t>(cfg_.vocabulary_size));
  // host_rows: host-pool slots pinned up front per lane (the pool grows on demand)
  for (int l = 0; l < lanes_; ++l)
    lane_[l].init(cfg_.cache_capacity, d_, owned_rows, cfg_.host_table_rows, umax);
  free_lb_.assign(lanes_, static_cast<int64_t>(cfg_.cache_capacity));
  if (world_ > 1 && cfg_.sync_mode == SFCTR_SYNC_ALLTOALL) {
    if (lanes_ != 1) fail(kConfig, "sync=alltoall needs one worker per process");
    if (W_ > 8) fail(kConfig, "sync=alltoall supports at most 8 workers (one NVSwitch box)");
    if (d_ % 4) fail(kConfig, "sync=alltoall needs dim % 4 == 0");
    a2a_ = true;
    xch_.init(W_, rank_, umax, d_);
    xch_.abort_flag = d_err_;
    CUDA_CHECK(cudaMalloc(&d_lvid_, sizeof(uint32_t) * n_local_));
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_totals_),
                             sizeof(int32_t) * Exchange::kTotals, 0));
    const char* np2p = std::getenv("SFCTR_NO_P2P");  // debugging: force NCCL send/recv
    if (!(np2p && np2p[0] == '1')) xch_.setup_p2p(d_G_, comm_, stream_);
    const char* ce = std::getenv("SFCTR_P2P_COPY_ENGINE");  // DMA copies instead of SM stores
    xch_.copy_engine = ce && ce[0] == '1';
    const char* nb = std::getenv("SFCTR_NCCL_BARRIER");
    xch_.nccl_barrier = nb && nb[0] == '1';
    // owner-sharded manager stage (same decision on every rank: the environment and the
    // collectively agreed peer access)
    const char* sh = std::getenv("SFCTR_SHARD_MANAGER");
    if (xch_.device_driven() && !xch_.nccl_barrier && cfg_.lookahead_depth == 1 &&
        !(sh && sh[0] == '0')) {
      shard_.init(W_, rank_, n_local_, umax);
      shard_.abort_flag = d_err_;
      sharded_ = shard_.setup_p2p(comm_, stream_);
      if (!sharded_) shard_.release();
    }
  }
  ensure_bias_tables(1024);
  CUDA_CHECK(cudaStreamSynchronize(stream_));
}

Trainer::~Trainer() {
  cudaSetDevice(dev_);
  try {
    dump_stamps();
    dump_phase_stamps();
  } catch (...) {
  }
  if (d_stamps_) cudaFree(d_stamps_);
  if (d_pst_) cudaFree(d_pst_);
  if (mstream_) cudaStreamSynchronize(mstream_);
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& l : lane_) l.release();
  csr_.release();
  tower_.release();
  towertc_.release();
  shard_.release();
  xch_.release();
  if (d_lvid_) cudaFree(d_lvid_);
  if (h_totals_) cudaFreeHost(h_totals_);
  vsi_.release();
  for (int k = 0; k < 2; ++k) {
    for (void* p : {static_cast<void*>(d_in_feat_set_[k]), static_cast<void*>(d_in_lab_set_[k]),
                    static_cast<void*>(d_in_win_set_[k]), static_cast<void*>(d_uniq_set_[k]),
                    static_cast<void*>(d_vid_set_[k]), static_cast<void*>(d_snap_[k]),
                    static_cast<void*>(d_loss_set_[k])})
      if (p) cudaFree(p);
    for (cudaEvent_t e : {prep_done_[k], train_done_[k]})
      if (e) cudaEventDestroy(e);
  }
  for (void* p : {static_cast<void*>(d_ids32_),
                  static_cast<void*>(d_gids_), static_cast<void*>(d_scalars_),
                  static_cast<void*>(d_wuniq_), static_cast<void*>(d_wvid_),
                  static_cast<void*>(d_G_), static_cast<void*>(d_dG_set_[0]),
                  static_cast<void*>(d_dG_set_[1]), static_cast<void*>(d_B_set_[0]),
                  static_cast<void*>(d_B_set_[1]), static_cast<void*>(d_X_),
                  static_cast<void*>(d_dX_), static_cast<void*>(d_fm_s_),
                  static_cast<void*>(d_fm_sqp_), static_cast<void*>(d_logits_),
                  static_cast<void*>(d_dense_), static_cast<void*>(d_dense_m_),
                  static_cast<void*>(d_dense_v_), static_cast<void*>(d_grads_),
                  static_cast<void*>(d_bc1_),
                  static_cast<void*>(d_bc2_), static_cast<void*>(d_acc_),
                  static_cast<void*>(d_err_),
                  })
    if (p) cudaFree(p);
  if (h_acc_) cudaFreeHost(h_acc_);
  if (h_scalars_) cudaFreeHost(h_scalars_);
  if (h_counts_) cudaFreeHost(h_counts_);
  if (h_loss_ring_) cudaFreeHost(h_loss_ring_);
  for (cudaEvent_t e : loss_ev_)
    if (e) cudaEventDestroy(e);
  for (auto e : ev_) cudaEventDestroy(e);
  if (dstream_) cudaStreamSynchronize(dstream_);
  idg_.release();
  for (cudaEvent_t e : {dense_ready_, dense_done_})
    if (e) cudaEventDestroy(e);
  if (dstream_) cudaStreamDestroy(dstream_);
  if (ustream_) {
    cudaStreamSynchronize(ustream_);
    cudaStreamDestroy(ustream_);
  }
  for (cudaEvent_t e : {dx_done_, upd_done_})
    if (e) cudaEventDestroy(e);
  if (mcomm_ && mcomm_ != comm_) ncclCommDestroy(mcomm_);
  if (comm_) ncclCommDestroy(comm_);
  if (mstream_ && mstream_ != stream_) cudaStreamDestroy(mstream_);
  if (cstream_) cudaStreamDestroy(cstream_);
  for (cudaEvent_t e : in_ready_)
    if (e) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
}

void Trainer::ensure_bias_tables(int64_t t_max) {
  if (t_max < bc_cap_) return;
  int64_t cap = std::max<int64_t>(1024, bc_cap_);
  while (cap <= t_max) cap *= 2;
  std::vector<float> b1(cap + 1), b2(cap + 1);
  for (int64_t t = 0; t <= cap; ++t) {  // 1 - beta^t in fp64, stored fp32
    b1[t] = static_cast<float>(1.0 - std::pow(cfg_.adam_beta1, static_cast<double>(t)));
    b2[t] = static_cast<float>(1.0 - std::pow(cfg_.adam_beta2, static_cast<double>(t)));
  }
  CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (d_bc1_) cudaFree(d_bc1_);
  if (d_bc2_) cudaFree(d_bc2_);
  CUDA_CHECK(cudaMalloc(&d_bc1_, sizeof(float) * (cap + 1)));
  CUDA_CHECK(cudaMalloc(&d_bc2_, sizeof(float) * (cap + 1)));
  CUDA_CHECK(cudaMemcpy(d_bc1_, b1.data(), sizeof(float) * (cap + 1), cudaMemcpyHostToDevice));
  CUDA_CHECK(cudaMemcpy(d_bc2_, b2.data(), sizeof(float) * (cap + 1), cudaMemcpyHostToDevice));
  bc_cap_ = cap;
}

namespace {

struct LaneCounters {
  const int32_t* c[8];
};

struct StepClear {
  int32_t* scalars;
  int32_t* cnt[8];
  int lanes;
};
// scalars[0] and [2, 8) ([1], the bad-id flag, is sticky until a host check has seen it);
// per lane counters [0, 2), [3, 5) and kCntOld
__global__ void step_clear_kernel(StepClear a) {
  pdl_wait();
  const int t = threadIdx.x;
  if (t < 8 && t != 1) a.scalars[t] = 0;
  const int l = t / 8, q = t % 8;
  if (l < a.lanes) {
    const int idx = q < 2 ? q : q < 4 ? q + 1 : q == 4 ? kCntOld : -1;
    if (idx >= 0) a.cnt[l][idx] = 0;
  }
}

// The step's tail in one launch: dense Adam over the P dense parameters (same math as
// dense_adam, tower.cu), the per-row Adam step counts of the rows sparse_adam just
// updated, the loss, and (host-wait-free steps) the step totals.
struct TailArgs {
  float *p, *m, *v;
  const float* g;
  int64_t n;
  float gs, lr, b1, b2, omb1, omb2, eps, bc1, bc2;
  const float* loss_sum;
  float inv_w;
  float* loss_out;
  int lanes;
  const uint32_t* own_slot[8];
  const int32_t* n_own[8];
  int32_t* steps[8];
  // W1's tf32 hi/lo parts in both tower layouts (nullptr: not maintained here)
  float *w_hi, *w_lo, *wt_hi, *wt_lo;
  int K, H, ldh, ldk;
  int64_t* acc;  // nullptr: no totals this step
  const int32_t* xtotals;  // owner-routed exchange plan totals (nullptr: none)
  int me;
  LaneCounters cnt;
  const int32_t* U;
  int W, d;
  int64_t P;
  const int32_t* bad;  // sticky bad-id flag: the step moves no state
  int32_t* gated;      // steps skipped that way
};

__global__ void tail_kernel(TailArgs a) {
  pdl_wait();
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (*a.bad) {
    if (tid == 0) {
      *a.gated += 1;
      *a.loss_out = __int_as_float(0x7fc00000);  // NaN: the step did not run
    }
    return;
  }
  for (int64_t i = tid; i < a.n; i += stride) {
    const float gi = a.g[i] * a.gs;
    const float mi = a.b1 * a.m[i] + a.omb1 * gi;
    const float vi = a.b2 * a.v[i] + a.omb2 * gi * gi;
    a.m[i] = mi;
    a.v[i] = vi;
    const float pn = a.p[i] - a.lr * (mi / a.bc1) / (sqrtf(vi / a.bc2) + a.eps);
    a.p[i] = pn;
    if (a.w_hi && i < static_cast<int64_t>(a.K) * a.H) {  // same split as prep_w1 (tc_tower.cu)
      const int k = static_cast<int>(i / a.H), j = static_cast<int>(i % a.H);
      const float h = tc::tf32_rna(pn), lo = tc::tf32_rna(pn - h);
      a.w_hi[static_cast<int64_t>(k) * a.ldh + j] = h;
      a.w_lo[static_cast<int64_t>(k) * a.ldh + j] = lo;
      a.wt_hi[static_cast<int64_t>(j) * a.ldk + k] = h;
      a.wt_lo[static_cast<int64_t>(j) * a.ldk + k] = lo;
    }
  }
  for (int l = 0; l < a.lanes; ++l) {
    const int32_t n = *a.n_own[l];
    for (int64_t j = tid; j < n; j += stride) a.steps[l][a.own_slot[l][j]] += 1;
  }
  if (tid == 0) {
    *a.loss_out = *a.loss_sum * a.inv_w;
    if (a.acc) {
      int64_t owned = 0, working = 0;
      for (int l = 0; l < a.lanes; ++l) {
        owned += a.cnt.c[l][kCntOwned];
        working += a.cnt.c[l][kCntWorking];
      }
      const int64_t U = *a.U;
      auto arb = [&](int64_t q) { return 2 * static_cast<int64_t>(a.W - 1) * q / a.W; };
      a.acc[0] += U;
      a.acc[1] += owned;
      a.acc[2] += working;
      a.acc[3] += static_cast<int64_t>(a.lanes) * (2 * arb(U * a.d * 4) + arb(a.P * 4));
      if (a.xtotals)  // rows pushed to / received from peers, both directions
        for (int w = 0; w < a.W; ++w)
          if (w != a.me) a.acc[4] += static_cast<int64_t>(a.xtotals[8 + w] + a.xtotals[w]) * a.d * 4;
    }
  }
}

// dG[0 : U*d) = 0 with U read on the device
__global__ void zero_rows_kernel(float4* __restrict__ p, const int32_t* __restrict__ U_ptr, int d4,
                                 int64_t bound) {
  const int64_t n = static_cast<int64_t>(*U_ptr) * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n && i < bound;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace

namespace {
__global__ void empty_kernel() { pdl_wait(); }
// SFCTR_STEP_TRACE=n: globaltimer stamps of the last n steps' stage boundaries (diagnostics)
__global__ void stamp_kernel(unsigned long long* p) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *p = t;
}
int step_trace_n() {
  static const int n = [] {
    const char* e = std::getenv("SFCTR_STEP_TRACE");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  return n;
}
// phase pass only: hold the stream for `ns` so the host enqueues the whole step behind it and
// every phase time is device time, not the host's issue time (SFCTR_PHASE_GATE_US)
__global__ void phase_gate_kernel(uint64_t ns) {
  uint64_t t0 = 0, t = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
uint64_t phase_gate_ns() {
  static const uint64_t ns = [] {
    const char* e = std::getenv("SFCTR_PHASE_GATE_US");
    return e ? static_cast<uint64_t>(std::max(0.0, std::atof(e)) * 1e3) : 0ull;
  }();
  return ns;
}
}  // namespace

void Trainer::stamp(int64_t step, int slot, cudaStream_t s) {
  const int n = step_trace_n();
  if (n <= 0) return;
  if (!d_stamps_) {
    CUDA_CHECK(cudaMalloc(&d_stamps_, sizeof(unsigned long long) * 4 * n));
    CUDA_CHECK(cudaMemset(d_stamps_, 0, sizeof(unsigned long long) * 4 * n));
  }
  stamp_kernel<<<1, 1, 0, s>>>(d_stamps_ + (step % n) * 4 + slot);
  CUDA_CHECK(cudaGetLastError());
  last_stamped_ = step;
}

void Trainer::dump_stamps() {
  const int n = step_trace_n();
  if (n <= 0 || !d_stamps_) return;
  std::vector<unsigned long long> h(4 * n);
  CUDA_CHECK(cudaDeviceSynchronize());
  CUDA_CHECK(cudaMemcpy(h.data(), d_stamps_, sizeof(unsigned long long) * 4 * n,
                        cudaMemcpyDeviceToHost));
  // steps last_stamped_ - n + 1 .. last_stamped_, in order
  fprintf(stderr, "step trace (us, rel. to the first manager start): step mgr_start mgr_end "
                  "train_start train_end | train_wait_for_mgr train_gap_after_prev\n");
  const int64_t first = std::max<int64_t>(0, last_stamped_ - n + 1);
  const unsigned long long t0 = h[(first % n) * 4];
  unsigned long long prev_end = 0;
  for (int64_t st = first; st <= last_stamped_; ++st) {
    const unsigned long long* r = h.data() + (st % n) * 4;
    auto us = [&](unsigned long long t) { return t ? (static_cast<double>(t) - t0) * 1e-3 : -1.0; };
    fprintf(stderr, "%5lld %9.1f %9.1f %9.1f %9.1f | %7.1f %7.1f\n", static_cast<long long>(st),
            us(r[0]), us(r[1]), us(r[2]), us(r[3]),
            r[2] > r[1] ? (static_cast<double>(r[2]) - r[1]) * 1e-3 : 0.0,
            prev_end && r[2] > prev_end ? (static_cast<double>(r[2]) - prev_end) * 1e-3 : 0.0);
    prev_end = r[3];
  }
}

// SFCTR_PHASE_STAMPS=n: outside the phase pass, every phase boundary also writes a
// globaltimer stamp (one 1-thread kernel each, so the run is perturbed by their launches);
// the destructor prints the mean device time per phase and stream over the last steps
// (diagnostics: the stage breakdown while both stages run concurrently)
void Trainer::phase_stamp(const char* name, cudaStream_t s) {
  static const int cap = [] {
    const char* e = std::getenv("SFCTR_PHASE_STAMPS");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  if (cap <= 0) return;
  if (!d_pst_) {
    CUDA_CHECK(cudaMalloc(&d_pst_, sizeof(unsigned long long) * cap));
    pst_cap_ = cap;
  }
  const int64_t i = pst_n_++;
  stamp_kernel<<<1, 1, 0, s>>>(d_pst_ + i % cap);
  CUDA_CHECK(cudaGetLastError());
  if (static_cast<int64_t>(pst_names_.size()) < cap) {
    pst_names_.emplace_back(name);
    pst_streams_.push_back(s);
  } else {
    pst_names_[i % cap] = name;
    pst_streams_[i % cap] = s;
  }
}

void Trainer::dump_phase_stamps() {
  if (!d_pst_ || pst_n_ < 2) return;
  const int cap = pst_cap_;
  std::vector<unsigned long long> h(cap);
  CUDA_CHECK(cudaDeviceSynchronize());
  CUDA_CHECK(cudaMemcpy(h.data(), d_pst_, sizeof(unsigned long long) * cap, cudaMemcpyDeviceToHost));
  const int64_t first = std::max<int64_t>(0, pst_n_ - cap);
  std::map<std::pair<cudaStream_t, std::string>, std::pair<double, int>> acc;
  std::map<cudaStream_t, unsigned long long> last;
  for (int64_t i = first; i < pst_n_; ++i) {
    const int q = static_cast<int>(i % cap);
    const cudaStream_t st = pst_streams_[q];
    const std::string& nm = pst_names_[q];
    auto it = last.find(st);
    if (it != last.end() && nm != "start") {
      auto& a = acc[{st, nm}];
      a.first += (static_cast<double>(h[q]) - it->second) * 1e-3;
      a.second += 1;
    }
    last[st] = h[q];
  }
  fprintf(stderr, "phase stamps (mean us per occurrence, concurrent run):\n");
  for (const auto& kv : acc)
    fprintf(stderr, "  %s %-24s %8.2f  (n=%d)\n",
            kv.first.first == mstream_ ? "mgr  " : kv.first.first == ustream_ ? "upd  " : "train",
            kv.first.second.c_str(), kv.second.first / kv.second.second, kv.second.second);
}

void Trainer::phase(const char* name, cudaStream_t s) {
  if (!timing_) {
    phase_stamp(name, s ? s : stream_);
    return;
  }
  if (!s) s = stream_;
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreate(&e));
  CUDA_CHECK(cudaEventRecord(e, s));
  ev_.push_back(e);
  ev_names_.emplace_back(name);
  ev_streams_.push_back(s);
}

// Sums, per phase name, the device time between consecutive phase events of
// every step recorded since the last call (events accumulate across steps so
// a timed region needs no extra host synchronisation). A phase spans from the
// previous event on the SAME stream (manager and training stages are timed
// separately in pipelined mode).
void Trainer::finish_phases() {
  if (ev_.size() < 2) return;
  sync_all();
  for (size_t i = 1; i < ev_.size(); ++i) {
    if (ev_names_[i] == "start") continue;
    size_t j = i;
    while (j > 0 && ev_streams_[j - 1] != ev_streams_[i]) --j;
    if (j == 0) continue;
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[j - 1], ev_[i]));
    auto it = std::find_if(phase_ms_.begin(), phase_ms_.end(),
                           [&](const auto& p) { return p.first == ev_names_[i]; });
    if (it == phase_ms_.end()) phase_ms_.emplace_back(ev_names_[i], ms);
    else it->second += ms;
  }
  for (auto e : ev_) cudaEventDestroy(e);
  ev_.clear();
  ev_names_.clear();
  ev_streams_.clear();
}

void Trainer::sync_all() {
  CUDA_CHECK(cudaSetDevice(dev_));
  if (mstream_ != stream_) CUDA_CHECK(cudaStreamSynchronize(mstream_));
  CUDA_CHECK(cudaStreamSynchronize(stream_));
}

namespace {
// U and every lane's counters as the manager stage left them: the training stage reads
// this copy, so the next step's manager may reset and advance the live counters
struct SnapArgs {
  const int32_t* U;
  const int32_t* cnt[8];
  int lanes;
  int32_t* out;
};
__global__ void snap_kernel(SnapArgs a) {
  pdl_wait();
  const int i = threadIdx.x;
  if (i == 0) a.out[0] = *a.U;
  if (i < kCntWords * a.lanes) a.out[1 + i] = a.cnt[i / kCntWords][i % kCntWords];
}
// Bad-id gate (sticky flag d_scalars_[1]): a batch with an id >= vocab moves no state. The
// VSI table was already reset behind the batch (select_owned); here the step is left with
// no uniques and no owned rows, so probe / admission / exchange / update_sparse / the
// dense update do nothing, and every position is pointed at table row 0 (own_slot[0] = 0,
// lpos[0] = 0 after the plan) so the training stage reads valid memory and discards it.
struct GatePtrs {
  uint32_t* own_slot[8];
};
__global__ void bad_id_gate_kernel(const int32_t* __restrict__ bad, int32_t* U, LaneCounters cnt,
                                   int lanes, uint32_t* __restrict__ vid, int64_t n, GatePtrs gp) {
  pdl_wait();
  if (!*bad) return;
  const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t i = i0; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) vid[i] = 0;
  if (i0 == 0) {
    *U = 0;
    for (int l = 0; l < lanes; ++l) {
      const_cast<int32_t*>(cnt.c[l])[kCntOwned] = 0;
      gp.own_slot[l][0] = 0;
    }
  }
}
__global__ void bad_id_gate_plan_kernel(const int32_t* __restrict__ bad, uint32_t* lpos) {
  pdl_wait();
  if (*bad) lpos[0] = 0;
}
}  // namespace

// Host-Manager stage of step t (Algorithm 1 l.2-7; manager_get + pull_parameters_to_host +
// push_parameters_to_cache): ids, VSI, MixCache, exchange plan, enqueued on
// the manager stream. The training stage of the same step must follow (train()) before the
// next step is prepared.
void Trainer::prepare(int64_t step, const uint64_t* d_features, const uint64_t* d_window) {
  CUDA_CHECK(cudaSetDevice(dev_));
  if (prep_.step >= 0)
    fail(kLogic, "step " + std::to_string(prep_.step) + " was prepared but not trained");
  const int64_t launches0 = g_launches;
  const int32_t t = static_cast<int32_t>(step);
  const uint32_t Wu = static_cast<uint32_t>(W_);
  // sm: manager stage (Data-Loader + Host-Manager of Fig. 4), sw: training stage. With
  // per-phase timing on, both stages go on one stream so every phase's time is its own.
  cudaStream_t sm = timing_ ? stream_ : mstream_, sw = stream_;
  const bool piped = pipelined_ && sm != sw;
  if (step < 0 || step >= (1ll << 23)) fail(kLogic, "step index out of the supported range");
  if (cfg_.lookahead_depth > 1 && !d_window)
    fail(kLogic, "lookahead > 1 needs the window batches");
  const int k = static_cast<int>(step & 1);  // buffer set of this step
  // the set's previous user (step t-2) must have finished training before it is refilled
  if (piped && train_pending_[k]) CUDA_CHECK(cudaStreamWaitEvent(sm, train_done_[k]));
  if (input_wait_) {  // host inputs staged on the copy stream (submit_host)
    CUDA_CHECK(cudaStreamWaitEvent(sm, in_ready_[k]));
    input_wait_ = false;
  }
  d_uniq_ = d_uniq_set_[k];
  d_vid_ = d_vid_set_[k];
  d_dG_ = d_dG_set_[k];
  d_B_ = d_B_set_[k];
  for (auto& L : lane_) L.use(k);
  if (a2a_) xch_.use(k);
  int32_t* snap = d_snap_[k];
  auto snap_cnt = [&](int l) { return snap + 1 + kCntWords * l; };
  if (timing_ && phase_gate_ns()) {
    phase_gate_kernel<<<1, 1, 0, sm>>>(phase_gate_ns());
    CUDA_LAUNCH_CHECK();
  }
  phase("start", sm);
  if (sm != sw) phase("start", sw);
  stamp(step, 0, sm);
  {  // per-step fields restart, running totals carry over
    sfctr_step_stats next{};
    next.total_steps = stats_.total_steps;
    next.total_working = stats_.total_working;
    next.total_evicted = stats_.total_evicted;
    next.total_filled_from_host = stats_.total_filled_from_host;
    next.total_kernel_launches = stats_.total_kernel_launches;
    next.total_unique = stats_.total_unique;
    next.total_owned = stats_.total_owned;
    next.total_nvlink_bytes = stats_.total_nvlink_bytes;
    next.total_pinned_waits = stats_.total_pinned_waits;
    stats_ = next;
  }

  // ==== manager stage (stream sm) ====
  // ---- Data-Loader: ids to u32, all-gather the global batch, VSI (Algorithm 1 l.2-3)
  // [1] (bad-id flag) is sticky until a host check has seen it
  // per-step scalars and per-lane counters cleared in one launch (kCntFromHost (index 2),
  // kCntFreeTop and kCntSeq carry over)
  {
    StepClear sc{};
    sc.scalars = d_scalars_;
    for (int l = 0; l < lanes_; ++l) sc.cnt[l] = lane_[l].counters;
    sc.lanes = lanes_;
    launch_pdl(step_clear_kernel, dim3(1), dim3(64), 0, sm, sc);
    CUDA_LAUNCH_CHECK();
  }
  const int32_t cap = static_cast<int32_t>(lane_[0].umax);
  struct HookCtx {
    Trainer* tr;
    cudaStream_t s;
  } hctx{this, sm};
  const PhaseHook mhook{[](void* c, const char* n) {
                          auto* h = static_cast<HookCtx*>(c);
                          h->tr->phase(n, h->s);
                        },
                        &hctx};
  const uint32_t* gids = d_ids32_;
  if (sharded_) {
    // ids routed to their owners; each owner's uniques in global first-appearance order
    // (own_k = identity, d_uniq_ = the owned features), the exchange plan and every rank's
    // position -> local-table row map (shard_.index(k) into shard_.rows(k)); U (all ranks)
    // lands in d_scalars_[0]
    shard_.run(d_features, cfg_.vocabulary_size, d_scalars_ + 1, k, xch_, d_uniq_, lane_[0].own_k,
               lane_[0].counters + kCntOwned, d_scalars_ + 0, sm, mhook);
    stats_.nvlink_bytes += n_local_ * 12;  // pairs out, local rows back
  } else if (world_ > 1 && idg_.p2p) {  // u64 -> u32 + peer stores into every rank's buffer
    gids = idg_.gather(d_features, cfg_.vocabulary_size, d_scalars_ + 1, k, sm);
    stats_.nvlink_bytes += n_local_ * 4;
  } else {
    ids_to_u32(d_features, d_ids32_, n_local_, cfg_.vocabulary_size, d_scalars_ + 1, sm);
    if (world_ > 1) {
      NCCL_CHECK(ncclAllGather(d_ids32_, d_gids_, static_cast<size_t>(n_local_), ncclUint32, mcomm_, sm));
      // every rank gates the step when any rank saw an id >= vocab
      NCCL_CHECK(ncclAllReduce(d_scalars_ + 1, d_scalars_ + 1, 1, ncclInt32, ncclMax, mcomm_, sm));
      gids = d_gids_;
      stats_.nvlink_bytes += n_local_ * 4;
    }
  }
  if (!sharded_) {
    phase("ids_allgather", sm);
    vsi_device(vsi_, gids, n_global_, d_uniq_, d_vid_, d_scalars_ + 0, sm, /*reset=*/false);
    phase("vsi", sm);
  }
  // ---- Host-Manager: MixCache per lane (Algorithm 1 l.4-7). The unique and
  // owned counts stay on the device (grids cover the batch-size bound), so the
  // step waits on the host only once, after the probe.
  for (int l = 0; l < lanes_ && !sharded_; ++l)
    lane_[l].select_owned(d_uniq_, d_scalars_ + 0, cap, Wu, static_cast<uint32_t>(lane0_ + l),
                          l == 0 && !vsi_.hashed32 ? vsi_.d_first : nullptr, sm);
  {
    LaneCounters lc{};
    GatePtrs gp{};
    for (int l = 0; l < lanes_; ++l) {
      lc.c[l] = lane_[l].counters;
      gp.own_slot[l] = lane_[l].own_slot;
    }
    // one block: the common case reads the flag and exits
    launch_pdl(bad_id_gate_kernel, dim3(1), dim3(256), 0, sm, d_scalars_ + 1, d_scalars_ + 0, lc, lanes_,
                                          d_vid_, sharded_ ? 0 : n_global_, gp);
    CUDA_LAUNCH_CHECK();
  }
  // window batches t+1..t+L-1 (needed_soon), one at a time through the window scratch
  const int nwin = cfg_.lookahead_depth - 1;
  for (int j = 0; j < nwin; ++j) {
    const uint64_t* wfeat = d_window + static_cast<size_t>(j) * n_local_;
    ids_to_u32(wfeat, d_ids32_, n_local_, cfg_.vocabulary_size, d_scalars_ + 1, sm);
    const uint32_t* wg = d_ids32_;
    if (world_ > 1) {
      NCCL_CHECK(ncclAllGather(d_ids32_, d_gids_, static_cast<size_t>(n_local_), ncclUint32, mcomm_, sm));
      NCCL_CHECK(ncclAllReduce(d_scalars_ + 1, d_scalars_ + 1, 1, ncclInt32, ncclMax, mcomm_, sm));
      wg = d_gids_;
    }
    vsi_device(vsi_, wg, n_global_, d_wuniq_, d_wvid_, d_scalars_ + 2, sm);
    for (int l = 0; l < lanes_; ++l)
      lane_[l].mark_window(d_wuniq_, d_scalars_ + 2, cap, Wu, static_cast<uint32_t>(lane0_ + l), t,
                           sm);
  }
  for (int l = 0; l < lanes_; ++l) lane_[l].probe(d_uniq_, cap, Wu, t, sm);
  phase("manage_probe", sm);
  // Host wait: needed for evictions (the LRU victim count), the capacity check and the
  // NCCL / exchange sizes. A step whose admissions provably fit the free slots
  // (free_lb_ >= the per-step admission bound umax) skips it when nothing else needs host
  // counts: one process, or the owner-routed exchange over peer stores (its layout is
  // derived on the device). Every kernel below reads the unique / owned / working counts
  // and the exchange plan from the device. In pipelined mode the wait is on the manager
  // stream only: the previous step keeps training meanwhile.
  const int64_t bound = lane_[0].umax;
  const bool xdev = a2a_ && xch_.device_driven();
  bool free_step = (world_ == 1 || xdev) && !no_free_steps_;
  // A lane whose cache holds its whole owned shard (C >= owned rows) can never run out of
  // slots: every admission is a non-resident owned row, so no step needs the host check
  for (int l = 0; l < lanes_ && free_step; ++l)
    free_step = lane_[l].C >= lane_[l].rows || free_lb_[l] >= bound;
  if (a2a_) {  // exchange plan (touched masks, send/receive positions), device only
    if (!sharded_) {  // (the sharded stage built it with the ids)
      xch_.plan(d_vid_, n_global_, static_cast<int64_t>(b_) * F_, d_uniq_, d_scalars_ + 0,
                lane_[0].own_k, lane_[0].counters + kCntOwned, sm, mhook);
      launch_pdl(bad_id_gate_plan_kernel, dim3(1), dim3(1), 0, sm, d_scalars_ + 1, xch_.lpos);
      CUDA_LAUNCH_CHECK();
    }
    if (!free_step)
      CUDA_CHECK(cudaMemcpyAsync(h_totals_, xch_.totals, sizeof(int32_t) * Exchange::kTotals,
                                 cudaMemcpyDeviceToHost, sm));
    phase("exchange_plan", sm);
  }
  int32_t U = 0;
  std::vector<int32_t> n_own(lanes_, static_cast<int32_t>(bound)), n_work(lanes_, 0);
  if (!free_step) {
    CUDA_CHECK(cudaMemcpyAsync(h_scalars_, d_scalars_, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, sm));
    for (int l = 0; l < lanes_; ++l)
      CUDA_CHECK(cudaMemcpyAsync(h_counts_ + kCntWords * l, lane_[l].counters,
                                 sizeof(int32_t) * kCntWords, cudaMemcpyDeviceToHost, sm));
    CUDA_CHECK(cudaStreamSynchronize(sm));
    U = h_scalars_[0];
    if (h_scalars_[1]) raise_bad_id(step);
    stats_.unique = U;
    for (int l = 0; l < lanes_; ++l) {
      CacheLane& L = lane_[l];
      const int32_t* hc = h_counts_ + kCntWords * l;
      n_own[l] = hc[kCntOwned];
      L.free_top = hc[kCntFreeTop];
      std::memcpy(&L.next_seq, hc + kCntSeq, sizeof(uint64_t));
      L.host.hi = static_cast<uint64_t>(hc[kCntHostNext]);  // host slots handed out so far
    }
    // capacity check before any state moves (push_parameters_to_cache deadlock)
    for (int l = 0; l < lanes_; ++l) {
      const int32_t* hc = h_counts_ + kCntWords * l;
      n_work[l] = n_own[l] > 0 ? hc[kCntWorking] : 0;
      const CacheLane& L = lane_[l];
      const int64_t occupied = static_cast<int64_t>(L.C) - L.free_top;
      const int64_t marked = hc[kCntMarked];
      const int64_t evictable = occupied - marked;
      if (n_work[l] > L.free_top + evictable)
        fail(kRun,
             "capacity deadlock on worker " + std::to_string(lane0_ + l) + ": need " +
                 std::to_string(n_work[l]) + " slots, " + std::to_string(L.free_top + evictable) +
                 " free or evictable (capacity=" + std::to_string(L.C) +
                 " occupied=" + std::to_string(occupied) + " free=" + std::to_string(L.free_top) +
                 " pinned=0 needed_soon=" + std::to_string(marked) + ")",
             step);
    }
    // Pipelined eviction safety (pinned => not evictable): step t-1 may
    // still be training on its rows (last_use == t-1). The sequential-mode victims are the
    // n_evict smallest (last_use, admit_seq) keys; when at least n_evict eligible slots
    // are older than t-1 those victims are all among them and eviction overlaps step t-1.
    // Otherwise the manager waits for step t-1 to finish first. Either way the victims,
    // and so every result, equal sequential mode's.
    bool selected = false;
    if (piped && train_pending_[k ^ 1]) {
      bool any = false;
      for (int l = 0; l < lanes_; ++l)
        if (n_work[l] > lane_[l].free_top) {
          lane_[l].victim_select(t, n_work[l] - lane_[l].free_top, sm);
          CUDA_CHECK(cudaMemcpyAsync(h_counts_ + kCntWords * l + kCntOld,
                                     lane_[l].counters + kCntOld, sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, sm));
          any = true;
        }
      if (any) {
        CUDA_CHECK(cudaStreamSynchronize(sm));
        selected = true;
        bool wait = false;
        for (int l = 0; l < lanes_; ++l)
          wait |= n_work[l] - lane_[l].free_top > h_counts_[kCntWords * l + kCntOld];
        if (wait) {
          CUDA_CHECK(cudaStreamWaitEvent(sm, train_done_[k ^ 1]));
          stats_.pinned_waits += 1;
        }
      }
    }
    std::pair<Trainer*, cudaStream_t> hook_ctx{this, sm};
    for (int l = 0; l < lanes_; ++l) {
      CacheLane& L = lane_[l];
      const int32_t n_evict = std::max<int32_t>(0, n_work[l] - L.free_top);
      L.evict_admit(n_evict, n_work[l], Wu, cfg_.seed, t, sm, selected && n_evict > 0,
                    PhaseHook{[](void* c, const char* nm) {
                                auto* h = static_cast<std::pair<Trainer*, cudaStream_t>*>(c);
                                h->first->phase(nm, h->second);
                              },
                              &hook_ctx});
      free_lb_[l] = static_cast<int64_t>(L.free_top) + n_evict - n_work[l];
      led_[0] += static_cast<int64_t>(n_work[l]) * d_ * 12;
      led_[1] += static_cast<int64_t>(n_evict) * d_ * 12;
      led_[3] += n_evict;
      stats_.owned += n_own[l];
      stats_.working += n_work[l];
      stats_.evicted += n_evict;
      stats_.pcie_d2h_bytes += static_cast<int64_t>(n_evict) * (3 * d_ + 1) * 4;
    }
  } else {
    for (int l = 0; l < lanes_; ++l) {
      lane_[l].admit(static_cast<int32_t>(bound), 0, Wu, cfg_.seed, t, sm);
      free_lb_[l] -= bound;
    }
  }
  {
    SnapArgs sa{};
    sa.U = d_scalars_ + 0;
    for (int l = 0; l < lanes_; ++l) sa.cnt[l] = lane_[l].counters;
    sa.lanes = lanes_;
    sa.out = snap;
    launch_pdl(snap_kernel, dim3(1), dim3(1 + kCntWords * 8), 0, sm, sa);
    CUDA_LAUNCH_CHECK();
  }
  // Clear this step's gradient table (its parity set) here, off the training stage's path:
  // one worker clears dG[0 : U) / B, the owner-routed exchange its local rows.
  if (early_clear_direct())
    zero_rows_b(snap + 1 + kCntOwned, static_cast<int32_t>(bound), d_, d_dG_, d_B_, sm);
  else if (xdev)
    xch_.zero_local_dev(d_dG_, sm, d_ % 4 == 0 && !tower_fused_ ? d_B_ : nullptr);
  phase("manage_evict_admit", sm);
  {  // experiment: SFCTR_MGR_EXTRA=k empty kernels on the manager stream (boundary cost)
    static const int extra = [] {
      const char* e = std::getenv("SFCTR_MGR_EXTRA");
      return e ? std::atoi(e) : 0;
    }();
    static const bool extra_pdl = std::getenv("SFCTR_MGR_EXTRA_PDL") != nullptr;
    for (int q = 0; q < extra; ++q) {
      if (extra_pdl) launch_pdl(empty_kernel, dim3(1), dim3(32), 0, sm);
      else empty_kernel<<<1, 32, 0, sm>>>();
    }
  }
  stamp(step, 1, sm);
  if (sm != sw) {
    CUDA_CHECK(cudaEventRecord(prep_done_[k], sm));
    prep_recorded_[k] = true;
  }
  prep_.step = step;
  prep_.k = k;
  prep_.sm = sm;
  prep_.free_step = free_step;
  prep_.xdev = xdev;
  prep_.U = U;
  prep_.n_own = n_own;
  prep_.launches0 = launches0;
}

// GPU-Worker stage of the prepared step t (Algorithm 1 l.9-14; gather_cache ...
// update_sparse), enqueued on the training stream behind its manager stage.
void Trainer::train(int64_t step, const uint8_t* d_labels, float* d_loss) {
  CUDA_CHECK(cudaSetDevice(dev_));
  if (prep_.step != step)
    fail(kLogic, "train(" + std::to_string(step) + ") without prepare(" + std::to_string(step) + ")");
  const int64_t launches0 = prep_.launches0;
  const int32_t t = static_cast<int32_t>(step);
  const int k = prep_.k;
  cudaStream_t sm = prep_.sm, sw = stream_;
  const bool free_step = prep_.free_step, xdev = prep_.xdev;
  const int32_t U = prep_.U;
  const std::vector<int32_t> n_own = prep_.n_own;
  prep_n_own0_ = n_own[0];
  prep_k_ = k;
  int32_t* snap = d_snap_[k];
  auto snap_cnt = [&](int l) { return snap + 1 + kCntWords * l; };
  prep_.step = -1;
  if (sm != sw) CUDA_CHECK(cudaStreamWaitEvent(sw, prep_done_[k]));
  stamp(step, 2, sw);
  (void)t;

  // ==== training stage (stream sw) ====
  cudaStream_t s = sw;
  // ---- GPU-Worker forward (Algorithm 1 l.9-11)
  const size_t ud = static_cast<size_t>(U) * d_;
  // rows of the table the lanes gather from: all U uniques (all-reduce scheme) or
  // only the ones this rank touches (owner-routed all-to-all)
  size_t table_rows = free_step ? static_cast<size_t>(n_global_) : static_cast<size_t>(U);
  // one worker: gather_cache writes every one of the U rows, so it zeroes dG as it goes
  const bool zero_in_gather = W_ == 1 && !a2a_ && d_ % 4 == 0;
  // one worker also defers segment_sum's -scale*gz*G term to sparse_adam (which reads the
  // same G row as emb[slot]): the scatter pass then does not re-gather G per position
  // (the owner-routed exchange over peer stores defers it too: the push to the owner and the
  // owner's reduction add it per local row, see FmDefer in exchange.cu)
  const bool defer_fm = (zero_in_gather || (xdev && d_ % 4 == 0)) && !tower_fused_ && !det_;
  // ... and the segment sum then runs inside the tower's dX GEMM epilogue (dX never hits HBM)
  const bool fuse_scatter = defer_fm && !tower_simt_ && H_ <= 64 && dx_scatter_fits(F_, d_);
  // ... and the forward reads the cache rows in place (own_k is the identity at W = 1, so
  // unique k's row is emb[own_slot[k]]): G is never materialised
  const bool direct_emb = defer_fm && zero_in_gather;
  // owner-routed: positions index the local table through lpos (no lvid pass); with the
  // sharded manager stage through the owners' replies (row = rows(k)[index(k)[i]])
  const bool remap_local = a2a_ && fuse_scatter && d_ % 4 == 0;
  if (a2a_) {
    if (!free_step) {
      xch_.set_counts(h_totals_);
      for (int w = 0; w < W_; ++w)  // rows this rank pushes / receives, both directions
        if (w != rank_) stats_.nvlink_bytes += (h_totals_[8 + w] + h_totals_[w]) * 4ll * d_;
    }
    if (xdev)
      xch_.forward_dev(lane_[0].own_k, lane_[0].own_slot, n_own[0], snap_cnt(0) + kCntOwned,
                       lane_[0].emb, s);
    else
      xch_.forward(lane_[0].own_k, lane_[0].own_slot, n_own[0], lane_[0].emb, d_G_, comm_, s,
                   /*barrier=*/false);
    phase("exchange_embed", s);
    if (xch_.p2p) xch_.barrier(comm_, s);
    phase("exchange_barrier", s);
    table_rows = free_step ? static_cast<size_t>(n_global_) : static_cast<size_t>(xch_.local_rows());
    // with the fused scatter the forward gather and the dX epilogue look the local row up
    // themselves (vid -> lpos[vid]); otherwise the local row of every position is materialised
    if (!remap_local && sharded_)
      xch_.local_vids(shard_.index(k), n_local_, d_lvid_, s, shard_.rows(k));
    else if (!remap_local)
      xch_.local_vids(d_vid_ + static_cast<size_t>(lane0_) * b_ * F_, n_local_, d_lvid_, s);
  } else {
    if (world_ > 1) CUDA_CHECK(cudaMemsetAsync(d_G_, 0, sizeof(float) * ud, s));
    // one worker: no G copy (gather_instances reads the cache rows through own_slot) and
    // dG / B were cleared by the manager stage
    if (!direct_emb) {
      for (int l = 0; l < lanes_; ++l)
        gather_cache(lane_[l].own_k, lane_[l].own_slot, n_own[l], snap_cnt(l) + kCntOwned,
                     lane_[l].emb, d_, d_G_, zero_in_gather ? d_dG_ : nullptr, s,
                     zero_in_gather ? d_B_ : nullptr);
      phase("gather_cache", s);
    }
    if (world_ > 1) {
      NCCL_CHECK(ncclAllReduce(d_G_, d_G_, ud, ncclFloat32, ncclSum, comm_, s));
      stats_.nvlink_bytes += static_cast<int64_t>(ud) * 4;
    }
    if (world_ > 1) phase("allreduce_embed", s);
  }
  // interworker ledger: the reference's accounting model, allreduce_bytes per
  // worker for each all-reduce, whatever the device scheme
  auto arb = [&](int64_t payload) { return 2 * static_cast<int64_t>(W_ - 1) * payload / W_; };
  if (!free_step) led_[2] += static_cast<int64_t>(lanes_) * arb(static_cast<int64_t>(ud) * 4);

  // ---- per lane: gather_instances, forward_backward, segment_sum (l.11-12)
  if (zero_in_gather) {
  } else if (xdev) {  // cleared by the manager stage
  } else if (free_step && d_ % 4 == 0)
    zero_rows_kernel<<<num_sms() * 8, 256, 0, s>>>(reinterpret_cast<float4*>(d_dG_), snap + 0,
                                             d_ / 4, n_global_ * (d_ / 4));
  else
    CUDA_CHECK(cudaMemsetAsync(d_dG_, 0, sizeof(float) * table_rows * d_, s));
  const float emb_scale = 1.f / static_cast<float>(W_);
  // Row update overlapped with dW1: once the dX GEMM has scattered every embedding gradient
  // (fused scatter, one lane), the row update only needs those gradients, so it runs on
  // ustream_ while GEMM3 and its reduction run here; the tail waits for it.
  const bool fork_update = fuse_scatter && !timing_ && !no_update_fork_ && lanes_ == 1 &&
                           !tower_fused_ && !tower_simt_ && (world_ == 1 || xdev);
  if (fork_update) ensure_bias_tables(steps_done_ + 2);  // may synchronise: before the fork
  struct ForkCtx {
    Trainer* tr;
    cudaStream_t s;
    int k;
    bool defer_fm;
    float scale;
  } fork_ctx{this, s, k, defer_fm, emb_scale};
  const PhaseHook after_dx =
      fork_update ? PhaseHook{[](void* c, const char*) {
                                auto* f = static_cast<ForkCtx*>(c);
                                Trainer* t = f->tr;
                                CUDA_CHECK(cudaEventRecord(t->dx_done_, f->s));
                                CUDA_CHECK(cudaStreamWaitEvent(t->ustream_, t->dx_done_));
                                t->launch_row_update(t->ustream_, f->k, t->a2a_, f->defer_fm,
                                                     f->scale, t->d_dG_);
                                CUDA_CHECK(cudaEventRecord(t->upd_done_, t->ustream_));
                              },
                              &fork_ctx}
                  : PhaseHook{};
  for (int l = 0; l < lanes_; ++l) {
    const uint32_t* vid = a2a_ && !remap_local ? d_lvid_
                          : sharded_            ? shard_.index(k)
                                                : d_vid_ + static_cast<size_t>(lane0_ + l) * b_ * F_;
    const uint32_t* remap = !remap_local ? nullptr : sharded_ ? shard_.rows(k) : xch_.lpos;
    const uint8_t* lab = d_labels + static_cast<size_t>(l) * b_;
    if (tower_fused_) {  // gather -> GEMM -> scatter-add, X / dX never materialised
      tower_forward_backward_fused(tower_, towertc_, d_G_, static_cast<int64_t>(table_rows), vid,
                                   lab, b_, F_, d_, d_dense_,
                                   d_logits_ + static_cast<size_t>(l) * b_, d_fm_s_, emb_scale,
                                   d_dG_, d_grads_, l > 0, s);
      phase("tower_fused", s);
      continue;
    }
    gather_instances(vid, b_, F_, d_, ldx_, direct_emb ? lane_[0].emb : d_G_, d_X_, d_fm_s_,
                     d_fm_sqp_, s, direct_emb ? lane_[0].own_slot : remap,
                     direct_emb ? 3 * d_ : d_);  // cache rows are [emb | m | v]
    phase("gather_instances", s);
    const DxScatter sc{vid, remap, d_fm_s_, tower_.gz, d_dG_, d_B_, F_, d_};
    if (tower_simt_)
      tower_forward_backward_simt(tower_, d_X_, d_fm_s_, d_fm_sqp_, lab, b_, F_, d_, d_dense_,
                                  d_logits_ + static_cast<size_t>(l) * b_, d_dX_, emb_scale,
                                  d_grads_, l > 0, s);
    else
      tower_forward_backward_tc(tower_, towertc_, d_X_, ldx_, d_fm_s_, d_fm_sqp_, lab, b_, F_, d_,
                                d_dense_, d_logits_ + static_cast<size_t>(l) * b_, d_dX_,
                                emb_scale, d_grads_, l > 0, s, w1_split_ready_,
                                PhaseHook{[](void* c, const char* n) {
                                             static_cast<Trainer*>(c)->phase(n);
                                           },
                                           this},
                                fuse_scatter ? &sc : nullptr, after_dx);
    phase(tower_simt_ ? "tower" : "tower_reduce", s);
    if (det_) {  // fixed-order (CSR) segment sum: bit-identical run to run
      int bits = 1;
      while (bits < 32 && (1ll << bits) < n_global_) ++bits;
      segment_sum_csr(csr_, vid, b_ * F_, F_, d_, ldx_, d_dX_, d_G_, d_fm_s_, tower_.gz, emb_scale,
                      d_dG_, bits, s);
      phase("segment_sum", s);
    } else if (!fuse_scatter) {
      segment_sum(vid, b_ * F_, F_, d_, ldx_, d_dX_, d_G_, d_fm_s_, tower_.gz, emb_scale, d_dG_, s,
                  defer_fm ? d_B_ : nullptr);
      phase("segment_sum", s);
    }
  }

  // ---- grad_synchronize (l.13)
  // The dense gradients are final here: with the flag-barrier exchange (no other NCCL call
  // on comm_ in this stage) their all-reduce runs on a side stream, overlapping the
  // embedding-gradient exchange; the tail waits for it.
  const bool dense_side = world_ > 1 && xdev && !xch_.nccl_barrier && !timing_;
  if (dense_side) {
    CUDA_CHECK(cudaEventRecord(dense_ready_, s));
    CUDA_CHECK(cudaStreamWaitEvent(dstream_, dense_ready_));
    NCCL_CHECK(ncclAllReduce(d_grads_, d_grads_, P_ + 1, ncclFloat32, ncclSum, comm_, dstream_));
    CUDA_CHECK(cudaEventRecord(dense_done_, dstream_));
    stats_.nvlink_bytes += static_cast<int64_t>(P_ + 1) * 4;
  }
  const float* grad_rows = d_dG_;
  bool fused_adam = false;  // owner reduction + sparse Adam fused (owner-routed, peer stores)
  if (fork_update) {
    // the row update is on ustream_ (push + barrier + owner reduction + Adam at W > 1)
  } else if (a2a_) {
    const bool xfm = xdev && defer_fm;
    if (xdev)
      xch_.backward_send_dev(d_dG_, s, xfm ? d_G_ : nullptr, xfm ? d_B_ : nullptr, emb_scale);
    else
      xch_.backward_send(d_dG_, comm_, s);
    phase("exchange_grad_send", s);
    if (xch_.p2p) xch_.barrier(comm_, s);
    phase("exchange_grad_barrier", s);
    if (xdev)  // reduce + update_sparse in one pass (the dense all-reduce goes first)
      fused_adam = true;
    else
      xch_.backward_reduce(lane_[0].own_k, n_own[0], d_dG_, s);
    grad_rows = xch_.gown;
  } else if (world_ > 1) {
    NCCL_CHECK(ncclAllReduce(d_dG_, d_dG_, ud, ncclFloat32, ncclSum, comm_, s));
    stats_.nvlink_bytes += static_cast<int64_t>(ud) * 4;
  }
  if (world_ > 1 && !dense_side) {
    NCCL_CHECK(ncclAllReduce(d_grads_, d_grads_, P_ + 1, ncclFloat32, ncclSum, comm_, s));
    stats_.nvlink_bytes += static_cast<int64_t>(P_ + 1) * 4;
  }
  if (!free_step)
    led_[2] += static_cast<int64_t>(lanes_) *
               (arb(static_cast<int64_t>(ud) * 4) + arb(static_cast<int64_t>(P_) * 4));
  if (world_ > 1) phase(a2a_ ? "exchange_grad" : "allreduce_grad", s);

  // ---- update_sparse (l.14) + dense Adam
  ensure_bias_tables(steps_done_ + 2);
  if (fork_update) {
    CUDA_CHECK(cudaStreamWaitEvent(s, upd_done_));
  } else if (fused_adam) {
    const bool xfm = defer_fm;
    Exchange::AdamRows ar{lane_[0].emb, lane_[0].mom, lane_[0].vel, lane_[0].own_slot,
                          lane_[0].steps, d_bc1_, d_bc2_,
                          static_cast<float>(cfg_.learning_rate),
                          static_cast<float>(cfg_.adam_beta1), static_cast<float>(cfg_.adam_beta2),
                          static_cast<float>(1.0 - cfg_.adam_beta1),
                          static_cast<float>(1.0 - cfg_.adam_beta2),
                          static_cast<float>(cfg_.adam_epsilon)};
    xch_.backward_reduce_adam_dev(lane_[0].own_k, n_own[0], snap_cnt(0) + kCntOwned, d_dG_, s,
                                  xfm ? d_B_ : nullptr, emb_scale, ar);
  }
  for (int l = 0; l < lanes_ && !fused_adam && !fork_update; ++l)
    sparse_adam(a2a_ ? nullptr : lane_[l].own_k, lane_[l].own_slot, n_own[l],
                snap_cnt(l) + kCntOwned, grad_rows, d_,
                lane_[l].emb,
                lane_[l].mom, lane_[l].vel, lane_[l].steps, d_bc1_, d_bc2_,
                static_cast<float>(cfg_.learning_rate), static_cast<float>(cfg_.adam_beta1),
                static_cast<float>(cfg_.adam_beta2), static_cast<float>(cfg_.adam_epsilon), s,
                /*inc_steps=*/false, defer_fm && !a2a_ ? d_B_ : nullptr, emb_scale);
  phase("sparse_adam", s);
  if (dense_side) CUDA_CHECK(cudaStreamWaitEvent(s, dense_done_));
  dense_steps_ += 1;
  const double bc1 = 1.0 - std::pow(cfg_.adam_beta1, static_cast<double>(dense_steps_));
  const double bc2 = 1.0 - std::pow(cfg_.adam_beta2, static_cast<double>(dense_steps_));
  {
    TailArgs a{};
    a.p = d_dense_;
    a.m = d_dense_m_;
    a.v = d_dense_v_;
    a.g = d_grads_;
    a.n = static_cast<int64_t>(P_);
    a.gs = 1.f / static_cast<float>(W_);
    a.lr = static_cast<float>(cfg_.learning_rate);
    a.b1 = static_cast<float>(cfg_.adam_beta1);
    a.b2 = static_cast<float>(cfg_.adam_beta2);
    a.omb1 = static_cast<float>(1.0 - cfg_.adam_beta1);
    a.omb2 = static_cast<float>(1.0 - cfg_.adam_beta2);
    a.eps = static_cast<float>(cfg_.adam_epsilon);
    a.bc1 = static_cast<float>(bc1);
    a.bc2 = static_cast<float>(bc2);
    a.loss_sum = d_grads_ + P_;
    a.inv_w = 1.f / static_cast<float>(W_);
    a.loss_out = d_loss ? d_loss : d_loss_set_[k];
    a.lanes = lanes_;
    for (int l = 0; l < lanes_; ++l) {
      a.own_slot[l] = lane_[l].own_slot;
      a.n_own[l] = snap_cnt(l) + kCntOwned;
      a.steps[l] = lane_[l].steps;
      a.cnt.c[l] = snap_cnt(l);
    }
    if (!tower_fused_ && !tower_simt_) {
      a.w_hi = towertc_.w_hi;
      a.w_lo = towertc_.w_lo;
      a.wt_hi = towertc_.wt_hi;
      a.wt_lo = towertc_.wt_lo;
      a.K = K_;
      a.H = H_;
      a.ldh = towertc_.ldh;
      a.ldk = towertc_.ldk;
    }
    a.acc = free_step ? d_acc_ : nullptr;
    a.xtotals = xdev ? xch_.totals : nullptr;
    a.me = rank_;
    a.U = snap + 0;
    a.W = W_;
    a.d = d_;
    a.P = static_cast<int64_t>(P_);
    a.bad = d_scalars_ + 1;
    a.gated = d_err_ + 1;
    launch_pdl(tail_kernel, dim3(num_sms() * 8), dim3(256), 0, s, a);  // one pass over the dense parameters and the rows
    CUDA_LAUNCH_CHECK();
    w1_split_ready_ = a.w_hi != nullptr;
  }
  phase("dense_adam", s);
  stamp(step, 3, s);
  if (pipelined_) {
    CUDA_CHECK(cudaEventRecord(train_done_[k], sw));
    train_pending_[k] = true;
  }
  if (free_step) {
    acc_pending_ = true;
    free_steps_ += 1;
  }
  last_step_free_ = free_step;
  steps_done_ += 1;
  stats_.kernel_launches = g_launches - launches0;
  stats_.total_steps += 1;
  if (!free_step) {  // free steps fold their device totals in at the next refresh()
    stats_.total_working += stats_.working;
    stats_.total_unique += stats_.unique;
    stats_.total_owned += stats_.owned;
  }
  stats_.total_evicted += stats_.evicted;
  stats_.total_nvlink_bytes += stats_.nvlink_bytes;
  stats_.total_kernel_launches += stats_.kernel_launches;
  stats_.total_pinned_waits += stats_.pinned_waits;
}

// The row update of one lane (W = 1: sparse Adam over the scattered gradients; owner-routed
// peer stores: push the partial gradient rows to their owners, flag barrier, fused owner
// reduction + Adam) on stream us.
void Trainer::launch_row_update(cudaStream_t us, int k, bool a2a, bool defer_fm, float emb_scale,
                                const float* grad_rows) {
  (void)k;
  const int32_t n_bound = prep_n_own0_;
  const int32_t* n_own_dev = d_snap_[prep_k_] + 1 + kCntOwned;
  if (a2a) {
    xch_.backward_send_dev(d_dG_, us, defer_fm ? d_G_ : nullptr, defer_fm ? d_B_ : nullptr,
                           emb_scale);
    xch_.barrier(comm_, us);
    Exchange::AdamRows ar{lane_[0].emb, lane_[0].mom, lane_[0].vel, lane_[0].own_slot,
                          lane_[0].steps, d_bc1_, d_bc2_,
                          static_cast<float>(cfg_.learning_rate),
                          static_cast<float>(cfg_.adam_beta1), static_cast<float>(cfg_.adam_beta2),
                          static_cast<float>(1.0 - cfg_.adam_beta1),
                          static_cast<float>(1.0 - cfg_.adam_beta2),
                          static_cast<float>(cfg_.adam_epsilon)};
    xch_.backward_reduce_adam_dev(lane_[0].own_k, n_bound, n_own_dev, d_dG_, us,
                                  defer_fm ? d_B_ : nullptr, emb_scale, ar);
    return;
  }
  sparse_adam(lane_[0].own_k, lane_[0].own_slot, n_bound, n_own_dev, grad_rows, d_, lane_[0].emb,
              lane_[0].mom, lane_[0].vel, lane_[0].steps, d_bc1_, d_bc2_,
              static_cast<float>(cfg_.learning_rate), static_cast<float>(cfg_.adam_beta1),
              static_cast<float>(cfg_.adam_beta2), static_cast<float>(cfg_.adam_epsilon), us,
              /*inc_steps=*/false, defer_fm ? d_B_ : nullptr, emb_scale);
}

void Trainer::step_device(int64_t step, const uint64_t* d_features, const uint8_t* d_labels,
                          const uint64_t* d_window, float* d_loss) {
  prepare(step, d_features, d_window);
  train(step, d_labels, d_loss);
}

// Folds the deferred device counters in: capacity errors flagged by kernels
// and the number of admissions that read a row back from the host table
// (cumulative on the device; the delta covers every step since the last call).
void Trainer::raise_bad_id(int64_t step) {
  sync_all();
  int32_t gated = 0;
  CUDA_CHECK(cudaMemcpy(&gated, d_err_ + 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemset(d_err_ + 1, 0, sizeof(int32_t)));
  CUDA_CHECK(cudaMemset(d_scalars_ + 1, 0, sizeof(int32_t)));
  dense_steps_ -= gated;  // the gated steps did not update the dense parameters
  fail(kLogic, "feature id >= vocabulary size in the batch (no state was changed)", step);
}

void Trainer::check_device_errors(int64_t step) {
  int32_t err[2] = {0, 0};
  CUDA_CHECK(cudaMemcpy(err, d_err_, sizeof(err), cudaMemcpyDeviceToHost));
  if (err[0])
    fail(kRun, "a peer rank did not arrive at an NVLink barrier within SFCTR_BARRIER_TIMEOUT_S (" +
                   std::to_string(barrier_timeout_ns() / 1000000000ull) + " s)",
         step);
  int32_t bad = 0;
  CUDA_CHECK(cudaMemcpy(&bad, d_scalars_ + 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (bad) raise_bad_id(step);
  int64_t cum = 0;
  for (int l = 0; l < lanes_; ++l) {
    int32_t c[kCntWords];
    CUDA_CHECK(cudaMemcpy(c, lane_[l].counters, sizeof(c), cudaMemcpyDeviceToHost));
    if (c[kCntError]) {
      const auto& L = lane_[l];
      fail(kRun,
           "capacity deadlock: fewer evictable slots than the working set needs (capacity=" +
               std::to_string(L.C) + " free=" + std::to_string(L.free_top) + ")",
           step);
    }
    cum += c[kCntFromHost];
  }
  const int64_t delta = cum - from_host_seen_;
  from_host_seen_ = cum;
  stats_.filled_from_host = delta;
  stats_.total_filled_from_host += delta;
  stats_.pcie_h2d_bytes = delta * (3 * d_ + 1) * 4;
}

void Trainer::submit_host(int64_t step, const uint64_t* features, const uint8_t* labels,
                          const uint64_t* window) {
  CUDA_CHECK(cudaSetDevice(dev_));
  const int k = static_cast<int>(step & 1);
  const int q = static_cast<int>(step % kLossRing);  // loss slot
  if (loss_step_[q] >= 0 && loss_step_[q] != step)
    fail(kLogic, "read the loss of step " + std::to_string(loss_step_[q]) +
                     " (loss_of) before submitting step " + std::to_string(step));
  // Staging set k was last read by step t-2: its ids / window by t-2's manager stage, its
  // labels by t-2's training stage. Pipelined: the copies run on their own stream as soon as
  // those readers are done (the ids usually long before step t-2 finishes training), and the
  // manager stage of step t waits for them. Otherwise they go on the manager's stream.
  const bool piped = pipelined_ && !timing_;
  cudaStream_t cs = piped ? cstream_ : stream_;
  if (piped && prep_recorded_[k]) CUDA_CHECK(cudaStreamWaitEvent(cs, prep_done_[k]));
  CUDA_CHECK(cudaMemcpyAsync(d_in_feat_set_[k], features, sizeof(uint64_t) * n_local_,
                             cudaMemcpyHostToDevice, cs));
  if (window && cfg_.lookahead_depth > 1)
    CUDA_CHECK(cudaMemcpyAsync(d_in_win_set_[k], window,
                               sizeof(uint64_t) * n_local_ * (cfg_.lookahead_depth - 1),
                               cudaMemcpyHostToDevice, cs));
  if (piped && train_pending_[k]) CUDA_CHECK(cudaStreamWaitEvent(cs, train_done_[k]));
  CUDA_CHECK(cudaMemcpyAsync(d_in_lab_set_[k], labels, static_cast<size_t>(lanes_) * b_,
                             cudaMemcpyHostToDevice, cs));
  if (piped) {
    CUDA_CHECK(cudaEventRecord(in_ready_[k], cs));
    input_wait_ = true;
  }
  step_device(step, d_in_feat_set_[k], d_in_lab_set_[k], window ? d_in_win_set_[k] : nullptr,
              d_loss_ring_ + q);  // the tail kernel writes the host slot (mapped memory)
  CUDA_CHECK(cudaEventRecord(loss_ev_[q], stream_));
  loss_step_[q] = step;
}

double Trainer::loss_of(int64_t step) {
  CUDA_CHECK(cudaSetDevice(dev_));
  const int q = static_cast<int>(step % kLossRing);
  if (loss_step_[q] != step)
    fail(kLogic, "no outstanding step " + std::to_string(step) + " (submit it first)");
  CUDA_CHECK(cudaEventSynchronize(loss_ev_[q]));
  loss_step_[q] = -1;
  check_device_errors(step);
  return static_cast<double>(h_loss_ring_[q]);
}

double Trainer::step_host(int64_t step, const uint64_t* features, const uint8_t* labels,
                          const uint64_t* window) {
  submit_host(step, features, labels, window);
  const double l = loss_of(step);
  refresh();
  finish_phases();
  return l;
}

void Trainer::refresh() {
  CUDA_CHECK(cudaSetDevice(dev_));
  sync_all();
  if (acc_pending_) {
    CUDA_CHECK(cudaMemcpy(h_acc_, d_acc_, sizeof(int64_t) * 8, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemset(d_acc_, 0, sizeof(int64_t) * 8));
    stats_.total_unique += h_acc_[0];
    stats_.total_owned += h_acc_[1];
    stats_.total_working += h_acc_[2];
    led_[0] += h_acc_[2] * d_ * 12;
    led_[2] += h_acc_[3];
    stats_.total_nvlink_bytes += h_acc_[4];
    acc_pending_ = false;
  }
  for (int l = 0; l < lanes_; ++l) {
    int32_t c[kCntWords];
    CUDA_CHECK(cudaMemcpy(c, lane_[l].counters, sizeof(c), cudaMemcpyDeviceToHost));
    lane_[l].free_top = c[kCntFreeTop];
    std::memcpy(&lane_[l].next_seq, c + kCntSeq, sizeof(uint64_t));
    free_lb_[l] = lane_[l].free_top;
    if (last_step_free_) {  // per-step counters of the last step, read back now
      if (l == 0) {
        int32_t U = 0;
        CUDA_CHECK(cudaMemcpy(&U, d_scalars_, sizeof(int32_t), cudaMemcpyDeviceToHost));
        stats_.unique = U;
        stats_.owned = stats_.working = 0;
      }
      stats_.owned += c[kCntOwned];
      stats_.working += c[kCntWorking];
    }
  }
}

sfctr_step_stats Trainer::stats() {
  refresh();
  stats_.total_free_steps = free_steps_;
  return stats_;
}

uint64_t Trainer::free_count(int lane) {
  refresh();
  return static_cast<uint64_t>(lane_.at(lane).free_top);
}

void Trainer::synchronize() {
  CUDA_CHECK(cudaSetDevice(dev_));
  sync_all();
  check_device_errors(steps_done_ - 1);
  refresh();
  finish_phases();
}

void Trainer::logits(float* out) {
  sync_all();
  CUDA_CHECK(cudaMemcpy(out, d_logits_, sizeof(float) * lanes_ * b_, cudaMemcpyDeviceToHost));
}

void Trainer::cache_slots(int lane, uint64_t* feature, int64_t* last_use, uint64_t* admit_seq,
                          uint64_t first, uint64_t count) {
  sync_all();
  const CacheLane& L = lane_.at(lane);
  if (first > L.C) first = L.C;
  if (count > L.C - first) count = L.C - first;
  std::vector<uint32_t> f(count);
  std::vector<int32_t> lu(count);
  CUDA_CHECK(cudaMemcpy(f.data(), L.slot_feat + first, sizeof(uint32_t) * count,
                        cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemcpy(lu.data(), L.last_use + first, sizeof(int32_t) * count,
                        cudaMemcpyDeviceToHost));
  if (admit_seq)
    CUDA_CHECK(cudaMemcpy(admit_seq, L.admit_seq + first, sizeof(uint64_t) * count,
                          cudaMemcpyDeviceToHost));
  for (uint64_t i = 0; i < count; ++i) {
    if (feature) feature[i] = f[i] == kEmpty ? ~0ull : f[i];
    if (last_use) last_use[i] = lu[i];
  }
}

namespace {
__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint64_t* __restrict__ idx,
                                  int64_t n, uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}
// rows [n x 3d] and step counts of cache slots `slots` (one warp per row)
__global__ void gather_slot_rows_kernel(const uint32_t* __restrict__ slots, int64_t n, int d3,
                                        const float* __restrict__ emb,
                                        const int32_t* __restrict__ steps, float* __restrict__ rows,
                                        int32_t* __restrict__ out_steps) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint32_t s = slots[w];
  for (int c = lane; c < d3; c += 32) rows[w * d3 + c] = emb[static_cast<size_t>(s) * d3 + c];
  if (lane == 0) out_steps[w] = steps[s];
}
}  // namespace

// Current state of owned rows wherever they live (cache slot or host pool): the index
// entries of the rows are gathered on the device, cache rows by a gather kernel (never a
// copy of the whole cache), host rows straight from the pinned slabs. kNever rows are
// reported through `never` (nullptr: a LogicError, as HostStore::peek of an absent row).
void Trainer::read_rows(int lane, const uint64_t* rows_idx, int64_t n, float* rows, int64_t* steps,
                        bool* never) {
  const CacheLane& L = lane_.at(lane);
  const int d3 = 3 * d_;
  if (n <= 0) return;
  uint64_t* d_idx = nullptr;
  uint32_t* d_where = nullptr;
  CUDA_CHECK(cudaMalloc(&d_idx, sizeof(uint64_t) * n));
  CUDA_CHECK(cudaMalloc(&d_where, sizeof(uint32_t) * n));
  std::vector<uint32_t> where(n);
  CUDA_CHECK(cudaMemcpy(d_idx, rows_idx, sizeof(uint64_t) * n, cudaMemcpyHostToDevice));
  gather_u32_kernel<<<ceil_div(n, 256), 256>>>(L.index, d_idx, n, d_where);
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpy(where.data(), d_where, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> slots;
  std::vector<int64_t> pos;
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t w = where[i];
    if (never) never[i] = w == kNever;
    if (w == kNever) {
      if (!never)
        fail(kLogic, "row " + std::to_string(rows_idx[i] * W_ + lane0_ + lane) +
                         " was never touched (HostStore::peek of an absent feature)");
      if (rows) std::memset(rows + i * d3, 0, sizeof(float) * d3);
      if (steps) steps[i] = 0;
    } else if (on_host(w)) {
      const uint32_t h = w & ~kHostBit;
      if (rows) std::memcpy(rows + i * d3, L.host.row_host(h), sizeof(float) * d3);
      if (steps) steps[i] = L.host.step_host(h);
    } else {
      slots.push_back(w);
      pos.push_back(i);
    }
  }
  if (!slots.empty()) {
    const int64_t m = static_cast<int64_t>(slots.size());
    uint32_t* d_slots = nullptr;
    float* d_rows = nullptr;
    int32_t* d_st = nullptr;
    CUDA_CHECK(cudaMalloc(&d_slots, sizeof(uint32_t) * m));
    CUDA_CHECK(cudaMalloc(&d_rows, sizeof(float) * m * d3));
    CUDA_CHECK(cudaMalloc(&d_st, sizeof(int32_t) * m));
    CUDA_CHECK(cudaMemcpy(d_slots, slots.data(), sizeof(uint32_t) * m, cudaMemcpyHostToDevice));
    gather_slot_rows_kernel<<<ceil_div(m * 32, 256), 256>>>(d_slots, m, d3, L.emb, L.steps, d_rows,
                                                            d_st);
    CUDA_LAUNCH_CHECK();
    std::vector<float> hr(static_cast<size_t>(m) * d3);
    std::vector<int32_t> hs(m);
    CUDA_CHECK(cudaMemcpy(hr.data(), d_rows, sizeof(float) * m * d3, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(hs.data(), d_st, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    for (int64_t q = 0; q < m; ++q) {
      if (rows) std::memcpy(rows + pos[q] * d3, hr.data() + q * d3, sizeof(float) * d3);
      if (steps) steps[pos[q]] = hs[q];
    }
    cudaFree(d_slots);
    cudaFree(d_rows);
    cudaFree(d_st);
  }
  cudaFree(d_idx);
  cudaFree(d_where);
}

void Trainer::peek_rows(int64_t n, const uint64_t* features, float* rows, int64_t* steps) {
  sync_all();
  std::vector<std::vector<uint64_t>> idx(lanes_);
  std::vector<std::vector<int64_t>> at(lanes_);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t f = features[i];
    if (f >= cfg_.vocabulary_size) fail(kLogic, "feature id >= vocabulary size");
    const int l = static_cast<int>(f % W_) - lane0_;
    if (l < 0 || l >= lanes_)
      fail(kLogic, "feature " + std::to_string(f) + " is owned by worker " +
                       std::to_string(f % W_) + ", not by this process");
    idx[l].push_back(f / W_);
    at[l].push_back(i);
  }
  const int d3 = 3 * d_;
  for (int l = 0; l < lanes_; ++l) {
    const int64_t m = static_cast<int64_t>(idx[l].size());
    if (!m) continue;
    std::vector<float> r(rows ? static_cast<size_t>(m) * d3 : 0);
    std::vector<int64_t> st(m);
    read_rows(l, idx[l].data(), m, rows ? r.data() : nullptr, st.data(), nullptr);
    for (int64_t q = 0; q < m; ++q) {
      if (rows) std::memcpy(rows + at[l][q] * d3, r.data() + q * d3, sizeof(float) * d3);
      if (steps) steps[at[l][q]] = st[q];
    }
  }
}

int64_t Trainer::snapshot(uint64_t* features, float* rows, int64_t* steps) {
  sync_all();
  // every touched owned row (index entry != kNever), sorted by feature
  std::vector<std::pair<uint64_t, std::pair<int, uint64_t>>> all;  // feature -> (lane, row)
  for (int l = 0; l < lanes_; ++l) {
    const CacheLane& L = lane_[l];
    std::vector<uint32_t> idx(L.rows);
    CUDA_CHECK(cudaMemcpy(idx.data(), L.index, sizeof(uint32_t) * L.rows, cudaMemcpyDeviceToHost));
    for (uint64_t r = 0; r < L.rows; ++r)
      if (idx[r] != kNever) all.push_back({r * W_ + (lane0_ + l), {l, r}});
  }
  std::sort(all.begin(), all.end());
  if (!features) return static_cast<int64_t>(all.size());
  const int d3 = 3 * d_;
  for (size_t i = 0; i < all.size(); ++i) features[i] = all[i].first;
  if (rows || steps) {
    std::vector<std::vector<uint64_t>> idx(lanes_);
    std::vector<std::vector<int64_t>> at(lanes_);
    for (size_t i = 0; i < all.size(); ++i) {
      idx[all[i].second.first].push_back(all[i].second.second);
      at[all[i].second.first].push_back(static_cast<int64_t>(i));
    }
    for (int l = 0; l < lanes_; ++l) {
      const int64_t m = static_cast<int64_t>(idx[l].size());
      if (!m) continue;
      std::vector<float> r(rows ? static_cast<size_t>(m) * d3 : 0);
      std::vector<int64_t> st(m);
      read_rows(l, idx[l].data(), m, rows ? r.data() : nullptr, st.data(), nullptr);
      for (int64_t q = 0; q < m; ++q) {
        if (rows) std::memcpy(rows + at[l][q] * d3, r.data() + q * d3, sizeof(float) * d3);
        if (steps) steps[at[l][q]] = st[q];
      }
    }
  }
  return static_cast<int64_t>(all.size());
}

void Trainer::dense_state(float* p, float* m, float* v, int64_t* step) {
  sync_all();
  if (p) CUDA_CHECK(cudaMemcpy(p, d_dense_, sizeof(float) * P_, cudaMemcpyDeviceToHost));
  if (m) CUDA_CHECK(cudaMemcpy(m, d_dense_m_, sizeof(float) * P_, cudaMemcpyDeviceToHost));
  if (v) CUDA_CHECK(cudaMemcpy(v, d_dense_v_, sizeof(float) * P_, cudaMemcpyDeviceToHost));
  if (step) *step = dense_steps_;
}

void Trainer::get_dense(float* w1, float* b1, float* w2, float* b2) {
  sync_all();
  const size_t kh = static_cast<size_t>(K_) * H_;
  if (w1) CUDA_CHECK(cudaMemcpy(w1, d_dense_, sizeof(float) * kh, cudaMemcpyDeviceToHost));
  if (b1) CUDA_CHECK(cudaMemcpy(b1, d_dense_ + kh, sizeof(float) * H_, cudaMemcpyDeviceToHost));
  if (w2) CUDA_CHECK(cudaMemcpy(w2, d_dense_ + kh + H_, sizeof(float) * H_, cudaMemcpyDeviceToHost));
  if (b2) CUDA_CHECK(cudaMemcpy(b2, d_dense_ + kh + 2 * H_, sizeof(float), cudaMemcpyDeviceToHost));
}

void Trainer::set_dense(const float* w1, const float* b1, const float* w2, const float* b2) {
  sync_all();
  w1_split_ready_ = false;
  const size_t kh = static_cast<size_t>(K_) * H_;
  if (w1) CUDA_CHECK(cudaMemcpy(d_dense_, w1, sizeof(float) * kh, cudaMemcpyHostToDevice));
  if (b1) CUDA_CHECK(cudaMemcpy(d_dense_ + kh, b1, sizeof(float) * H_, cudaMemcpyHostToDevice));
  if (w2) CUDA_CHECK(cudaMemcpy(d_dense_ + kh + H_, w2, sizeof(float) * H_, cudaMemcpyHostToDevice));
  if (b2) CUDA_CHECK(cudaMemcpy(d_dense_ + kh + 2 * H_, b2, sizeof(float), cudaMemcpyHostToDevice));
}

void Trainer::ledger(int64_t out[4]) {
  refresh();
  for (int i = 0; i < 4; ++i) out[i] = led_[i];
}

}  // namespace sfb
