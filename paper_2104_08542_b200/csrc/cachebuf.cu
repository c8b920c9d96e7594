// The standalone device CacheBuffer (cache_buffer.hpp:40-86 / cache_buffer.cpp) with its
// HostStore (host_store.hpp:61-92) and the MixCache manager step, for
// callers that drive the cache themselves (sfctr_cache_* in include/sfctr_b200.h). Same
// device structures as the trainer's lanes (CacheLane): HBM slot rows [emb | m | v], the
// LIFO free stack, the owned-row index, the lazy pinned host pool, the LRU selection.
//
// Flags: pinned is a per-slot byte; needed_soon is mark[s] == epoch_, the step of the last
// manager step (prepare() recomputes needed_soon from the lookahead window, as the manager
// does), so set_needed_soon / admit stamp the current epoch. Batched operations follow
// the reference's one-at-a-time semantics: they apply in list order and stop at the first
// feature the reference would throw on (LogicError after the preceding ones took effect).
#include "cachebuf.h"

#include <algorithm>
#include <cstring>
#include <unordered_set>

namespace sfb {

namespace {

__global__ void stamp_kernel(const uint32_t* __restrict__ slots, int32_t n, int32_t* mark,
                             int32_t epoch, uint8_t* __restrict__ pinned) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  mark[slots[i]] = epoch;  // CacheBuffer::admit: needed_soon = true, pinned = false
  pinned[slots[i]] = 0;
}

// mode 0 touch(step), 1 pin(on), 2 needed_soon(on)
__global__ void flag_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                            const uint32_t* __restrict__ index, int mode, int32_t arg,
                            int32_t epoch, int32_t* __restrict__ last_use,
                            uint8_t* __restrict__ pinned, int32_t* __restrict__ mark) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = index[static_cast<uint32_t>(feats[i]) / W];
  if (mode == 0) {
    if (arg > last_use[s]) last_use[s] = arg;  // cache_buffer.cpp:69-72
  } else if (mode == 1) {
    pinned[s] = arg ? 1 : 0;
  } else {
    if (arg) mark[s] = epoch;
    else if (mark[s] == epoch) mark[s] = -1;
  }
}

__global__ void slot_of_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                               const uint32_t* __restrict__ index, uint32_t C,
                               int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = index[static_cast<uint32_t>(feats[i]) / W];
  out[i] = s < C ? static_cast<int64_t>(s) : -1;
}

// occupied, pinned, needed_soon over the occupied slots
__global__ void occupancy_kernel(uint32_t C, const uint32_t* __restrict__ slot_feat,
                                 const uint8_t* __restrict__ pinned,
                                 const int32_t* __restrict__ mark, int32_t epoch,
                                 unsigned long long* __restrict__ out) {
  unsigned long long o = 0, p = 0, nd = 0;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < C; s += gridDim.x * blockDim.x) {
    if (slot_feat[s] == kEmpty) continue;
    ++o;
    p += pinned[s] ? 1 : 0;
    nd += mark[s] == epoch ? 1 : 0;
  }
  for (int off = 16; off > 0; off >>= 1) {
    o += __shfl_xor_sync(0xFFFFFFFFu, o, off);
    p += __shfl_xor_sync(0xFFFFFFFFu, p, off);
    nd += __shfl_xor_sync(0xFFFFFFFFu, nd, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (o) atomicAdd(out + 0, o);
    if (p) atomicAdd(out + 1, p);
    if (nd) atomicAdd(out + 2, nd);
  }
}

__global__ void gather_rows_kernel(const uint64_t* __restrict__ feats, int32_t n, uint32_t W,
                                   const uint32_t* __restrict__ index, uint32_t C, int d3,
                                   const float* __restrict__ emb, const int32_t* __restrict__ steps,
                                   HostTab host, float* __restrict__ rows,
                                   int32_t* __restrict__ out_steps,
                                   unsigned long long* __restrict__ err) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint32_t where = index[static_cast<uint32_t>(feats[w]) / W];
  if (where == kNever) {
    if (lane == 0) atomicMin(err, (static_cast<unsigned long long>(w) << 8) | 5);
    return;
  }
  const float* src;
  int32_t st;
  if (where < C) {
    src = emb + static_cast<size_t>(where) * d3;
    st = steps[where];
  } else {
    src = host.row(where & ~kHostBit, d3);
    st = *host.step(where & ~kHostBit);
  }
  for (int c = lane; c < d3; c += 32) rows[w * d3 + c] = src[c];
  if (lane == 0) out_steps[w] = st;
}

}  // namespace

DeviceCache::DeviceCache(uint64_t capacity, int dim, uint64_t seed, uint64_t key_space,
                         int num_workers, int worker, int64_t max_batch, uint64_t host_reserve,
                         int device)
    : W_(num_workers), w_(worker), d_(dim), dev_(device), seed_(seed), key_space_(key_space),
      max_batch_(max_batch) {
  if (capacity == 0) fail(kLogic, "cache buffer needs at least one slot");  // cache_buffer.cpp:24
  if (capacity >= 0x7FFFFFF0ull) fail(kConfig, "capacity must fit 31-bit slots");
  if (dim <= 0) fail(kConfig, "dim must be positive");
  if (num_workers <= 0 || worker < 0 || worker >= num_workers)
    fail(kConfig, "worker must be in [0, num_workers)");
  if (key_space == 0 || key_space >= 0xFFFFFFF0ull)
    fail(kConfig, "key_space must be in (0, 2^32 - 16)");
  if (max_batch <= 0 || max_batch >= (1ll << 31)) fail(kConfig, "max_batch must be positive");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(kCuda, "no CUDA device available (the device path has no CPU fallback)");
  }
  CUDA_CHECK(cudaSetDevice(device));
  CUDA_CHECK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
  const uint64_t rows = (key_space + W_ - 1) / W_;
  L_.init(capacity, dim, rows, host_reserve, max_batch);
  L_.use(0);
  CUDA_CHECK(cudaMalloc(&pinned_, L_.C));
  CUDA_CHECK(cudaMemset(pinned_, 0, L_.C));
  CUDA_CHECK(cudaMalloc(&d_feats_, sizeof(uint64_t) * max_batch));
  CUDA_CHECK(cudaMalloc(&d_ids32_, sizeof(uint32_t) * max_batch));
  CUDA_CHECK(cudaMalloc(&d_win32_, sizeof(uint32_t) * max_batch));
  CUDA_CHECK(cudaMalloc(&d_scal_, sizeof(int32_t) * 4));
  CUDA_CHECK(cudaMemset(d_scal_, 0, sizeof(int32_t) * 4));
  CUDA_CHECK(cudaMalloc(&d_err_, sizeof(unsigned long long)));
  CUDA_CHECK(cudaMalloc(&d_occ_, sizeof(unsigned long long) * 4));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_cnt_), sizeof(int32_t) * kCntWords, 0));
  CUDA_CHECK(cudaDeviceSynchronize());
}

DeviceCache::~DeviceCache() {
  cudaSetDevice(dev_);
  if (s_) cudaStreamSynchronize(s_);
  L_.release();
  for (void* p : {static_cast<void*>(pinned_), static_cast<void*>(d_feats_),
                  static_cast<void*>(d_ids32_), static_cast<void*>(d_win32_),
                  static_cast<void*>(d_scal_), static_cast<void*>(d_err_),
                  static_cast<void*>(d_occ_)})
    if (p) cudaFree(p);
  if (h_cnt_) cudaFreeHost(h_cnt_);
  if (s_) cudaStreamDestroy(s_);
}

// features -> d_feats_ (host-validated: < key_space, owned by this worker)
void DeviceCache::to_device(int64_t n, const uint64_t* features, bool owned_check) {
  if (n > max_batch_)
    fail(kLogic, "batch of " + std::to_string(n) + " ids exceeds max_batch " +
                     std::to_string(max_batch_));
  for (int64_t i = 0; i < n && owned_check; ++i) {
    if (features[i] >= key_space_)
      fail(kLogic, "feature " + std::to_string(features[i]) + " >= key_space");
    if (features[i] % W_ != static_cast<uint64_t>(w_))
      fail(kLogic, "feature " + std::to_string(features[i]) + " is owned by worker " +
                       std::to_string(features[i] % W_) + ", not " + std::to_string(w_));
  }
  if (n > 0)
    CUDA_CHECK(cudaMemcpyAsync(d_feats_, features, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s_));
}

void DeviceCache::refresh_counters() {
  CUDA_CHECK(cudaMemcpyAsync(h_cnt_, L_.counters, sizeof(int32_t) * kCntWords,
                             cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  L_.free_top = h_cnt_[kCntFreeTop];
  std::memcpy(&L_.next_seq, h_cnt_ + kCntSeq, sizeof(uint64_t));
  L_.host.hi = static_cast<uint64_t>(h_cnt_[kCntHostNext]);
  if (h_cnt_[kCntError]) fail(kRun, "capacity deadlock in the device cache: " + occupancy_diagnostics());
}

namespace {
// first position of a repeated feature (the reference's second op on it throws), or n
int64_t first_repeat(int64_t n, const uint64_t* f) {
  std::unordered_set<uint64_t> seen;
  for (int64_t i = 0; i < n; ++i)
    if (!seen.insert(f[i]).second) return i;
  return n;
}
const char* err_text(int code) {
  switch (code) {
    case 1: return "already resident";
    case 2: return "not resident";
    case 3: return "pinned";
    case 4: return "inside the lookahead window";
    default: return "without state";
  }
}
}  // namespace

void DeviceCache::admit(int64_t n, const uint64_t* features, int64_t step, uint64_t* slots_out) {
  CUDA_CHECK(cudaSetDevice(dev_));
  refresh_counters();
  to_device(n, features, true);
  // the prefix the reference admits before it throws: a repeat, a resident feature, or
  // the first admission with no free slot left
  int64_t stop = first_repeat(n, features);
  CUDA_CHECK(cudaMemsetAsync(d_err_, 0xFF, sizeof(unsigned long long), s_));
  L_.check_list(d_feats_, static_cast<int32_t>(n), W_, pinned_, epoch_, 0, d_err_, s_);
  unsigned long long err = ~0ull;
  CUDA_CHECK(cudaMemcpyAsync(&err, d_err_, sizeof(err), cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  int code = 1;
  if (err != ~0ull && static_cast<int64_t>(err >> 8) < stop) stop = static_cast<int64_t>(err >> 8);
  std::string why;
  if (stop < n) why = "feature " + std::to_string(features[stop]) + " already resident";
  if (stop > L_.free_top) {
    stop = L_.free_top;
    why = "admit with no free slot; evict first";
    code = 0;
  }
  (void)code;
  if (step > max_step_) max_step_ = step;
  const int32_t t = static_cast<int32_t>(step);
  L_.admit_list(d_feats_, static_cast<int32_t>(stop), W_, seed_, t, s_);
  // admitted: needed_soon (mark = epoch), unpinned; own_slot[j] = slot of position j
  if (stop > 0) {
    stamp_kernel<<<ceil_div(stop, 256), 256, 0, s_>>>(L_.own_slot, static_cast<int32_t>(stop),
                                                      L_.mark, epoch_, pinned_);
    CUDA_LAUNCH_CHECK();
    if (slots_out) {
      std::vector<uint32_t> sl(stop);
      CUDA_CHECK(cudaMemcpyAsync(sl.data(), L_.own_slot, sizeof(uint32_t) * stop,
                                 cudaMemcpyDeviceToHost, s_));
      CUDA_CHECK(cudaStreamSynchronize(s_));
      for (int64_t i = 0; i < stop; ++i) slots_out[i] = sl[i];
    }
  }
  refresh_counters();
  if (stop < n) fail(kLogic, why);
}

void DeviceCache::evict(int64_t n, const uint64_t* features) {
  CUDA_CHECK(cudaSetDevice(dev_));
  refresh_counters();
  to_device(n, features, true);
  int64_t stop = first_repeat(n, features);
  int code = 2;  // a repeat is a non-resident feature by then
  CUDA_CHECK(cudaMemsetAsync(d_err_, 0xFF, sizeof(unsigned long long), s_));
  L_.check_list(d_feats_, static_cast<int32_t>(n), W_, pinned_, epoch_, 2, d_err_, s_);
  unsigned long long err = ~0ull;
  CUDA_CHECK(cudaMemcpyAsync(&err, d_err_, sizeof(err), cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  if (err != ~0ull && static_cast<int64_t>(err >> 8) <= stop) {
    stop = static_cast<int64_t>(err >> 8);
    code = static_cast<int>(err & 0xFF);
  }
  L_.evict_list(d_feats_, static_cast<int32_t>(stop), W_, s_);
  refresh_counters();
  if (stop < n) {  // cache_buffer.cpp:57-60 messages
    const std::string f = std::to_string(features[stop]);
    if (code == 2) fail(kLogic, "evicting non-resident feature " + f);
    if (code == 3) fail(kLogic, "evicting pinned feature " + f);
    fail(kLogic, "evicting feature " + f + " inside the lookahead window");
  }
}

namespace {
void flag_op(CacheLane& L, cudaStream_t s, const uint64_t* d_feats, int64_t n, uint32_t W,
             int mode, int32_t arg, int32_t epoch, uint8_t* pinned) {
  if (n <= 0) return;
  flag_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_feats, static_cast<int32_t>(n), W, L.index, mode,
                                               arg, epoch, L.last_use, pinned, L.mark);
  CUDA_LAUNCH_CHECK();
}
}  // namespace

// touch / pin / set_needed_soon: slot_of() throws for a non-resident feature
// (cache_buffer.cpp:31-35), after the preceding ones took effect
#define SFB_RESIDENT_PREFIX(MODE, ARG)                                                     \
  CUDA_CHECK(cudaSetDevice(dev_));                                                         \
  to_device(n, features, true);                                                            \
  CUDA_CHECK(cudaMemsetAsync(d_err_, 0xFF, sizeof(unsigned long long), s_));               \
  L_.check_list(d_feats_, static_cast<int32_t>(n), W_, pinned_, epoch_, 1, d_err_, s_);    \
  unsigned long long err = ~0ull;                                                          \
  CUDA_CHECK(cudaMemcpyAsync(&err, d_err_, sizeof(err), cudaMemcpyDeviceToHost, s_));      \
  CUDA_CHECK(cudaStreamSynchronize(s_));                                                   \
  const int64_t stop = err == ~0ull ? n : static_cast<int64_t>(err >> 8);                  \
  flag_op(L_, s_, d_feats_, stop, W_, MODE, ARG, epoch_, pinned_);                         \
  CUDA_CHECK(cudaStreamSynchronize(s_));                                                   \
  if (stop < n) fail(kLogic, "feature " + std::to_string(features[stop]) + " not resident");

void DeviceCache::touch(int64_t n, const uint64_t* features, int64_t step) {
  if (step > max_step_) max_step_ = step;
  SFB_RESIDENT_PREFIX(0, static_cast<int32_t>(step))
}
void DeviceCache::pin(int64_t n, const uint64_t* features, bool on) {
  SFB_RESIDENT_PREFIX(1, on ? 1 : 0)
}
void DeviceCache::set_needed_soon(int64_t n, const uint64_t* features, bool on) {
  SFB_RESIDENT_PREFIX(2, on ? 1 : 0)
}
#undef SFB_RESIDENT_PREFIX

void DeviceCache::slot_of(int64_t n, const uint64_t* features, int64_t* out) {
  CUDA_CHECK(cudaSetDevice(dev_));
  to_device(n, features, true);
  if (n <= 0) return;
  int64_t* d_out = nullptr;
  CUDA_CHECK(cudaMalloc(&d_out, sizeof(int64_t) * n));
  slot_of_kernel<<<ceil_div(n, 256), 256, 0, s_>>>(d_feats_, static_cast<int32_t>(n), W_, L_.index,
                                                   static_cast<uint32_t>(L_.C), d_out);
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(out, d_out, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  cudaFree(d_out);
}

uint64_t DeviceCache::free_count() {
  CUDA_CHECK(cudaSetDevice(dev_));
  refresh_counters();
  return static_cast<uint64_t>(L_.free_top);
}

void DeviceCache::slots(uint64_t* feature, int64_t* last_use, uint64_t* admit_seq,
                        uint8_t* pinned, uint8_t* needed_soon) {
  CUDA_CHECK(cudaSetDevice(dev_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  const uint64_t C = L_.C;
  std::vector<uint32_t> f(C);
  std::vector<int32_t> lu(C), mk(C);
  CUDA_CHECK(cudaMemcpy(f.data(), L_.slot_feat, sizeof(uint32_t) * C, cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemcpy(lu.data(), L_.last_use, sizeof(int32_t) * C, cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemcpy(mk.data(), L_.mark, sizeof(int32_t) * C, cudaMemcpyDeviceToHost));
  if (admit_seq)
    CUDA_CHECK(cudaMemcpy(admit_seq, L_.admit_seq, sizeof(uint64_t) * C, cudaMemcpyDeviceToHost));
  if (pinned) CUDA_CHECK(cudaMemcpy(pinned, pinned_, C, cudaMemcpyDeviceToHost));
  for (uint64_t i = 0; i < C; ++i) {
    const bool occ = f[i] != kEmpty;
    if (feature) feature[i] = occ ? f[i] : ~0ull;
    if (last_use) last_use[i] = lu[i];
    if (needed_soon) needed_soon[i] = occ && mk[i] == epoch_ ? 1 : 0;
    if (pinned && !occ) pinned[i] = 0;
  }
}

void DeviceCache::occupancy(uint64_t out[5]) {
  CUDA_CHECK(cudaSetDevice(dev_));
  CUDA_CHECK(cudaMemsetAsync(d_occ_, 0, sizeof(unsigned long long) * 4, s_));
  occupancy_kernel<<<std::max(1, std::min(ceil_div(static_cast<int64_t>(L_.C), 256), num_sms() * 4)),
                     256, 0, s_>>>(static_cast<uint32_t>(L_.C), L_.slot_feat, pinned_, L_.mark,
                                   epoch_, reinterpret_cast<unsigned long long*>(d_occ_));
  CUDA_LAUNCH_CHECK();
  unsigned long long h[4] = {0, 0, 0, 0};
  CUDA_CHECK(cudaMemcpyAsync(h, d_occ_, sizeof(h), cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  out[0] = L_.C;
  out[1] = h[0];
  out[2] = L_.C - h[0];
  out[3] = h[1];
  out[4] = h[2];
}

std::string DeviceCache::occupancy_diagnostics() {  // cache_buffer.cpp:81-92 format
  uint64_t o[5];
  occupancy(o);
  return "capacity=" + std::to_string(o[0]) + " occupied=" + std::to_string(o[1]) +
         " free=" + std::to_string(o[2]) + " pinned=" + std::to_string(o[3]) +
         " needed_soon=" + std::to_string(o[4]);
}

void DeviceCache::peek(int64_t n, const uint64_t* features, float* rows, int64_t* steps) {
  CUDA_CHECK(cudaSetDevice(dev_));
  to_device(n, features, true);
  if (n <= 0) return;
  const int d3 = 3 * d_;
  float* d_rows = nullptr;
  int32_t* d_st = nullptr;
  CUDA_CHECK(cudaMalloc(&d_rows, sizeof(float) * n * d3));
  CUDA_CHECK(cudaMalloc(&d_st, sizeof(int32_t) * n));
  CUDA_CHECK(cudaMemsetAsync(d_err_, 0xFF, sizeof(unsigned long long), s_));
  gather_rows_kernel<<<ceil_div(n * 32, 256), 256, 0, s_>>>(
      d_feats_, static_cast<int32_t>(n), W_, L_.index, static_cast<uint32_t>(L_.C), d3, L_.emb,
      L_.steps, L_.host.tab(), d_rows, d_st, d_err_);
  CUDA_LAUNCH_CHECK();
  unsigned long long err = ~0ull;
  std::vector<int32_t> st(n);
  CUDA_CHECK(cudaMemcpyAsync(&err, d_err_, sizeof(err), cudaMemcpyDeviceToHost, s_));
  if (rows)
    CUDA_CHECK(cudaMemcpyAsync(rows, d_rows, sizeof(float) * n * d3, cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaMemcpyAsync(st.data(), d_st, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s_));
  CUDA_CHECK(cudaStreamSynchronize(s_));
  cudaFree(d_rows);
  cudaFree(d_st);
  if (err != ~0ull)  // HostStore::peek of an absent feature (host_store.cpp:35-39)
    fail(kLogic, "feature " + std::to_string(features[err >> 8]) + " has no state");
  if (steps)
    for (int64_t i = 0; i < n; ++i) steps[i] = st[i];
}

void DeviceCache::prepare(int64_t step, int64_t n_global, const uint64_t* global_ids,
                          int64_t n_window, const uint64_t* window_ids, int64_t out[5]) {
  CUDA_CHECK(cudaSetDevice(dev_));
  if (step < 0 || step >= (1ll << 23)) fail(kLogic, "step index out of the supported range");
  if (epoch_ >= 0 && step <= epoch_)
    fail(kLogic, "prepare steps must increase (step " + std::to_string(step) + " after " +
                     std::to_string(epoch_) + ")");
  if (step < max_step_) fail(kLogic, "prepare step is older than a touched step");
  for (int64_t i = 0; i < n_global; ++i)
    if (global_ids[i] >= key_space_) fail(kLogic, "feature id >= key_space");
  if (n_global > max_batch_ || n_window > max_batch_) fail(kLogic, "more ids than max_batch");
  refresh_counters();
  const int32_t t = static_cast<int32_t>(step);
  epoch_ = t;  // needed_soon restarts: the window below and the hits / admissions re-stamp it
  max_step_ = step;
  const int32_t ng = static_cast<int32_t>(n_global);
  if (ng > 0) {
    CUDA_CHECK(cudaMemcpyAsync(d_feats_, global_ids, sizeof(uint64_t) * ng, cudaMemcpyHostToDevice,
                               s_));
    ids_to_u32(d_feats_, d_ids32_, ng, key_space_, d_scal_ + 1, s_);
  }
  const int32_t hs[3] = {ng, 0, static_cast<int32_t>(n_window)};
  CUDA_CHECK(cudaMemcpyAsync(d_scal_, hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
  // per-step counters; the free-stack height, admit_seq, host slots and from-host carry over
  CUDA_CHECK(cudaMemsetAsync(L_.counters, 0, sizeof(int32_t) * 2, s_));
  CUDA_CHECK(cudaMemsetAsync(L_.counters + 3, 0, sizeof(int32_t) * 2, s_));
  const int32_t from_host0 = h_cnt_[kCntFromHost];
  const uint32_t Wu = static_cast<uint32_t>(W_), wu = static_cast<uint32_t>(w_);
  const int32_t cap = std::max<int32_t>(1, ng);
  L_.select_owned(d_ids32_, d_scal_ + 0, cap, Wu, wu, nullptr, s_);
  if (n_window > 0) {
    CUDA_CHECK(cudaMemcpyAsync(d_feats_, window_ids, sizeof(uint64_t) * n_window,
                               cudaMemcpyHostToDevice, s_));
    ids_to_u32(d_feats_, d_win32_, n_window, key_space_, d_scal_ + 1, s_);
    L_.mark_window(d_win32_, d_scal_ + 2, static_cast<int32_t>(n_window), Wu, wu, t, s_);
  }
  L_.probe(d_ids32_, cap, Wu, t, s_);
  refresh_counters();
  const int32_t n_own = h_cnt_[kCntOwned];
  const int32_t n_work = n_own > 0 ? h_cnt_[kCntWorking] : 0;
  const int32_t n_evict = std::max<int32_t>(0, n_work - L_.free_top);
  if (n_evict > 0) {  // capacity check before any state moves
    L_.victim_select(t, n_evict, s_, pinned_);
    refresh_counters();
    if (h_cnt_[kCntSelTotal] < n_evict)
      fail(kRun,
           "capacity deadlock on worker " + std::to_string(w_) + ": need " +
               std::to_string(n_work) + " slots, " +
               std::to_string(L_.free_top + h_cnt_[kCntSelTotal]) +
               " free or evictable (" + occupancy_diagnostics() + ")",
           step);
  }
  L_.evict_admit(n_evict, n_work, Wu, seed_, t, s_, n_evict > 0, PhaseHook{}, pinned_);
  refresh_counters();
  if (out) {
    out[0] = n_own;
    out[1] = n_own - n_work;
    out[2] = n_work;
    out[3] = n_evict;
    out[4] = h_cnt_[kCntFromHost] - from_host0;
  }
}

}  // namespace sfb
