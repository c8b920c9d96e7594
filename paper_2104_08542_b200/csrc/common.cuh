// Shared host/device plumbing for the sm_100a kernels: error types that map
// onto the reference's exception classes (include/sfctr/error.hpp:28-56),
// CUDA/NCCL check macros, and the counter-based RNG of rng.hpp:27-84 in a
// form that is bit-exact on the device.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

namespace sfb {

// Status codes of include/sfctr_b200.h.
enum Status : int { kOk = 0, kConfig = 1, kData = 2, kLogic = 3, kRun = 4, kCuda = 5, kNccl = 6 };

struct Error : std::runtime_error {
  int status;
  int64_t step;
  Error(int s, const std::string& m, int64_t st = -1) : std::runtime_error(m), status(s), step(st) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg, int64_t step = -1) {
  throw Error(status, msg, step);
}

#define SFB_CHECK(cond, msg)                                                              \
  do {                                                                                    \
    if (!(cond))                                                                          \
      ::sfb::fail(::sfb::kLogic, std::string("check failed: ") + #cond + " (" + (msg) + ")"); \
  } while (0)

#define CUDA_CHECK(expr)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      ::sfb::fail(::sfb::kCuda, std::string(#expr) + ": " + cudaGetErrorString(e_) + " at " + \
                                    __FILE__ + ":" + std::to_string(__LINE__));           \
  } while (0)

// kernels launched by this thread (the bench's gpu_launches claim); CUB
// primitives add their own kernel counts at the call site
extern thread_local int64_t g_launches;
#define CUDA_LAUNCH_CHECK()          \
  do {                               \
    ++::sfb::g_launches;             \
    CUDA_CHECK(cudaGetLastError());  \
  } while (0)

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// SM count of the current device (148 on B200), read once per device: grids are sized in
// waves of it rather than a hard-coded count (MIG slices and other parts differ)
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 0;
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// ---------------- rng.hpp:27-56 (host + device) ----------------
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ inline uint64_t splitmix_mix(uint64_t z) {  // rng.hpp:38-41
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t splitmix_next(uint64_t& s) {  // rng.hpp:36-42
  s += kGolden;
  return splitmix_mix(s);
}

inline uint64_t fnv1a64(const char* p, size_t n) {  // rng.hpp:27-34
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<uint8_t>(p[i]);
    h *= 0x100000001b3ull;
  }
  return h;
}
inline uint64_t fnv1a64(const std::string& s) { return fnv1a64(s.data(), s.size()); }

// derive_seed(base, label, index) with fnv1a64(label) precomputed (rng.hpp:49-56).
__host__ __device__ inline uint64_t derive_seed_h(uint64_t base, uint64_t label_hash,
                                                  uint64_t index) {
  uint64_t state = base ^ label_hash;
  state ^= kGolden * (index + 1);
  uint64_t out = splitmix_next(state);
  out = splitmix_next(state) ^ out;
  return out;
}

#ifdef __CUDACC__
// Rng::next_unit (rng.hpp:67): exact in fp64.
__device__ __forceinline__ double unit_from(uint64_t x) {
  return __dmul_rn(static_cast<double>(x >> 11), 0x1.0p-53);
}
// Rng::next_uniform(lo, hi) = lo + (hi - lo) * unit, rounded step by step as
// the host does (no FMA contraction, rng.hpp:70).
__device__ __forceinline__ double uniform_from(uint64_t x, double lo, double hi) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), unit_from(x)));
}
#endif

#ifdef __CUDACC__
// a / b for the flat-index kernels: a 32-bit divide (a few instructions) instead of the
// ~70-instruction 64-bit one whenever the index fits, which it does at every shipped size
__device__ __forceinline__ int64_t idiv(int64_t a, int b) {
  return a <= 0xFFFFFFFFll ? static_cast<int64_t>(static_cast<uint32_t>(a) / static_cast<uint32_t>(b))
                           : a / b;
}
#endif

#ifdef __CUDACC__
// NVLink flag barrier between the W ranks of one box (peer[w] = rank w's flag words, mapped
// over CUDA IPC): rank `me` stores `epoch` into slot me of every peer's words (release,
// system scope) and waits until every peer's store into its own slot has arrived (acquire).
// Spinning backs off with __nanosleep. A peer that does not arrive within timeout_ns (global
// timer) makes the barrier give up and raise *abort_flag instead of trapping: the host
// reports a RunError at its next check, and a peer that is merely slow (host-side work,
// a debugger) no longer takes down every other rank's CUDA context.
__device__ inline void flag_barrier_wait(uint64_t* const* peer, int W, int me, uint64_t epoch,
                                         uint64_t timeout_ns, int32_t* abort_flag) {
  const int w = threadIdx.x;
  if (w >= W || w == me) return;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer[w] + me), "l"(epoch) : "memory");
  const uint64_t* mine = peer[me] + w;
  uint64_t v = 0, t0 = 0, now = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      if (abort_flag) atomicExch(abort_flag, 1);
      break;
    }
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
}
#endif

// Programmatic dependent launch (PDL) between consecutive kernels of the training stream:
// a kernel launched with launch_pdl() may start (prologue: barrier init, TMEM allocation,
// tensor-map prefetch) while its predecessor drains; pdl_wait() blocks until the predecessor
// has completed and its writes are visible, so it must precede every read of the
// predecessor's outputs. pdl_trigger() lets the successor launch before this grid exits.
// Both are no-ops for a kernel launched without the attribute. SFCTR_NO_PDL=1 disables it.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SFCTR_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
#endif

// Grid of a manager-stage kernel (grid-stride loops inside): at most SFCTR_MGR_CTAS_PER_SM
// CTAs per SM when set (default 0 = uncapped). Measured at cfg2 N = 1: a cap of 2 made the
// step slower (25.9 vs 27.5 M samples/s): the capped CTAs live longer and the block
// scheduler packs them onto a subset of SMs, which then cannot take a persistent training
// GEMM CTA. The training GEMMs take their work items dynamically instead (tc_ts.cuh).
inline int mgr_grid(int64_t want) {
  static const int per = [] {
    const char* e = std::getenv("SFCTR_MGR_CTAS_PER_SM");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  const int64_t cap = per > 0 ? static_cast<int64_t>(num_sms()) * per : want;
  return static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
}

// barrier timeout: SFCTR_BARRIER_TIMEOUT_S seconds (default 600)
inline uint64_t barrier_timeout_ns() {
  static const uint64_t ns = [] {
    double s = 600;
    if (const char* e = std::getenv("SFCTR_BARRIER_TIMEOUT_S")) s = std::atof(e);
    if (!(s > 0)) s = 600;
    return static_cast<uint64_t>(s * 1e9);
  }();
  return ns;
}

// Slot / index sentinels of the device MixCache. index[r] of owned row r is a cache slot
// (< kHostBit: capacities stay below 2^31), kNever, or kHostBit | h: the row lives in host
// slot h of the pinned host pool (HostStore, host_store.hpp:61-92).
constexpr uint32_t kEmpty = 0xFFFFFFFFu;     // slot_feature of a free slot
constexpr uint32_t kNever = 0xFFFFFFFFu;     // index[r]: row never touched (lazy init on admit)
constexpr uint32_t kHostBit = 0x80000000u;   // index[r] = kHostBit | host slot
constexpr uint32_t kNoHost = 0xFFFFFFFFu;    // slot_host[s]: the row has no host slot yet
__host__ __device__ inline bool on_host(uint32_t where) {
  return (where & kHostBit) && where != kNever;
}

}  // namespace sfb
