// Global-batch id all-gather over NVLink peer stores (the Data-Loader's exchange, Algorithm 1
// l.2-3; PAPER.md:294 fn.: every GPU sees the global batch). One kernel converts this rank's
// u64 ids to u32 (vocabulary range check, criteo/generator ids are < 2^32) and stores them
// straight into every rank's global-batch buffer at offset rank * n, then a flag barrier
// publishes them. It replaces ncclAllGather on the manager stream: a 1.3 MB-per-rank NCCL
// all-gather costs ~45 us at W = 4, mostly protocol latency.
//
// Buffers are double-buffered by step parity: rank A may run step t+1's manager stage while
// rank B still reads step t's global batch; a rank cannot be two steps ahead because every
// training step ends in NVLink barriers.
#include "idgather.h"

namespace sfb {

namespace {

struct PeerIds {
  uint32_t* dst[8];
};

// vec (host-decided): n and off multiples of 4 and `in` 16-byte aligned
__global__ void __launch_bounds__(256) push_ids_kernel(const uint64_t* __restrict__ in, int64_t n,
                                                       uint64_t limit, int32_t* __restrict__ bad,
                                                       PeerIds pd, int W, int64_t off, bool vec) {
  pdl_wait();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (vec) {  // 4 ids per thread: two 16 B loads, one 16 B store per destination
    const int64_t n4 = n >> 2;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n4; q += stride) {
      const ulonglong2 a = reinterpret_cast<const ulonglong2*>(in)[2 * q];
      const ulonglong2 b = reinterpret_cast<const ulonglong2*>(in)[2 * q + 1];
      const bool over = a.x >= limit || a.y >= limit || b.x >= limit || b.y >= limit;
      if (over) *bad = 1;
      const uint4 v = make_uint4(a.x < limit ? static_cast<uint32_t>(a.x) : 0u,
                                 a.y < limit ? static_cast<uint32_t>(a.y) : 0u,
                                 b.x < limit ? static_cast<uint32_t>(b.x) : 0u,
                                 b.y < limit ? static_cast<uint32_t>(b.y) : 0u);
#pragma unroll
      for (int w = 0; w < 8; ++w)  // static peer index: pd stays in the parameter bank
        if (w < W) reinterpret_cast<uint4*>(pd.dst[w] + off)[q] = v;
    }
  } else {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
      const uint64_t a = in[i];
      if (a >= limit) *bad = 1;
      const uint32_t v = a < limit ? static_cast<uint32_t>(a) : 0u;
#pragma unroll
      for (int w = 0; w < 8; ++w)
        if (w < W) pd.dst[w][off + i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

struct PeerFlags {
  uint64_t* peer[8];
};

// The exchange's flag barrier protocol (flag_barrier_wait, common.cuh) on its own flags and
// epochs, with one addition: bit 63 of the published word carries this rank's bad-id flag
// (an id >= vocab in its batch), so every rank leaves the barrier knowing whether ANY rank
// saw one and gates the step the same way (Trainer::prepare: no state moves).
constexpr uint64_t kBadBit = 1ull << 63;
__global__ void id_barrier_kernel(PeerFlags pf, int W, int me, uint64_t epoch, uint64_t timeout_ns,
                                  int32_t* abort_flag, int32_t* bad) {
  pdl_wait();
  const int w = threadIdx.x;
  if (w >= W || w == me) return;
  const uint64_t word = epoch | (*bad ? kBadBit : 0ull);
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pf.peer[w] + me), "l"(word) : "memory");
  const uint64_t* mine = pf.peer[me] + w;
  uint64_t v = 0, t0 = 0, now = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 32;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if ((v & ~kBadBit) >= epoch) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      if (abort_flag) atomicExch(abort_flag, 1);
      return;
    }
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
  if (v & kBadBit) atomicExch(bad, 1);
}

}  // namespace

void IdGather::init(int W_, int me_, int64_t n_) {
  release();
  W = W_;
  me = me_;
  n = n_;
  for (int k = 0; k < 2; ++k) CUDA_CHECK(cudaMalloc(&gids[k], sizeof(uint32_t) * W * n));
}

void IdGather::release() {
  if (p2p)
    for (int w = 0; w < W; ++w) {
      if (w == me) continue;
      for (int k = 0; k < 2; ++k)
        if (peer_gids[k][w]) cudaIpcCloseMemHandle(peer_gids[k][w]);
      if (peer_flags[w]) cudaIpcCloseMemHandle(peer_flags[w]);
    }
  for (void* p : {static_cast<void*>(gids[0]), static_cast<void*>(gids[1]),
                  static_cast<void*>(flags)})
    if (p) cudaFree(p);
  *this = IdGather();
}

bool IdGather::setup_p2p(ncclComm_t comm, cudaStream_t s) {
  // the peer tables hold 8 ranks (one NVSwitch box): larger worlds keep the NCCL
  // all-gather (W is the same on every rank, so all of them return here together)
  if (W > 8) return false;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  int* d_x = nullptr;
  CUDA_CHECK(cudaMalloc(&d_x, sizeof(int) * (W + 1)));
  CUDA_CHECK(cudaMemcpyAsync(d_x + me, &dev, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_x + me, d_x, 1, ncclInt32, comm, s));
  std::vector<int> devs(W);
  CUDA_CHECK(cudaMemcpyAsync(devs.data(), d_x, sizeof(int) * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  int ok = 1;
  for (int w = 0; w < W; ++w) {
    if (w == me) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, devs[w]) != cudaSuccess || !can) ok = 0;
  }
  cudaGetLastError();
  CUDA_CHECK(cudaMemcpyAsync(d_x + W, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllReduce(d_x + W, d_x + W, 1, ncclInt32, ncclMin, comm, s));
  CUDA_CHECK(cudaMemcpyAsync(&ok, d_x + W, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_x);
  if (!ok) return false;
  CUDA_CHECK(cudaMalloc(&flags, sizeof(uint64_t) * 8));
  CUDA_CHECK(cudaMemset(flags, 0, sizeof(uint64_t) * 8));
  cudaIpcMemHandle_t mine[3];
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[0], gids[0]));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[1], gids[1]));
  CUDA_CHECK(cudaIpcGetMemHandle(&mine[2], flags));
  const size_t hb = sizeof(mine);
  uint8_t* d_h = nullptr;
  CUDA_CHECK(cudaMalloc(&d_h, hb * W));
  CUDA_CHECK(cudaMemcpyAsync(d_h + hb * me, mine, hb, cudaMemcpyHostToDevice, s));
  NCCL_CHECK(ncclAllGather(d_h + hb * me, d_h, hb, ncclUint8, comm, s));
  std::vector<cudaIpcMemHandle_t> all(3 * W);
  CUDA_CHECK(cudaMemcpyAsync(all.data(), d_h, hb * W, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(d_h);
  for (int w = 0; w < W; ++w) {
    if (w == me) {
      peer_gids[0][w] = gids[0];
      peer_gids[1][w] = gids[1];
      peer_flags[w] = flags;
      continue;
    }
    void* p[3] = {nullptr, nullptr, nullptr};
    for (int q = 0; q < 3; ++q)
      CUDA_CHECK(cudaIpcOpenMemHandle(&p[q], all[3 * w + q], cudaIpcMemLazyEnablePeerAccess));
    peer_gids[0][w] = static_cast<uint32_t*>(p[0]);
    peer_gids[1][w] = static_cast<uint32_t*>(p[1]);
    peer_flags[w] = static_cast<uint64_t*>(p[2]);
  }
  p2p = true;
  return true;
}

const uint32_t* IdGather::gather(const uint64_t* d_ids, uint64_t limit, int32_t* d_bad, int k,
                                 cudaStream_t s) {
  PeerIds pd{};
  for (int w = 0; w < W; ++w) pd.dst[w] = peer_gids[k][w];
  const bool vec = (n & 3) == 0 && ((static_cast<int64_t>(me) * n) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(d_ids) & 15) == 0;
  const int64_t units = vec ? n / 4 : n;
  launch_pdl(push_ids_kernel, dim3(std::max(1, std::min(ceil_div(units, 256), num_sms() * 2))), dim3(256), 0, s, d_ids, n, limit, d_bad, pd, W, static_cast<int64_t>(me) * n, vec);
  CUDA_LAUNCH_CHECK();
  PeerFlags pf{};
  for (int w = 0; w < W; ++w) pf.peer[w] = peer_flags[w];
  launch_pdl(id_barrier_kernel, dim3(1), dim3(32), 0, s, pf, W, me, ++epoch, barrier_timeout_ns(), abort_flag, d_bad);
  CUDA_LAUNCH_CHECK();
  return gids[k];
}

}  // namespace sfb
