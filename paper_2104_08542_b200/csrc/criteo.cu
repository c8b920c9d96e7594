// Criteo TSV ingest on the device, bit-exact with CriteoReader (core/src/criteo.cpp:27-98):
// lines "label \t 13 numerics \t 26 categorical tokens", '\r' stripped, empty lines
// skipped, exactly 40 tab-separated columns, label "0" or "1", each categorical token
// hashed with 64-bit FNV-1a (rng.hpp:27-34) modulo the vocabulary, an empty token -> 0.
//
// The input streams through two pinned chunk buffers; a line cut by a chunk boundary is
// carried into the next chunk. Three stages overlap: the host reads chunk c+1 while the
// copy stream moves chunk c over PCIe and the compute stream parses chunk c-1. Nothing
// in the loop waits for a device count: per chunk, on the device,
//   1. nl_count:  per 4 KB tile, (lines << 32 | non-empty lines) — a line is empty when
//                 only an optional '\r' precedes its '\n' (a 2-byte look-back)
//   2. scan of the packed tile counts (CUB, u64)
//   3. nl_write:  nlpos[line] = its '\n', rowline[row] = line of every non-empty line
//   4. parse:     one warp per non-empty line (grid-stride over the device row count);
//                 tab positions by warp ballots over 32-byte windows, column-count / label
//                 validation, lanes 0..25 hash one token each; rows land after the previous
//                 chunks' rows (device running base), the smallest malformed line number
//                 is kept with atomicMin
//   5. advance:   running base += this chunk's rows / lines
// The host checks the error word once at the end and formats the reference's DataError
// for that line from the input bytes (criteo.cpp:59-68; message text only).
// The parsed table stays in HBM ([rows x 26] u32 ids + u8 labels) and read_batch gathers
// a (wrapping) global batch from it (criteo.cpp:81-98).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <exception>
#include <fstream>
#include <thread>
#include <vector>

#include "criteo.h"

namespace sfb {

namespace {

constexpr int kTileThreads = 256;
constexpr int kTileBytes = kTileThreads * 16;  // 4 KB of the chunk per block
constexpr unsigned long long kNoError = ~0ull;

__device__ __forceinline__ int nl_in(const uint4 v, uint32_t valid_mask16, uint16_t* bits) {
  // bit b of *bits = byte b of the 16 is '\n' (and inside the chunk)
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (((w[q] >> (8 * b)) & 0xFFu) == '\n') m |= 1u << (4 * q + b);
  m &= valid_mask16;
  *bits = static_cast<uint16_t>(m);
  return __popc(m);
}

__device__ __forceinline__ uint4 load16(const uint8_t* __restrict__ buf, int64_t off, int64_t n,
                                        uint32_t* valid) {
  if (off + 16 <= n) {
    *valid = 0xFFFFu;
    return *reinterpret_cast<const uint4*>(buf + off);
  }
  uint8_t tmp[16];
  uint32_t v = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    tmp[b] = off + b < n ? buf[off + b] : 0;
    if (off + b < n) v |= 1u << b;
  }
  *valid = v;
  uint4 r;
  memcpy(&r, tmp, 16);
  return r;
}

// The line ending at '\n' position p (chunks start at a line start) is empty when nothing
// but an optional '\r' precedes it since the previous '\n' (criteo.cpp:43-44).
__device__ __forceinline__ bool empty_line_at(const uint8_t* __restrict__ buf, int64_t p) {
  if (p == 0) return true;
  const uint8_t b1 = buf[p - 1];
  if (b1 == '\n') return true;
  return b1 == '\r' && (p == 1 || buf[p - 2] == '\n');
}

// lines / non-empty lines among the thread's 16 bytes, packed (lines << 32 | rows)
__device__ __forceinline__ uint64_t thread_counts(const uint8_t* __restrict__ buf, int64_t off,
                                                  int64_t n, uint16_t* bits, uint16_t* keep) {
  *bits = 0;
  *keep = 0;
  if (off >= n) return 0;
  uint32_t valid;
  const int nl = nl_in(load16(buf, off, n, &valid), valid, bits);
  int rows = 0;
  uint16_t b2 = *bits;
  while (b2) {
    const int b = __ffs(b2) - 1;
    b2 &= b2 - 1;
    if (!empty_line_at(buf, off + b)) {
      ++rows;
      *keep |= static_cast<uint16_t>(1u << b);
    }
  }
  return (static_cast<uint64_t>(nl) << 32) | static_cast<uint32_t>(rows);
}

__global__ void __launch_bounds__(kTileThreads) nl_count_kernel(const uint8_t* __restrict__ buf,
                                                                int64_t n,
                                                                uint64_t* __restrict__ tile_cnt) {
  using Reduce = cub::BlockReduce<uint64_t, kTileThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  uint16_t bits, keep;
  const uint64_t c = thread_counts(
      buf, static_cast<int64_t>(blockIdx.x) * kTileBytes + threadIdx.x * 16, n, &bits, &keep);
  const uint64_t tot = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

// nlpos[line] = position of its '\n'; rowline[row] = line of every non-empty line
__global__ void __launch_bounds__(kTileThreads) nl_write_kernel(const uint8_t* __restrict__ buf,
                                                                int64_t n,
                                                                const uint64_t* __restrict__ tile_off,
                                                                uint32_t* __restrict__ nlpos,
                                                                uint32_t* __restrict__ rowline) {
  using Scan = cub::BlockScan<uint64_t, kTileThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t off = static_cast<int64_t>(blockIdx.x) * kTileBytes + threadIdx.x * 16;
  uint16_t bits, keep;
  const uint64_t c = thread_counts(buf, off, n, &bits, &keep);
  uint64_t pre;
  Scan(tmp).ExclusiveSum(c, pre);
  pre += tile_off[blockIdx.x];
  uint32_t line = static_cast<uint32_t>(pre >> 32), row = static_cast<uint32_t>(pre);
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    nlpos[line] = static_cast<uint32_t>(off + b);
    if ((keep >> b) & 1u) rowline[row++] = line;
    ++line;
  }
}

// One warp per non-empty line (grid-stride; the chunk's row count is read on the device).
// base[0] / base[1] = rows / lines of the previous chunks; err = smallest bad line (1-based)
__global__ void __launch_bounds__(256) parse_kernel(
    const uint8_t* __restrict__ buf, const uint32_t* __restrict__ nlpos,
    const uint32_t* __restrict__ rowline, const uint64_t* __restrict__ chunk_tot,
    const uint64_t* __restrict__ base, int64_t cap_rows, uint64_t vocab,
    uint32_t* __restrict__ feat, uint8_t* __restrict__ lab, unsigned long long* __restrict__ err) {
  __shared__ uint32_t tabs[8][40];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nrows = static_cast<uint32_t>(*chunk_tot);
  const uint64_t row0 = base[0], line0 = base[1];
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t j = rowline[r];
    const uint32_t start = j == 0 ? 0u : nlpos[j - 1] + 1;
    uint32_t end = nlpos[j];
    if (buf[end - 1] == '\r') --end;
    uint32_t ntabs = 0;
    for (uint32_t p = start; p < end; p += 32) {
      const uint32_t q = p + lane;
      const bool tab = q < end && buf[q] == '\t';
      const unsigned m = __ballot_sync(0xFFFFFFFFu, tab);
      if (tab) {
        const uint32_t k = ntabs + __popc(m & ((1u << lane) - 1u));
        if (k < 40) tabs[wib][k] = q;
      }
      ntabs += __popc(m);
    }
    __syncwarp();
    // criteo.cpp:59-68: 40 columns, label "0" | "1"
    const bool bad = ntabs != 39 ||
                     !(tabs[wib][0] == start + 1 && (buf[start] == '0' || buf[start] == '1'));
    const uint64_t row = row0 + r;
    if (bad || row >= static_cast<uint64_t>(cap_rows)) {  // (row >= cap implies a bad line)
      if (lane == 0 && bad) atomicMin(err, static_cast<unsigned long long>(line0 + j + 1));
      __syncwarp();
      continue;
    }
    if (lane == 0) lab[row] = buf[start] == '1' ? 1 : 0;
    if (lane < 26) {  // criteo.cpp:69-76
      const uint32_t a = tabs[wib][13 + lane] + 1;
      const uint32_t b = lane == 25 ? end : tabs[wib][14 + lane];
      uint32_t id = 0;
      if (b > a) {
        uint64_t h = 0xcbf29ce484222325ull;  // fnv1a64 (rng.hpp:27-34)
        for (uint32_t i = a; i < b; ++i) {
          h ^= buf[i];
          h *= 0x100000001b3ull;
        }
        id = static_cast<uint32_t>(h % vocab);
      }
      feat[row * 26 + lane] = id;
    }
    __syncwarp();
  }
}

__global__ void advance_base_kernel(const uint64_t* __restrict__ chunk_tot, uint64_t* base) {
  const uint64_t t = *chunk_tot;
  base[0] += static_cast<uint32_t>(t);
  base[1] += t >> 32;
}

__global__ void read_batch_kernel(const uint32_t* __restrict__ feat,
                                  const uint8_t* __restrict__ lab, int64_t total, int64_t first,
                                  int32_t nrows, uint64_t* __restrict__ out_f,
                                  uint8_t* __restrict__ out_l) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(nrows) * 26) return;
  const int64_t r = i / 26, f = i - r * 26;
  const int64_t src = (first + r) % total;  // criteo.cpp:88-96 wrap-around
  out_f[i] = feat[src * 26 + f];
  if (f == 0) out_l[r] = lab[src];
}

// The reference's own message for a malformed line (criteo.cpp:59-68), from its bytes.
std::string line_error(const std::string& name, int64_t lineno, std::string line) {
  if (!line.empty() && line.back() == '\r') line.pop_back();
  size_t cols = 1;
  for (char ch : line) cols += ch == '\t';
  if (cols != 40)
    return name + ":" + std::to_string(lineno) + ": expected 40 tab-separated columns, got " +
           std::to_string(cols);
  return name + ":" + std::to_string(lineno) + ": label must be 0 or 1, got '" +
         line.substr(0, line.find('\t')) + "'";
}

}  // namespace

void CriteoTable::init(uint64_t vocabulary, int fields, int64_t byte_bound, size_t chunk) {
  if (fields != 26)  // criteo.cpp:31-34
    fail(kConfig, "criteo format has 26 categorical fields; fields=" + std::to_string(fields) +
                      " was configured");
  if (vocabulary == 0 || vocabulary >= (1ull << 32))
    fail(kConfig, "criteo ingest needs 0 < vocab < 2^32");
  vocab = vocabulary;
  chunk_bytes = chunk;
  // a data line holds at least 39 tabs + a label + '\n'
  cap_rows = byte_bound / 41 + 2;
  CUDA_CHECK(cudaMalloc(&d_feat, sizeof(uint32_t) * 26 * cap_rows));
  CUDA_CHECK(cudaMalloc(&d_lab, cap_rows));
  const int64_t maxlines = static_cast<int64_t>(chunk) + 2;
  tiles_cap = (static_cast<int64_t>(chunk) + kTileBytes) / kTileBytes + 2;
  for (int k = 0; k < 2; ++k) {
    CUDA_CHECK(cudaMalloc(&d_buf[k], chunk + 16));
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_buf[k]), chunk + 16, 0));
    CUDA_CHECK(cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&parsed[k], cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaMalloc(&d_tile, sizeof(uint64_t) * 2 * tiles_cap));
  CUDA_CHECK(cudaMalloc(&d_nlpos, sizeof(uint32_t) * maxlines));
  CUDA_CHECK(cudaMalloc(&d_rowline, sizeof(uint32_t) * maxlines));
  CUDA_CHECK(cudaMalloc(&d_state, sizeof(uint64_t) * 4));  // base rows, base lines, err
  CUDA_CHECK(cudaMemset(d_state, 0, sizeof(uint64_t) * 2));
  CUDA_CHECK(cudaMemset(d_state + 2, 0xFF, sizeof(uint64_t)));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_state), sizeof(uint64_t) * 4, 0));
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<const uint64_t*>(nullptr),
                                static_cast<uint64_t*>(nullptr), static_cast<int>(tiles_cap));
  CUDA_CHECK(cudaMalloc(&d_scan, scan_bytes));
  CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreate(&ev0));
  CUDA_CHECK(cudaEventCreate(&ev1));
  CUDA_CHECK(cudaDeviceSynchronize());
}

void CriteoTable::release() {
  for (void* p : {static_cast<void*>(d_feat), static_cast<void*>(d_lab),
                  static_cast<void*>(d_buf[0]), static_cast<void*>(d_buf[1]),
                  static_cast<void*>(d_tile), static_cast<void*>(d_nlpos),
                  static_cast<void*>(d_rowline), static_cast<void*>(d_state), d_scan})
    if (p) cudaFree(p);
  for (char* p : {h_buf[0], h_buf[1]})
    if (p) cudaFreeHost(p);
  if (h_state) cudaFreeHost(h_state);
  for (cudaEvent_t e : {ev0, ev1, copied[0], copied[1], parsed[0], parsed[1]})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {stream, copy_stream})
    if (s) cudaStreamDestroy(s);
  *this = CriteoTable();
}

// Enqueues h_buf[k][0, n) (complete lines, the last one '\n'-terminated): H2D on the copy
// stream (after the parse that last read d_buf[k]), parse on the compute stream.
void CriteoTable::enqueue_chunk(int k, size_t n) {
  CUDA_CHECK(cudaStreamWaitEvent(copy_stream, parsed[k]));
  CUDA_CHECK(cudaMemcpyAsync(d_buf[k], h_buf[k], n, cudaMemcpyHostToDevice, copy_stream));
  CUDA_CHECK(cudaEventRecord(copied[k], copy_stream));
  cudaStream_t s = stream;
  CUDA_CHECK(cudaStreamWaitEvent(s, copied[k]));
  const int64_t N = static_cast<int64_t>(n);
  const int tiles = static_cast<int>((N + kTileBytes - 1) / kTileBytes);
  uint64_t* tile_cnt = d_tile;
  uint64_t* tile_off = d_tile + tiles_cap;
  nl_count_kernel<<<tiles + 1, kTileThreads, 0, s>>>(d_buf[k], N, tile_cnt);  // +1: zero sentinel
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, tile_cnt, tile_off, tiles + 1, s));
  nl_write_kernel<<<tiles, kTileThreads, 0, s>>>(d_buf[k], N, tile_off, d_nlpos, d_rowline);
  CUDA_LAUNCH_CHECK();
  // tile_off[tiles] = (lines << 32 | rows) of the chunk
  parse_kernel<<<num_sms() * 8, 256, 0, s>>>(d_buf[k], d_nlpos, d_rowline, tile_off + tiles, d_state,
                                       cap_rows, vocab, d_feat, d_lab,
                                       reinterpret_cast<unsigned long long*>(d_state + 2));
  CUDA_LAUNCH_CHECK();
  advance_base_kernel<<<1, 1, 0, s>>>(tile_off + tiles, d_state);
  CUDA_LAUNCH_CHECK();
  CUDA_CHECK(cudaEventRecord(parsed[k], s));
  bytes += static_cast<int64_t>(n);
}

// Host stage: bytes [off, off + n) of the source into pinned memory, split over host
// threads (a single memcpy / pread stream tops out near 5-10 GB/s, below PCIe).
static void parallel_read(const ByteReader& read_at, char* dst, size_t off, size_t n) {
  const size_t kMinPart = 4ull << 20;
  const int parts = static_cast<int>(std::min<size_t>(16, std::max<size_t>(1, n / kMinPart)));
  if (parts == 1) {
    read_at(dst, off, n);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(parts);
  const size_t per = (n + parts - 1) / parts;
  for (int p = 0; p < parts; ++p) {
    const size_t a = p * per, e = std::min(n, a + per);
    if (a < e)
      th.emplace_back([&, a, e, p] {
        try {
          read_at(dst + a, off + a, e - a);
        } catch (...) {
          errs[p] = std::current_exception();
        }
      });
  }
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void CriteoTable::ingest(const ByteReader& read_at, size_t total, const std::string& name) {
  size_t carry = 0;  // bytes of an unfinished line at the start of the next buffer
  size_t off = 0;    // next unread source byte
  int k = 0;
  int64_t chunks = 0;
  CUDA_CHECK(cudaEventRecord(ev0, stream));
  for (;;) {
    // h_buf[k] was last sent two chunks ago: its copy must be done before it is refilled
    if (chunks >= 2) CUDA_CHECK(cudaEventSynchronize(copied[k]));
    const size_t got = std::min(chunk_bytes - carry, total - off);
    parallel_read(read_at, h_buf[k] + carry, off, got);
    off += got;
    size_t n = carry + got;
    const bool eof = off == total;
    if (n == 0) break;
    size_t cut = n;  // parse [0, cut): complete lines only
    if (!eof) {
      const char* nl = static_cast<const char*>(memrchr(h_buf[k], '\n', n));
      if (!nl)
        fail(kData, name + ": a line is longer than the " + std::to_string(chunk_bytes) +
                        "-byte ingest chunk");
      cut = static_cast<size_t>(nl - h_buf[k]) + 1;
    } else if (h_buf[k][n - 1] != '\n') {  // last line without a newline (std::getline reads it)
      h_buf[k][n++] = '\n';
      cut = n;
    }
    const size_t rest = n - cut;
    const int o = k ^ 1;
    if (rest) {  // the other buffer's previous copy must be done before the carry lands in it
      if (chunks >= 1) CUDA_CHECK(cudaEventSynchronize(copied[o]));
      memcpy(h_buf[o], h_buf[k] + cut, rest);
    }
    enqueue_chunk(k, cut);
    ++chunks;
    carry = rest;
    k = o;
    if (eof) break;
  }
  CUDA_CHECK(cudaEventRecord(ev1, stream));
  CUDA_CHECK(cudaMemcpyAsync(h_state, d_state, sizeof(uint64_t) * 3, cudaMemcpyDeviceToHost, stream));
  CUDA_CHECK(cudaStreamSynchronize(stream));
  float ms = 0;
  CUDA_CHECK(cudaEventElapsedTime(&ms, ev0, ev1));
  parse_ms += ms;
  rows = static_cast<int64_t>(h_state[0]);
  lines = static_cast<int64_t>(h_state[1]);
  if (h_state[2] != kNoError) {  // first malformed line: the reference's message for it
    const int64_t bad = static_cast<int64_t>(h_state[2]);
    std::string line;  // bytes of line `bad` (1-based), found by a sequential host scan
    int64_t lineno = 1;
    std::vector<char> blk(1 << 20);
    for (size_t p = 0; p < total && lineno <= bad; p += blk.size()) {
      const size_t m = std::min(blk.size(), total - p);
      read_at(blk.data(), p, m);
      for (size_t i = 0; i < m && lineno <= bad; ++i) {
        if (blk[i] == '\n') ++lineno;
        else if (lineno == bad) line.push_back(blk[i]);
      }
    }
    fail(kData, line_error(name, bad, line));
  }
  if (rows == 0) fail(kData, name + ": no data rows");  // criteo.cpp:78
}

void CriteoTable::read_batch(int64_t step, int32_t global_rows, int32_t row0, int32_t nrows,
                             uint64_t* d_features, uint8_t* d_labels, cudaStream_t s) const {
  if (rows == 0) fail(kLogic, "criteo table is empty");
  if (row0 < 0 || nrows < 0 || row0 + nrows > global_rows) fail(kLogic, "rows outside the batch");
  const int64_t first = (step * static_cast<int64_t>(global_rows) + row0) % rows;
  if (nrows == 0) return;
  read_batch_kernel<<<ceil_div(static_cast<int64_t>(nrows) * 26, 256), 256, 0, s>>>(
      d_feat, d_lab, rows, first, nrows, d_features, d_labels);
  CUDA_LAUNCH_CHECK();
}

}  // namespace sfb
