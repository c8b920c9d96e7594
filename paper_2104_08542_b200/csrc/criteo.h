// Criteo TSV ingest on the device (criteo.cu) — CriteoReader (core/include/sfctr/criteo.hpp:37-58).
#pragma once

#include <functional>
#include <string>

#include "ops.h"

namespace sfb {

// reads source bytes [off, off + n) into dst (thread-safe: called from several threads)
using ByteReader = std::function<void(char* dst, size_t off, size_t n)>;

struct CriteoTable {
  uint64_t vocab = 0;
  int64_t rows = 0, lines = 0, bytes = 0;  // parsed data rows, all lines, bytes
  double parse_ms = 0;                     // device span of the ingest (first chunk -> last parse)
  int64_t cap_rows = 0;
  size_t chunk_bytes = 0;
  uint32_t* d_feat = nullptr;  // [cap_rows x 26] hashed ids (vocab < 2^32)
  uint8_t* d_lab = nullptr;    // [cap_rows]
  // chunk pipeline: host read | H2D (copy_stream) | parse (stream)
  char* h_buf[2] = {nullptr, nullptr};      // pinned
  uint8_t* d_buf[2] = {nullptr, nullptr};
  cudaEvent_t copied[2] = {nullptr, nullptr}, parsed[2] = {nullptr, nullptr};
  int64_t tiles_cap = 0;
  uint64_t* d_tile = nullptr;                // [2 x tiles_cap] packed counts / offsets
  uint32_t *d_nlpos = nullptr, *d_rowline = nullptr;
  uint64_t* d_state = nullptr;               // running rows, running lines, first bad line
  uint64_t* h_state = nullptr;
  void* d_scan = nullptr;
  size_t scan_bytes = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // byte_bound: total input size (bounds the row count); chunk: streaming unit
  void init(uint64_t vocab, int fields, int64_t byte_bound, size_t chunk = 64ull << 20);
  void release();
  void ingest(const ByteReader& read_at, size_t total, const std::string& name);
  void enqueue_chunk(int k, size_t n);
  // rows [row0, row0 + nrows) of global batch `step` (global_rows rows), wrapping at the end
  void read_batch(int64_t step, int32_t global_rows, int32_t row0, int32_t nrows,
                  uint64_t* d_features, uint8_t* d_labels, cudaStream_t s) const;
};

}  // namespace sfb
