// sfctr_b200.hpp — header-only C++ façade over the C-ABI (sfctr_b200.h) that
// keeps the reference's C++ vocabulary: it consumes and produces the
// reference's own types (sfctr::RawBatch / DedupBatch / FeatureId,
// include/sfctr/batch.hpp, types.hpp) and throws the reference's exception
// classes (include/sfctr/error.hpp:28-56). Build with
// -I/path/to/reference/proj/core/include and link libsfctr_b200.so.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "sfctr/batch.hpp"
#include "sfctr/error.hpp"
#include "sfctr/host_store.hpp"
#include "sfctr_b200.h"

namespace sfctr {
namespace b200 {

class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

// status code -> the reference's exception class (error.hpp:28-56)
inline void check(int status) {
  if (status == SFCTR_OK) return;
  const std::string msg = sfctr_last_error();
  switch (status) {
    case SFCTR_ERR_CONFIG: throw ConfigError(msg);
    case SFCTR_ERR_DATA: throw DataError(msg);
    case SFCTR_ERR_LOGIC: throw LogicError(msg);
    case SFCTR_ERR_RUN: throw RunError(sfctr_last_error_step(), msg);
    default: throw CudaError(msg);
  }
}

struct Config {  // SimConfig (config.hpp:42-71) + B200 keys
  sfctr_config c;
  Config() { sfctr_config_default(&c); }
  Config& set(const std::string& key, const std::string& value) {  // apply_config_entry
    check(sfctr_config_apply(&c, key.c_str(), value.c_str()));
    return *this;
  }
  Config& load(const std::string& path) {  // load_config_file
    check(sfctr_config_load(&c, path.c_str()));
    return *this;
  }
  void validate() const { check(sfctr_config_validate(&c)); }
};

// SyntheticGenerator (generator.hpp:35-62) on the device
class Generator {
 public:
  explicit Generator(const Config& cfg, int device = 0) : cfg_(cfg) {
    check(sfctr_generator_create(&cfg_.c, device, &g_));
  }
  ~Generator() { sfctr_generator_destroy(g_); }
  Generator(const Generator&) = delete;
  Generator& operator=(const Generator&) = delete;

  RawBatch generate(std::int64_t step) const {  // generator.cpp:82-108
    RawBatch b;
    b.rows = cfg_.c.num_workers * cfg_.c.batch_size_per_worker;
    b.fields = cfg_.c.num_fields;
    std::vector<std::uint64_t> f(static_cast<std::size_t>(b.rows) * b.fields);
    b.labels.resize(b.rows);
    check(sfctr_generator_generate(g_, step, 0, b.rows, f.data(), b.labels.data()));
    b.features.reserve(f.size());
    for (auto v : f) b.features.emplace_back(v);
    return b;
  }
  std::uint64_t shard_start(int field) const { return sfctr_generator_shard_start(g_, field); }

 private:
  Config cfg_;
  sfctr_generator* g_ = nullptr;
};

inline std::vector<double> initial_embedding(std::uint64_t seed, FeatureId f, int dim,
                                             int device = 0) {  // generator.hpp:62
  std::vector<double> out(dim);
  check(sfctr_initial_embedding(seed, f.value, dim, device, out.data()));
  return out;
}

// DedupBatch virtual_sparse_id(const RawBatch&, int) (vsi.hpp:29), on the device, for any
// FeatureId: key_space defaults to max id + 1 (direct-mapped first-position table) while
// that stays below 2^31, else the hashed table (arbitrary u64 ids).
inline DedupBatch virtual_sparse_id(const RawBatch& batch, int num_workers, int device = 0,
                                    std::uint64_t key_space = 0) {
  const std::size_t n = batch.features.size();
  std::vector<std::uint64_t> ids(n);
  std::uint64_t mx = 0;
  for (std::size_t i = 0; i < n; ++i) {
    ids[i] = batch.features[i].value;
    mx = ids[i] > mx ? ids[i] : mx;
  }
  if (!key_space && mx < (1ull << 31)) key_space = mx + 1;
  sfctr_vsi* v = nullptr;
  check(sfctr_vsi_create(device, key_space, static_cast<std::int64_t>(n ? n : 1), &v));
  std::vector<std::uint64_t> g(n ? n : 1), vid(n ? n : 1);
  std::vector<std::int32_t> rr(2 * (num_workers > 0 ? num_workers : 1));
  std::int64_t u = 0;
  const int st = sfctr_virtual_sparse_id(v, ids.data(), batch.rows, batch.fields, num_workers,
                                         g.data(), vid.data(), &u, rr.data());
  sfctr_vsi_destroy(v);
  check(st);
  DedupBatch d;
  d.rows = batch.rows;
  d.fields = batch.fields;
  d.labels = batch.labels;
  d.global_ids.reserve(u);
  for (std::int64_t k = 0; k < u; ++k) d.global_ids.emplace_back(g[k]);
  d.virtual_ids.reserve(n);
  for (std::size_t i = 0; i < n; ++i) d.virtual_ids.emplace_back(vid[i]);
  for (int w = 0; w < num_workers; ++w) d.worker_row_ranges.push_back({rr[2 * w], rr[2 * w + 1]});
  return d;
}

// CacheBuffer (cache_buffer.hpp:40-86) of one worker with its HostStore and the manager
// step, on the device: the reference's member functions, SlotId / FeatureId / ParamEntry
// in and out, the reference's exceptions. evict() returns the evicted entry (fp32 state
// widened to the reference's fp64 ParamEntry) after it went to the host pool.
class CacheBuffer {
 public:
  CacheBuffer(std::uint64_t capacity, int dim, std::uint64_t seed, std::uint64_t key_space,
              int num_workers = 1, int worker = 0, std::int64_t max_batch = 1 << 16,
              int device = 0)
      : dim_(dim), capacity_(capacity) {
    check(sfctr_cache_create(capacity, dim, seed, key_space, num_workers, worker, max_batch, 0,
                             device, &c_));
  }
  ~CacheBuffer() { sfctr_cache_destroy(c_); }
  CacheBuffer(const CacheBuffer&) = delete;
  CacheBuffer& operator=(const CacheBuffer&) = delete;

  std::uint64_t capacity() const { return capacity_; }
  std::size_t free_count() const {
    std::uint64_t n = 0;
    check(sfctr_cache_free_count(c_, &n));
    return static_cast<std::size_t>(n);
  }
  std::size_t occupied_count() const { return capacity_ - free_count(); }
  bool resident(FeatureId f) const { return raw_slot(f) >= 0; }
  SlotId slot_of(FeatureId f) const {  // cache_buffer.cpp:31-35
    const std::int64_t s = raw_slot(f);
    if (s < 0) throw LogicError("feature " + std::to_string(f.value) + " not resident");
    return SlotId{static_cast<std::uint64_t>(s)};
  }
  SlotId admit(FeatureId f, std::int64_t step) {  // admit(f, host.take(f), step)
    std::uint64_t slot = 0;
    check(sfctr_cache_admit(c_, 1, &f.value, step, &slot));
    return SlotId{slot};
  }
  ParamEntry evict(FeatureId f) {  // host.put(f, evict(f)); returns the entry
    check(sfctr_cache_evict(c_, 1, &f.value));
    std::vector<float> row(3 * static_cast<std::size_t>(dim_));
    std::int64_t steps = 0;
    check(sfctr_cache_peek(c_, 1, &f.value, row.data(), &steps));
    ParamEntry e(dim_);
    for (std::size_t i = 0; i < row.size(); ++i) e.data[i] = row[i];
    e.adam_steps = steps;
    return e;
  }
  void touch(FeatureId f, std::int64_t step) { check(sfctr_cache_touch(c_, 1, &f.value, step)); }
  void pin(FeatureId f) { check(sfctr_cache_pin(c_, 1, &f.value, 1)); }
  void unpin(FeatureId f) { check(sfctr_cache_pin(c_, 1, &f.value, 0)); }
  void set_needed_soon(FeatureId f, bool value) {
    check(sfctr_cache_set_needed_soon(c_, 1, &f.value, value ? 1 : 0));
  }
  std::string occupancy_diagnostics() const {
    char buf[256];
    check(sfctr_cache_occupancy_diagnostics(c_, buf, sizeof(buf)));
    return buf;
  }
  // manager_get + pull + push for this worker: owned, hits, admitted,
  // evicted, refilled
  std::vector<std::int64_t> prepare(std::int64_t step, const std::vector<FeatureId>& global_ids,
                                    const std::vector<FeatureId>& window = {}) {
    std::vector<std::uint64_t> g(global_ids.size()), w(window.size());
    for (std::size_t i = 0; i < g.size(); ++i) g[i] = global_ids[i].value;
    for (std::size_t i = 0; i < w.size(); ++i) w[i] = window[i].value;
    std::vector<std::int64_t> out(5);
    check(sfctr_cache_prepare(c_, step, static_cast<std::int64_t>(g.size()), g.data(),
                              static_cast<std::int64_t>(w.size()), w.data(), out.data()));
    return out;
  }
  sfctr_cache* handle() { return c_; }

 private:
  std::int64_t raw_slot(FeatureId f) const {
    std::int64_t s = -1;
    check(sfctr_cache_slot_of(c_, 1, &f.value, &s));
    return s;
  }
  int dim_;
  std::uint64_t capacity_;
  sfctr_cache* c_ = nullptr;
};

// HostStore + CacheBuffer per worker + worker ops: one BSP step per call.
class Trainer {
 public:
  Trainer(const Config& cfg, int rank = 0, int world = 1, const std::uint8_t* nccl_id = nullptr,
          int device = 0)
      : cfg_(cfg) {
    check(sfctr_trainer_create(&cfg_.c, rank, world, nccl_id, device, &t_));
  }
  ~Trainer() { sfctr_trainer_destroy(t_); }
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  // this process's rows of global batch `step`
  double step(std::int64_t step, const RawBatch& rows) {
    std::vector<std::uint64_t> f(rows.features.size());
    for (std::size_t i = 0; i < f.size(); ++i) f[i] = rows.features[i].value;
    double loss = 0;
    check(sfctr_trainer_step(t_, step, f.data(), rows.labels.data(), nullptr, &loss));
    return loss;
  }
  // HostStore::snapshot_sorted (host_store.hpp:85-86): feature -> (emb|m|v fp32, adam_steps)
  std::map<std::uint64_t, std::pair<std::vector<float>, std::int64_t>> snapshot() {
    std::int64_t n = 0;
    check(sfctr_trainer_snapshot(t_, &n, nullptr, nullptr, nullptr));
    const int d3 = 3 * cfg_.c.embedding_dim;
    std::vector<std::uint64_t> f(n ? n : 1);
    std::vector<float> rows(static_cast<std::size_t>(n ? n : 1) * d3);
    std::vector<std::int64_t> st(n ? n : 1);
    check(sfctr_trainer_snapshot(t_, &n, f.data(), rows.data(), st.data()));
    std::map<std::uint64_t, std::pair<std::vector<float>, std::int64_t>> out;
    for (std::int64_t i = 0; i < n; ++i)
      out.emplace(f[i], std::make_pair(std::vector<float>(rows.begin() + i * d3,
                                                          rows.begin() + (i + 1) * d3),
                                       st[i]));
    return out;
  }
  // TransferLedger (ledger.hpp:60-63): h2w, w2h, interworker, swap_events
  std::vector<std::int64_t> ledger() {
    std::vector<std::int64_t> out(4);
    check(sfctr_trainer_ledger(t_, out.data()));
    return out;
  }
  // pipelined driving (one step in flight): submit, then loss of the previous step
  void submit(std::int64_t step, const RawBatch& rows) {
    auto& f = staged_[step & 1];
    f.first.resize(rows.features.size());
    for (std::size_t i = 0; i < f.first.size(); ++i) f.first[i] = rows.features[i].value;
    f.second = rows.labels;
    check(sfctr_trainer_submit(t_, step, f.first.data(), f.second.data(), nullptr));
  }
  double loss(std::int64_t step) {
    double l = 0;
    check(sfctr_trainer_loss(t_, step, &l));
    return l;
  }
  sfctr_trainer* handle() { return t_; }

 private:
  Config cfg_;
  sfctr_trainer* t_ = nullptr;
  // host inputs of the (at most two) submitted steps, alive until their loss is read
  std::pair<std::vector<std::uint64_t>, std::vector<std::uint8_t>> staged_[2];
};

// CriteoReader (criteo.hpp:37-58): the TSV is parsed and hashed on the device at
// construction; read_batch(step) returns the wrapping global batch (criteo.cpp:81-98).
class CriteoReader {
 public:
  static constexpr int kNumericColumns = 13;
  static constexpr int kCategoricalColumns = 26;
  CriteoReader(const std::string& path, const Config& cfg, int device = 0) : cfg_(cfg) {
    check(sfctr_criteo_open(path.c_str(), &cfg_.c, device, &r_));
  }
  ~CriteoReader() { sfctr_criteo_destroy(r_); }
  CriteoReader(const CriteoReader&) = delete;
  CriteoReader& operator=(const CriteoReader&) = delete;
  RawBatch read_batch(std::int64_t step) const {
    RawBatch b;
    b.rows = cfg_.c.num_workers * cfg_.c.batch_size_per_worker;
    b.fields = kCategoricalColumns;
    std::vector<std::uint64_t> f(static_cast<std::size_t>(b.rows) * b.fields);
    b.labels.resize(b.rows);
    check(sfctr_criteo_read_batch(r_, step, 0, b.rows, f.data(), b.labels.data()));
    b.features.reserve(f.size());
    for (auto v : f) b.features.emplace_back(v);
    return b;
  }
  std::int64_t row_count() const { return sfctr_criteo_row_count(r_); }
  static std::uint64_t token_hash(const std::string& token) {
    return sfctr_criteo_token_hash(token.data(), token.size());
  }

 private:
  Config cfg_;
  sfctr_criteo* r_ = nullptr;
};

}  // namespace b200
}  // namespace sfctr
