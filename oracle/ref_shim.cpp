// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the reference's own compiled translation units
// (/root/reference/proj/core/src/*.cpp, built in place by oracle/build_ref.sh
// into oracle/_ref/libsfctr_ref.so). It exposes the reference's present
// primitives — rng.hpp, generator.cpp, vsi.cpp, host_store.cpp,
// cache_buffer.cpp, comm.hpp, config.cpp — to Python (ctypes) so that the C
// restatement in oracle/sfctr_oracle.c can be pinned against the real
// reference, and so that golden vectors can be regenerated
// (tests/golden/make_golden.py).
//
// No reference source is copied here: this file only #includes the
// reference headers through -I/root/reference/proj/core/include.

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sfctr/cache_buffer.hpp"
#include "sfctr/comm.hpp"
#include "sfctr/config.hpp"
#include "sfctr/criteo.hpp"
#include "sfctr/generator.hpp"
#include "sfctr/host_store.hpp"
#include "sfctr/rng.hpp"
#include "sfctr/vsi.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const sfctr::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const sfctr::DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const sfctr::LogicError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

sfctr::SimConfig make_cfg(int workers, int dim, int fields, int batch, std::uint64_t vocab,
                          std::uint64_t seed, double zipf) {
  sfctr::SimConfig c;
  c.num_workers = workers;
  c.embedding_dim = dim;
  c.num_fields = fields;
  c.batch_size_per_worker = batch;
  c.vocabulary_size = vocab;
  c.seed = seed;
  c.zipf_exponent = zipf;
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_fnv1a64(const char* bytes, std::size_t n) {
  return sfctr::fnv1a64(std::string_view(bytes, n));
}

std::uint64_t ref_derive_seed(std::uint64_t base, const char* label, std::uint64_t index) {
  return sfctr::derive_seed(base, label, index);
}

std::int64_t ref_allreduce_bytes(std::int64_t payload, int workers) {
  std::int64_t out = -1;
  guarded([&] { out = sfctr::allreduce_bytes(payload, workers); });
  return out;
}

void ref_initial_embedding(std::uint64_t seed, std::uint64_t feature, int dim, double* out) {
  auto v = sfctr::initial_embedding(seed, sfctr::FeatureId{feature}, dim);
  std::memcpy(out, v.data(), sizeof(double) * dim);
}

double ref_truth_weight(std::uint64_t seed, std::uint64_t feature) {
  return sfctr::SyntheticGenerator::truth_weight(seed, sfctr::FeatureId{feature});
}

// ---- SyntheticGenerator (generator.cpp) ----
void* ref_gen_create(int workers, int fields, int batch, std::uint64_t vocab, std::uint64_t seed,
                     double zipf) {
  sfctr::SyntheticGenerator* g = nullptr;
  int rc = guarded([&] {
    g = new sfctr::SyntheticGenerator(make_cfg(workers, 16, fields, batch, vocab, seed, zipf));
  });
  return rc == 0 ? g : nullptr;
}
void ref_gen_destroy(void* g) { delete static_cast<sfctr::SyntheticGenerator*>(g); }

void ref_gen_generate(void* g, std::int64_t step, std::uint64_t* features, std::uint8_t* labels) {
  auto b = static_cast<sfctr::SyntheticGenerator*>(g)->generate(step);
  for (std::size_t i = 0; i < b.features.size(); ++i) features[i] = b.features[i].value;
  std::memcpy(labels, b.labels.data(), b.labels.size());
}

std::uint64_t ref_gen_shard_start(void* g, int field) {
  return static_cast<sfctr::SyntheticGenerator*>(g)->shard_start(field);
}

// ---- virtual_sparse_id (vsi.cpp) ----
// Returns U (>=0) or -(status) on a reference exception.
std::int64_t ref_vsi(const std::uint64_t* features, const std::uint8_t* labels, int rows,
                     int fields, int workers, std::uint64_t* global_ids, std::uint64_t* vids,
                     int* row_ranges /* 2*workers */) {
  std::int64_t u = 0;
  int rc = guarded([&] {
    sfctr::RawBatch b;
    b.rows = rows;
    b.fields = fields;
    b.features.resize(static_cast<std::size_t>(rows) * fields);
    for (std::size_t i = 0; i < b.features.size(); ++i) b.features[i] = sfctr::FeatureId{features[i]};
    b.labels.assign(labels, labels + rows);
    auto d = sfctr::virtual_sparse_id(b, workers);
    u = d.unique_count();
    for (std::int64_t k = 0; k < u; ++k) global_ids[k] = d.global_ids[k].value;
    for (std::size_t i = 0; i < d.virtual_ids.size(); ++i) vids[i] = d.virtual_ids[i].value;
    for (int w = 0; w < workers; ++w) {
      row_ranges[2 * w] = d.worker_row_ranges[w].begin;
      row_ranges[2 * w + 1] = d.worker_row_ranges[w].end;
    }
  });
  return rc == 0 ? u : -rc;
}

// ---- HostStore + CacheBuffer (host_store.cpp, cache_buffer.cpp) ----
struct RefCache {
  sfctr::HostStore host;
  sfctr::CacheBuffer cb;
  int dim;
  RefCache(std::uint64_t seed, int d, std::uint64_t cap) : host(seed, d), cb(cap, d), dim(d) {}
};

void* ref_cache_create(std::uint64_t seed, int dim, std::uint64_t capacity) {
  RefCache* c = nullptr;
  int rc = guarded([&] { c = new RefCache(seed, dim, capacity); });
  return rc == 0 ? c : nullptr;
}
void ref_cache_destroy(void* c) { delete static_cast<RefCache*>(c); }

// take from host (lazy init) and admit; returns slot or -(status)
std::int64_t ref_cache_admit(void* cp, std::uint64_t f, std::int64_t step) {
  auto* c = static_cast<RefCache*>(cp);
  std::int64_t slot = 0;
  int rc = guarded([&] {
    sfctr::FeatureId id{f};
    slot = static_cast<std::int64_t>(c->cb.admit(id, c->host.take(id), step).value);
  });
  return rc == 0 ? slot : -rc;
}
// evict back into host; returns 0 or status
int ref_cache_evict(void* cp, std::uint64_t f) {
  auto* c = static_cast<RefCache*>(cp);
  return guarded([&] {
    sfctr::FeatureId id{f};
    c->host.put(id, c->cb.evict(id));
  });
}
int ref_cache_touch(void* cp, std::uint64_t f, std::int64_t step) {
  auto* c = static_cast<RefCache*>(cp);
  return guarded([&] { c->cb.touch(sfctr::FeatureId{f}, step); });
}
int ref_cache_pin(void* cp, std::uint64_t f, int on) {
  auto* c = static_cast<RefCache*>(cp);
  return guarded([&] {
    if (on) c->cb.pin(sfctr::FeatureId{f});
    else c->cb.unpin(sfctr::FeatureId{f});
  });
}
int ref_cache_set_needed_soon(void* cp, std::uint64_t f, int on) {
  auto* c = static_cast<RefCache*>(cp);
  return guarded([&] { c->cb.set_needed_soon(sfctr::FeatureId{f}, on != 0); });
}
std::int64_t ref_cache_slot_of(void* cp, std::uint64_t f) {
  auto* c = static_cast<RefCache*>(cp);
  std::int64_t s = 0;
  int rc = guarded([&] { s = static_cast<std::int64_t>(c->cb.slot_of(sfctr::FeatureId{f}).value); });
  return rc == 0 ? s : -rc;
}
std::uint64_t ref_cache_free_count(void* cp) { return static_cast<RefCache*>(cp)->cb.free_count(); }
std::uint64_t ref_cache_host_size(void* cp) { return static_cast<RefCache*>(cp)->host.size(); }
// slot table dump: feature (UINT64_MAX if empty), last_use, admit_seq
void ref_cache_slots(void* cp, std::uint64_t* feature, std::int64_t* last_use,
                     std::uint64_t* admit_seq) {
  auto* c = static_cast<RefCache*>(cp);
  const auto& s = c->cb.slots();
  for (std::size_t i = 0; i < s.size(); ++i) {
    feature[i] = s[i].occupied ? s[i].feature.value : ~std::uint64_t{0};
    last_use[i] = s[i].last_use;
    admit_seq[i] = s[i].admit_seq;
  }
}
// host row (embedding|momentum|velocity, 3*dim) of a host-resident feature
int ref_cache_host_row(void* cp, std::uint64_t f, double* out, std::int64_t* steps) {
  auto* c = static_cast<RefCache*>(cp);
  return guarded([&] {
    const auto& e = c->host.peek(sfctr::FeatureId{f});
    std::memcpy(out, e.data.data(), sizeof(double) * e.data.size());
    *steps = e.adam_steps;
  });
}

// ---- SimConfig (config.cpp) ----
int ref_config_check(const char* key, const char* value, int validate_after) {
  return guarded([&] {
    sfctr::SimConfig c;
    if (key) sfctr::apply_config_entry(c, key, value);
    if (validate_after) c.validate();
  });
}

// ---- CriteoReader (criteo.cpp) ----
// Returns a reader or nullptr (status in *rc: 1 ConfigError, 2 DataError; ref_last_error()).
void* ref_criteo_open(const char* path, int fields, std::uint64_t vocab, int workers, int batch,
                      int* rc) {
  sfctr::CriteoReader* r = nullptr;
  *rc = guarded([&] {
    r = new sfctr::CriteoReader(path, make_cfg(workers, 16, fields, batch, vocab, 7, 1.2));
  });
  return *rc == 0 ? r : nullptr;
}
void ref_criteo_destroy(void* r) { delete static_cast<sfctr::CriteoReader*>(r); }
std::int64_t ref_criteo_rows(void* r) { return static_cast<sfctr::CriteoReader*>(r)->row_count(); }
void ref_criteo_read_batch(void* r, std::int64_t step, std::uint64_t* features,
                           std::uint8_t* labels) {
  auto b = static_cast<sfctr::CriteoReader*>(r)->read_batch(step);
  for (std::size_t i = 0; i < b.features.size(); ++i) features[i] = b.features[i].value;
  std::memcpy(labels, b.labels.data(), b.labels.size());
}
std::uint64_t ref_criteo_token_hash(const char* token, std::size_t n) {
  return sfctr::CriteoReader::token_hash(std::string(token, n));
}

}  // extern "C"
