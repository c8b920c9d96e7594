// extern "C" boundary (include/sfctr_b200.h). Every entry point catches the
// engine's sfb::Error and maps it to a status code + thread-local message,
// mirroring the reference's exception classes (error.hpp:28-56).
#include <cstring>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <functional>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>

#include "cachebuf.h"
#include "criteo.h"
#include "trainer.h"

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_step = -1;

template <typename F>
int guarded(F&& f) {
  try {
    g_err.clear();
    g_err_step = -1;
    f();
    return sfb::kOk;
  } catch (const sfb::Error& e) {
    g_err = e.what();
    g_err_step = e.step;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return sfb::kRun;
  } catch (const std::exception& e) {
    g_err = e.what();
    return sfb::kLogic;
  }
}

uint64_t parse_u64(const std::string& key, const std::string& value) {  // config.cpp:84-96
  try {
    size_t pos = 0;
    if (!value.empty() && value[0] == '-') throw std::invalid_argument("negative");
    const uint64_t v = std::stoull(value, &pos);
    if (pos != value.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    sfb::fail(sfb::kConfig, "config key '" + key + "': cannot parse '" + value + "' as an integer");
  }
}
int parse_int(const std::string& key, const std::string& value) {  // config.cpp:98-104
  const uint64_t v = parse_u64(key, value);
  if (v > (1ull << 30))
    sfb::fail(sfb::kConfig, "config key '" + key + "': value '" + value + "' out of range");
  return static_cast<int>(v);
}
double parse_double(const std::string& key, const std::string& value) {  // config.cpp:106-113
  try {
    size_t pos = 0;
    const double v = std::stod(value, &pos);
    if (pos != value.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    sfb::fail(sfb::kConfig, "config key '" + key + "': cannot parse '" + value + "' as a number");
  }
}

void apply_entry(sfctr_config& c, const std::string& key, const std::string& value) {
  // config.cpp:115-159 (same keys), plus the B200 keys sync / host_rows
  if (key == "workers") c.num_workers = parse_int(key, value);
  else if (key == "dim") c.embedding_dim = parse_int(key, value);
  else if (key == "fields") c.num_fields = parse_int(key, value);
  else if (key == "batch_size") c.batch_size_per_worker = parse_int(key, value);
  else if (key == "vocab") c.vocabulary_size = parse_u64(key, value);
  else if (key == "cache_capacity") c.cache_capacity = parse_u64(key, value);
  else if (key == "lookahead") c.lookahead_depth = parse_int(key, value);
  else if (key == "strategy") {
    if (value == "host") c.strategy = SFCTR_STRATEGY_HOST;
    else if (value == "prefetch") c.strategy = SFCTR_STRATEGY_PREFETCH;
    else if (value == "cache") c.strategy = SFCTR_STRATEGY_CACHE;
    else sfb::fail(sfb::kConfig, "unknown strategy '" + value + "' (expected host, prefetch or cache)");
  } else if (key == "seed") c.seed = parse_u64(key, value);
  else if (key == "lr") c.learning_rate = parse_double(key, value);
  else if (key == "beta1") c.adam_beta1 = parse_double(key, value);
  else if (key == "beta2") c.adam_beta2 = parse_double(key, value);
  else if (key == "epsilon") c.adam_epsilon = parse_double(key, value);
  else if (key == "zipf") c.zipf_exponent = parse_double(key, value);
  else if (key == "hidden") c.hidden_dim = parse_int(key, value);
  else if (key == "data") {  // config.cpp:146-154
    if (value == "synthetic") {
      c.data_source = SFCTR_DATA_SYNTHETIC;
      c.criteo_path[0] = 0;
    } else if (value.rfind("criteo:", 0) == 0) {
      const std::string path = value.substr(7);
      if (path.size() >= SFCTR_PATH_MAX) sfb::fail(sfb::kConfig, "config key 'data': path too long");
      c.data_source = SFCTR_DATA_CRITEO;
      std::memcpy(c.criteo_path, path.c_str(), path.size() + 1);
    } else {
      sfb::fail(sfb::kConfig, "config key 'data': expected 'synthetic' or 'criteo:<path>'");
    }
  } else if (key == "deterministic") {
    if (value == "1" || value == "true") c.deterministic = 1;
    else if (value == "0" || value == "false") c.deterministic = 0;
    else sfb::fail(sfb::kConfig, "config key 'deterministic': expected 0 or 1");
  } else if (key == "sync") {
    if (value == "allreduce") c.sync_mode = SFCTR_SYNC_ALLREDUCE;
    else if (value == "alltoall") c.sync_mode = SFCTR_SYNC_ALLTOALL;
    else sfb::fail(sfb::kConfig, "config key 'sync': expected allreduce or alltoall");
  } else if (key == "host_rows") c.host_table_rows = parse_u64(key, value);
  else if (key == "mode") {  // run_mode_from_string (config.cpp:49-53)
    if (value == "pipelined") c.run_mode = SFCTR_MODE_PIPELINED;
    else if (value == "sequential") c.run_mode = SFCTR_MODE_SEQUENTIAL;
    else sfb::fail(sfb::kConfig, "unknown mode '" + value + "' (expected pipelined or sequential)");
  }
  else sfb::fail(sfb::kConfig, "unknown config key '" + key + "'");
}

struct DeviceScope {  // every compute entry point needs a usable device
  explicit DeviceScope(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      sfb::fail(sfb::kCuda, "no CUDA device available (the device path has no CPU fallback)");
    }
    CUDA_CHECK(cudaSetDevice(device));
  }
};

}  // namespace

struct sfctr_generator {
  int device;
  sfb::GenTables tables;
  int32_t global_rows;
  cudaStream_t stream;
  uint64_t* d_feat = nullptr;
  uint8_t* d_lab = nullptr;
  int64_t cap = 0;
};

struct sfctr_criteo {
  int device;
  int32_t global_rows;
  sfb::CriteoTable table;
  ~sfctr_criteo() {
    cudaSetDevice(device);
    table.release();
  }
};

struct sfctr_vsi {
  int device;
  sfb::VsiScratch scratch;
  cudaStream_t stream;
  uint64_t* d_in = nullptr;
  uint32_t* d_ids = nullptr;
  uint32_t* d_gids = nullptr;
  uint32_t* d_vids = nullptr;
  uint64_t* d_out64 = nullptr;
  int32_t* d_scal = nullptr;
};

struct sfctr_trainer {
  std::unique_ptr<sfb::Trainer> t;
};

struct sfctr_batch_source {  // the configured DataSource behind one read interface
  sfctr_generator* gen = nullptr;
  sfctr_criteo* criteo = nullptr;
};

struct sfctr_cache {
  std::unique_ptr<sfb::DeviceCache> c;
};

extern "C" {

const char* sfctr_last_error(void) { return g_err.c_str(); }
int64_t sfctr_last_error_step(void) { return g_err_step; }
int sfctr_abi_version(void) { return SFCTR_B200_ABI_VERSION; }

void sfctr_config_default(sfctr_config* c) {  // config.hpp:44-71
  std::memset(c, 0, sizeof(*c));
  c->num_workers = 4;
  c->embedding_dim = 16;
  c->num_fields = 26;
  c->batch_size_per_worker = 256;
  c->vocabulary_size = 100000;
  c->cache_capacity = 8192;
  c->lookahead_depth = 1;
  c->strategy = SFCTR_STRATEGY_CACHE;
  c->seed = 7;
  c->learning_rate = 1e-3;
  c->adam_beta1 = 0.9;
  c->adam_beta2 = 0.999;
  c->adam_epsilon = 1e-8;
  c->zipf_exponent = 1.2;
  c->hidden_dim = 64;
  c->sync_mode = SFCTR_SYNC_ALLREDUCE;
  c->host_table_rows = 0;
  c->run_mode = SFCTR_MODE_SEQUENTIAL;
  c->data_source = SFCTR_DATA_SYNTHETIC;
  c->criteo_path[0] = 0;
  c->deterministic = 0;
}

int sfctr_config_validate(const sfctr_config* c) {
  return guarded([&] { sfb::validate_config(*c); });
}

int sfctr_config_apply(sfctr_config* c, const char* key, const char* value) {
  return guarded([&] { apply_entry(*c, key ? key : "", value ? value : ""); });
}

int sfctr_config_load(sfctr_config* c, const char* path) {  // config.cpp:161-187
  return guarded([&] {
    std::ifstream in(path);
    if (!in) sfb::fail(sfb::kConfig, std::string("cannot open config file: ") + path);
    std::string line;
    int lineno = 0;
    auto strip = [](const std::string& s) {
      const auto b = s.find_first_not_of(" \t\r");
      if (b == std::string::npos) return std::string();
      const auto e = s.find_last_not_of(" \t\r");
      return s.substr(b, e - b + 1);
    };
    while (std::getline(in, line)) {
      ++lineno;
      const auto hash = line.find('#');
      if (hash != std::string::npos) line.erase(hash);
      const std::string t = strip(line);
      if (t.empty()) continue;
      const auto eq = t.find('=');
      if (eq == std::string::npos)
        sfb::fail(sfb::kConfig, std::string(path) + ":" + std::to_string(lineno) + ": expected key=value");
      apply_entry(*c, strip(t.substr(0, eq)), strip(t.substr(eq + 1)));
    }
  });
}

uint64_t sfctr_fnv1a64(const char* bytes, size_t n) { return sfb::fnv1a64(bytes, n); }

uint64_t sfctr_derive_seed(uint64_t base, const char* label, uint64_t index) {
  return sfb::derive_seed_h(base, sfb::fnv1a64(label, std::strlen(label)), index);
}

int64_t sfctr_allreduce_bytes(int64_t payload, int w) {  // comm.hpp:36-41
  if (w < 1 || payload < 0) {
    g_err = w < 1 ? "all-reduce needs at least one participant" : "negative payload";
    return -1;
  }
  return 2 * static_cast<int64_t>(w - 1) * payload / w;
}

int sfctr_device_count(int* count) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return sfb::kOk;
}

// ---------------- Criteo ingest (CriteoReader, criteo.hpp:37-58) ----------------
namespace {

void criteo_common(const sfctr_config* cfg, int device, int64_t bytes, sfctr_criteo** out,
                   const std::function<void(sfb::CriteoTable&)>& fill) {
  if (!cfg || !out) sfb::fail(sfb::kLogic, "null argument");
  DeviceScope ds(device);
  auto r = std::make_unique<sfctr_criteo>();
  r->device = device;
  r->global_rows = cfg->num_workers * cfg->batch_size_per_worker;
  if (r->global_rows <= 0) sfb::fail(sfb::kConfig, "bad batch shape");
  size_t chunk = std::min<size_t>(64ull << 20, std::max<int64_t>(bytes + 64, 1 << 16));
  if (const char* e = std::getenv("SFCTR_CRITEO_CHUNK"))  // tests: force multi-chunk streaming
    chunk = std::max<size_t>(std::strtoull(e, nullptr, 10), 4096);
  r->table.init(cfg->vocabulary_size, cfg->num_fields, bytes, chunk);
  fill(r->table);
  *out = r.release();
}
}  // namespace

int sfctr_criteo_open(const char* path, const sfctr_config* cfg, int device, sfctr_criteo** out) {
  return guarded([&] {
    if (!path) sfb::fail(sfb::kLogic, "null path");
    if (cfg && cfg->num_fields != 26)  // criteo.cpp:31-34 (before the file is touched)
      sfb::fail(sfb::kConfig, "criteo format has 26 categorical fields; fields=" +
                                  std::to_string(cfg->num_fields) + " was configured");
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) sfb::fail(sfb::kConfig, std::string("cannot open criteo file: ") + path);
    struct stat st {};
    if (fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
      ::close(fd);
      sfb::fail(sfb::kConfig, std::string("cannot open criteo file: ") + path);
    }
    const size_t bytes = static_cast<size_t>(st.st_size);
    auto read_at = [fd, path](char* dst, size_t off, size_t n) {
      while (n) {
        const ssize_t r = ::pread(fd, dst, n, static_cast<off_t>(off));
        if (r <= 0) sfb::fail(sfb::kData, std::string("read error in ") + path);
        dst += r;
        off += static_cast<size_t>(r);
        n -= static_cast<size_t>(r);
      }
    };
    try {
      criteo_common(cfg, device, static_cast<int64_t>(bytes), out,
                    [&](sfb::CriteoTable& t) { t.ingest(read_at, bytes, path); });
    } catch (...) {
      ::close(fd);
      throw;
    }
    ::close(fd);
  });
}

int sfctr_criteo_open_buffer(const char* data, size_t n, const char* name, const sfctr_config* cfg,
                             int device, sfctr_criteo** out) {
  return guarded([&] {
    if (!data && n) sfb::fail(sfb::kLogic, "null data");
    auto read_at = [data](char* dst, size_t off, size_t m) { std::memcpy(dst, data + off, m); };
    criteo_common(cfg, device, static_cast<int64_t>(n), out,
                  [&](sfb::CriteoTable& t) { t.ingest(read_at, n, name ? name : "<buffer>"); });
  });
}

void sfctr_criteo_destroy(sfctr_criteo* r) { delete r; }

int64_t sfctr_criteo_row_count(const sfctr_criteo* r) { return r ? r->table.rows : -1; }

uint64_t sfctr_criteo_token_hash(const char* token, size_t n) { return sfb::fnv1a64(token, n); }

int sfctr_criteo_read_batch_device(sfctr_criteo* r, int64_t step, int32_t row0, int32_t nrows,
                                   uint64_t* d_features, uint8_t* d_labels, void* stream) {
  return guarded([&] {
    DeviceScope ds(r->device);
    r->table.read_batch(step, r->global_rows, row0, nrows, d_features, d_labels,
                        static_cast<cudaStream_t>(stream));
  });
}

int sfctr_criteo_read_batch(sfctr_criteo* r, int64_t step, int32_t row0, int32_t nrows,
                            uint64_t* features, uint8_t* labels) {
  return guarded([&] {
    DeviceScope ds(r->device);
    uint64_t* df = nullptr;
    uint8_t* dl = nullptr;
    CUDA_CHECK(cudaMalloc(&df, sizeof(uint64_t) * 26 * std::max(nrows, 1)));
    CUDA_CHECK(cudaMalloc(&dl, std::max(nrows, 1)));
    try {
      r->table.read_batch(step, r->global_rows, row0, nrows, df, dl, r->table.stream);
      CUDA_CHECK(cudaMemcpyAsync(features, df, sizeof(uint64_t) * 26 * nrows,
                                 cudaMemcpyDeviceToHost, r->table.stream));
      CUDA_CHECK(cudaMemcpyAsync(labels, dl, nrows, cudaMemcpyDeviceToHost, r->table.stream));
      CUDA_CHECK(cudaStreamSynchronize(r->table.stream));
    } catch (...) {
      cudaFree(df);
      cudaFree(dl);
      throw;
    }
    cudaFree(df);
    cudaFree(dl);
  });
}

int sfctr_criteo_stats(const sfctr_criteo* r, int64_t* bytes, int64_t* lines, double* parse_ms) {
  return guarded([&] {
    if (bytes) *bytes = r->table.bytes;
    if (lines) *lines = r->table.lines;
    if (parse_ms) *parse_ms = r->table.parse_ms;
  });
}

// ---------------- generator ----------------
int sfctr_generator_create(const sfctr_config* cfg, int device, sfctr_generator** out) {
  *out = nullptr;
  return guarded([&] {
    DeviceScope ds(device);
    auto g = std::make_unique<sfctr_generator>();
    g->device = device;
    g->global_rows = cfg->num_workers * cfg->batch_size_per_worker;
    if (cfg->num_fields <= 0 || g->global_rows <= 0) sfb::fail(sfb::kConfig, "bad generator shape");
    g->tables.build(cfg->num_fields, cfg->vocabulary_size, cfg->seed, cfg->zipf_exponent);
    CUDA_CHECK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    *out = g.release();
  });
}

void sfctr_generator_destroy(sfctr_generator* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  g->tables.release();
  cudaFree(g->d_feat);
  cudaFree(g->d_lab);
  cudaStreamDestroy(g->stream);
  delete g;
}

int sfctr_generator_generate_device(sfctr_generator* g, int64_t step, int32_t row0, int32_t nrows,
                                    uint64_t* d_features, uint8_t* d_labels, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(g->device));
    if (row0 < 0 || nrows < 0 || row0 + nrows > g->global_rows)
      sfb::fail(sfb::kLogic, "row range outside the global batch");
    sfb::generate_rows(g->tables, step, row0, nrows, d_features, d_labels,
                       static_cast<cudaStream_t>(stream));
  });
}

int sfctr_generator_generate(sfctr_generator* g, int64_t step, int32_t row0, int32_t nrows,
                             uint64_t* features, uint8_t* labels) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(g->device));
    if (row0 < 0 || nrows < 0 || row0 + nrows > g->global_rows)
      sfb::fail(sfb::kLogic, "row range outside the global batch");
    const int64_t n = static_cast<int64_t>(nrows) * g->tables.fields;
    if (n > g->cap) {
      cudaFree(g->d_feat);
      cudaFree(g->d_lab);
      CUDA_CHECK(cudaMalloc(&g->d_feat, sizeof(uint64_t) * std::max<int64_t>(n, 1)));
      CUDA_CHECK(cudaMalloc(&g->d_lab, std::max<int32_t>(nrows, 1)));
      g->cap = n;
    }
    sfb::generate_rows(g->tables, step, row0, nrows, g->d_feat, g->d_lab, g->stream);
    CUDA_CHECK(cudaMemcpyAsync(features, g->d_feat, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost,
                               g->stream));
    CUDA_CHECK(cudaMemcpyAsync(labels, g->d_lab, nrows, cudaMemcpyDeviceToHost, g->stream));
    CUDA_CHECK(cudaStreamSynchronize(g->stream));
  });
}

uint64_t sfctr_generator_shard_start(const sfctr_generator* g, int32_t field) {
  return g->tables.shard_starts.at(field);
}

int sfctr_initial_embedding(uint64_t seed, uint64_t feature, int32_t dim, int device, double* out) {
  return guarded([&] {
    DeviceScope ds(device);
    double* d = nullptr;
    CUDA_CHECK(cudaMalloc(&d, sizeof(double) * dim));
    sfb::initial_embedding_device(seed, feature, dim, d, nullptr);
    CUDA_CHECK(cudaMemcpy(out, d, sizeof(double) * dim, cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

// ---------------- batch source (config key `data`) ----------------
int sfctr_batch_source_create(const sfctr_config* cfg, int device, sfctr_batch_source** out) {
  *out = nullptr;
  return guarded([&] {
    sfb::validate_config(*cfg);
    auto b = std::make_unique<sfctr_batch_source>();
    int st = 0;
    if (cfg->data_source == SFCTR_DATA_CRITEO)
      st = sfctr_criteo_open(cfg->criteo_path, cfg, device, &b->criteo);
    else
      st = sfctr_generator_create(cfg, device, &b->gen);
    if (st) sfb::fail(st, g_err);
    *out = b.release();
  });
}
void sfctr_batch_source_destroy(sfctr_batch_source* b) {
  if (!b) return;
  if (b->gen) sfctr_generator_destroy(b->gen);
  if (b->criteo) sfctr_criteo_destroy(b->criteo);
  delete b;
}
int sfctr_batch_source_read(sfctr_batch_source* b, int64_t step, int32_t row0, int32_t nrows,
                            uint64_t* features, uint8_t* labels) {
  return b->criteo ? sfctr_criteo_read_batch(b->criteo, step, row0, nrows, features, labels)
                   : sfctr_generator_generate(b->gen, step, row0, nrows, features, labels);
}
int sfctr_batch_source_read_device(sfctr_batch_source* b, int64_t step, int32_t row0,
                                   int32_t nrows, uint64_t* d_features, uint8_t* d_labels,
                                   void* stream) {
  return b->criteo ? sfctr_criteo_read_batch_device(b->criteo, step, row0, nrows, d_features,
                                                    d_labels, stream)
                   : sfctr_generator_generate_device(b->gen, step, row0, nrows, d_features,
                                                     d_labels, stream);
}

// ---------------- VSI ----------------
int sfctr_vsi_create(int device, uint64_t key_space, int64_t max_ids, sfctr_vsi** out) {
  *out = nullptr;
  return guarded([&] {
    DeviceScope ds(device);
    if (key_space >= 0xFFFFFFF0ull)
      sfb::fail(sfb::kConfig, "key_space must be below 2^32-16 (0 = arbitrary u64 ids, hashed)");
    auto v = std::make_unique<sfctr_vsi>();
    v->device = device;
    v->scratch.init(key_space, max_ids);
    const int64_t n = std::max<int64_t>(max_ids, 1);
    CUDA_CHECK(cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaMalloc(&v->d_in, sizeof(uint64_t) * n));
    CUDA_CHECK(cudaMalloc(&v->d_ids, sizeof(uint32_t) * n));
    CUDA_CHECK(cudaMalloc(&v->d_gids, sizeof(uint32_t) * n));
    CUDA_CHECK(cudaMalloc(&v->d_vids, sizeof(uint32_t) * n));
    CUDA_CHECK(cudaMalloc(&v->d_out64, sizeof(uint64_t) * n));
    CUDA_CHECK(cudaMalloc(&v->d_scal, sizeof(int32_t) * 4));
    *out = v.release();
  });
}

void sfctr_vsi_destroy(sfctr_vsi* v) {
  if (!v) return;
  cudaSetDevice(v->device);
  v->scratch.release();
  for (void* p : {static_cast<void*>(v->d_in), static_cast<void*>(v->d_ids),
                  static_cast<void*>(v->d_gids), static_cast<void*>(v->d_vids),
                  static_cast<void*>(v->d_out64), static_cast<void*>(v->d_scal)})
    cudaFree(p);
  cudaStreamDestroy(v->stream);
  delete v;
}

int sfctr_virtual_sparse_id(sfctr_vsi* v, const uint64_t* features, int32_t rows, int32_t fields,
                            int32_t num_workers, uint64_t* global_ids, uint64_t* virtual_ids,
                            int64_t* unique_count, int32_t* row_ranges) {
  return guarded([&] {
    // vsi.cpp:24-31 checks, same order and class (LogicError)
    SFB_CHECK(rows > 0 && fields > 0, "empty batch");
    SFB_CHECK(num_workers > 0 && rows % num_workers == 0, "rows must split evenly across workers");
    const int64_t n = static_cast<int64_t>(rows) * fields;
    SFB_CHECK(n <= v->scratch.cap, "batch larger than the VSI context's max_ids");
    CUDA_CHECK(cudaSetDevice(v->device));
    cudaStream_t s = v->stream;
    CUDA_CHECK(cudaMemsetAsync(v->d_scal, 0, sizeof(int32_t) * 4, s));
    CUDA_CHECK(cudaMemcpyAsync(v->d_in, features, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
    if (v->scratch.key_space == 0) {  // arbitrary u64 ids: hashed first-position table
      sfb::vsi_device_hashed(v->scratch, v->d_in, n, v->d_out64, v->d_vids, v->d_scal, s);
      int32_t u = 0;
      CUDA_CHECK(cudaMemcpyAsync(&u, v->d_scal, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      CUDA_CHECK(cudaMemcpyAsync(global_ids, v->d_out64, sizeof(uint64_t) * u,
                                 cudaMemcpyDeviceToHost, s));
      sfb::u32_to_u64(v->d_vids, v->d_in, n, s);
      CUDA_CHECK(cudaMemcpyAsync(virtual_ids, v->d_in, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost,
                                 s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      *unique_count = u;
      if (row_ranges) {
        const int per = rows / num_workers;  // vsi.cpp:48-52
        for (int w = 0; w < num_workers; ++w) {
          row_ranges[2 * w] = w * per;
          row_ranges[2 * w + 1] = (w + 1) * per;
        }
      }
      return;
    }
    sfb::ids_to_u32(v->d_in, v->d_ids, n, v->scratch.key_space, v->d_scal + 1, s);
    int32_t bad = 0;
    CUDA_CHECK(cudaMemcpyAsync(&bad, v->d_scal + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    SFB_CHECK(!bad, "feature id outside the VSI key space");
    sfb::vsi_device(v->scratch, v->d_ids, n, v->d_gids, v->d_vids, v->d_scal, s);
    int32_t u = 0;
    CUDA_CHECK(cudaMemcpyAsync(&u, v->d_scal, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    sfb::u32_to_u64(v->d_gids, v->d_out64, u, s);
    CUDA_CHECK(cudaMemcpyAsync(global_ids, v->d_out64, sizeof(uint64_t) * u, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    sfb::u32_to_u64(v->d_vids, v->d_out64, n, s);
    CUDA_CHECK(cudaMemcpyAsync(virtual_ids, v->d_out64, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    *unique_count = u;
    if (row_ranges) {
      const int per = rows / num_workers;  // vsi.cpp:48-52
      for (int w = 0; w < num_workers; ++w) {
        row_ranges[2 * w] = w * per;
        row_ranges[2 * w + 1] = (w + 1) * per;
      }
    }
  });
}

int sfctr_virtual_sparse_id_device(sfctr_vsi* v, const uint32_t* d_ids, int64_t n,
                                   uint32_t* d_global_ids, uint32_t* d_virtual_ids,
                                   int32_t* d_unique, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(v->device));
    SFB_CHECK(v->scratch.key_space > 0, "the u32 device entry needs a context with a key space");
    sfb::vsi_device(v->scratch, d_ids, n, d_global_ids, d_virtual_ids, d_unique,
                    static_cast<cudaStream_t>(stream));
  });
}

// ---------------- trainer ----------------
int sfctr_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    NCCL_CHECK(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
  });
}

int sfctr_trainer_create(const sfctr_config* cfg, int32_t rank, int32_t world,
                         const uint8_t* nccl_id, int device, sfctr_trainer** out) {
  *out = nullptr;
  return guarded([&] {
    auto t = std::make_unique<sfctr_trainer>();
    t->t = std::make_unique<sfb::Trainer>(*cfg, rank, world, nccl_id, device);
    *out = t.release();
  });
}

void sfctr_trainer_destroy(sfctr_trainer* t) { delete t; }

// ---- standalone device CacheBuffer + HostStore + manager (cachebuf.h) ----
int sfctr_cache_create(uint64_t capacity, int32_t dim, uint64_t seed, uint64_t key_space,
                       int32_t num_workers, int32_t worker, int64_t max_batch,
                       uint64_t host_reserve, int device, sfctr_cache** out) {
  return guarded([&] {
    SFB_CHECK(out != nullptr, "out");
    auto* c = new sfctr_cache;
    try {
      c->c = std::make_unique<sfb::DeviceCache>(capacity, dim, seed, key_space, num_workers,
                                                worker, max_batch, host_reserve, device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}
void sfctr_cache_destroy(sfctr_cache* c) { delete c; }
int sfctr_cache_admit(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t step,
                      uint64_t* slots) {
  return guarded([&] { c->c->admit(n, features, step, slots); });
}
int sfctr_cache_evict(sfctr_cache* c, int64_t n, const uint64_t* features) {
  return guarded([&] { c->c->evict(n, features); });
}
int sfctr_cache_touch(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t step) {
  return guarded([&] { c->c->touch(n, features, step); });
}
int sfctr_cache_pin(sfctr_cache* c, int64_t n, const uint64_t* features, int32_t pinned) {
  return guarded([&] { c->c->pin(n, features, pinned != 0); });
}
int sfctr_cache_set_needed_soon(sfctr_cache* c, int64_t n, const uint64_t* features,
                                int32_t value) {
  return guarded([&] { c->c->set_needed_soon(n, features, value != 0); });
}
int sfctr_cache_slot_of(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t* slots) {
  return guarded([&] { c->c->slot_of(n, features, slots); });
}
int sfctr_cache_free_count(sfctr_cache* c, uint64_t* out) {
  return guarded([&] { *out = c->c->free_count(); });
}
int sfctr_cache_slots(sfctr_cache* c, uint64_t* feature, int64_t* last_use, uint64_t* admit_seq,
                      uint8_t* pinned, uint8_t* needed_soon) {
  return guarded([&] { c->c->slots(feature, last_use, admit_seq, pinned, needed_soon); });
}
int sfctr_cache_occupancy(sfctr_cache* c, uint64_t out[5]) {
  return guarded([&] { c->c->occupancy(out); });
}
int sfctr_cache_occupancy_diagnostics(sfctr_cache* c, char* buf, size_t cap) {
  return guarded([&] {
    const std::string d = c->c->occupancy_diagnostics();
    if (buf && cap) {
      std::strncpy(buf, d.c_str(), cap - 1);
      buf[cap - 1] = 0;
    }
  });
}
int sfctr_cache_peek(sfctr_cache* c, int64_t n, const uint64_t* features, float* rows,
                     int64_t* steps) {
  return guarded([&] { c->c->peek(n, features, rows, steps); });
}
int sfctr_cache_prepare(sfctr_cache* c, int64_t step, int64_t n_global, const uint64_t* global_ids,
                        int64_t n_window, const uint64_t* window_ids, int64_t out[5]) {
  return guarded([&] { c->c->prepare(step, n_global, global_ids, n_window, window_ids, out); });
}

int sfctr_trainer_step(sfctr_trainer* t, int64_t step, const uint64_t* features,
                       const uint8_t* labels, const uint64_t* window, double* loss) {
  return guarded([&] {
    const double l = t->t->step_host(step, features, labels, window);
    if (!std::isfinite(l)) sfb::fail(sfb::kRun, "non-finite loss", step);
    if (loss) *loss = l;
  });
}

int sfctr_trainer_step_device(sfctr_trainer* t, int64_t step, const uint64_t* d_features,
                              const uint8_t* d_labels, const uint64_t* d_window, float* d_loss) {
  return guarded([&] { t->t->step_device(step, d_features, d_labels, d_window, d_loss); });
}

int sfctr_trainer_prepare(sfctr_trainer* t, int64_t step, const uint64_t* d_features,
                          const uint64_t* d_window) {
  return guarded([&] { t->t->prepare(step, d_features, d_window); });
}

int sfctr_trainer_train(sfctr_trainer* t, int64_t step, const uint8_t* d_labels, float* d_loss) {
  return guarded([&] { t->t->train(step, d_labels, d_loss); });
}

int sfctr_trainer_submit(sfctr_trainer* t, int64_t step, const uint64_t* features,
                         const uint8_t* labels, const uint64_t* window) {
  return guarded([&] { t->t->submit_host(step, features, labels, window); });
}

int sfctr_trainer_loss(sfctr_trainer* t, int64_t step, double* loss) {
  return guarded([&] {
    const double l = t->t->loss_of(step);
    if (!std::isfinite(l)) sfb::fail(sfb::kRun, "non-finite loss", step);
    if (loss) *loss = l;
  });
}

int sfctr_trainer_synchronize(sfctr_trainer* t) {
  return guarded([&] { t->t->synchronize(); });
}

void* sfctr_trainer_stream(sfctr_trainer* t) { return t->t->stream(); }

int sfctr_trainer_logits(sfctr_trainer* t, float* out) {
  return guarded([&] { t->t->logits(out); });
}

int sfctr_trainer_cache_slots(sfctr_trainer* t, int32_t lane, uint64_t* feature, int64_t* last_use,
                              uint64_t* admit_seq) {
  return guarded([&] {
    SFB_CHECK(lane >= 0 && lane < t->t->lanes(), "lane out of range");
    t->t->cache_slots(lane, feature, last_use, admit_seq);
  });
}

int sfctr_trainer_cache_slots_range(sfctr_trainer* t, int32_t lane, uint64_t first, uint64_t count,
                                    uint64_t* feature, int64_t* last_use, uint64_t* admit_seq) {
  return guarded([&] {
    SFB_CHECK(lane >= 0 && lane < t->t->lanes(), "lane out of range");
    t->t->cache_slots(lane, feature, last_use, admit_seq, first, count);
  });
}

int sfctr_trainer_peek_rows(sfctr_trainer* t, int64_t n, const uint64_t* features, float* rows,
                            int64_t* steps) {
  return guarded([&] {
    SFB_CHECK(n >= 0 && (n == 0 || features), "features");
    t->t->peek_rows(n, features, rows, steps);
  });
}

int sfctr_trainer_dense_state(sfctr_trainer* t, float* params, float* m, float* v,
                              int64_t* step) {
  return guarded([&] { t->t->dense_state(params, m, v, step); });
}

int sfctr_trainer_free_count(sfctr_trainer* t, int32_t lane, uint64_t* out) {
  return guarded([&] {
    SFB_CHECK(lane >= 0 && lane < t->t->lanes(), "lane out of range");
    *out = t->t->free_count(lane);
  });
}

int sfctr_trainer_snapshot(sfctr_trainer* t, int64_t* count, uint64_t* features, float* rows,
                           int64_t* steps) {
  return guarded([&] { *count = t->t->snapshot(features, rows, steps); });
}

int sfctr_trainer_get_dense(sfctr_trainer* t, float* w1, float* b1, float* w2, float* b2) {
  return guarded([&] { t->t->get_dense(w1, b1, w2, b2); });
}

int sfctr_trainer_set_dense(sfctr_trainer* t, const float* w1, const float* b1, const float* w2,
                            const float* b2) {
  return guarded([&] { t->t->set_dense(w1, b1, w2, b2); });
}

int sfctr_trainer_ledger(sfctr_trainer* t, int64_t out[4]) {
  return guarded([&] { t->t->ledger(out); });
}

int sfctr_trainer_stats(sfctr_trainer* t, sfctr_step_stats* out) {
  return guarded([&] { *out = t->t->stats(); });
}

int sfctr_trainer_set_timing(sfctr_trainer* t, int enabled) {
  return guarded([&] { t->t->set_timing(enabled != 0); });
}

int sfctr_trainer_phase_times(sfctr_trainer* t, int32_t max_phases, char* names, float* ms,
                              int32_t* n_phases) {
  return guarded([&] {
    const auto& p = t->t->phase_times();
    const int n = std::min<int>(max_phases, static_cast<int>(p.size()));
    for (int i = 0; i < n; ++i) {
      std::strncpy(names + 32 * i, p[i].first.c_str(), 31);
      names[32 * i + 31] = 0;
      ms[i] = p[i].second;
    }
    *n_phases = static_cast<int32_t>(p.size());
  });
}

// ---------------- standalone model op ----------------
int sfctr_model_forward_backward(int device, int32_t rows, int32_t fields, int32_t dim,
                                 int32_t hidden, const float* x, const uint8_t* labels,
                                 const float* w1, const float* b1, const float* w2,
                                 const float* b2, double* loss, float* logits, float* dx,
                                 float* dw1, float* db1, float* dw2, float* db2) {
  return guarded([&] {
    DeviceScope ds(device);
    SFB_CHECK(rows > 0 && fields > 0 && dim > 0 && hidden > 0, "bad model shape");
    const int K = fields * dim, H = hidden;
    const size_t P = static_cast<size_t>(K) * H + 2 * H + 1;
    const int ldx = sfb::tower_ldx(K);
    const size_t rk = static_cast<size_t>(rows) * ldx;
    float *d_x, *d_dx, *d_dense, *d_g, *d_s, *d_sq, *d_lg;
    uint8_t* d_y;
    CUDA_CHECK(cudaMalloc(&d_x, sizeof(float) * rk));
    CUDA_CHECK(cudaMalloc(&d_dx, sizeof(float) * rk));
    CUDA_CHECK(cudaMalloc(&d_dense, sizeof(float) * P));
    CUDA_CHECK(cudaMalloc(&d_g, sizeof(float) * (P + 1)));
    CUDA_CHECK(cudaMalloc(&d_s, sizeof(float) * rows * dim));
    CUDA_CHECK(cudaMalloc(&d_sq, sizeof(float) * rows * dim));
    CUDA_CHECK(cudaMalloc(&d_lg, sizeof(float) * rows));
    CUDA_CHECK(cudaMalloc(&d_y, rows));
    CUDA_CHECK(cudaMemset(d_x, 0, sizeof(float) * rk));
    CUDA_CHECK(cudaMemcpy2D(d_x, sizeof(float) * ldx, x, sizeof(float) * K, sizeof(float) * K, rows,
                            cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(d_y, labels, rows, cudaMemcpyHostToDevice));
    const size_t kh = static_cast<size_t>(K) * H;
    CUDA_CHECK(cudaMemcpy(d_dense, w1, sizeof(float) * kh, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(d_dense + kh, b1, sizeof(float) * H, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(d_dense + kh + H, w2, sizeof(float) * H, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(d_dense + kh + 2 * H, b2, sizeof(float), cudaMemcpyHostToDevice));
    sfb::TowerBufs tb;
    sfb::TowerTC tt;
    tb.init(rows, K, H, dim);
    tt.init(rows, K, H, dim);
    sfb::fm_sums(d_x, rows, fields, dim, ldx, d_s, d_sq, nullptr);
    sfb::tower_forward_backward_tc(tb, tt, d_x, ldx, d_s, d_sq, d_y, rows, fields, dim, d_dense,
                                   d_lg, d_dx, 1.f, d_g, false, nullptr);
    sfb::fm_grad_add(d_x, rows, fields, dim, ldx, d_s, tb.gz, 1.f, d_dx, nullptr);
    CUDA_CHECK(cudaDeviceSynchronize());
    std::vector<float> g(P + 1);
    CUDA_CHECK(cudaMemcpy(g.data(), d_g, sizeof(float) * (P + 1), cudaMemcpyDeviceToHost));
    if (loss) *loss = g[P];
    if (logits) CUDA_CHECK(cudaMemcpy(logits, d_lg, sizeof(float) * rows, cudaMemcpyDeviceToHost));
    if (dx)
      CUDA_CHECK(cudaMemcpy2D(dx, sizeof(float) * K, d_dx, sizeof(float) * ldx, sizeof(float) * K,
                              rows, cudaMemcpyDeviceToHost));
    if (dw1) std::memcpy(dw1, g.data(), sizeof(float) * kh);
    if (db1) std::memcpy(db1, g.data() + kh, sizeof(float) * H);
    if (dw2) std::memcpy(dw2, g.data() + kh + H, sizeof(float) * H);
    if (db2) *db2 = g[kh + 2 * H];
    tt.release();
    tb.release();
    for (void* p : {static_cast<void*>(d_x), static_cast<void*>(d_dx), static_cast<void*>(d_dense),
                    static_cast<void*>(d_g), static_cast<void*>(d_s), static_cast<void*>(d_sq),
                    static_cast<void*>(d_lg), static_cast<void*>(d_y)})
      cudaFree(p);
  });
}

}  // extern "C"
