/*
 * TEST INFRASTRUCTURE ONLY — the CPU parity oracle (see sfctr_oracle.h).
 *
 * Plain C11 restatement of the reference path in fp64. Every function cites
 * the reference file:line (paths relative to /root/reference/proj/core/ for
 * the C++ sources, /root/reference/ for SPEC.md) it follows. The product
 * never links this file.
 */
#include "sfctr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[512];
const char* orc_last_error(void) { return g_err; }

/* ======================= rng.hpp:27-84 ======================= */

uint64_t orc_fnv1a64(const char* bytes, size_t n) { /* rng.hpp:27-34 */
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= (uint8_t)bytes[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

static inline uint64_t splitmix64_next(uint64_t* state) { /* rng.hpp:36-42 */
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t orc_derive_seed(uint64_t base, const char* label, uint64_t index) { /* rng.hpp:49-56 */
  uint64_t state = base ^ orc_fnv1a64(label, strlen(label));
  state ^= 0x9e3779b97f4a7c15ull * (index + 1);
  uint64_t out = splitmix64_next(&state);
  out = splitmix64_next(&state) ^ out;
  return out;
}

/* Rng::next_unit / next_uniform / next_bernoulli (rng.hpp:67-80) */
static inline double rng_unit(uint64_t* st) {
  return (double)(splitmix64_next(st) >> 11) * 0x1.0p-53;
}
static inline double rng_uniform(uint64_t* st, double lo, double hi) {
  return lo + (hi - lo) * rng_unit(st);
}

double orc_truth_weight(uint64_t seed, uint64_t feature) { /* generator.cpp:77-80 */
  uint64_t st = orc_derive_seed(seed, "truth", feature);
  return rng_uniform(&st, -1.0, 1.0);
}

void orc_initial_embedding(uint64_t seed, uint64_t feature, int dim, double* out) {
  /* generator.cpp:110-115 */
  uint64_t st = orc_derive_seed(seed, "embed", feature);
  for (int i = 0; i < dim; ++i) out[i] = rng_uniform(&st, -0.01, 0.01);
}

int64_t orc_allreduce_bytes(int64_t payload, int workers) { /* comm.hpp:36-41 */
  if (workers < 1 || payload < 0) return -1;
  const int64_t w = workers;
  return 2 * (w - 1) * payload / w;
}

/* ======================= generator.cpp:32-108 ======================= */

struct orc_gen {
  int rows, fields;
  uint64_t vocab, seed, base;
  double zipf;
  uint64_t* shard_starts; /* fields + 1 */
  double* cdf_base;       /* shard size == base */
  double* cdf_big;        /* shard size == base + 1 (may be NULL) */
};

static double* build_cdf(uint64_t k, double s) { /* generator.cpp:52-61 */
  double* cdf = (double*)malloc(sizeof(double) * (k ? k : 1));
  double total = 0;
  for (uint64_t i = 0; i < k; ++i) {
    total += pow((double)(i + 1), -s);
    cdf[i] = total;
  }
  for (uint64_t i = 0; i < k; ++i) cdf[i] /= total;
  return cdf;
}

orc_gen* orc_gen_create(int global_rows, int fields, uint64_t vocab, uint64_t seed, double zipf) {
  if (vocab < (uint64_t)fields) return NULL; /* generator.cpp:35-36 */
  orc_gen* g = (orc_gen*)calloc(1, sizeof(orc_gen));
  g->rows = global_rows;
  g->fields = fields;
  g->vocab = vocab;
  g->seed = seed;
  g->zipf = zipf;
  g->shard_starts = (uint64_t*)malloc(sizeof(uint64_t) * (fields + 1));
  const uint64_t base = vocab / fields, rem = vocab % fields; /* generator.cpp:40-46 */
  g->base = base;
  g->shard_starts[0] = 0;
  for (int f = 0; f < fields; ++f)
    g->shard_starts[f + 1] = g->shard_starts[f] + base + ((uint64_t)f < rem ? 1 : 0);
  g->cdf_base = build_cdf(base, zipf);
  g->cdf_big = rem ? build_cdf(base + 1, zipf) : NULL;
  return g;
}

void orc_gen_destroy(orc_gen* g) {
  if (!g) return;
  free(g->shard_starts);
  free(g->cdf_base);
  free(g->cdf_big);
  free(g);
}

uint64_t orc_gen_shard_start(const orc_gen* g, int field) { return g->shard_starts[field]; }

static uint64_t sample_rank(const orc_gen* g, double unit, int field) { /* generator.cpp:70-75 */
  const uint64_t k = g->shard_starts[field + 1] - g->shard_starts[field];
  const double* cdf = (k == g->base) ? g->cdf_base : g->cdf_big;
  /* std::upper_bound: first index with cdf[i] > unit */
  uint64_t lo = 0, hi = k;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (cdf[mid] > unit) hi = mid;
    else lo = mid + 1;
  }
  if (lo == k) --lo;
  return lo;
}

void orc_gen_generate_rows(const orc_gen* g, int64_t step, int row0, int nrows, uint64_t* features,
                           uint8_t* labels) {
  /* generator.cpp:82-108. The reference draws one sequential Rng stream,
   * F+1 draws per row; splitmix64 is counter based, so row r's stream starts
   * at state seed_b + r*(F+1)*golden (random access). */
  const int F = g->fields;
  const uint64_t seed_b = orc_derive_seed(g->seed, "batch", (uint64_t)step);
  const double truth_scale = 2.5 / sqrt((double)F); /* generator.cpp:28,93 */
  for (int i = 0; i < nrows; ++i) {
    const int r = row0 + i;
    uint64_t st = seed_b + (uint64_t)r * (uint64_t)(F + 1) * 0x9e3779b97f4a7c15ull;
    double logit = 0;
    for (int f = 0; f < F; ++f) {
      const uint64_t rank = sample_rank(g, rng_unit(&st), f);
      const uint64_t feat = g->shard_starts[f] + rank;
      features[(size_t)i * F + f] = feat;
      logit += orc_truth_weight(g->seed, feat);
    }
    const double p = 1.0 / (1.0 + exp(-truth_scale * logit));
    labels[i] = rng_unit(&st) < p ? 1 : 0;
  }
}

/* ======================= u64 -> i64 hash map (linear probing) ======================= */

typedef struct {
  uint64_t* keys;
  int64_t* vals;
  uint8_t* used;
  size_t cap, size;
} hmap;

static inline uint64_t hmix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  return x;
}

static void hm_init(hmap* m, size_t want) {
  size_t cap = 16;
  while (cap < want * 2) cap <<= 1;
  m->cap = cap;
  m->size = 0;
  m->keys = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  m->vals = (int64_t*)malloc(sizeof(int64_t) * cap);
  m->used = (uint8_t*)calloc(cap, 1);
}
static void hm_free(hmap* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
}
static int64_t* hm_find(const hmap* m, uint64_t k) {
  size_t i = hmix(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) return &m->vals[i];
    i = (i + 1) & (m->cap - 1);
  }
  return NULL;
}
static void hm_put(hmap* m, uint64_t k, int64_t v);
static void hm_grow(hmap* m) {
  hmap n;
  hm_init(&n, m->cap);
  for (size_t i = 0; i < m->cap; ++i)
    if (m->used[i]) hm_put(&n, m->keys[i], m->vals[i]);
  hm_free(m);
  *m = n;
}
/* inserts or overwrites */
static void hm_put(hmap* m, uint64_t k, int64_t v) {
  if ((m->size + 1) * 2 > m->cap) hm_grow(m);
  size_t i = hmix(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) {
      m->vals[i] = v;
      return;
    }
    i = (i + 1) & (m->cap - 1);
  }
  m->used[i] = 1;
  m->keys[i] = k;
  m->vals[i] = v;
  m->size++;
}
/* backward-shift deletion */
static int hm_erase(hmap* m, uint64_t k) {
  size_t i = hmix(k) & (m->cap - 1);
  while (m->used[i] && m->keys[i] != k) i = (i + 1) & (m->cap - 1);
  if (!m->used[i]) return 0;
  size_t j = i;
  for (;;) {
    j = (j + 1) & (m->cap - 1);
    if (!m->used[j]) break;
    size_t home = hmix(m->keys[j]) & (m->cap - 1);
    /* can entry j move into hole i? yes unless home lies cyclically in (i, j] */
    int in_range = (i <= j) ? (home > i && home <= j) : (home > i || home <= j);
    if (in_range) continue;
    m->keys[i] = m->keys[j];
    m->vals[i] = m->vals[j];
    i = j;
  }
  m->used[i] = 0;
  m->size--;
  return 1;
}

/* ======================= vsi.cpp:23-54 ======================= */

int64_t orc_vsi(const uint64_t* features, int rows, int fields, int workers, uint64_t* global_ids,
                uint64_t* virtual_ids) {
  if (!(rows > 0 && fields > 0)) { /* vsi.cpp:24 */
    snprintf(g_err, sizeof g_err, "empty batch");
    return -3;
  }
  if (!(workers > 0 && rows % workers == 0)) { /* vsi.cpp:30-31 */
    snprintf(g_err, sizeof g_err, "rows must split evenly across workers");
    return -3;
  }
  const size_t n = (size_t)rows * fields;
  hmap first;
  hm_init(&first, n);
  int64_t u = 0;
  for (size_t i = 0; i < n; ++i) { /* vsi.cpp:41-46: first-appearance order */
    int64_t* v = hm_find(&first, features[i]);
    if (!v) {
      hm_put(&first, features[i], u);
      global_ids[u] = features[i];
      virtual_ids[i] = (uint64_t)u;
      ++u;
    } else {
      virtual_ids[i] = (uint64_t)*v;
    }
  }
  hm_free(&first);
  return u;
}

/* ======================= DeepFM-lite ======================= */

static void uniform_stream(uint64_t seed, const char* label, double a, double* out, size_t n) {
  uint64_t st = orc_derive_seed(seed, label, 0);
  for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&st, -a, a);
}

void orc_dense_init(uint64_t seed, int K, int h, double* w1, double* b1, double* w2, double* b2) {
  uniform_stream(seed, "dense_w1", sqrt(6.0 / (double)(K + h)), w1, (size_t)K * h);
  uniform_stream(seed, "dense_w2", sqrt(6.0 / (double)(h + 1)), w2, (size_t)h);
  for (int j = 0; j < h; ++j) b1[j] = 0;
  *b2 = 0;
}

#define ORC_CHUNKS 16 /* fixed row chunks: summation order independent of threads */
#define P_CLAMP 1e-7

/* dxabs / dabs (tests only, may be NULL): the same sums over |terms| — the condition
 * scale of every gradient entry (dxabs [rows, F*d]; dabs [P] = |W1| | |b1| | |w2| | |b2|
 * parts, summed over rows and divided like the gradients).
 * dxamb / damb (with dxabs / dabs): the gradient mass behind ReLU decisions that fp32 does
 * not determine — hidden units with |hpre| <= 1e-5 (|b1| + sum_k |x_k w_kj|), whose
 * derivative may legitimately come out either way on the device: sum of |gz w2_j w_kj|
 * (dx) and |x_k gz w2_j|, |gz w2_j| (W1, b1) over those units. *n_amb counts them. */
#define AMB_RTOL 1e-5
static double model_core(const double* x, const uint8_t* labels, int rows, int fields, int dim,
                         int hidden, const double* w1, const double* b1, const double* w2,
                         double b2, double* logits, double* dx, double* dw1, double* db1,
                         double* dw2, double* db2, int num_threads, double* dxabs, double* dabs,
                         double* dxamb, double* damb, int64_t* n_amb) {
  const int K = fields * dim, H = hidden;
  const int want_dense = (dw1 != NULL);
  const int want_abs = want_dense && dabs != NULL;
  double loss_chunk[ORC_CHUNKS] = {0};
  double* pw1 = want_dense ? (double*)calloc((size_t)ORC_CHUNKS * K * H, sizeof(double)) : NULL;
  double* pv = want_dense ? (double*)calloc((size_t)ORC_CHUNKS * (2 * H + 1), sizeof(double)) : NULL;
  double* paw1 = want_abs ? (double*)calloc((size_t)ORC_CHUNKS * K * H, sizeof(double)) : NULL;
  double* pav = want_abs ? (double*)calloc((size_t)ORC_CHUNKS * (2 * H + 1), sizeof(double)) : NULL;
  double* pmw1 = want_abs ? (double*)calloc((size_t)ORC_CHUNKS * K * H, sizeof(double)) : NULL;
  double* pmv = want_abs ? (double*)calloc((size_t)ORC_CHUNKS * H, sizeof(double)) : NULL;
  int64_t amb_chunk[ORC_CHUNKS] = {0};
  const double inv_rows = 1.0 / (double)rows;
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int c = 0; c < ORC_CHUNKS; ++c) {
    const int r0 = (int)((int64_t)rows * c / ORC_CHUNKS), r1 = (int)((int64_t)rows * (c + 1) / ORC_CHUNKS);
    double* hpre = (double*)malloc(sizeof(double) * H);
    double* dh = (double*)malloc(sizeof(double) * H);
    double* s = (double*)malloc(sizeof(double) * dim);
    double* sa = (double*)malloc(sizeof(double) * dim);
    double* hsc = (double*)malloc(sizeof(double) * H);
    double* da = (double*)malloc(sizeof(double) * H); /* |gz w2_j| of ambiguous units, else 0 */
    double lsum = 0;
    for (int r = r0; r < r1; ++r) {
      const double* xr = x + (size_t)r * K;
      /* MLP hidden: h = b1 + x.W1 (k ascending) */
      for (int j = 0; j < H; ++j) hpre[j] = b1[j];
      for (int k = 0; k < K; ++k) {
        const double xv = xr[k];
        const double* wk = w1 + (size_t)k * H;
        for (int j = 0; j < H; ++j) hpre[j] += xv * wk[j];
      }
      double mlp = b2;
      for (int j = 0; j < H; ++j) mlp += (hpre[j] > 0 ? hpre[j] : 0) * w2[j];
      /* FM second order: sum_{i<j} <v_i,v_j> = 0.5 (|sum v|^2 - sum |v|^2) */
      double sq = 0;
      for (int c2 = 0; c2 < dim; ++c2) s[c2] = sa[c2] = 0;
      for (int f = 0; f < fields; ++f)
        for (int c2 = 0; c2 < dim; ++c2) {
          const double v = xr[f * dim + c2];
          s[c2] += v;
          sa[c2] += fabs(v);
          sq += v * v;
        }
      double ss = 0;
      for (int c2 = 0; c2 < dim; ++c2) ss += s[c2] * s[c2];
      const double fm = 0.5 * (ss - sq);
      const double z = fm + mlp;
      if (logits) logits[r] = z;
      const double p = 1.0 / (1.0 + exp(-z));
      const double y = labels[r] ? 1.0 : 0.0;
      const int clamped = (p < P_CLAMP) || (p > 1.0 - P_CLAMP);
      const double pc = p < P_CLAMP ? P_CLAMP : (p > 1.0 - P_CLAMP ? 1.0 - P_CLAMP : p);
      lsum += -(y * log(pc) + (1.0 - y) * log(1.0 - pc));
      /* d(mean loss)/dz; zero where the clamp is active */
      const double gz = clamped ? 0.0 : (p - y) * inv_rows;
      for (int j = 0; j < H; ++j) dh[j] = hpre[j] > 0 ? gz * w2[j] : 0.0;
      int any_amb = 0;
      if (dxabs) {
        for (int j = 0; j < H; ++j) hsc[j] = fabs(b1[j]);
        for (int k = 0; k < K; ++k) {
          const double xv = fabs(xr[k]);
          const double* wk = w1 + (size_t)k * H;
          for (int j = 0; j < H; ++j) hsc[j] += xv * fabs(wk[j]);
        }
        for (int j = 0; j < H; ++j) {
          const int amb = fabs(hpre[j]) <= AMB_RTOL * hsc[j];
          da[j] = amb ? fabs(gz * w2[j]) : 0.0;
          any_amb |= amb && da[j] > 0;
          amb_chunk[c] += amb;
        }
      }
      if (dx) {
        double* dxr = dx + (size_t)r * K;
        for (int k = 0; k < K; ++k) {
          const double* wk = w1 + (size_t)k * H;
          double acc = 0;
          for (int j = 0; j < H; ++j) acc += dh[j] * wk[j];
          const int c2 = k % dim;
          dxr[k] = acc + gz * (s[c2] - xr[k]);
          if (dxabs) {
            double aa = 0, am = 0;
            for (int j = 0; j < H; ++j) aa += fabs(dh[j] * wk[j]);
            if (any_amb)
              for (int j = 0; j < H; ++j) am += da[j] * fabs(wk[j]);
            dxabs[(size_t)r * K + k] = aa + fabs(gz) * (sa[c2] + fabs(xr[k]));
            dxamb[(size_t)r * K + k] = am;
          }
        }
      }
      if (want_dense) {
        double* cw1 = pw1 + (size_t)c * K * H;
        double* cv = pv + (size_t)c * (2 * H + 1);
        for (int k = 0; k < K; ++k) {
          const double xv = xr[k];
          double* wk = cw1 + (size_t)k * H;
          for (int j = 0; j < H; ++j) wk[j] += xv * dh[j];
        }
        for (int j = 0; j < H; ++j) {
          cv[j] += dh[j];                                       /* db1 */
          cv[H + j] += gz * (hpre[j] > 0 ? hpre[j] : 0);        /* dw2 */
        }
        cv[2 * H] += gz; /* db2 */
        if (want_abs) {
          double* aw1 = paw1 + (size_t)c * K * H;
          double* av = pav + (size_t)c * (2 * H + 1);
          for (int k = 0; k < K; ++k) {
            const double xv = fabs(xr[k]);
            double* wk = aw1 + (size_t)k * H;
            for (int j = 0; j < H; ++j) wk[j] += xv * fabs(dh[j]);
          }
          for (int j = 0; j < H; ++j) {
            av[j] += fabs(dh[j]);
            av[H + j] += fabs(gz) * (hpre[j] > 0 ? hpre[j] : 0);
          }
          av[2 * H] += fabs(gz);
          if (any_amb) {
            double* mw1 = pmw1 + (size_t)c * K * H;
            for (int k = 0; k < K; ++k) {
              const double xv = fabs(xr[k]);
              double* wk = mw1 + (size_t)k * H;
              for (int j = 0; j < H; ++j) wk[j] += xv * da[j];
            }
            double* mv = pmv + (size_t)c * H;
            for (int j = 0; j < H; ++j) mv[j] += da[j];
          }
        }
      }
    }
    loss_chunk[c] = lsum;
    free(hpre);
    free(dh);
    free(s);
    free(sa);
    free(hsc);
    free(da);
  }
  double loss = 0;
  for (int c = 0; c < ORC_CHUNKS; ++c) loss += loss_chunk[c];
  if (want_dense) {
    memset(dw1, 0, sizeof(double) * K * H);
    if (db1) memset(db1, 0, sizeof(double) * H);
    if (dw2) memset(dw2, 0, sizeof(double) * H);
    if (db2) *db2 = 0;
    for (int c = 0; c < ORC_CHUNKS; ++c) {
      const double* cw1 = pw1 + (size_t)c * K * H;
      for (size_t i = 0; i < (size_t)K * H; ++i) dw1[i] += cw1[i];
      const double* cv = pv + (size_t)c * (2 * H + 1);
      for (int j = 0; j < H; ++j) {
        if (db1) db1[j] += cv[j];
        if (dw2) dw2[j] += cv[H + j];
      }
      if (db2) *db2 += cv[2 * H];
    }
    free(pw1);
    free(pv);
  }
  if (want_abs) {
    memset(dabs, 0, sizeof(double) * ((size_t)K * H + 2 * H + 1));
    memset(damb, 0, sizeof(double) * ((size_t)K * H + 2 * H + 1));
    for (int c = 0; c < ORC_CHUNKS; ++c) {
      const double* aw1 = paw1 + (size_t)c * K * H;
      const double* mw1 = pmw1 + (size_t)c * K * H;
      for (size_t i = 0; i < (size_t)K * H; ++i) {
        dabs[i] += aw1[i];
        damb[i] += mw1[i];
      }
      const double* av = pav + (size_t)c * (2 * H + 1);
      for (int j = 0; j < 2 * H + 1; ++j) dabs[(size_t)K * H + j] += av[j];
      const double* mv = pmv + (size_t)c * H;
      for (int j = 0; j < H; ++j) damb[(size_t)K * H + j] += mv[j];
    }
    free(paw1);
    free(pav);
    free(pmw1);
    free(pmv);
  }
  if (n_amb) {
    *n_amb = 0;
    for (int c = 0; c < ORC_CHUNKS; ++c) *n_amb += amb_chunk[c];
  }
  return loss * inv_rows;
}

double orc_model_fwd_bwd(const double* x, const uint8_t* labels, int rows, int fields, int dim,
                         int hidden, const double* w1, const double* b1, const double* w2,
                         double b2, double* logits, double* dx, double* dw1, double* db1,
                         double* dw2, double* db2, int num_threads) {
  return model_core(x, labels, rows, fields, dim, hidden, w1, b1, w2, b2, logits, dx, dw1, db1,
                    dw2, db2, num_threads, NULL, NULL, NULL, NULL, NULL);
}

/* ======================= HostStore / CacheBuffer / manager ======================= */

typedef struct {
  double* data; /* [emb | momentum | velocity], 3*dim — host_store.hpp:33-54 */
  int64_t steps;
} entry_t;

typedef struct { /* cache_buffer.hpp:42-50 */
  int occupied, pinned, needed_soon;
  uint64_t feature;
  int64_t last_use;
  uint64_t admit_seq;
  entry_t entry;
} slot_t;

typedef struct {
  slot_t* slots;
  uint64_t cap;
  hmap index;     /* feature -> slot */
  uint64_t* free_; /* LIFO free list, lower slots at the back (cache_buffer.cpp:27-28) */
  uint64_t nfree;
  uint64_t next_seq;
} cache_t;

typedef struct {
  hmap table; /* feature -> index into rows/steps pools */
  entry_t* pool;
  size_t pool_n, pool_cap;
  int64_t* free_ids;
  size_t nfree_ids, free_cap;
  int dim;
  uint64_t seed;
} host_t;

static void host_init(host_t* h, uint64_t seed, int dim) { /* host_store.cpp:23 */
  memset(h, 0, sizeof *h);
  hm_init(&h->table, 1024);
  h->dim = dim;
  h->seed = seed;
}
static void host_free(host_t* h) {
  for (size_t i = 0; i < h->table.cap; ++i)
    if (h->table.used[i]) free(h->pool[h->table.vals[i]].data);
  free(h->pool);
  free(h->free_ids);
  hm_free(&h->table);
}
/* HostStore::take (host_store.cpp:41-45) with lazy get_or_init (:25-33) */
static entry_t host_take(host_t* h, uint64_t f) {
  int64_t* v = hm_find(&h->table, f);
  entry_t e;
  if (!v) {
    e.data = (double*)calloc((size_t)3 * h->dim, sizeof(double));
    e.steps = 0;
    orc_initial_embedding(h->seed, f, h->dim, e.data);
    return e;
  }
  const int64_t id = *v;
  e = h->pool[id];
  hm_erase(&h->table, f);
  if (h->nfree_ids == h->free_cap) {
    h->free_cap = h->free_cap ? 2 * h->free_cap : 1024;
    h->free_ids = (int64_t*)realloc(h->free_ids, sizeof(int64_t) * h->free_cap);
  }
  h->free_ids[h->nfree_ids++] = id;
  return e;
}
/* HostStore::put (host_store.cpp:47-50): conservation */
static int host_put(host_t* h, uint64_t f, entry_t e) {
  if (hm_find(&h->table, f)) {
    snprintf(g_err, sizeof g_err, "feature %llu already host-resident (conservation violated)",
             (unsigned long long)f);
    return -1;
  }
  int64_t id;
  if (h->nfree_ids) id = h->free_ids[--h->nfree_ids];
  else {
    if (h->pool_n == h->pool_cap) {
      h->pool_cap = h->pool_cap ? 2 * h->pool_cap : 1024;
      h->pool = (entry_t*)realloc(h->pool, sizeof(entry_t) * h->pool_cap);
    }
    id = (int64_t)h->pool_n++;
  }
  h->pool[id] = e;
  hm_put(&h->table, f, id);
  return 0;
}

static void cache_init(cache_t* c, uint64_t cap) { /* cache_buffer.cpp:23-30 */
  c->cap = cap;
  c->slots = (slot_t*)calloc(cap, sizeof(slot_t));
  for (uint64_t i = 0; i < cap; ++i) c->slots[i].last_use = -1;
  c->free_ = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  c->nfree = 0;
  for (uint64_t i = cap; i-- > 0;) c->free_[c->nfree++] = i;
  hm_init(&c->index, cap);
  c->next_seq = 0;
}
static void cache_free(cache_t* c) {
  for (uint64_t i = 0; i < c->cap; ++i)
    if (c->slots[i].occupied) free(c->slots[i].entry.data);
  free(c->slots);
  free(c->free_);
  hm_free(&c->index);
}
static int64_t cache_slot_of(const cache_t* c, uint64_t f) {
  const int64_t* v = hm_find(&c->index, f);
  return v ? *v : -1;
}
/* CacheBuffer::admit (cache_buffer.cpp:38-53) */
static int64_t cache_admit(cache_t* c, uint64_t f, entry_t e, int64_t step) {
  if (c->nfree == 0) {
    snprintf(g_err, sizeof g_err, "admit with no free slot; evict first");
    return -1;
  }
  const uint64_t idx = c->free_[--c->nfree];
  slot_t* s = &c->slots[idx];
  s->occupied = 1;
  s->pinned = 0;
  s->needed_soon = 1;
  s->feature = f;
  s->last_use = step;
  s->admit_seq = c->next_seq++;
  s->entry = e;
  hm_put(&c->index, f, (int64_t)idx);
  return (int64_t)idx;
}
/* CacheBuffer::evict (cache_buffer.cpp:55-67) with the eviction-safety asserts */
static int cache_evict(cache_t* c, uint64_t f, entry_t* out) {
  const int64_t idx = cache_slot_of(c, f);
  if (idx < 0) {
    snprintf(g_err, sizeof g_err, "evicting non-resident feature %llu", (unsigned long long)f);
    return -1;
  }
  slot_t* s = &c->slots[idx];
  if (s->pinned || s->needed_soon) {
    snprintf(g_err, sizeof g_err, "evicting %s feature %llu",
             s->pinned ? "pinned" : "lookahead-needed", (unsigned long long)f);
    return -1;
  }
  *out = s->entry;
  s->occupied = 0;
  s->entry.data = NULL;
  c->free_[c->nfree++] = (uint64_t)idx;
  hm_erase(&c->index, f);
  return 0;
}

typedef struct {
  int64_t last_use;
  uint64_t admit_seq;
  uint64_t slot;
} victim_t;
static int victim_cmp(const void* a, const void* b) {
  const victim_t* x = (const victim_t*)a;
  const victim_t* y = (const victim_t*)b;
  if (x->last_use != y->last_use) return x->last_use < y->last_use ? -1 : 1;
  if (x->admit_seq != y->admit_seq) return x->admit_seq < y->admit_seq ? -1 : 1;
  return 0;
}

typedef struct {
  int64_t h2w, w2h, inter, swaps; /* ledger.hpp:60-63 */
} ledger_t;

/*
 * manager_get + pull_parameters_to_host + push_parameters_to_cache for one
 * worker, in the fixed order DESIGN.md §MixCache states:
 *  1. needed_soon := owned resident features of the window batches (cleared
 *     elsewhere);
 *  2. working := owned features of batch t not resident, in global_ids order;
 *     resident owned features are touched (cache_buffer.cpp:69-72);
 *  3. evict max(0, |working| - free) victims, the eligible slots
 *     (occupied, !pinned, !needed_soon) with the smallest (last_use,
 *     admit_seq), oldest first (host.put(evict(f)));
 *  4. admit working in order (admit(f, host.take(f), t)).
 * `owned` = owned features of batch t (global_ids order); `window` = owned
 * features of every window batch (t..t+L-1), duplicates allowed.
 * Returns number of evictions or -1 (LogicError) / -2 (capacity deadlock).
 */
static int64_t manage_worker(cache_t* c, host_t* h, ledger_t* led, int dim, int64_t step,
                             const uint64_t* owned, int64_t n_owned, const uint64_t* window,
                             int64_t n_window, uint64_t* evicted_out) {
  for (uint64_t i = 0; i < c->cap; ++i) c->slots[i].needed_soon = 0;
  for (int64_t i = 0; i < n_window; ++i) {
    const int64_t s = cache_slot_of(c, window[i]);
    if (s >= 0) c->slots[s].needed_soon = 1;
  }
  uint64_t* working = (uint64_t*)malloc(sizeof(uint64_t) * (n_owned ? n_owned : 1));
  int64_t nw = 0;
  for (int64_t i = 0; i < n_owned; ++i) {
    const int64_t s = cache_slot_of(c, owned[i]);
    if (s >= 0) {
      if (step > c->slots[s].last_use) c->slots[s].last_use = step;
    } else {
      working[nw++] = owned[i];
    }
  }
  int64_t need = nw - (int64_t)c->nfree;
  int64_t nev = 0;
  if (need > 0) {
    victim_t* el = (victim_t*)malloc(sizeof(victim_t) * c->cap);
    int64_t ne = 0;
    for (uint64_t i = 0; i < c->cap; ++i) {
      const slot_t* s = &c->slots[i];
      if (s->occupied && !s->pinned && !s->needed_soon)
        el[ne++] = (victim_t){s->last_use, s->admit_seq, i};
    }
    if (ne < need) {
      uint64_t pinned = 0, needed = 0, occ = 0;
      for (uint64_t i = 0; i < c->cap; ++i)
        if (c->slots[i].occupied) {
          ++occ;
          pinned += c->slots[i].pinned;
          needed += c->slots[i].needed_soon;
        }
      snprintf(g_err, sizeof g_err,
               "step %lld: capacity deadlock: need %lld slots, %lld evictable "
               "(capacity=%llu occupied=%llu free=%llu pinned=%llu needed_soon=%llu)",
               (long long)step, (long long)nw, (long long)(ne + c->nfree),
               (unsigned long long)c->cap, (unsigned long long)occ,
               (unsigned long long)c->nfree, (unsigned long long)pinned,
               (unsigned long long)needed);
      free(el);
      free(working);
      return -2;
    }
    qsort(el, (size_t)ne, sizeof(victim_t), victim_cmp);
    for (int64_t i = 0; i < need; ++i) {
      const uint64_t f = c->slots[el[i].slot].feature;
      entry_t e;
      if (cache_evict(c, f, &e) || host_put(h, f, e)) {
        free(el);
        free(working);
        return -1;
      }
      if (evicted_out) evicted_out[nev] = f;
      ++nev;
    }
    free(el);
    led->w2h += nev * dim * 12;
    led->swaps += nev;
  }
  for (int64_t i = 0; i < nw; ++i) {
    if (cache_admit(c, working[i], host_take(h, working[i]), step) < 0) {
      free(working);
      return -1;
    }
  }
  led->h2w += nw * dim * 12;
  free(working);
  return nev;
}

int64_t orc_manager_example(uint64_t capacity, const uint64_t* resident, int n_resident,
                            const uint64_t* pinned, int n_pinned, const uint64_t* next, int n_next,
                            uint64_t* slots_out, uint64_t* evicted_out) {
  cache_t c;
  host_t h;
  ledger_t led = {0, 0, 0, 0};
  cache_init(&c, capacity);
  host_init(&h, 7, 2);
  for (int i = 0; i < n_resident; ++i) cache_admit(&c, resident[i], host_take(&h, resident[i]), 0);
  for (int i = 0; i < n_pinned; ++i) {
    const int64_t s = cache_slot_of(&c, pinned[i]);
    if (s >= 0) c.slots[s].pinned = 1;
  }
  const int64_t nev = manage_worker(&c, &h, &led, 2, 1, next, n_next, next, n_next, evicted_out);
  for (uint64_t i = 0; i < capacity; ++i)
    slots_out[i] = c.slots[i].occupied ? c.slots[i].feature : UINT64_MAX;
  cache_free(&c);
  host_free(&h);
  return nev < 0 ? -1 : nev;
}

/* ======================= the simulated system ======================= */

void orc_config_default(orc_config* c) { /* config.hpp:44-71 */
  c->num_workers = 4;
  c->embedding_dim = 16;
  c->num_fields = 26;
  c->batch_size_per_worker = 256;
  c->vocabulary_size = 100000;
  c->cache_capacity = 8192;
  c->lookahead_depth = 1;
  c->seed = 7;
  c->learning_rate = 1e-3;
  c->adam_beta1 = 0.9;
  c->adam_beta2 = 0.999;
  c->adam_epsilon = 1e-8;
  c->zipf_exponent = 1.2;
  c->hidden_dim = 64;
  c->num_threads = 1;
}

struct orc_sim {
  orc_config cfg;
  int W, d, F, b, H, K;
  host_t host;
  cache_t* caches;
  ledger_t led;
  double *w1, *b1, *w2, b2;                    /* dense parameters */
  double *mw1, *vw1, *mb1, *vb1, *mw2, *vw2, mb2, vb2; /* dense Adam state */
  int64_t dense_steps;
  int64_t last_u;
  /* tests: the last step's summed gradients and their condition scales (sums of |terms|) */
  int keep_grads;
  double *last_g, *last_gabs, *last_dg, *last_dgabs, *last_gamb, *last_dgamb;
  int64_t last_amb;
};

orc_sim* orc_sim_create(const orc_config* cfg) {
  if (cfg->num_workers <= 0 || cfg->embedding_dim <= 0 || cfg->num_fields <= 0 ||
      cfg->batch_size_per_worker <= 0 || cfg->cache_capacity == 0 || cfg->hidden_dim <= 0 ||
      cfg->lookahead_depth <= 0) {
    snprintf(g_err, sizeof g_err, "invalid config");
    return NULL;
  }
  orc_sim* s = (orc_sim*)calloc(1, sizeof(orc_sim));
  s->cfg = *cfg;
  s->W = cfg->num_workers;
  s->d = cfg->embedding_dim;
  s->F = cfg->num_fields;
  s->b = cfg->batch_size_per_worker;
  s->H = cfg->hidden_dim;
  s->K = s->F * s->d;
  host_init(&s->host, cfg->seed, s->d);
  s->caches = (cache_t*)calloc(s->W, sizeof(cache_t));
  for (int w = 0; w < s->W; ++w) cache_init(&s->caches[w], cfg->cache_capacity);
  const size_t kh = (size_t)s->K * s->H;
  s->w1 = (double*)calloc(kh, sizeof(double));
  s->mw1 = (double*)calloc(kh, sizeof(double));
  s->vw1 = (double*)calloc(kh, sizeof(double));
  s->b1 = (double*)calloc(s->H, sizeof(double));
  s->mb1 = (double*)calloc(s->H, sizeof(double));
  s->vb1 = (double*)calloc(s->H, sizeof(double));
  s->w2 = (double*)calloc(s->H, sizeof(double));
  s->mw2 = (double*)calloc(s->H, sizeof(double));
  s->vw2 = (double*)calloc(s->H, sizeof(double));
  orc_dense_init(cfg->seed, s->K, s->H, s->w1, s->b1, s->w2, &s->b2);
  return s;
}

void orc_sim_destroy(orc_sim* s) {
  if (!s) return;
  free(s->last_g); free(s->last_gabs); free(s->last_dg); free(s->last_dgabs);
  free(s->last_gamb); free(s->last_dgamb);
  for (int w = 0; w < s->W; ++w) cache_free(&s->caches[w]);
  free(s->caches);
  host_free(&s->host);
  free(s->w1); free(s->mw1); free(s->vw1);
  free(s->b1); free(s->mb1); free(s->vb1);
  free(s->w2); free(s->mw2); free(s->vw2);
  free(s);
}

/* standard bias-corrected Adam on n values with step count t */
static void adam(double* theta, double* m, double* v, const double* g, size_t n, int64_t t,
                 const orc_config* c) {
  const double b1 = c->adam_beta1, b2 = c->adam_beta2;
  const double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  for (size_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    const double mh = m[i] / bc1, vh = v[i] / bc2;
    theta[i] -= c->learning_rate * mh / (sqrt(vh) + c->adam_epsilon);
  }
}

int orc_sim_step(orc_sim* s, int64_t step, const uint64_t* features, const uint8_t* labels,
                 const uint64_t* window_features, int window_batches, double* loss_out,
                 double* worker_losses, double* logits) {
  const int W = s->W, d = s->d, F = s->F, b = s->b, H = s->H, K = s->K;
  const int B = W * b;
  const size_t N = (size_t)B * F;
  int rc = 0;
  /* 1. VSI (Algorithm 1 l.3; vsi.cpp:23-54) */
  uint64_t* gids = (uint64_t*)malloc(sizeof(uint64_t) * N);
  uint64_t* vids = (uint64_t*)malloc(sizeof(uint64_t) * N);
  const int64_t U = orc_vsi(features, B, F, W, gids, vids);
  if (U < 0) {
    free(gids);
    free(vids);
    return 3;
  }
  s->last_u = U;
  /* window: owned features of batches t..t+L-1 (batch t itself first) */
  int nwin = 1 + (window_features ? window_batches : 0);
  uint64_t* wgids = (uint64_t*)malloc(sizeof(uint64_t) * N * nwin);
  int64_t wtot = 0;
  memcpy(wgids, gids, sizeof(uint64_t) * U);
  wtot = U;
  for (int j = 0; j + 1 < nwin; ++j) {
    uint64_t* tmpv = (uint64_t*)malloc(sizeof(uint64_t) * N);
    const int64_t u2 = orc_vsi(window_features + (size_t)j * N, B, F, W, wgids + wtot, tmpv);
    free(tmpv);
    if (u2 > 0) wtot += u2;
  }
  /* 2. manage each worker (Algorithm 1 l.4-7) */
  uint64_t* owned = (uint64_t*)malloc(sizeof(uint64_t) * (U ? U : 1));
  uint64_t* wowned = (uint64_t*)malloc(sizeof(uint64_t) * (wtot ? wtot : 1));
  for (int w = 0; w < W && rc == 0; ++w) {
    int64_t no = 0, nwo = 0;
    for (int64_t k = 0; k < U; ++k)
      if (gids[k] % (uint64_t)W == (uint64_t)w) owned[no++] = gids[k]; /* shard_owner */
    for (int64_t k = 0; k < wtot; ++k)
      if (wgids[k] % (uint64_t)W == (uint64_t)w) wowned[nwo++] = wgids[k];
    const int64_t r = manage_worker(&s->caches[w], &s->host, &s->led, d, step, owned, no, wowned,
                                    nwo, NULL);
    if (r == -2) rc = 4;
    else if (r < 0) rc = 3;
    /* pin the batch's owned features until update_sparse */
    for (int64_t i = 0; i < no && rc == 0; ++i)
      s->caches[w].slots[cache_slot_of(&s->caches[w], owned[i])].pinned = 1;
  }
  free(wgids);
  free(wowned);
  if (rc) {
    free(gids); free(vids); free(owned);
    return rc;
  }
  /* 3-4. gather_cache + forward all-reduce, ordered sum over workers.
   * Every row has exactly one nonzero contribution, so the sum equals the owner's row. */
  double* gce = (double*)calloc((size_t)U * d, sizeof(double));
  for (int w = 0; w < W; ++w)
    for (int64_t k = 0; k < U; ++k) {
      if (gids[k] % (uint64_t)W != (uint64_t)w) continue;
      const slot_t* sl = &s->caches[w].slots[cache_slot_of(&s->caches[w], gids[k])];
      for (int c = 0; c < d; ++c) gce[(size_t)k * d + c] += sl->entry.data[c];
    }
  s->led.inter += (int64_t)W * orc_allreduce_bytes(U * d * 4, W);
  /* 5-7. per worker: gather_instances, forward_backward, segment_sum */
  double* gcg = (double*)calloc((size_t)U * d, sizeof(double));
  double* lcg = (double*)malloc(sizeof(double) * (size_t)U * d);
  const size_t P = (size_t)K * H + 2 * H + 1;
  double* dsum = (double*)calloc(P, sizeof(double));
  double* dw = (double*)malloc(sizeof(double) * P);
  double* x = (double*)malloc(sizeof(double) * (size_t)b * K);
  double* dx = (double*)malloc(sizeof(double) * (size_t)b * K);
  const int ka = s->keep_grads;
  double* dxa = ka ? (double*)malloc(sizeof(double) * (size_t)b * K) : NULL;
  double* gca = ka ? (double*)calloc((size_t)U * d, sizeof(double)) : NULL;
  double* dwa = ka ? (double*)malloc(sizeof(double) * P) : NULL;
  double* dsa = ka ? (double*)calloc(P, sizeof(double)) : NULL;
  double* dxm = ka ? (double*)malloc(sizeof(double) * (size_t)b * K) : NULL;
  double* gcm = ka ? (double*)calloc((size_t)U * d, sizeof(double)) : NULL;
  double* dwm = ka ? (double*)malloc(sizeof(double) * P) : NULL;
  double* dsm = ka ? (double*)calloc(P, sizeof(double)) : NULL;
  int64_t amb_total = 0;
  double lossum = 0;
  for (int w = 0; w < W; ++w) {
    const int r0 = w * b; /* contiguous even split, vsi.cpp:48-52 */
    int64_t amb_w = 0;
    for (int r = 0; r < b; ++r)
      for (int f = 0; f < F; ++f) {
        const uint64_t v = vids[(size_t)(r0 + r) * F + f];
        memcpy(x + (size_t)r * K + (size_t)f * d, gce + v * d, sizeof(double) * d);
      }
    const double lw = model_core(x, labels + r0, b, F, d, H, s->w1, s->b1, s->w2, s->b2,
                                 logits ? logits + r0 : NULL, dx, dw, dw + (size_t)K * H,
                                 dw + (size_t)K * H + H, dw + (size_t)K * H + 2 * H,
                                 s->cfg.num_threads, dxa, dwa, dxm, dwm, &amb_w);
    amb_total += amb_w;
    if (!isfinite(lw)) {
      snprintf(g_err, sizeof g_err, "step %lld: non-finite loss", (long long)step);
      rc = 4;
    }
    if (worker_losses) worker_losses[w] = lw;
    lossum += lw;
    /* segment_sum in position order; embedding gradients of the
     * global-mean loss: each worker's contribution is scaled by 1/W */
    memset(lcg, 0, sizeof(double) * (size_t)U * d);
    const double scale = 1.0 / (double)W;
    for (int r = 0; r < b; ++r)
      for (int f = 0; f < F; ++f) {
        const uint64_t v = vids[(size_t)(r0 + r) * F + f];
        const double* g = dx + (size_t)r * K + (size_t)f * d;
        for (int c = 0; c < d; ++c) lcg[v * d + c] += g[c] * scale;
        if (ka) {
          const double* ga = dxa + (size_t)r * K + (size_t)f * d;
          const double* gm = dxm + (size_t)r * K + (size_t)f * d;
          for (int c = 0; c < d; ++c) {
            gca[v * d + c] += ga[c] * scale;
            gcm[v * d + c] += gm[c] * scale;
          }
        }
      }
    /* grad_synchronize: ordered sum over workers */
    for (size_t i = 0; i < (size_t)U * d; ++i) gcg[i] += lcg[i];
    for (size_t i = 0; i < P; ++i) dsum[i] += dw[i];
    if (ka)
      for (size_t i = 0; i < P; ++i) {
        dsa[i] += dwa[i];
        dsm[i] += dwm[i];
      }
  }
  s->led.inter += (int64_t)W * (orc_allreduce_bytes(U * d * 4, W) +
                                orc_allreduce_bytes((int64_t)P * 4, W));
  /* 8. update_sparse: lazy Adam on owned rows, per-feature step count, then unpin */
  for (int w = 0; w < W; ++w)
    for (int64_t k = 0; k < U; ++k) {
      if (gids[k] % (uint64_t)W != (uint64_t)w) continue;
      slot_t* sl = &s->caches[w].slots[cache_slot_of(&s->caches[w], gids[k])];
      entry_t* e = &sl->entry;
      e->steps += 1;
      adam(e->data, e->data + d, e->data + 2 * d, gcg + (size_t)k * d, (size_t)d, e->steps, &s->cfg);
      sl->pinned = 0;
    }
  /* dense: mean over workers, then Adam with the global step */
  for (size_t i = 0; i < P; ++i) dsum[i] /= (double)W;
  if (ka) {
    for (size_t i = 0; i < P; ++i) {
      dsa[i] /= (double)W;
      dsm[i] /= (double)W;
    }
    free(s->last_g); free(s->last_gabs); free(s->last_dg); free(s->last_dgabs);
    free(s->last_gamb); free(s->last_dgamb);
    s->last_gamb = gcm;
    s->last_dgamb = dsm;
    s->last_amb = amb_total;
    free(dxm);
    free(dwm);
    s->last_g = (double*)malloc(sizeof(double) * (size_t)U * d);
    memcpy(s->last_g, gcg, sizeof(double) * (size_t)U * d);
    s->last_gabs = gca;
    s->last_dg = (double*)malloc(sizeof(double) * P);
    memcpy(s->last_dg, dsum, sizeof(double) * P);
    s->last_dgabs = dsa;
    free(dxa);
    free(dwa);
  }
  s->dense_steps += 1;
  adam(s->w1, s->mw1, s->vw1, dsum, (size_t)K * H, s->dense_steps, &s->cfg);
  adam(s->b1, s->mb1, s->vb1, dsum + (size_t)K * H, (size_t)H, s->dense_steps, &s->cfg);
  adam(s->w2, s->mw2, s->vw2, dsum + (size_t)K * H + H, (size_t)H, s->dense_steps, &s->cfg);
  adam(&s->b2, &s->mb2, &s->vb2, dsum + (size_t)K * H + 2 * H, 1, s->dense_steps, &s->cfg);
  if (loss_out) *loss_out = lossum / (double)W;
  free(gids); free(vids); free(owned);
  free(gce); free(gcg); free(lcg); free(dsum); free(dw); free(x); free(dx);
  return rc;
}

void orc_sim_cache_slots(const orc_sim* s, int worker, uint64_t* feature, int64_t* last_use,
                         uint64_t* admit_seq) {
  const cache_t* c = &s->caches[worker];
  for (uint64_t i = 0; i < c->cap; ++i) {
    feature[i] = c->slots[i].occupied ? c->slots[i].feature : UINT64_MAX;
    if (last_use) last_use[i] = c->slots[i].last_use;
    if (admit_seq) admit_seq[i] = c->slots[i].admit_seq;
  }
}

uint64_t orc_sim_free_count(const orc_sim* s, int worker) { return s->caches[worker].nfree; }

typedef struct {
  uint64_t f;
  const entry_t* e;
} snap_t;
static int snap_cmp(const void* a, const void* b) {
  const uint64_t x = ((const snap_t*)a)->f, y = ((const snap_t*)b)->f;
  return x < y ? -1 : (x > y);
}

int64_t orc_sim_snapshot(const orc_sim* s, uint64_t* features, double* rows, int64_t* steps) {
  size_t n = s->host.table.size;
  for (int w = 0; w < s->W; ++w) n += s->caches[w].index.size;
  if (!features) return (int64_t)n;
  snap_t* all = (snap_t*)malloc(sizeof(snap_t) * (n ? n : 1));
  size_t m = 0;
  for (size_t i = 0; i < s->host.table.cap; ++i)
    if (s->host.table.used[i])
      all[m++] = (snap_t){s->host.table.keys[i], &s->host.pool[s->host.table.vals[i]]};
  for (int w = 0; w < s->W; ++w)
    for (uint64_t i = 0; i < s->caches[w].cap; ++i)
      if (s->caches[w].slots[i].occupied)
        all[m++] = (snap_t){s->caches[w].slots[i].feature, &s->caches[w].slots[i].entry};
  qsort(all, m, sizeof(snap_t), snap_cmp);
  const int d3 = 3 * s->d;
  for (size_t i = 0; i < m; ++i) {
    features[i] = all[i].f;
    if (rows) memcpy(rows + i * d3, all[i].e->data, sizeof(double) * d3);
    if (steps) steps[i] = all[i].e->steps;
  }
  free(all);
  return (int64_t)m;
}

void orc_sim_dense(const orc_sim* s, double* w1, double* b1, double* w2, double* b2) {
  memcpy(w1, s->w1, sizeof(double) * (size_t)s->K * s->H);
  memcpy(b1, s->b1, sizeof(double) * s->H);
  memcpy(w2, s->w2, sizeof(double) * s->H);
  *b2 = s->b2;
}

void orc_sim_set_dense(orc_sim* s, const double* w1, const double* b1, const double* w2,
                       const double* b2) {
  memcpy(s->w1, w1, sizeof(double) * (size_t)s->K * s->H);
  memcpy(s->b1, b1, sizeof(double) * s->H);
  memcpy(s->w2, w2, sizeof(double) * s->H);
  s->b2 = *b2;
}

void orc_sim_ledger(const orc_sim* s, int64_t out[4]) {
  out[0] = s->led.h2w;
  out[1] = s->led.w2h;
  out[2] = s->led.inter;
  out[3] = s->led.swaps;
}

int64_t orc_sim_last_unique(const orc_sim* s) { return s->last_u; }

/* ======================= criteo.cpp:27-98 ======================= */
int64_t orc_criteo_parse(const char* data, size_t n, uint64_t vocab, uint64_t* features,
                         uint8_t* labels, int64_t cap_rows, int64_t* err_line, char* err_msg,
                         size_t msg_cap) {
  int64_t rows = 0, lineno = 0;
  size_t pos = 0;
  while (pos < n) { /* std::getline over '\n' (criteo.cpp:41-45) */
    const char* nl = memchr(data + pos, '\n', n - pos);
    size_t end = nl ? (size_t)(nl - data) : n;
    const size_t next = nl ? end + 1 : n;
    ++lineno;
    if (end > pos && data[end - 1] == '\r') --end;
    if (end == pos) { pos = next; continue; }
    size_t tabs[40];
    size_t ntab = 0;
    for (size_t i = pos; i < end; ++i)
      if (data[i] == '\t') { if (ntab < 40) tabs[ntab] = i; ++ntab; }
    if (ntab != 39) { /* criteo.cpp:59-63 */
      *err_line = lineno;
      snprintf(err_msg, msg_cap, "expected 40 tab-separated columns, got %zu", ntab + 1);
      return -1;
    }
    if (!(tabs[0] == pos + 1 && (data[pos] == '0' || data[pos] == '1'))) { /* :64-68 */
      *err_line = lineno;
      snprintf(err_msg, msg_cap, "label must be 0 or 1, got '%.*s'", (int)(tabs[0] - pos),
               data + pos);
      return -1;
    }
    if (rows >= cap_rows) return -3;
    labels[rows] = data[pos] == '1' ? 1 : 0;
    for (int f = 0; f < 26; ++f) { /* :69-76 */
      const size_t a = tabs[13 + f] + 1, b = f == 25 ? end : tabs[14 + f];
      features[rows * 26 + f] = b > a ? orc_fnv1a64(data + a, b - a) % vocab : 0;
    }
    ++rows;
    pos = next;
  }
  if (rows == 0) return -2; /* :78 */
  return rows;
}

void orc_criteo_read_batch(const uint64_t* features, const uint8_t* labels, int64_t rows,
                           int64_t step, int global_rows, uint64_t* out_f, uint8_t* out_l) {
  int64_t src = (step * global_rows) % rows; /* criteo.cpp:88-96 */
  for (int r = 0; r < global_rows; ++r) {
    out_l[r] = labels[src];
    for (int f = 0; f < 26; ++f) out_f[(size_t)r * 26 + f] = features[src * 26 + f];
    src = (src + 1) % rows;
  }
}

/* ---- state access for per-step parity from identical state (tests only) ----
 * The row of feature f lives in its owner's cache (f mod W) or the host table; a
 * never-touched feature has no state (returns -1). */
static entry_t* find_entry(orc_sim* s, uint64_t f) {
  cache_t* c = &s->caches[f % (uint64_t)s->W];
  const int64_t slot = cache_slot_of(c, f);
  if (slot >= 0) return &c->slots[slot].entry;
  int64_t* v = hm_find(&s->host.table, f);
  return v ? &s->host.pool[*v] : NULL;
}

int64_t orc_sim_get_rows(orc_sim* s, int64_t n, const uint64_t* features, double* rows,
                         int64_t* steps) {
  const int d3 = 3 * s->d;
  int64_t absent = 0;
  for (int64_t i = 0; i < n; ++i) {
    const entry_t* e = find_entry(s, features[i]);
    if (!e) {  /* never touched: no state yet */
      ++absent;
      if (rows) memset(rows + i * d3, 0, sizeof(double) * d3);
      if (steps) steps[i] = -1;
      continue;
    }
    if (rows) memcpy(rows + i * d3, e->data, sizeof(double) * d3);
    if (steps) steps[i] = e->steps;
  }
  return absent;
}

int orc_sim_set_rows(orc_sim* s, int64_t n, const uint64_t* features, const double* rows,
                     const int64_t* steps) {
  const int d3 = 3 * s->d;
  for (int64_t i = 0; i < n; ++i) {
    entry_t* e = find_entry(s, features[i]);
    if (!e) {
      snprintf(g_err, sizeof g_err, "feature %llu has no state", (unsigned long long)features[i]);
      return -1;
    }
    if (rows) memcpy(e->data, rows + i * d3, sizeof(double) * d3);
    if (steps) e->steps = steps[i];
  }
  return 0;
}

/* dense parameters and Adam moments, each [P] = W1 | b1 | w2 | b2, and the dense step */
static void dense_io(orc_sim* s, double* p, double* m, double* v, int64_t* step, int set) {
  const size_t kh = (size_t)s->K * s->H, H = (size_t)s->H;
  double* bufs[3] = {p, m, v};
  double* w1s[3] = {s->w1, s->mw1, s->vw1};
  double* b1s[3] = {s->b1, s->mb1, s->vb1};
  double* w2s[3] = {s->w2, s->mw2, s->vw2};
  double* b2s[3] = {&s->b2, &s->mb2, &s->vb2};
  for (int q = 0; q < 3; ++q) {
    double* b = bufs[q];
    if (!b) continue;
    double* parts[4] = {w1s[q], b1s[q], w2s[q], b2s[q]};
    const size_t lens[4] = {kh, H, H, 1};
    size_t off = 0;
    for (int k = 0; k < 4; ++k) {
      if (set) memcpy(parts[k], b + off, sizeof(double) * lens[k]);
      else memcpy(b + off, parts[k], sizeof(double) * lens[k]);
      off += lens[k];
    }
  }
  if (step) {
    if (set) s->dense_steps = *step;
    else *step = s->dense_steps;
  }
}
void orc_sim_get_dense_state(orc_sim* s, double* p, double* m, double* v, int64_t* step) {
  dense_io(s, p, m, v, step, 0);
}
void orc_sim_set_dense_state(orc_sim* s, const double* p, const double* m, const double* v,
                             const int64_t* step) {
  dense_io(s, (double*)p, (double*)m, (double*)v, (int64_t*)step, 1);
}

void orc_sim_keep_grads(orc_sim* s, int on) { s->keep_grads = on; }

/* the last step's summed embedding gradients g [U*d] (global_ids order) with their
 * condition scales gabs (sums of |terms|), and the dense gradients (worker mean) dg [P]
 * with dgabs [P]; gamb / dgamb: the gradient mass behind fp32-undetermined ReLU decisions
 * (model_core), n_amb: how many (row, unit) decisions were undetermined; 0, or -1 when
 * keep_grads was off */
int orc_sim_last_grads(const orc_sim* s, double* g, double* gabs, double* dg, double* dgabs,
                       double* gamb, double* dgamb, int64_t* n_amb) {
  if (!s->last_g) return -1;
  const size_t ud = (size_t)s->last_u * s->d, P = (size_t)s->K * s->H + 2 * s->H + 1;
  if (g) memcpy(g, s->last_g, sizeof(double) * ud);
  if (gabs) memcpy(gabs, s->last_gabs, sizeof(double) * ud);
  if (dg) memcpy(dg, s->last_dg, sizeof(double) * P);
  if (dgabs) memcpy(dgabs, s->last_dgabs, sizeof(double) * P);
  if (gamb) memcpy(gamb, s->last_gamb, sizeof(double) * ud);
  if (dgamb) memcpy(dgamb, s->last_dgamb, sizeof(double) * P);
  if (n_amb) *n_amb = s->last_amb;
  return 0;
}
