/*
 * TEST INFRASTRUCTURE ONLY — the CPU parity oracle.
 *
 * A plain-C restatement of the ScaleFreeCTR reference path
 * (/root/reference/proj/core + SPEC.md) in fp64 with a fixed, documented
 * reduction order. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it; the product
 * (paper_2104_08542_b200/) never links or calls it.
 *
 * Pinning: the present reference primitives (rng, generator, initial
 * embedding, VSI, HostStore/CacheBuffer slot semantics, allreduce_bytes) are
 * checked bit-for-bit against the reference's own compiled TUs
 * (oracle/_ref/libsfctr_ref.so, built by oracle/build_ref.sh) and against
 * committed golden vectors (tests/golden/). The manager, DeepFM-lite model
 * and worker ops are MISSING from the reference (core/CMakeLists.txt:10-12
 * lists manager.cpp/model.cpp/worker_ops.cpp, none exist); they are restated
 * from SPEC.md:179-358 and pinned only by the SPEC's worked examples
 * and a
 * finite-difference gradient check — "parity partially unpinned" for those
 * rows.
 */
#ifndef SFCTR_ORACLE_H
#define SFCTR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:27-84 ---- */
uint64_t orc_fnv1a64(const char* bytes, size_t n);
uint64_t orc_derive_seed(uint64_t base, const char* label, uint64_t index);
double orc_truth_weight(uint64_t seed, uint64_t feature);
void orc_initial_embedding(uint64_t seed, uint64_t feature, int dim, double* out);
int64_t orc_allreduce_bytes(int64_t payload, int workers);

/* ---- criteo.cpp:27-98 (CriteoReader) ----
 * Parses a whole TSV held in memory: rows = data lines (empty / "\r"-only lines
 * skipped), features [rows*26] = fnv1a64(token) % vocab (0 for an empty token),
 * labels [rows]. Returns rows (>= 0), or -1 with *err_line (1-based, counting every
 * line) and err_msg (the reference's text after "path:line: ") for the first malformed
 * line, or -2 when there is no data row. Capacity: cap_rows rows. */
int64_t orc_criteo_parse(const char* data, size_t n, uint64_t vocab, uint64_t* features,
                         uint8_t* labels, int64_t cap_rows, int64_t* err_line, char* err_msg,
                         size_t msg_cap);
/* read_batch(step): global_rows rows starting at (step*global_rows) % rows, wrapping */
void orc_criteo_read_batch(const uint64_t* features, const uint8_t* labels, int64_t rows,
                           int64_t step, int global_rows, uint64_t* out_f, uint8_t* out_l);

/* ---- generator.cpp:32-108 ---- */
typedef struct orc_gen orc_gen;
orc_gen* orc_gen_create(int global_rows, int fields, uint64_t vocab, uint64_t seed, double zipf);
void orc_gen_destroy(orc_gen* g);
/* rows [row0, row0+nrows) of generate(step); the whole batch is row0=0, nrows=global_rows */
void orc_gen_generate_rows(const orc_gen* g, int64_t step, int row0, int nrows, uint64_t* features,
                           uint8_t* labels);
uint64_t orc_gen_shard_start(const orc_gen* g, int field);

/* ---- vsi.cpp:23-54 ---- returns U, or -3 (LogicError) on a failed check */
int64_t orc_vsi(const uint64_t* features, int rows, int fields, int workers, uint64_t* global_ids,
                uint64_t* virtual_ids);

/* ---- the simulated training system, sequential BSP mode ---- */
typedef struct orc_config {
  int num_workers;
  int embedding_dim;
  int num_fields;
  int batch_size_per_worker;
  uint64_t vocabulary_size;
  uint64_t cache_capacity;
  int lookahead_depth;
  uint64_t seed;
  double learning_rate, adam_beta1, adam_beta2, adam_epsilon;
  double zipf_exponent;
  int hidden_dim;
  int num_threads; /* model fwd/bwd threads; results do not depend on it */
} orc_config;

void orc_config_default(orc_config* c); /* config.hpp:42-71 defaults */

typedef struct orc_sim orc_sim;
orc_sim* orc_sim_create(const orc_config* cfg);
void orc_sim_destroy(orc_sim* s);
const char* orc_last_error(void);

/*
 * One BSP step over a global batch (rows = W*b): VSI, per-worker manage
 * (evict-then-admit), gather_cache, forward all-reduce, gather_instances,
 * forward_backward, segment_sum, grad all-reduce, lazy sparse Adam, dense
 * Adam. `window_*` optionally pass the lookahead batches t+1..t+L-1 (raw
 * features, same shape) for the needed_soon rule; NULL = only batch t.
 * Outputs: mean loss; per-worker losses [W]; logits [rows] (may be NULL).
 * Returns 0, or a nonzero status (3 LogicError, 4 RunError) with
 * orc_last_error() set.
 */
int orc_sim_step(orc_sim* s, int64_t step, const uint64_t* features, const uint8_t* labels,
                 const uint64_t* window_features, int window_batches, double* loss_out,
                 double* worker_losses, double* logits);

/* cache slot dump of one worker: feature per slot (UINT64_MAX = empty), last_use, admit_seq */
void orc_sim_cache_slots(const orc_sim* s, int worker, uint64_t* feature, int64_t* last_use,
                         uint64_t* admit_seq);
uint64_t orc_sim_free_count(const orc_sim* s, int worker);
/* every feature ever touched (host or cache), sorted: returns the count; when
 * the out pointers are non-NULL they receive features [n], rows [n*3d] =
 * embedding|momentum|velocity, steps [n] */
int64_t orc_sim_snapshot(const orc_sim* s, uint64_t* features, double* rows, int64_t* steps);
/* dense parameters: W1 [K*h] row-major (k, j), b1 [h], w2 [h], b2 [1] */
void orc_sim_dense(const orc_sim* s, double* w1, double* b1, double* w2, double* b2);
void orc_sim_set_dense(orc_sim* s, const double* w1, const double* b1, const double* w2,
                       const double* b2);
/* ledger.hpp:60-63: host_to_worker, worker_to_host, interworker, swap_events */
void orc_sim_ledger(const orc_sim* s, int64_t out[4]);
/* last step's VSI unique count */
int64_t orc_sim_last_unique(const orc_sim* s);

/* Per-step parity from identical state: read / overwrite the [emb|m|v] rows and adam
 * step counts of touched features (wherever they live), and the dense parameters with
 * their Adam moments ([P] = W1 | b1 | w2 | b2) and the dense step. get_rows returns the
 * number of features without state (zero rows, step -1); set_rows returns 0, or -1 for a
 * feature without state. */
int64_t orc_sim_get_rows(orc_sim* s, int64_t n, const uint64_t* features, double* rows,
                         int64_t* steps);
int orc_sim_set_rows(orc_sim* s, int64_t n, const uint64_t* features, const double* rows,
                     const int64_t* steps);
void orc_sim_get_dense_state(orc_sim* s, double* p, double* m, double* v, int64_t* step);
void orc_sim_set_dense_state(orc_sim* s, const double* p, const double* m, const double* v,
                             const int64_t* step);

/* keep the next steps' gradients and their condition scales (sums of |terms| over every
 * addition that forms them) for orc_sim_last_grads: g / gabs [U*d] in global_ids order,
 * dense dg / dgabs [P] (worker mean); gamb / dgamb: the gradient mass behind ReLU
 * decisions fp32 does not determine (|hpre| <= 1e-5 (|b1| + sum |x w|)), n_amb: their
 * count. Returns -1 when nothing was kept. */
void orc_sim_keep_grads(orc_sim* s, int on);
int orc_sim_last_grads(const orc_sim* s, double* g, double* gabs, double* dg, double* dgabs,
                       double* gamb, double* dgamb, int64_t* n_amb);

/* initial dense parameters: W1 ~ U(-a,a), a = sqrt(6/(K+h)),
 * stream derive_seed(seed,"dense_w1",0); w2 ~ U(-a2,a2), a2 = sqrt(6/(h+1)),
 * stream "dense_w2"; b1 = b2 = 0 */
void orc_dense_init(uint64_t seed, int K, int h, double* w1, double* b1, double* w2, double* b2);

/*
 * DeepFM-lite forward+backward on one worker's rows (SPEC.md:261-264,
 * 292-300, 342). X [rows, F*d]; returns the mean BCE; grad outputs are
 * d(mean loss)/d(.) — dx [rows, F*d], dw1 [K*h], db1 [h], dw2 [h], db2 [1];
 * logits [rows]. Any output pointer may be NULL except dx when dense grads are
 * wanted.
 */
double orc_model_fwd_bwd(const double* x, const uint8_t* labels, int rows, int fields, int dim,
                         int hidden, const double* w1, const double* b1, const double* w2,
                         double b2, double* logits, double* dx, double* dw1, double* db1,
                         double* dw2, double* db2, int num_threads);

/*
 * The MixCache manager on a standalone cache (the SPEC.md:195 worked
 * example): builds a cache of `capacity` slots, admits `resident` in order at
 * step 0, pins `pinned`, then runs one manage step for `next` (window = next)
 * at step 1 with the evict-then-admit order. Writes the final slot->feature
 * table (UINT64_MAX empty) and returns the number of evictions, or -1.
 */
int64_t orc_manager_example(uint64_t capacity, const uint64_t* resident, int n_resident,
                            const uint64_t* pinned, int n_pinned, const uint64_t* next, int n_next,
                            uint64_t* slots_out, uint64_t* evicted_out);

#ifdef __cplusplus
}
#endif
#endif
