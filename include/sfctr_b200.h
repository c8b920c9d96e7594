/*
 * sfctr_b200.h — C-ABI of the B200-native ScaleFreeCTR embedding hot path.
 *
 * Plain C: opaque handles, plain pointers and sizes, status codes; no torch
 * or C++ types. Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core/ unless they start with
 * SPEC.md). The reference is a C++ library whose error convention is four
 * exception classes (include/sfctr/error.hpp:28-56); they map to status
 * codes 1-4 here, with the message in sfctr_last_error() (thread-local) and
 * the failing step of a RunError in sfctr_last_error_step(). The header-only
 * C++ facade include/sfctr_b200.hpp rethrows them as the same classes.
 *
 * All compute runs as hand-written sm_100a CUDA kernels; there is no CPU
 * fallback: without a usable CUDA device every compute entry point returns
 * SFCTR_ERR_CUDA.
 */
#ifndef SFCTR_B200_H
#define SFCTR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFCTR_B200_ABI_VERSION 2

typedef enum sfctr_status {
  SFCTR_OK = 0,
  SFCTR_ERR_CONFIG = 1, /* sfctr::ConfigError  (error.hpp:28-31) */
  SFCTR_ERR_DATA = 2,   /* sfctr::DataError    (error.hpp:34-37) */
  SFCTR_ERR_LOGIC = 3,  /* sfctr::LogicError   (error.hpp:42-45; SFCTR_CHECK) */
  SFCTR_ERR_RUN = 4,    /* sfctr::RunError     (error.hpp:48-56; carries the step) */
  SFCTR_ERR_CUDA = 5,   /* CUDA runtime failure / no device */
  SFCTR_ERR_NCCL = 6    /* NCCL failure */
} sfctr_status;

/* Message of the last failing call on this thread ("" if none). */
const char* sfctr_last_error(void);
/* Step index carried by the last SFCTR_ERR_RUN on this thread (-1 if none). */
int64_t sfctr_last_error_step(void);
int sfctr_abi_version(void);

/* ---------------------------------------------------------------------
 * Configuration — SimConfig (include/sfctr/config.hpp:42-83)
 * ------------------------------------------------------------------- */
enum { SFCTR_STRATEGY_HOST = 0, SFCTR_STRATEGY_PREFETCH = 1, SFCTR_STRATEGY_CACHE = 2 };
enum { SFCTR_SYNC_ALLREDUCE = 0, SFCTR_SYNC_ALLTOALL = 1 };
/* RunMode (config.hpp:30): pipelined overlaps the manager stage of step t+1 with the
 * training of step t; results are identical to sequential. */
enum { SFCTR_MODE_SEQUENTIAL = 0, SFCTR_MODE_PIPELINED = 1 };
/* DataSource (config.hpp:33-36, config key `data`: synthetic | criteo:<path>) */
enum { SFCTR_DATA_SYNTHETIC = 0, SFCTR_DATA_CRITEO = 1 };
#define SFCTR_PATH_MAX 1024

typedef struct sfctr_config {
  /* reference fields, config.hpp:44-71 (same defaults) */
  int32_t num_workers;           /* W  (workers)         default 4 */
  int32_t embedding_dim;         /* d  (dim)             default 16 */
  int32_t num_fields;            /* F  (fields)          default 26 */
  int32_t batch_size_per_worker; /* b  (batch_size)      default 256 */
  uint64_t vocabulary_size;      /* n  (vocab)           default 100000 */
  uint64_t cache_capacity;       /* C  (cache_capacity)  default 8192 slots / worker */
  int32_t lookahead_depth;       /* L  (lookahead)       default 1 */
  int32_t strategy;              /*    (strategy)        default cache; only cache is on the device path */
  uint64_t seed;                 /*    (seed)            default 7 */
  double learning_rate;          /*    (lr)              default 1e-3 */
  double adam_beta1;             /*    (beta1)           default 0.9 */
  double adam_beta2;             /*    (beta2)           default 0.999 */
  double adam_epsilon;           /*    (epsilon)         default 1e-8 */
  double zipf_exponent;          /*    (zipf)            default 1.2 */
  int32_t hidden_dim;            /* h  (hidden)          default 64 */
  /* B200 extensions (config keys in parentheses) */
  int32_t sync_mode;             /* (sync) allreduce (reference scheme) | alltoall (owner-routed) */
  uint64_t host_table_rows;      /* (host_rows) host-pool rows pinned up front per worker (the pool
                                    of evicted rows grows on demand beyond it); 0 = none */
  int32_t run_mode;              /* (mode) sequential | pipelined — RunMode, config.hpp:30 */
  /* reference fields, config.hpp:69-71 */
  int32_t data_source;           /* (data) synthetic | criteo:<path> */
  char criteo_path[SFCTR_PATH_MAX];
  /* (deterministic) 1: fixed-order gradient sums (segment sum in ascending position order
   * per unique, no atomics): bit-identical results run to run. Slower. */
  int32_t deterministic;
} sfctr_config;

void sfctr_config_default(sfctr_config* cfg);
/* SimConfig::validate (config.cpp:55-78) + B200 limits; SFCTR_ERR_CONFIG on failure. */
int sfctr_config_validate(const sfctr_config* cfg);
/* apply_config_entry (config.cpp:115-159), same keys/grammar plus the B200 keys. */
int sfctr_config_apply(sfctr_config* cfg, const char* key, const char* value);
/* load_config_file (config.cpp:161-187): key=value lines, '#' comments. */
int sfctr_config_load(sfctr_config* cfg, const char* path);

/* ---------------------------------------------------------------------
 * core helpers — rng.hpp:27-56, comm.hpp:36-41, generator.cpp:110-115
 * ------------------------------------------------------------------- */
uint64_t sfctr_fnv1a64(const char* bytes, size_t n);
uint64_t sfctr_derive_seed(uint64_t base, const char* label, uint64_t index);
/* allreduce_bytes(payload, W); -1 + SFCTR_ERR_LOGIC semantics on bad input */
int64_t sfctr_allreduce_bytes(int64_t payload_bytes, int num_workers);

/* Number of visible CUDA devices (0 when none). */
int sfctr_device_count(int* count);

/* ---------------------------------------------------------------------
 * Synthetic batch ingest — SyntheticGenerator (generator.hpp:35-62)
 * Device kernels reproduce generate(step) bit-for-bit; rows may be any
 * sub-range of the global batch (the RNG is counter based), so each rank
 * synthesises only its own rows.
 * ------------------------------------------------------------------- */
typedef struct sfctr_generator sfctr_generator;
/* SyntheticGenerator(config) — uses workers, batch_size, fields, vocab, seed, zipf. */
int sfctr_generator_create(const sfctr_config* cfg, int device, sfctr_generator** out);
void sfctr_generator_destroy(sfctr_generator* g);
/* generate(step) rows [row0, row0+nrows) into HOST buffers: features [nrows*F], labels [nrows]. */
int sfctr_generator_generate(sfctr_generator* g, int64_t step, int32_t row0, int32_t nrows,
                             uint64_t* features, uint8_t* labels);
/* Same into DEVICE buffers on `stream` (cudaStream_t; NULL = legacy default), asynchronous. */
int sfctr_generator_generate_device(sfctr_generator* g, int64_t step, int32_t row0, int32_t nrows,
                                    uint64_t* d_features, uint8_t* d_labels, void* stream);
/* shard_start(field) (generator.hpp:42) */
uint64_t sfctr_generator_shard_start(const sfctr_generator* g, int32_t field);
/* initial_embedding(seed, feature, dim) (generator.hpp:62), computed by the device kernel. */
int sfctr_initial_embedding(uint64_t seed, uint64_t feature, int32_t dim, int device, double* out);

/* ---------------------------------------------------------------------
 * Criteo ingest — CriteoReader (criteo.hpp:37-58, criteo.cpp:25-98)
 * TSV "label \t 13 numerics \t 26 categorical tokens" parsed and hashed on the device
 * (fnv1a64(token) % vocab, empty token -> 0), bit-exact with the reference. The whole
 * file is parsed at open (streamed through pinned chunks); malformed lines are
 * SFCTR_ERR_DATA with the reference's "path:line: ..." message; a missing file or
 * fields != 26 is SFCTR_ERR_CONFIG. Batches of num_workers * batch_size_per_worker rows
 * wrap around at the end of the file (read_batch, criteo.cpp:81-98).
 * ------------------------------------------------------------------- */
typedef struct sfctr_criteo sfctr_criteo;
int sfctr_criteo_open(const char* path, const sfctr_config* cfg, int device, sfctr_criteo** out);
/* the same over bytes already in memory; `name` replaces the path in messages */
int sfctr_criteo_open_buffer(const char* data, size_t n, const char* name, const sfctr_config* cfg,
                             int device, sfctr_criteo** out);
void sfctr_criteo_destroy(sfctr_criteo* r);
int64_t sfctr_criteo_row_count(const sfctr_criteo* r);           /* row_count() */
uint64_t sfctr_criteo_token_hash(const char* token, size_t n);   /* token_hash() */
/* rows [row0, row0+nrows) of batch `step`: features [nrows*26] u64, labels [nrows] */
int sfctr_criteo_read_batch(sfctr_criteo* r, int64_t step, int32_t row0, int32_t nrows,
                            uint64_t* features, uint8_t* labels);
int sfctr_criteo_read_batch_device(sfctr_criteo* r, int64_t step, int32_t row0, int32_t nrows,
                                   uint64_t* d_features, uint8_t* d_labels, void* stream);
/* bytes and lines parsed; device span of the ingest, first chunk copy to last parse (ms) */
int sfctr_criteo_stats(const sfctr_criteo* r, int64_t* bytes, int64_t* lines, double* parse_ms);

/* ---------------------------------------------------------------------
 * Batch source — the pipeline's data loader over the configured DataSource (config key
 * `data`, config.cpp:146-154): the SyntheticGenerator or the CriteoReader (criteo_path),
 * same read interface (rows [row0, row0+nrows) of global batch `step`).
 * ------------------------------------------------------------------- */
typedef struct sfctr_batch_source sfctr_batch_source;
int sfctr_batch_source_create(const sfctr_config* cfg, int device, sfctr_batch_source** out);
void sfctr_batch_source_destroy(sfctr_batch_source* b);
int sfctr_batch_source_read(sfctr_batch_source* b, int64_t step, int32_t row0, int32_t nrows,
                            uint64_t* features, uint8_t* labels);
int sfctr_batch_source_read_device(sfctr_batch_source* b, int64_t step, int32_t row0,
                                   int32_t nrows, uint64_t* d_features, uint8_t* d_labels,
                                   void* stream);

/* ---------------------------------------------------------------------
 * Virtual Sparse Id — virtual_sparse_id(const RawBatch&, int) (vsi.hpp:29)
 * ------------------------------------------------------------------- */
typedef struct sfctr_vsi sfctr_vsi;
/* key_space: every feature id must be < key_space (the vocabulary size): a direct-mapped
 * first-position table of 4 B per key; key_space = 0: arbitrary u64 ids (any FeatureId the
 * reference accepts, vsi.cpp:23-54) through a hashed table of ~16 B per id slot.
 * max_ids: the largest rows*fields that will be passed. */
int sfctr_vsi_create(int device, uint64_t key_space, int64_t max_ids, sfctr_vsi** out);
void sfctr_vsi_destroy(sfctr_vsi* v);
/* HOST buffers. global_ids [>= unique], virtual_ids [rows*fields] (first-appearance
 * order, bit-exact with vsi.cpp:41-46), row_ranges [2*num_workers] (vsi.cpp:48-52).
 * Errors: SFCTR_ERR_LOGIC for the reference's SFCTR_CHECKs (empty batch, uneven split)
 * and for ids >= key_space. */
int sfctr_virtual_sparse_id(sfctr_vsi* v, const uint64_t* features, int32_t rows, int32_t fields,
                            int32_t num_workers, uint64_t* global_ids, uint64_t* virtual_ids,
                            int64_t* unique_count, int32_t* row_ranges);
/* DEVICE buffers, asynchronous on `stream` (contexts with key_space > 0): ids are u32
 * feature ids (< key_space);
 * writes d_global_ids [U] (u32), d_virtual_ids [n] (u32) and *d_unique (int32, device). */
int sfctr_virtual_sparse_id_device(sfctr_vsi* v, const uint32_t* d_ids, int64_t n,
                                   uint32_t* d_global_ids, uint32_t* d_virtual_ids,
                                   int32_t* d_unique, void* stream);

/* ---------------------------------------------------------------------
 * Trainer — the Host-Manager + GPU-Worker of Algorithm 1:
 * HostStore (host_store.hpp:61-92) as a pinned host table, CacheBuffer
 * (cache_buffer.hpp:40-86) as an HBM slot pool per worker, the MixCache
 * manager, worker ops, DeepFM-lite
 * (SPEC.md:261-264), TransferLedger (ledger.hpp:27-64).
 *
 * One process drives `num_workers / world` worker lanes on one GPU; lanes of
 * different processes exchange over NCCL (world > 1). world = 1 with
 * num_workers = W runs all W lanes on one device (the reference's in-process
 * lanes).
 * ------------------------------------------------------------------- */
typedef struct sfctr_trainer sfctr_trainer;

/* 128-byte ncclUniqueId for rank 0 to broadcast (world > 1). */
int sfctr_nccl_unique_id(uint8_t out[128]);
int sfctr_trainer_create(const sfctr_config* cfg, int32_t rank, int32_t world,
                         const uint8_t* nccl_id, int device, sfctr_trainer** out);
void sfctr_trainer_destroy(sfctr_trainer* t);

/* One BSP training step (Algorithm 1 l.2-14) over this process's rows of
 * global batch `step`: rows = (num_workers/world) * batch_size_per_worker,
 * row-major features [rows*F] and labels [rows] in HOST memory (pinned or
 * pageable). Returns the global mean logloss in *loss.
 * window_features: the same process's rows of batches step+1..step+L-1
 * ((L-1)*rows*F ids, NULL when L == 1) for the needed_soon rule. */
int sfctr_trainer_step(sfctr_trainer* t, int64_t step, const uint64_t* features,
                       const uint8_t* labels, const uint64_t* window_features, double* loss);
/* Same with DEVICE inputs (u64 features, u8 labels) already resident in HBM;
 * enqueues the step on the trainer's stream. d_loss (device float, may be NULL)
 * receives the loss. The call returns after launching (one host-side wait for
 * the unique/working counts happens inside). */
int sfctr_trainer_step_device(sfctr_trainer* t, int64_t step, const uint64_t* d_features,
                              const uint8_t* d_labels, const uint64_t* d_window_features,
                              float* d_loss);
/* The device step split into its two stages (Algorithm 1): prepare = Host-Manager
 * (all-gather ids, virtual_sparse_id, manager_get + pull_parameters_to_host +
 * push_parameters_to_cache, exchange plan), train = GPU-Worker
 * (gather_cache ... update_sparse). Both only enqueue. prepare(t) must
 * be followed by train(t) before prepare(t+1) (else SFCTR_ERR_LOGIC); in pipelined mode
 * prepare(t+1) runs on the manager stream while train(t) is still executing.
 * sfctr_trainer_step_device(t) == prepare(t) + train(t). */
int sfctr_trainer_prepare(sfctr_trainer* t, int64_t step, const uint64_t* d_features,
                          const uint64_t* d_window_features);
int sfctr_trainer_train(sfctr_trainer* t, int64_t step, const uint8_t* d_labels, float* d_loss);
/* The host-buffer step split in two, for a driver that keeps steps in flight
 * (pipelined mode overlaps the manager stage of step t+1 with step t's training):
 * submit enqueues the H2D copies of the inputs and the step (whose last kernel stores the
 * loss straight into a mapped pinned slot: no D2H copy on the stream), and returns; loss waits for that step's loss. At most four submitted steps may be
 * outstanding: read the loss of step t before submitting step t+4 (else LOGIC). The
 * host input buffers must stay untouched until the step's loss has been read. */
int sfctr_trainer_submit(sfctr_trainer* t, int64_t step, const uint64_t* features,
                         const uint8_t* labels, const uint64_t* window_features);
int sfctr_trainer_loss(sfctr_trainer* t, int64_t step, double* loss);
/* Waits for the trainer's stream; reports deferred device-side errors. */
int sfctr_trainer_synchronize(sfctr_trainer* t);
/* cudaStream_t the trainer launches on */
void* sfctr_trainer_stream(sfctr_trainer* t);

/* Last step's logits (pre-sigmoid model output) for this process's rows [rows]. */
int sfctr_trainer_logits(sfctr_trainer* t, float* out);
/* Slot table of a LOCAL lane (0..lanes-1): feature per slot (UINT64_MAX = empty),
 * last_use, admit_seq — CacheBuffer::slots() (cache_buffer.hpp:63). */
int sfctr_trainer_cache_slots(sfctr_trainer* t, int32_t lane, uint64_t* feature,
                              int64_t* last_use, uint64_t* admit_seq);
/* The same for slots [first, first + count) only (clamped to the capacity): large caches
 * need not be copied whole. */
int sfctr_trainer_cache_slots_range(sfctr_trainer* t, int32_t lane, uint64_t first, uint64_t count,
                                    uint64_t* feature, int64_t* last_use, uint64_t* admit_seq);
/* Free-slot count of a local lane (CacheBuffer::free_count, cache_buffer.hpp:56). */
int sfctr_trainer_free_count(sfctr_trainer* t, int32_t lane, uint64_t* out);
/* HostStore::snapshot_sorted (host_store.hpp:85-86) over every feature this
 * process owns (host table and caches): call with NULL buffers to get *count,
 * then again with features [count], rows [count*3d] (embedding|momentum|
 * velocity, fp32), steps [count]. */
int sfctr_trainer_snapshot(sfctr_trainer* t, int64_t* count, uint64_t* features, float* rows,
                           int64_t* steps);
/* HostStore::peek (host_store.hpp:69-70) for n features owned by this process, wherever
 * their state lives (HBM cache slot or host pool): rows [n*3d] = embedding|momentum|
 * velocity (fp32), steps [n] (adam_steps). A feature that was never touched, or that
 * another process owns, is SFCTR_ERR_LOGIC. */
int sfctr_trainer_peek_rows(sfctr_trainer* t, int64_t n, const uint64_t* features, float* rows,
                            int64_t* steps);
/* Dense parameters and their Adam state, each [P] = w1 [F*d*h] | b1 [h] | w2 [h] | b2 [1],
 * and the dense Adam step (any pointer may be NULL). */
int sfctr_trainer_dense_state(sfctr_trainer* t, float* params, float* m, float* v,
                              int64_t* step);
/* Dense (replicated) parameters: w1 [F*d*h] row-major (k, j), b1 [h], w2 [h], b2 [1]. */
int sfctr_trainer_get_dense(sfctr_trainer* t, float* w1, float* b1, float* w2, float* b2);
int sfctr_trainer_set_dense(sfctr_trainer* t, const float* w1, const float* b1, const float* w2,
                            const float* b2);
/* TransferLedger counters (ledger.hpp:60-63), summed over this process's lanes:
 * host_to_worker, worker_to_host, interworker, swap_events. */
int sfctr_trainer_ledger(sfctr_trainer* t, int64_t out[4]);

typedef struct sfctr_step_stats {
  int64_t unique;          /* U of the last global batch */
  int64_t owned;           /* owned uniques, summed over local lanes */
  int64_t working;         /* admitted (cache misses) */
  int64_t evicted;         /* evicted to the host table */
  int64_t filled_from_host;/* admissions that read a row back over PCIe */
  int64_t pcie_h2d_bytes;  /* actual row bytes read from the pinned host table */
  int64_t pcie_d2h_bytes;  /* actual row bytes written back to the pinned host table */
  int64_t nvlink_bytes;    /* bytes this process handed to NCCL in the last step */
  int64_t kernel_launches; /* kernels launched by the last step */
  /* running totals since creation (deferred device counters are folded in at
   * every sfctr_trainer_synchronize / host-buffer step) */
  int64_t total_steps;
  int64_t total_working;
  int64_t total_evicted;
  int64_t total_filled_from_host;
  int64_t total_kernel_launches;
  int64_t total_unique;
  int64_t total_owned;
  int64_t total_nvlink_bytes;
  int64_t total_free_steps; /* steps that ran without a mid-step host wait */
  int64_t pinned_waits;     /* pipelined: 1 if the last step's eviction had to wait for the
                               previous step's rows to be unpinned */
  int64_t total_pinned_waits;
} sfctr_step_stats;
int sfctr_trainer_stats(sfctr_trainer* t, sfctr_step_stats* out);

/* Per-phase device timing of the last step (CUDA events on the trainer's stream),
 * enabled by sfctr_trainer_set_timing(t, 1). Names: see DESIGN.md §Kernels. */
int sfctr_trainer_set_timing(sfctr_trainer* t, int enabled);
int sfctr_trainer_phase_times(sfctr_trainer* t, int32_t max_phases, char* names /* max*32 */,
                              float* ms, int32_t* n_phases);

/* ---------------------------------------------------------------------
 * Standalone device MixCache of ONE worker — CacheBuffer (cache_buffer.hpp:40-86) with its
 * HostStore (host_store.hpp:61-92, a lazy pinned host pool of evicted rows) and the manager
 * step, for callers that drive the cache themselves. The worker owns
 * features f < key_space with f % num_workers == worker (shard_owner); rows
 * are [emb | m | v] (dim each, fp32) + adam_steps, lazily initialised with
 * initial_embedding(seed, f, dim) on first admission (HostStore::get_or_init).
 *
 * Batched operations take HOST arrays of n features and apply in list order with the
 * reference's one-at-a-time semantics: they stop at the first feature the reference
 * would throw on and return SFCTR_ERR_LOGIC with its message (cache_buffer.cpp), the
 * preceding features having taken effect. n <= max_batch per call.
 * ------------------------------------------------------------------- */
typedef struct sfctr_cache sfctr_cache;
/* CacheBuffer(capacity, dim) + HostStore(seed, dim); host_reserve pins host-pool rows up
 * front (the pool grows on demand) */
int sfctr_cache_create(uint64_t capacity, int32_t dim, uint64_t seed, uint64_t key_space,
                       int32_t num_workers, int32_t worker, int64_t max_batch,
                       uint64_t host_reserve, int device, sfctr_cache** out);
void sfctr_cache_destroy(sfctr_cache* c);
/* admit(f, host.take(f), step) (cache_buffer.cpp:38-53): needed_soon set, unpinned;
 * slots (nullable) [n] receive the SlotIds */
int sfctr_cache_admit(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t step,
                      uint64_t* slots);
/* host.put(f, evict(f)) (cache_buffer.cpp:55-67): non-resident / pinned / needed_soon is
 * SFCTR_ERR_LOGIC */
int sfctr_cache_evict(sfctr_cache* c, int64_t n, const uint64_t* features);
int sfctr_cache_touch(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t step);
/* pin (pinned != 0) / unpin */
int sfctr_cache_pin(sfctr_cache* c, int64_t n, const uint64_t* features, int32_t pinned);
int sfctr_cache_set_needed_soon(sfctr_cache* c, int64_t n, const uint64_t* features,
                                int32_t value);
/* slot_of: SlotId per feature, -1 when not resident (resident() == slot >= 0) */
int sfctr_cache_slot_of(sfctr_cache* c, int64_t n, const uint64_t* features, int64_t* slots);
int sfctr_cache_free_count(sfctr_cache* c, uint64_t* out);
/* slots(): per slot feature (UINT64_MAX = free), last_use, admit_seq, pinned, needed_soon
 * (any pointer may be NULL) */
int sfctr_cache_slots(sfctr_cache* c, uint64_t* feature, int64_t* last_use, uint64_t* admit_seq,
                      uint8_t* pinned, uint8_t* needed_soon);
/* capacity, occupied, free, pinned, needed_soon; and occupancy_diagnostics() text */
int sfctr_cache_occupancy(sfctr_cache* c, uint64_t out[5]);
int sfctr_cache_occupancy_diagnostics(sfctr_cache* c, char* buf, size_t cap);
/* HostStore::peek / slot(s).entry: rows [n*3d] (emb|m|v) + steps [n], cache or host */
int sfctr_cache_peek(sfctr_cache* c, int64_t n, const uint64_t* features, float* rows,
                     int64_t* steps);
/* One manager step for this worker (manager_get + pull_parameters_to_host +
 * push_parameters_to_cache): global_ids [n_global] = the step's
 * DedupBatch::global_ids (all workers'; the owned ones are taken in order), window_ids
 * [n_window] = every feature of the lookahead batches t..t+L-1 (duplicates allowed, may
 * be empty). needed_soon := resident window features; hits touched; misses admitted in
 * global_ids order after evicting the LRU (last_use, admit_seq) slots that are neither
 * pinned nor needed_soon. Capacity shortfall is SFCTR_ERR_RUN before anything moves.
 * Steps must increase. out (nullable) [5]: owned, hits, admitted, evicted, refilled from
 * the host pool. */
int sfctr_cache_prepare(sfctr_cache* c, int64_t step, int64_t n_global, const uint64_t* global_ids,
                        int64_t n_window, const uint64_t* window_ids, int64_t out[5]);

/* ---------------------------------------------------------------------
 * DeepFM-lite forward_backward on the device, standalone:
 * x [rows, F*d] fp32 host, labels [rows]; dense params as above. Outputs
 * (host, any may be NULL): loss (mean BCE), logits [rows], dx [rows, F*d]
 * = d(mean loss)/dx, dw1 [F*d*h], db1 [h], dw2 [h], db2 [1].
 * ------------------------------------------------------------------- */
int sfctr_model_forward_backward(int device, int32_t rows, int32_t fields, int32_t dim,
                                 int32_t hidden, const float* x, const uint8_t* labels,
                                 const float* w1, const float* b1, const float* w2,
                                 const float* b2, double* loss, float* logits, float* dx,
                                 float* dw1, float* db1, float* dw2, float* db2);

#ifdef __cplusplus
}
#endif
#endif /* SFCTR_B200_H */
