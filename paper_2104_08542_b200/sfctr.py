"""ctypes binding of the C-ABI (include/sfctr_b200.h).

This is the Python-side mirror of the reference's C++ interface
(/root/reference/proj/core/include/sfctr/*.hpp) for the hot path: the same
names (``virtual_sparse_id``, ``SyntheticGenerator.generate``,
``initial_embedding``, ``allreduce_bytes``, the trainer's step / snapshot /
ledger), the same argument meaning, and the reference's exception classes
(error.hpp:28-56) raised from the ABI's status codes.

All compute goes through ``libsfctr_b200.so`` (hand-written sm_100a kernels).
There is no fallback: if the library is missing, importing the binding
raises, and on a machine without a GPU every compute call raises CudaError.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsfctr_b200.so")


class SfctrError(RuntimeError):
    status = -1


class ConfigError(SfctrError):  # error.hpp:28-31
    status = 1


class DataError(SfctrError):  # error.hpp:34-37
    status = 2


class LogicError(SfctrError):  # error.hpp:42-45
    status = 3


class RunError(SfctrError):  # error.hpp:48-56
    status = 4

    def __init__(self, msg, step=-1):
        super().__init__(msg)
        self.step = step


class CudaError(SfctrError):
    status = 5


class NcclError(SfctrError):
    status = 6


_ERRORS = {1: ConfigError, 2: DataError, 3: LogicError, 4: RunError, 5: CudaError, 6: NcclError}

STRATEGY = {"host": 0, "prefetch": 1, "cache": 2}
SYNC = {"allreduce": 0, "alltoall": 1}


class Config(C.Structure):
    """sfctr_config — SimConfig (config.hpp:42-71) + B200 keys."""

    _fields_ = [
        ("num_workers", C.c_int32),
        ("embedding_dim", C.c_int32),
        ("num_fields", C.c_int32),
        ("batch_size_per_worker", C.c_int32),
        ("vocabulary_size", C.c_uint64),
        ("cache_capacity", C.c_uint64),
        ("lookahead_depth", C.c_int32),
        ("strategy", C.c_int32),
        ("seed", C.c_uint64),
        ("learning_rate", C.c_double),
        ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double),
        ("adam_epsilon", C.c_double),
        ("zipf_exponent", C.c_double),
        ("hidden_dim", C.c_int32),
        ("sync_mode", C.c_int32),
        ("host_table_rows", C.c_uint64),
        ("run_mode", C.c_int32),
        ("data_source", C.c_int32),
        ("criteo_path", C.c_char * 1024),
        ("deterministic", C.c_int32),
    ]

    def __init__(self, **kw):
        super().__init__()
        lib().sfctr_config_default(C.byref(self))
        for k, v in kw.items():
            setattr(self, k, v)

    def apply(self, key, value):
        _check(lib().sfctr_config_apply(C.byref(self), key.encode(), str(value).encode()))
        return self

    def load(self, path):
        _check(lib().sfctr_config_load(C.byref(self), path.encode()))
        return self

    def validate(self):
        _check(lib().sfctr_config_validate(C.byref(self)))
        return self

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class StepStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "unique", "owned", "working", "evicted", "filled_from_host", "pcie_h2d_bytes",
        "pcie_d2h_bytes", "nvlink_bytes", "kernel_launches", "total_steps", "total_working",
        "total_evicted", "total_filled_from_host", "total_kernel_launches", "total_unique",
        "total_owned", "total_nvlink_bytes", "total_free_steps", "pinned_waits",
        "total_pinned_waits")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None

P = C.c_void_p
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

# (name, restype, argtypes) — kept in sync with include/sfctr_b200.h; the
# CPU test suite checks that every declared symbol is exported.
SIGNATURES = [
    ("sfctr_last_error", C.c_char_p, []),
    ("sfctr_last_error_step", C.c_int64, []),
    ("sfctr_abi_version", C.c_int, []),
    ("sfctr_config_default", None, [P]),
    ("sfctr_config_validate", C.c_int, [P]),
    ("sfctr_config_apply", C.c_int, [P, C.c_char_p, C.c_char_p]),
    ("sfctr_config_load", C.c_int, [P, C.c_char_p]),
    ("sfctr_fnv1a64", C.c_uint64, [C.c_char_p, C.c_size_t]),
    ("sfctr_derive_seed", C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64]),
    ("sfctr_allreduce_bytes", C.c_int64, [C.c_int64, C.c_int]),
    ("sfctr_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("sfctr_generator_create", C.c_int, [P, C.c_int, C.POINTER(P)]),
    ("sfctr_generator_destroy", None, [P]),
    ("sfctr_generator_generate", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, P, P]),
    ("sfctr_generator_generate_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, P, P, P]),
    ("sfctr_generator_shard_start", C.c_uint64, [P, C.c_int32]),
    ("sfctr_initial_embedding", C.c_int, [C.c_uint64, C.c_uint64, C.c_int32, C.c_int, f64p]),
    ("sfctr_batch_source_create", C.c_int, [P, C.c_int, C.POINTER(P)]),
    ("sfctr_batch_source_destroy", None, [P]),
    ("sfctr_batch_source_read", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, u64p, u8p]),
    ("sfctr_batch_source_read_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, P, P, P]),
    ("sfctr_vsi_create", C.c_int, [C.c_int, C.c_uint64, C.c_int64, C.POINTER(P)]),
    ("sfctr_vsi_destroy", None, [P]),
    ("sfctr_virtual_sparse_id", C.c_int,
     [P, u64p, C.c_int32, C.c_int32, C.c_int32, u64p, u64p, C.POINTER(C.c_int64), i32p]),
    ("sfctr_virtual_sparse_id_device", C.c_int, [P, P, C.c_int64, P, P, P, P]),
    ("sfctr_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("sfctr_trainer_create", C.c_int, [P, C.c_int32, C.c_int32, C.c_char_p, C.c_int, C.POINTER(P)]),
    ("sfctr_trainer_destroy", None, [P]),
    ("sfctr_trainer_step", C.c_int, [P, C.c_int64, P, P, P, C.POINTER(C.c_double)]),
    ("sfctr_trainer_step_device", C.c_int, [P, C.c_int64, P, P, P, P]),
    ("sfctr_trainer_submit", C.c_int, [P, C.c_int64, P, P, P]),
    ("sfctr_trainer_prepare", C.c_int, [P, C.c_int64, P, P]),
    ("sfctr_trainer_train", C.c_int, [P, C.c_int64, P, P]),
    ("sfctr_criteo_open", C.c_int, [C.c_char_p, P, C.c_int, C.POINTER(P)]),
    ("sfctr_criteo_open_buffer", C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, P, C.c_int,
                                           C.POINTER(P)]),
    ("sfctr_criteo_destroy", None, [P]),
    ("sfctr_criteo_row_count", C.c_int64, [P]),
    ("sfctr_criteo_token_hash", C.c_uint64, [C.c_char_p, C.c_size_t]),
    ("sfctr_criteo_read_batch", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, u64p, u8p]),
    ("sfctr_criteo_read_batch_device", C.c_int, [P, C.c_int64, C.c_int32, C.c_int32, P, P, P]),
    ("sfctr_criteo_stats", C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double)]),
    ("sfctr_trainer_loss", C.c_int, [P, C.c_int64, C.POINTER(C.c_double)]),
    ("sfctr_trainer_synchronize", C.c_int, [P]),
    ("sfctr_trainer_stream", P, [P]),
    ("sfctr_trainer_logits", C.c_int, [P, f32p]),
    ("sfctr_trainer_cache_slots", C.c_int, [P, C.c_int32, u64p, i64p, u64p]),
    ("sfctr_trainer_cache_slots_range", C.c_int,
     [P, C.c_int32, C.c_uint64, C.c_uint64, u64p, i64p, u64p]),
    ("sfctr_trainer_peek_rows", C.c_int, [P, C.c_int64, u64p, P, P]),
    ("sfctr_trainer_dense_state", C.c_int, [P, P, P, P, C.POINTER(C.c_int64)]),
    ("sfctr_trainer_free_count", C.c_int, [P, C.c_int32, C.POINTER(C.c_uint64)]),
    ("sfctr_trainer_snapshot", C.c_int, [P, C.POINTER(C.c_int64), P, P, P]),
    ("sfctr_trainer_get_dense", C.c_int, [P, f32p, f32p, f32p, f32p]),
    ("sfctr_trainer_set_dense", C.c_int, [P, f32p, f32p, f32p, f32p]),
    ("sfctr_trainer_ledger", C.c_int, [P, i64p]),
    ("sfctr_trainer_stats", C.c_int, [P, C.POINTER(StepStats)]),
    ("sfctr_trainer_set_timing", C.c_int, [P, C.c_int]),
    ("sfctr_trainer_phase_times", C.c_int, [P, C.c_int32, C.c_char_p, f32p, C.POINTER(C.c_int32)]),
    ("sfctr_cache_create", C.c_int, [C.c_uint64, C.c_int32, C.c_uint64, C.c_uint64, C.c_int32,
                                     C.c_int32, C.c_int64, C.c_uint64, C.c_int, C.POINTER(P)]),
    ("sfctr_cache_destroy", None, [P]),
    ("sfctr_cache_admit", C.c_int, [P, C.c_int64, u64p, C.c_int64, P]),
    ("sfctr_cache_evict", C.c_int, [P, C.c_int64, u64p]),
    ("sfctr_cache_touch", C.c_int, [P, C.c_int64, u64p, C.c_int64]),
    ("sfctr_cache_pin", C.c_int, [P, C.c_int64, u64p, C.c_int32]),
    ("sfctr_cache_set_needed_soon", C.c_int, [P, C.c_int64, u64p, C.c_int32]),
    ("sfctr_cache_slot_of", C.c_int, [P, C.c_int64, u64p, i64p]),
    ("sfctr_cache_free_count", C.c_int, [P, C.POINTER(C.c_uint64)]),
    ("sfctr_cache_slots", C.c_int, [P, P, P, P, P, P]),
    ("sfctr_cache_occupancy", C.c_int, [P, u64p]),
    ("sfctr_cache_occupancy_diagnostics", C.c_int, [P, C.c_char_p, C.c_size_t]),
    ("sfctr_cache_peek", C.c_int, [P, C.c_int64, u64p, P, P]),
    ("sfctr_cache_prepare", C.c_int, [P, C.c_int64, C.c_int64, P, C.c_int64, P, i64p]),
    ("sfctr_model_forward_backward", C.c_int,
     [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p, u8p, f32p, f32p, f32p, f32p,
      C.POINTER(C.c_double), P, P, P, P, P, P]),
]


def lib():
    """Load libsfctr_b200.so; raises loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C paper_2104_08542_b200` "
                          "(there is no fallback implementation)")
    L = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc):
    if rc == 0:
        return
    L = lib()
    msg = L.sfctr_last_error().decode(errors="replace")
    cls = _ERRORS.get(rc, SfctrError)
    if cls is RunError:
        raise RunError(msg, L.sfctr_last_error_step())
    raise cls(msg)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ---------------- core helpers ----------------

def fnv1a64(data: bytes) -> int:  # rng.hpp:27-34
    return lib().sfctr_fnv1a64(data, len(data))


def derive_seed(base: int, label: str, index: int = 0) -> int:  # rng.hpp:49-56
    return lib().sfctr_derive_seed(base, label.encode(), index)


def allreduce_bytes(payload: int, workers: int) -> int:  # comm.hpp:36-41
    r = lib().sfctr_allreduce_bytes(payload, workers)
    if r < 0:
        raise LogicError(lib().sfctr_last_error().decode())
    return r


def device_count() -> int:
    n = C.c_int(0)
    lib().sfctr_device_count(C.byref(n))
    return n.value


def initial_embedding(seed: int, feature: int, dim: int, device: int = 0) -> np.ndarray:
    """initial_embedding(seed, FeatureId, dim) (generator.hpp:62), computed on the GPU."""
    out = np.zeros(dim, np.float64)
    _check(lib().sfctr_initial_embedding(seed, feature, dim, device, out))
    return out


# ---------------- generator ----------------

class SyntheticGenerator:
    """SyntheticGenerator(config) (generator.hpp:35-62) on the device."""

    def __init__(self, config: Config, device: int = 0):
        self.config = config
        self.fields = config.num_fields
        self.global_rows = config.num_workers * config.batch_size_per_worker
        h = P()
        _check(lib().sfctr_generator_create(C.byref(config), device, C.byref(h)))
        self._h = h

    def generate(self, step, row0=0, nrows=None):
        """RawBatch generate(step) (generator.cpp:82-108): rows [row0, row0+nrows)."""
        n = self.global_rows - row0 if nrows is None else nrows
        f = np.zeros(n * self.fields, np.uint64)
        y = np.zeros(n, np.uint8)
        _check(lib().sfctr_generator_generate(self._h, step, row0, n, _ptr(f), _ptr(y)))
        return f, y

    def generate_device(self, step, row0, nrows, d_features, d_labels, stream=None):
        _check(lib().sfctr_generator_generate_device(self._h, step, row0, nrows, d_features,
                                                     d_labels, stream))

    def shard_start(self, field):
        return lib().sfctr_generator_shard_start(self._h, field)

    def close(self):
        if getattr(self, "_h", None):
            lib().sfctr_generator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------- VSI ----------------

class BatchSource:
    """The configured DataSource (config key `data`, config.cpp:146-154): the synthetic
    generator or the Criteo TSV at criteo_path, one read interface."""

    def __init__(self, config: Config, device: int = 0):
        self._h = P()
        self.fields = config.num_fields
        self.global_rows = config.num_workers * config.batch_size_per_worker
        _check(lib().sfctr_batch_source_create(C.byref(config), device, C.byref(self._h)))

    def read(self, step, row0=0, nrows=None):
        n = self.global_rows if nrows is None else nrows
        f = np.zeros(n * self.fields, np.uint64)
        y = np.zeros(n, np.uint8)
        _check(lib().sfctr_batch_source_read(self._h, step, row0, n, f, y))
        return f, y

    def read_device(self, step, row0, nrows, d_features, d_labels, stream=None):
        _check(lib().sfctr_batch_source_read_device(self._h, step, row0, nrows, d_features,
                                                    d_labels, stream))

    def close(self):
        if self._h:
            lib().sfctr_batch_source_destroy(self._h)
            self._h = P()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class VirtualSparseId:
    """Device context for virtual_sparse_id (vsi.hpp:29)."""

    def __init__(self, key_space: int, max_ids: int, device: int = 0):
        h = P()
        _check(lib().sfctr_vsi_create(device, key_space, max_ids, C.byref(h)))
        self._h = h
        self.max_ids = max_ids

    def __call__(self, features, rows, fields, num_workers=1):
        """Returns (global_ids [U] u64, virtual_ids [rows*fields] u64, row_ranges [W,2])."""
        feats = np.ascontiguousarray(features, np.uint64)
        n = rows * fields
        g = np.zeros(max(n, 1), np.uint64)
        v = np.zeros(max(n, 1), np.uint64)
        rr = np.zeros(2 * max(num_workers, 1), np.int32)
        u = C.c_int64(0)
        _check(lib().sfctr_virtual_sparse_id(self._h, feats if feats.size else np.zeros(1, np.uint64),
                                             rows, fields, num_workers, g, v, C.byref(u), rr))
        return g[:u.value].copy(), v[:n].copy(), rr.reshape(-1, 2)

    def device_call(self, d_ids, n, d_gids, d_vids, d_unique, stream=None):
        _check(lib().sfctr_virtual_sparse_id_device(self._h, d_ids, n, d_gids, d_vids, d_unique,
                                                    stream))

    def close(self):
        if getattr(self, "_h", None):
            lib().sfctr_vsi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def virtual_sparse_id(features, rows, fields, num_workers=1, key_space=None, device=0):
    """One-shot DedupBatch virtual_sparse_id(const RawBatch&, int) (vsi.hpp:29)."""
    feats = np.ascontiguousarray(features, np.uint64)
    if key_space is None:  # direct-mapped below 2^31 ids, else the hashed table (any u64)
        mx = int(feats.max()) if feats.size else 0
        ks = mx + 1 if mx < (1 << 31) else 0
    else:
        ks = int(key_space)
    v = VirtualSparseId(ks, max(rows * fields, 1), device)
    try:
        return v(feats, rows, fields, num_workers)
    finally:
        v.close()


# ---------------- trainer ----------------

def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().sfctr_nccl_unique_id(buf))
    return buf.raw


class Trainer:
    """Host-Manager + GPU-Worker lanes of one process."""

    def __init__(self, config: Config, rank=0, world=1, nccl_id=None, device=0):
        self.config = config
        self.rank, self.world = rank, world
        self.lanes = config.num_workers // world
        self.rows = self.lanes * config.batch_size_per_worker
        self.fields = config.num_fields
        self.dim = config.embedding_dim
        self.hidden = config.hidden_dim
        h = P()
        _check(lib().sfctr_trainer_create(C.byref(config), rank, world, nccl_id, device,
                                          C.byref(h)))
        self._h = h

    def step(self, step, features, labels, window=None):
        """One BSP step on this process's rows (HOST buffers); returns the mean logloss."""
        f = np.ascontiguousarray(features, np.uint64)
        y = np.ascontiguousarray(labels, np.uint8)
        assert f.size == self.rows * self.fields and y.size == self.rows
        w = None if window is None else np.ascontiguousarray(window, np.uint64)
        loss = C.c_double(0)
        _check(lib().sfctr_trainer_step(self._h, step, _ptr(f), _ptr(y), _ptr(w), C.byref(loss)))
        return loss.value

    def submit(self, step, features, labels, window=None):
        """Enqueue one step on HOST buffers without waiting (read it back with loss()).
        The arrays must stay alive and unchanged until loss(step) returns."""
        f = np.ascontiguousarray(features, np.uint64)
        y = np.ascontiguousarray(labels, np.uint8)
        assert f.size == self.rows * self.fields and y.size == self.rows
        w = None if window is None else np.ascontiguousarray(window, np.uint64)
        self._keep = getattr(self, "_keep", {})
        self._keep[step] = (f, y, w)
        _check(lib().sfctr_trainer_submit(self._h, step, _ptr(f), _ptr(y), _ptr(w)))

    def loss(self, step):
        l = C.c_double(0)
        try:
            _check(lib().sfctr_trainer_loss(self._h, step, C.byref(l)))
        finally:
            getattr(self, "_keep", {}).pop(step, None)
        return l.value

    def prepare_device(self, step, d_features, d_window=None):
        """Host-Manager stage of `step` (device buffers), enqueued."""
        _check(lib().sfctr_trainer_prepare(self._h, step, d_features, d_window))

    def train_device(self, step, d_labels, d_loss=None):
        """GPU-Worker stage of the prepared `step`, enqueued."""
        _check(lib().sfctr_trainer_train(self._h, step, d_labels, d_loss))

    def step_device(self, step, d_features, d_labels, d_window=None, d_loss=None):
        _check(lib().sfctr_trainer_step_device(self._h, step, d_features, d_labels, d_window,
                                               d_loss))

    def synchronize(self):
        _check(lib().sfctr_trainer_synchronize(self._h))

    @property
    def stream(self):
        return lib().sfctr_trainer_stream(self._h)

    def logits(self):
        out = np.zeros(self.rows, np.float32)
        _check(lib().sfctr_trainer_logits(self._h, out))
        return out

    def cache_slots(self, lane=0, first=0, count=None):
        """CacheBuffer::slots() of a local lane (slot -> feature, last_use, admit_seq);
        first / count select a slot range (large caches)."""
        C_ = self.config.cache_capacity
        if count is None and first == 0:
            f = np.zeros(C_, np.uint64)
            lu = np.zeros(C_, np.int64)
            seq = np.zeros(C_, np.uint64)
            _check(lib().sfctr_trainer_cache_slots(self._h, lane, f, lu, seq))
            return f, lu, seq
        n = max(0, min(C_ - first, C_ if count is None else count))
        f = np.zeros(max(n, 1), np.uint64)
        lu = np.zeros(max(n, 1), np.int64)
        seq = np.zeros(max(n, 1), np.uint64)
        _check(lib().sfctr_trainer_cache_slots_range(self._h, lane, first, n, f, lu, seq))
        return f[:n], lu[:n], seq[:n]

    def peek_rows(self, features):
        """HostStore::peek for features owned by this process: (rows [n, 3d] fp32 =
        emb|m|v, adam steps [n])."""
        f = np.ascontiguousarray(features, np.uint64).ravel()
        rows = np.zeros((max(f.size, 1), 3 * self.dim), np.float32)
        st = np.zeros(max(f.size, 1), np.int64)
        _check(lib().sfctr_trainer_peek_rows(self._h, f.size, f, _ptr(rows), _ptr(st)))
        return rows[:f.size], st[:f.size]

    def dense_state(self):
        """(params, m, v) each [P] = W1 | b1 | w2 | b2 (fp32), and the dense Adam step."""
        P_ = self.fields * self.dim * self.hidden + 2 * self.hidden + 1
        p, m, v = (np.zeros(P_, np.float32) for _ in range(3))
        st = C.c_int64(0)
        _check(lib().sfctr_trainer_dense_state(self._h, _ptr(p), _ptr(m), _ptr(v), C.byref(st)))
        return p, m, v, st.value

    def free_count(self, lane=0):
        n = C.c_uint64(0)
        _check(lib().sfctr_trainer_free_count(self._h, lane, C.byref(n)))
        return n.value

    def snapshot(self):
        """HostStore::snapshot_sorted over this process's rows: (features, rows[n,3d], steps)."""
        n = C.c_int64(0)
        _check(lib().sfctr_trainer_snapshot(self._h, C.byref(n), None, None, None))
        f = np.zeros(max(n.value, 1), np.uint64)
        r = np.zeros((max(n.value, 1), 3 * self.dim), np.float32)
        s = np.zeros(max(n.value, 1), np.int64)
        _check(lib().sfctr_trainer_snapshot(self._h, C.byref(n), _ptr(f), _ptr(r), _ptr(s)))
        return f[:n.value], r[:n.value], s[:n.value]

    def get_dense(self):
        K = self.fields * self.dim
        w1 = np.zeros(K * self.hidden, np.float32)
        b1 = np.zeros(self.hidden, np.float32)
        w2 = np.zeros(self.hidden, np.float32)
        b2 = np.zeros(1, np.float32)
        _check(lib().sfctr_trainer_get_dense(self._h, w1, b1, w2, b2))
        return w1, b1, w2, b2

    def set_dense(self, w1, b1, w2, b2):
        c = lambda a: np.ascontiguousarray(a, np.float32).ravel()  # noqa: E731
        _check(lib().sfctr_trainer_set_dense(self._h, c(w1), c(b1), c(w2), c(b2)))

    def ledger(self):
        out = np.zeros(4, np.int64)
        _check(lib().sfctr_trainer_ledger(self._h, out))
        return {"host_to_worker": int(out[0]), "worker_to_host": int(out[1]),
                "interworker": int(out[2]), "swap_events": int(out[3])}

    def stats(self):
        s = StepStats()
        _check(lib().sfctr_trainer_stats(self._h, C.byref(s)))
        return s.as_dict()

    def set_timing(self, on=True):
        _check(lib().sfctr_trainer_set_timing(self._h, 1 if on else 0))

    def phase_times(self):
        n = C.c_int32(0)
        names = C.create_string_buffer(64 * 32)
        ms = np.zeros(64, np.float32)
        _check(lib().sfctr_trainer_phase_times(self._h, 64, names, ms, C.byref(n)))
        out = []
        for i in range(min(n.value, 64)):
            nm = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
            out.append((nm, float(ms[i])))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().sfctr_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CacheBuffer:
    """One worker's device MixCache: CacheBuffer (cache_buffer.hpp:40-86) + HostStore
    (host_store.hpp:61-92) + the manager step, sfctr_cache_* in
    include/sfctr_b200.h. Feature arguments are sequences of owned feature ids; batched
    calls apply in order and raise LogicError where the reference would, after the
    preceding features took effect."""

    def __init__(self, capacity, dim, seed=7, key_space=1 << 20, num_workers=1, worker=0,
                 max_batch=1 << 16, host_reserve=0, device=0):
        self._h = P()
        self.capacity, self.dim = capacity, dim
        _check(lib().sfctr_cache_create(capacity, dim, seed, key_space, num_workers, worker,
                                        max_batch, host_reserve, device, C.byref(self._h)))

    @staticmethod
    def _f(features):
        return np.ascontiguousarray(np.atleast_1d(np.asarray(features, np.uint64)))

    def admit(self, features, step):
        f = self._f(features)
        slots = np.zeros(max(f.size, 1), np.uint64)
        _check(lib().sfctr_cache_admit(self._h, f.size, f, step, _ptr(slots)))
        return slots[:f.size]

    def evict(self, features):
        f = self._f(features)
        _check(lib().sfctr_cache_evict(self._h, f.size, f))

    def touch(self, features, step):
        f = self._f(features)
        _check(lib().sfctr_cache_touch(self._h, f.size, f, step))

    def pin(self, features):
        f = self._f(features)
        _check(lib().sfctr_cache_pin(self._h, f.size, f, 1))

    def unpin(self, features):
        f = self._f(features)
        _check(lib().sfctr_cache_pin(self._h, f.size, f, 0))

    def set_needed_soon(self, features, value=True):
        f = self._f(features)
        _check(lib().sfctr_cache_set_needed_soon(self._h, f.size, f, 1 if value else 0))

    def slot_of(self, features):
        f = self._f(features)
        out = np.zeros(max(f.size, 1), np.int64)
        _check(lib().sfctr_cache_slot_of(self._h, f.size, f, out))
        return out[:f.size]

    def resident(self, feature):
        return int(self.slot_of([feature])[0]) >= 0

    def free_count(self):
        n = C.c_uint64(0)
        _check(lib().sfctr_cache_free_count(self._h, C.byref(n)))
        return n.value

    def slots(self):
        """(feature [UINT64_MAX = free], last_use, admit_seq, pinned, needed_soon) per slot"""
        n = self.capacity
        f, lu, seq = np.zeros(n, np.uint64), np.zeros(n, np.int64), np.zeros(n, np.uint64)
        pin, nd = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        _check(lib().sfctr_cache_slots(self._h, _ptr(f), _ptr(lu), _ptr(seq), _ptr(pin), _ptr(nd)))
        return f, lu, seq, pin, nd

    def occupancy(self):
        out = np.zeros(5, np.uint64)
        _check(lib().sfctr_cache_occupancy(self._h, out))
        return dict(zip(("capacity", "occupied", "free", "pinned", "needed_soon"),
                        (int(x) for x in out)))

    def occupancy_diagnostics(self):
        buf = C.create_string_buffer(256)
        _check(lib().sfctr_cache_occupancy_diagnostics(self._h, buf, 256))
        return buf.value.decode()

    def peek(self, features):
        f = self._f(features)
        rows = np.zeros((max(f.size, 1), 3 * self.dim), np.float32)
        st = np.zeros(max(f.size, 1), np.int64)
        _check(lib().sfctr_cache_peek(self._h, f.size, f, _ptr(rows), _ptr(st)))
        return rows[:f.size], st[:f.size]

    def prepare(self, step, global_ids, window_ids=None):
        g = self._f(global_ids)
        w = self._f(window_ids) if window_ids is not None and len(window_ids) else None
        out = np.zeros(5, np.int64)
        _check(lib().sfctr_cache_prepare(self._h, step, g.size, _ptr(g), 0 if w is None else w.size,
                                         _ptr(w), out))
        return dict(zip(("owned", "hits", "admitted", "evicted", "refilled"), (int(x) for x in out)))

    def close(self):
        if self._h:
            lib().sfctr_cache_destroy(self._h)
            self._h = P()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def model_forward_backward(x, labels, w1, b1, w2, b2, fields, dim, hidden, device=0):
    """DeepFM-lite forward_backward on the device."""
    x = np.ascontiguousarray(x, np.float32)
    rows = x.shape[0]
    K = fields * dim
    logits = np.zeros(rows, np.float32)
    dx = np.zeros((rows, K), np.float32)
    dw1 = np.zeros(K * hidden, np.float32)
    db1 = np.zeros(hidden, np.float32)
    dw2 = np.zeros(hidden, np.float32)
    db2 = np.zeros(1, np.float32)
    loss = C.c_double(0)
    c = lambda a: np.ascontiguousarray(a, np.float32).ravel()  # noqa: E731
    _check(lib().sfctr_model_forward_backward(
        device, rows, fields, dim, hidden, x.ravel(), np.ascontiguousarray(labels, np.uint8),
        c(w1), c(b1), c(w2), c(b2), C.byref(loss), _ptr(logits), _ptr(dx), _ptr(dw1), _ptr(db1),
        _ptr(dw2), _ptr(db2)))
    return {"loss": loss.value, "logits": logits, "dx": dx, "dw1": dw1, "db1": db1, "dw2": dw2,
            "db2": float(db2[0])}


class CriteoReader:
    """CriteoReader (criteo.hpp:37-58) on the device: the TSV is parsed and hashed by the
    sm_100a kernels at construction; read_batch(step) returns the wrapping global batch."""

    kNumericColumns = 13
    kCategoricalColumns = 26

    def __init__(self, path, config: Config, device=0, _buffer=None, _name=None):
        self.config = config
        self.global_rows = config.num_workers * config.batch_size_per_worker
        h = P()
        if _buffer is None:
            _check(lib().sfctr_criteo_open(str(path).encode(), C.byref(config), device,
                                           C.byref(h)))
        else:
            _check(lib().sfctr_criteo_open_buffer(_buffer, len(_buffer),
                                                  (_name or "<buffer>").encode(),
                                                  C.byref(config), device, C.byref(h)))
        self._h = h

    @classmethod
    def from_bytes(cls, data: bytes, config: Config, name="<buffer>", device=0):
        return cls(None, config, device, _buffer=data, _name=name)

    @staticmethod
    def token_hash(token) -> int:
        b = token.encode() if isinstance(token, str) else bytes(token)
        return lib().sfctr_criteo_token_hash(b, len(b))

    def row_count(self) -> int:
        return lib().sfctr_criteo_row_count(self._h)

    def read_batch(self, step, row0=0, nrows=None):
        n = self.global_rows - row0 if nrows is None else nrows
        f = np.zeros(n * 26, np.uint64)
        y = np.zeros(n, np.uint8)
        _check(lib().sfctr_criteo_read_batch(self._h, step, row0, n, f, y))
        return f, y

    def read_batch_device(self, step, row0, nrows, d_features, d_labels, stream=None):
        _check(lib().sfctr_criteo_read_batch_device(self._h, step, row0, nrows, d_features,
                                                    d_labels, stream))

    def stats(self):
        b, l, ms = C.c_int64(0), C.c_int64(0), C.c_double(0)
        _check(lib().sfctr_criteo_stats(self._h, C.byref(b), C.byref(l), C.byref(ms)))
        return {"bytes": b.value, "lines": l.value, "parse_ms": ms.value}

    def close(self):
        if self._h:
            lib().sfctr_criteo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
