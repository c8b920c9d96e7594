"""ctypes loaders for the TEST-ONLY oracle libraries.

- ``oracle/liboracle.so``: the C restatement (oracle/sfctr_oracle.c).
- ``oracle/_ref/libsfctr_ref.so``: the reference's own TUs + shim, built by
  oracle/build_ref.sh where /root/reference exists (it travels to the GPU
  box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product never does.
"""
import ctypes as C
import hashlib
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsfctr_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class OrcConfig(C.Structure):
    _fields_ = [
        ("num_workers", C.c_int),
        ("embedding_dim", C.c_int),
        ("num_fields", C.c_int),
        ("batch_size_per_worker", C.c_int),
        ("vocabulary_size", C.c_uint64),
        ("cache_capacity", C.c_uint64),
        ("lookahead_depth", C.c_int),
        ("seed", C.c_uint64),
        ("learning_rate", C.c_double),
        ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double),
        ("adam_epsilon", C.c_double),
        ("zipf_exponent", C.c_double),
        ("hidden_dim", C.c_int),
        ("num_threads", C.c_int),
    ]


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_oracle = None


def oracle():
    global _oracle
    if _oracle is not None:
        return _oracle
    if not os.path.exists(ORACLE_SO):
        raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
    L = C.CDLL(ORACLE_SO)
    _sig(L, "orc_fnv1a64", C.c_uint64, [C.c_char_p, C.c_size_t])
    _sig(L, "orc_derive_seed", C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64])
    _sig(L, "orc_truth_weight", C.c_double, [C.c_uint64, C.c_uint64])
    _sig(L, "orc_initial_embedding", None, [C.c_uint64, C.c_uint64, C.c_int, f64p])
    _sig(L, "orc_allreduce_bytes", C.c_int64, [C.c_int64, C.c_int])
    _sig(L, "orc_gen_create", C.c_void_p, [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_double])
    _sig(L, "orc_gen_destroy", None, [C.c_void_p])
    _sig(L, "orc_gen_generate_rows", None, [C.c_void_p, C.c_int64, C.c_int, C.c_int, u64p, u8p])
    _sig(L, "orc_gen_shard_start", C.c_uint64, [C.c_void_p, C.c_int])
    _sig(L, "orc_vsi", C.c_int64, [u64p, C.c_int, C.c_int, C.c_int, u64p, u64p])
    _sig(L, "orc_config_default", None, [C.POINTER(OrcConfig)])
    _sig(L, "orc_sim_create", C.c_void_p, [C.POINTER(OrcConfig)])
    _sig(L, "orc_sim_destroy", None, [C.c_void_p])
    _sig(L, "orc_last_error", C.c_char_p, [])
    _sig(L, "orc_sim_step", C.c_int,
         [C.c_void_p, C.c_int64, u64p, u8p, C.c_void_p, C.c_int, C.POINTER(C.c_double),
          C.c_void_p, C.c_void_p])
    _sig(L, "orc_sim_cache_slots", None, [C.c_void_p, C.c_int, u64p, i64p, u64p])
    _sig(L, "orc_sim_free_count", C.c_uint64, [C.c_void_p, C.c_int])
    _sig(L, "orc_sim_snapshot", C.c_int64, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
    _sig(L, "orc_sim_dense", None, [C.c_void_p, f64p, f64p, f64p, f64p])
    _sig(L, "orc_sim_set_dense", None, [C.c_void_p, f64p, f64p, f64p, f64p])
    _sig(L, "orc_sim_ledger", None, [C.c_void_p, i64p])
    _sig(L, "orc_sim_get_rows", C.c_int64, [C.c_void_p, C.c_int64, u64p, C.c_void_p, C.c_void_p])
    _sig(L, "orc_sim_set_rows", C.c_int, [C.c_void_p, C.c_int64, u64p, C.c_void_p, C.c_void_p])
    _sig(L, "orc_sim_keep_grads", None, [C.c_void_p, C.c_int])
    _sig(L, "orc_sim_last_grads", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_int64)])
    _sig(L, "orc_sim_get_dense_state", None,
         [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)])
    _sig(L, "orc_sim_set_dense_state", None,
         [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)])
    _sig(L, "orc_sim_last_unique", C.c_int64, [C.c_void_p])
    _sig(L, "orc_dense_init", None, [C.c_uint64, C.c_int, C.c_int, f64p, f64p, f64p, f64p])
    _sig(L, "orc_model_fwd_bwd", C.c_double,
         [f64p, u8p, C.c_int, C.c_int, C.c_int, C.c_int, f64p, f64p, f64p, C.c_double,
          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int])
    _sig(L, "orc_manager_example", C.c_int64,
         [C.c_uint64, u64p, C.c_int, u64p, C.c_int, u64p, C.c_int, u64p, u64p])
    _sig(L, "orc_criteo_parse", C.c_int64,
         [C.c_char_p, C.c_size_t, C.c_uint64, u64p, u8p, C.c_int64, C.POINTER(C.c_int64),
          C.c_char_p, C.c_size_t])
    _sig(L, "orc_criteo_read_batch", None,
         [u64p, u8p, C.c_int64, C.c_int64, C.c_int, u64p, u8p])
    _oracle = L
    return L


_ref = None


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is not None:
        return _ref
    L = C.CDLL(REF_SO)
    _sig(L, "ref_last_error", C.c_char_p, [])
    _sig(L, "ref_fnv1a64", C.c_uint64, [C.c_char_p, C.c_size_t])
    _sig(L, "ref_derive_seed", C.c_uint64, [C.c_uint64, C.c_char_p, C.c_uint64])
    _sig(L, "ref_allreduce_bytes", C.c_int64, [C.c_int64, C.c_int])
    _sig(L, "ref_initial_embedding", None, [C.c_uint64, C.c_uint64, C.c_int, f64p])
    _sig(L, "ref_truth_weight", C.c_double, [C.c_uint64, C.c_uint64])
    _sig(L, "ref_gen_create", C.c_void_p,
         [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_double])
    _sig(L, "ref_gen_destroy", None, [C.c_void_p])
    _sig(L, "ref_gen_generate", None, [C.c_void_p, C.c_int64, u64p, u8p])
    _sig(L, "ref_vsi", C.c_int64, [u64p, u8p, C.c_int, C.c_int, C.c_int, u64p, u64p, i32p])
    _sig(L, "ref_cache_create", C.c_void_p, [C.c_uint64, C.c_int, C.c_uint64])
    _sig(L, "ref_cache_destroy", None, [C.c_void_p])
    _sig(L, "ref_cache_admit", C.c_int64, [C.c_void_p, C.c_uint64, C.c_int64])
    _sig(L, "ref_cache_evict", C.c_int, [C.c_void_p, C.c_uint64])
    _sig(L, "ref_cache_touch", C.c_int, [C.c_void_p, C.c_uint64, C.c_int64])
    _sig(L, "ref_cache_pin", C.c_int, [C.c_void_p, C.c_uint64, C.c_int])
    _sig(L, "ref_cache_set_needed_soon", C.c_int, [C.c_void_p, C.c_uint64, C.c_int])
    _sig(L, "ref_cache_slot_of", C.c_int64, [C.c_void_p, C.c_uint64])
    _sig(L, "ref_cache_free_count", C.c_uint64, [C.c_void_p])
    _sig(L, "ref_cache_host_size", C.c_uint64, [C.c_void_p])
    _sig(L, "ref_cache_slots", None, [C.c_void_p, u64p, i64p, u64p])
    _sig(L, "ref_cache_host_row", C.c_int, [C.c_void_p, C.c_uint64, f64p, C.POINTER(C.c_int64)])
    _sig(L, "ref_config_check", C.c_int, [C.c_char_p, C.c_char_p, C.c_int])
    _sig(L, "ref_criteo_open", C.c_void_p,
         [C.c_char_p, C.c_int, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int)])
    _sig(L, "ref_criteo_destroy", None, [C.c_void_p])
    _sig(L, "ref_criteo_rows", C.c_int64, [C.c_void_p])
    _sig(L, "ref_criteo_read_batch", None, [C.c_void_p, C.c_int64, u64p, u8p])
    _sig(L, "ref_criteo_token_hash", C.c_uint64, [C.c_char_p, C.c_size_t])
    _ref = L
    return L


# ---------------- convenience wrappers ----------------

def oracle_generate(rows, fields, vocab, seed, zipf, step, row0=0, nrows=None):
    L = oracle()
    g = L.orc_gen_create(rows, fields, vocab, seed, zipf)
    try:
        n = rows if nrows is None else nrows
        f = np.zeros(n * fields, np.uint64)
        y = np.zeros(n, np.uint8)
        L.orc_gen_generate_rows(g, step, row0, n, f, y)
        return f, y
    finally:
        L.orc_gen_destroy(g)


def ref_generate(workers, fields, batch, vocab, seed, zipf, step):
    L = ref()
    g = L.ref_gen_create(workers, fields, batch, vocab, seed, zipf)
    try:
        rows = workers * batch
        f = np.zeros(rows * fields, np.uint64)
        y = np.zeros(rows, np.uint8)
        L.ref_gen_generate(g, step, f, y)
        return f, y
    finally:
        L.ref_gen_destroy(g)


def oracle_vsi(features, rows, fields, workers=1):
    L = oracle()
    gids = np.zeros(rows * fields, np.uint64)
    vids = np.zeros(rows * fields, np.uint64)
    u = L.orc_vsi(np.ascontiguousarray(features, np.uint64), rows, fields, workers, gids, vids)
    if u < 0:
        raise RuntimeError(L.orc_last_error().decode())
    return gids[:u].copy(), vids


def ref_vsi(features, labels, rows, fields, workers=1):
    L = ref()
    gids = np.zeros(rows * fields, np.uint64)
    vids = np.zeros(rows * fields, np.uint64)
    rr = np.zeros(2 * workers, np.int32)
    u = L.ref_vsi(np.ascontiguousarray(features, np.uint64), np.ascontiguousarray(labels, np.uint8),
                  rows, fields, workers, gids, vids, rr)
    if u < 0:
        raise RuntimeError(L.ref_last_error().decode())
    return gids[:u].copy(), vids, rr


def fnv_digest(*arrays):
    """FNV-1a over the little-endian bytes of the arrays, in order."""
    h = 0xcbf29ce484222325
    for a in arrays:
        for byte in np.ascontiguousarray(a).view(np.uint8).tobytes():
            h ^= byte
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv_digest_fast(*arrays):
    L = oracle()
    buf = b"".join(np.ascontiguousarray(a).view(np.uint8).tobytes() for a in arrays)
    return L.orc_fnv1a64(buf, len(buf))


# ---------------- Criteo TSV (criteo.cpp) ----------------

def make_criteo_tsv(rows, seed=0, edge_cases=True):
    """Synthetic Criteo-format bytes: label, 13 numerics, 26 hex tokens per line, with
    the reader's edge cases mixed in (empty categorical cells, CRLF endings, empty and
    "\r"-only lines, long and non-hex tokens, no final newline)."""
    rng = np.random.default_rng(seed)
    out = []
    for r in range(rows):
        lab = str(int(rng.integers(0, 2)))
        nums = [str(int(x)) if rng.random() > 0.2 else "" for x in rng.integers(0, 5000, 13)]
        cats = []
        for f in range(26):
            u = rng.random()
            if edge_cases and u < 0.08:
                cats.append("")
            elif edge_cases and u < 0.1:
                cats.append("tok_" + "x" * int(rng.integers(1, 40)))
            else:
                cats.append("%08x" % int(rng.integers(0, 1 << 32)))
        line = "\t".join([lab] + nums + cats)
        if edge_cases and rng.random() < 0.1:
            line += "\r"
        out.append(line)
        if edge_cases and rng.random() < 0.03:
            out.append("" if rng.random() < 0.5 else "\r")
    data = "\n".join(out)
    if not edge_cases or rng.random() < 0.5:
        data += "\n"
    return data.encode()


def oracle_criteo(data, vocab):
    """(features [rows*26] u64, labels [rows] u8) or raises ValueError(line, message)."""
    O = oracle()
    cap = data.count(b"\n") + 2
    f = np.zeros(cap * 26, np.uint64)
    y = np.zeros(cap, np.uint8)
    line = C.c_int64(0)
    msg = C.create_string_buffer(512)
    rows = O.orc_criteo_parse(data, len(data), vocab, f, y, cap, C.byref(line), msg, 512)
    if rows == -1:
        raise ValueError(line.value, msg.value.decode())
    if rows == -2:
        raise ValueError(0, "no data rows")
    return f[:rows * 26].copy(), y[:rows].copy()


def u64_golden_batches(golden):
    """the golden u64 batches (tests/golden/make_golden.py: same rng calls)"""
    rng = np.random.default_rng(2026)
    out = []
    for rec in golden["vsi_u64_examples"]:
        rows, F = rec["rows"], rec["fields"]
        pool = np.concatenate([rng.integers(0, 1 << 62, 40, dtype=np.uint64) * np.uint64(3),
                               np.array([0, 1, (1 << 32) - 1, 1 << 32, (1 << 64) - 1,
                                         (1 << 64) - 2], np.uint64)])
        f = pool[rng.integers(0, pool.size, rows * F)]
        assert hashlib.sha256(f.tobytes()).hexdigest() == rec["features_sha256"]
        if "features" in rec:
            assert [str(int(x)) for x in f] == rec["features"]
        out.append((rec, f))
    return out
