"""CPU tests of the parity oracle (oracle/sfctr_oracle.c).

The oracle is pinned two ways: against committed golden vectors produced by
the reference's own compiled code (tests/golden/make_golden.py), and — where
the prebuilt oracle/_ref library is present — directly against the reference
TUs on fresh random inputs. The SPEC.md worked examples and acceptance
properties that concern the hot path are checked here on the
oracle; the GPU tests then compare the device path with this oracle.
"""
import hashlib
import struct

import numpy as np
import pytest

from oracle_lib import (OrcConfig, oracle, oracle_generate, oracle_vsi, ref, ref_available,
                        ref_generate, ref_vsi)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


def dhex(x):
    return struct.pack("<d", float(x)).hex()


# ---------------- golden vectors (reference output) ----------------

def test_rng_golden(golden):
    O = oracle()
    for s, h in golden["fnv1a64"].items():
        assert format(O.orc_fnv1a64(s.encode(), len(s)), "016x") == h
    for base, label, idx, h in golden["derive_seed"]:
        assert format(O.orc_derive_seed(base, label.encode(), idx), "016x") == h
    for f, want in golden["initial_embedding_seed7_d80"].items():
        v = np.zeros(80)
        O.orc_initial_embedding(7, int(f), 80, v)
        assert [dhex(x) for x in v] == want
    for f, want in golden["truth_weight_seed7"].items():
        assert dhex(O.orc_truth_weight(7, int(f))) == want
    for p, w, want in golden["allreduce_bytes"]:
        assert O.orc_allreduce_bytes(p, w) == want


def test_generator_and_vsi_golden(golden):
    for rec in golden["batches"]:
        if rec["workers"] * rec["batch"] * rec["fields"] > 400_000:
            continue  # cfg2 W=2 covered on the GPU side
        rows = rec["workers"] * rec["batch"]
        f, y = oracle_generate(rows, rec["fields"], rec["vocab"], rec["seed"], rec["zipf"],
                               rec["step"])
        assert sha(f) == rec["features_sha256"], rec["name"]
        assert sha(y) == rec["labels_sha256"], rec["name"]
        g, v = oracle_vsi(f, rows, rec["fields"], rec["workers"])
        assert len(g) == rec["unique"]
        assert sha(g) == rec["global_ids_sha256"]
        assert sha(v) == rec["virtual_ids_sha256"]


def test_generator_random_access_rows(golden):
    rec = next(r for r in golden["batches"] if r["name"] == "mini_w4" and r["step"] == 5)
    rows = rec["workers"] * rec["batch"]
    full, yf = oracle_generate(rows, 26, rec["vocab"], 7, 1.2, 5)
    parts = [oracle_generate(rows, 26, rec["vocab"], 7, 1.2, 5, row0=r0, nrows=256)
             for r0 in range(0, rows, 256)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), full)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), yf)


def test_vsi_spec_examples(golden):
    # SPEC.md:132-134 / PAPER.md:292
    for ex in golden["vsi_examples"]:
        g, v = oracle_vsi(np.array(ex["features"], np.uint64), ex["rows"], ex["fields"])
        assert g.tolist() == ex["global_ids"]
        assert v.tolist() == ex["virtual_ids"]
    g, v = oracle_vsi(np.array([1, 3, 2, 2, 3, 1], np.uint64), 2, 3)
    assert g.tolist() == [1, 3, 2] and v.tolist() == [0, 1, 2, 2, 1, 0]


def test_vsi_checks():
    O = oracle()
    z = np.zeros(4, np.uint64)
    assert O.orc_vsi(z, 0, 2, 1, z, z) == -3  # empty batch (vsi.cpp:24)
    assert O.orc_vsi(z, 3, 1, 2, z, z) == -3  # uneven split (vsi.cpp:30)


# ---------------- oracle vs the reference TUs on fresh inputs ----------------

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_vsi_roundtrip_property_vs_reference():
    """SPEC acceptance 1: roundtrip over many random batches, equal to the reference."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        rows = int(rng.integers(1, 40))
        fields = int(rng.integers(1, 8))
        vocab = int(rng.integers(1, 200))
        f = rng.integers(0, vocab, rows * fields).astype(np.uint64)
        g, v = oracle_vsi(f, rows, fields)
        assert np.array_equal(g[v.astype(np.int64)], f)
        assert len(np.unique(f)) == len(g)
        g2, v2, _ = ref_vsi(f, np.zeros(rows, np.uint8), rows, fields)
        assert np.array_equal(g, g2) and np.array_equal(v, v2)


@needs_ref
def test_generator_vs_reference_random_configs():
    rng = np.random.default_rng(1)
    for _ in range(6):
        W = int(rng.integers(1, 4))
        F = int(rng.integers(1, 30))
        b = int(rng.integers(1, 64))
        vocab = int(rng.integers(F, 50_000))
        zipf = float(rng.uniform(0, 2))
        step = int(rng.integers(0, 1000))
        fo, yo = oracle_generate(W * b, F, vocab, 99, zipf, step)
        fr, yr = ref_generate(W, F, b, vocab, 99, zipf, step)
        assert np.array_equal(fo, fr) and np.array_equal(yo, yr)


@needs_ref
def test_cache_trace_reference(golden):
    """The reference CacheBuffer trace (LIFO free list, low slots first) is what
    the oracle's cache reproduces: replay it through the reference and compare."""
    tr = golden["cache_trace"]
    R = ref()
    c = R.ref_cache_create(tr["seed"], tr["dim"], tr["capacity"])
    for op in tr["ops"]:
        if op[0] == "admit":
            assert R.ref_cache_admit(c, op[1], op[2]) == op[3]
        elif op[0] == "evict":
            R.ref_cache_set_needed_soon(c, op[1], 0)
            assert R.ref_cache_evict(c, op[1]) == op[3]
        else:
            R.ref_cache_touch(c, op[1], op[2])
    R.ref_cache_destroy(c)


# ---------------- MixCache manager ----------------

def test_mixcache_paper_example():
    """SPEC.md:195 / PAPER.md:312-318: final cache [7,3,2,5,4,6,12,13,14,15,9,8], 1 evicted."""
    O = oracle()
    res = np.array([1, 3, 2, 5, 4, 6, 12, 13, 14, 15, 9], np.uint64)
    pinned = np.array([3, 2, 5, 4], np.uint64)
    nxt = np.array([6, 7, 8], np.uint64)
    slots = np.zeros(12, np.uint64)
    ev = np.zeros(12, np.uint64)
    n = O.orc_manager_example(12, res, len(res), pinned, len(pinned), nxt, len(nxt), slots, ev)
    assert n == 1 and ev[0] == 1
    assert slots.tolist() == [7, 3, 2, 5, 4, 6, 12, 13, 14, 15, 9, 8]


def test_mixcache_trivial_examples():
    O = oracle()
    slots = np.zeros(12, np.uint64)
    ev = np.zeros(12, np.uint64)
    e = np.zeros(1, np.uint64)
    # cold start: working {10, 20}, nothing evicted
    n = O.orc_manager_example(12, e, 0, e, 0, np.array([10, 20], np.uint64), 2, slots, ev)
    assert n == 0 and slots[:2].tolist() == [10, 20]
    # fully resident: nothing moves
    r = np.array([1, 2, 3], np.uint64)
    n = O.orc_manager_example(3, r, 3, e, 0, r, 3, slots[:3].copy(), ev)
    assert n == 0


def make_cfg(**kw):
    c = OrcConfig()
    oracle().orc_config_default(c)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def run_oracle(cfg, steps, window=False):
    import ctypes as C
    O = oracle()
    s = O.orc_sim_create(C.byref(cfg))
    assert s
    W, b, F = cfg.num_workers, cfg.batch_size_per_worker, cfg.num_fields
    losses = []
    L = cfg.lookahead_depth
    for t in range(steps):
        f, y = oracle_generate(W * b, F, cfg.vocabulary_size, cfg.seed, cfg.zipf_exponent, t)
        win = None
        if window and L > 1:
            win = np.concatenate([oracle_generate(W * b, F, cfg.vocabulary_size, cfg.seed,
                                                  cfg.zipf_exponent, t + j)[0]
                                  for j in range(1, L)])
        loss = C.c_double()
        rc = O.orc_sim_step(s, t, f, y, win.ctypes.data if win is not None else None,
                            L - 1 if win is not None else 0, C.byref(loss), None, None)
        assert rc == 0, O.orc_last_error()
        losses.append(loss.value)
    return s, losses


def test_ledger_spec_arithmetic():
    """push {7,8} at d=80 -> 1920 B; pull {1} -> 960 B, 1 swap."""
    import ctypes as C
    O = oracle()
    cfg = make_cfg(num_workers=1, embedding_dim=80, num_fields=1, batch_size_per_worker=2,
                   vocabulary_size=100, cache_capacity=2, hidden_dim=2)
    s = O.orc_sim_create(C.byref(cfg))
    led = np.zeros(4, np.int64)
    loss = C.c_double()
    assert O.orc_sim_step(s, 0, np.array([7, 8], np.uint64), np.array([0, 1], np.uint8), None, 0,
                          C.byref(loss), None, None) == 0
    O.orc_sim_ledger(s, led)
    assert led[0] == 1920 and led[1] == 0
    # next batch {1, 8}: 8 resident, 1 new -> evict LRU 7 (960 B), admit 1 (960 B)
    assert O.orc_sim_step(s, 1, np.array([1, 8], np.uint64), np.array([0, 1], np.uint8), None, 0,
                          C.byref(loss), None, None) == 0
    O.orc_sim_ledger(s, led)
    assert led[0] == 1920 + 960 and led[1] == 960 and led[3] == 1
    O.orc_sim_destroy(s)


def test_capacity_deadlock_reported():
    import ctypes as C
    O = oracle()
    cfg = make_cfg(num_workers=1, embedding_dim=4, num_fields=3, batch_size_per_worker=2,
                   vocabulary_size=100, cache_capacity=4, hidden_dim=2)
    s = O.orc_sim_create(C.byref(cfg))
    loss = C.c_double()
    rc = O.orc_sim_step(s, 0, np.arange(6, dtype=np.uint64), np.zeros(2, np.uint8), None, 0,
                        C.byref(loss), None, None)
    assert rc == 4 and b"capacity deadlock" in O.orc_last_error()
    O.orc_sim_destroy(s)


# ---------------- DeepFM-lite ----------------

def test_model_finite_difference():
    """SPEC acceptance 6: gradients vs central differences, rel < 1e-4 (d=2, F=2, h=3)."""
    O = oracle()
    rng = np.random.default_rng(5)
    F, d, H, rows = 2, 2, 3, 3
    K = F * d
    for _ in range(20):
        x = rng.normal(0, 0.5, (rows, K))
        y = rng.integers(0, 2, rows).astype(np.uint8)
        w1 = rng.normal(0, 0.7, K * H)
        b1 = rng.normal(0, 0.3, H)
        w2 = rng.normal(0, 0.7, H)
        b2 = float(rng.normal(0, 0.3))
        dx = np.zeros(rows * K)
        dw1 = np.zeros(K * H)
        db1 = np.zeros(H)
        dw2 = np.zeros(H)
        db2 = np.zeros(1)

        def loss(x_, w1_, b1_, w2_, b2_):
            return O.orc_model_fwd_bwd(np.ascontiguousarray(x_.ravel()), y, rows, F, d, H, w1_,
                                       b1_, w2_, b2_, None, None, None, None, None, None, 1)

        O.orc_model_fwd_bwd(x.ravel(), y, rows, F, d, H, w1, b1, w2, b2, None, dx.ctypes.data,
                            dw1.ctypes.data, db1.ctypes.data, dw2.ctypes.data, db2.ctypes.data, 1)
        eps = 1e-6

        def fd(vec, i, fn):
            a = vec.copy()
            b = vec.copy()
            a[i] += eps
            b[i] -= eps
            return (fn(a) - fn(b)) / (2 * eps)

        def close(an, num):
            return abs(an - num) <= 1e-4 * max(abs(an), abs(num)) + 1e-9

        xf = x.ravel()
        for i in range(xf.size):
            assert close(dx[i], fd(xf, i, lambda v: loss(v, w1, b1, w2, b2)))
        for i in range(w1.size):
            assert close(dw1[i], fd(w1, i, lambda v: loss(xf, v, b1, w2, b2)))
        for i in range(H):
            assert close(db1[i], fd(b1, i, lambda v: loss(xf, w1, v, w2, b2)))
            assert close(dw2[i], fd(w2, i, lambda v: loss(xf, w1, b1, v, b2)))
        assert close(db2[0], (loss(xf, w1, b1, w2, b2 + eps) - loss(xf, w1, b1, w2, b2 - eps)) / (2 * eps))


def test_model_loss_examples():
    """p = 0.5 -> ln 2; p = y -> ~0 with the clamp."""
    O = oracle()
    F, d, H = 1, 1, 1
    x = np.zeros(1)
    w = np.zeros(1)
    l = O.orc_model_fwd_bwd(x, np.array([1], np.uint8), 1, F, d, H, w, w, w, 0.0, None, None,
                            None, None, None, None, 1)
    assert abs(l - np.log(2)) < 1e-12
    l = O.orc_model_fwd_bwd(x, np.array([1], np.uint8), 1, F, d, H, w, w, w, 40.0, None, None,
                            None, None, None, None, 1)
    assert l <= 1e-6


def test_adam_spec_example():
    """fresh feature, g = 1, lr = 1e-3 -> moves by -0.000999999..."""
    b1, b2, eps, lr = 0.9, 0.999, 1e-8, 1e-3
    m = (1 - b1) * 1.0
    v = (1 - b2) * 1.0
    step = lr * (m / (1 - b1)) / (np.sqrt(v / (1 - b2)) + eps)
    assert abs(step - 0.000999999990) < 1e-12


# ---------------- system properties ----------------

def oracle_snapshot(s, d):
    import ctypes as C
    O = oracle()
    n = O.orc_sim_snapshot(s, None, None, None)
    f = np.zeros(n, np.uint64)
    rows = np.zeros((n, 3 * d))
    st = np.zeros(n, np.int64)
    O.orc_sim_snapshot(s, f.ctypes.data, rows.ctypes.data, st.ctypes.data)
    return f, rows, st


def test_worker_count_invariance():
    """SPEC acceptance 4 (shortened): W in {1,2,4}, same global batches -> same parameters."""
    outs = []
    for W in (1, 2, 4):
        cfg = make_cfg(num_workers=W, batch_size_per_worker=256 // W, num_fields=8,
                       embedding_dim=4, vocabulary_size=2000, cache_capacity=4000, hidden_dim=8)
        s, losses = run_oracle(cfg, 5)
        f, rows, st = oracle_snapshot(s, 4)
        outs.append((losses, f, rows, st))
        oracle().orc_sim_destroy(s)
    for losses, f, rows, st in outs[1:]:
        assert np.allclose(losses, outs[0][0], rtol=1e-9)
        assert np.array_equal(f, outs[0][1]) and np.array_equal(st, outs[0][3])
        assert np.max(np.abs(rows - outs[0][2])) < 1e-9


def test_cache_equals_no_eviction():
    """Cache == Host equivalence (SPEC acceptance 3, shortened): a cache small enough to
    evict every step gives the same trajectory as one that never evicts."""
    res = []
    for cap in (60, 100000):
        cfg = make_cfg(num_workers=2, batch_size_per_worker=8, num_fields=6, embedding_dim=4,
                       vocabulary_size=3000, cache_capacity=cap, hidden_dim=4)
        s, losses = run_oracle(cfg, 8)
        f, rows, st = oracle_snapshot(s, 4)
        led = np.zeros(4, np.int64)
        oracle().orc_sim_ledger(s, led)
        res.append((losses, f, rows, st, led))
        oracle().orc_sim_destroy(s)
    assert res[0][4][3] > 0 and res[1][4][3] == 0  # swaps only with the small cache
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])


def test_cache_size_monotonicity():
    """SPEC acceptance 8: swap traffic non-increasing in capacity."""
    swaps = []
    for cap in (70, 140, 400):
        cfg = make_cfg(num_workers=1, batch_size_per_worker=16, num_fields=4, embedding_dim=2,
                       vocabulary_size=1000, cache_capacity=cap, hidden_dim=2)
        s, _ = run_oracle(cfg, 12)
        led = np.zeros(4, np.int64)
        oracle().orc_sim_ledger(s, led)
        swaps.append(led[1])
        oracle().orc_sim_destroy(s)
    assert swaps[0] >= swaps[1] >= swaps[2]


def test_vsi_volume_dominance():
    """SPEC acceptance 11: H2W bytes with VSI <= without, equality iff no duplicates."""
    for zipf in (0.0, 1.2, 2.0):
        f, y = oracle_generate(512, 26, 100_000, 7, zipf, 0)
        g, _ = oracle_vsi(f, 512, 26)
        assert len(g) <= f.size
        assert len(g) == len(np.unique(f))
    f = np.arange(64, dtype=np.uint64)
    g, _ = oracle_vsi(f, 8, 8)
    assert len(g) == 64


def test_lookahead_protects_window():
    """needed_soon: with L=2 the manager never evicts a feature of batch t+1."""
    cfg = make_cfg(num_workers=1, batch_size_per_worker=8, num_fields=4, embedding_dim=2,
                   vocabulary_size=400, cache_capacity=80, hidden_dim=2, lookahead_depth=2)
    s, losses = run_oracle(cfg, 10, window=True)
    assert all(np.isfinite(losses))
    oracle().orc_sim_destroy(s)


def test_eviction_safety_fuzz():
    """SPEC acceptance 7 (shortened): random schedules never trip the eviction-safety
    asserts (status 3); the only allowed failure is a reported capacity deadlock (4)."""
    import ctypes as C
    O = oracle()
    rng = np.random.default_rng(3)
    deadlocks = 0
    for trial in range(300):
        W = int(rng.integers(1, 4))
        b = int(rng.integers(1, 6))
        F = int(rng.integers(1, 5))
        vocab = int(rng.integers(F + 1, 200))
        cap = int(rng.integers(1, 3 * W * b * F + 2))
        cfg = make_cfg(num_workers=W, batch_size_per_worker=b, num_fields=F, embedding_dim=2,
                       vocabulary_size=vocab, cache_capacity=cap, hidden_dim=2,
                       zipf_exponent=float(rng.uniform(0, 2)), seed=trial)
        s = O.orc_sim_create(C.byref(cfg))
        for t in range(4):
            f, y = oracle_generate(W * b, F, vocab, trial, cfg.zipf_exponent, t)
            loss = C.c_double()
            rc = O.orc_sim_step(s, t, f, y, None, 0, C.byref(loss), None, None)
            assert rc in (0, 4), O.orc_last_error()
            if rc == 4:
                assert b"capacity deadlock" in O.orc_last_error()
                deadlocks += 1
                break
        O.orc_sim_destroy(s)
    assert 0 < deadlocks < 300


def test_oracle_vsi_u64_golden(golden):
    """the oracle's VSI on arbitrary u64 ids equals the reference's (golden digests)"""
    from oracle_lib import u64_golden_batches
    for rec, f in u64_golden_batches(golden):
        g, v = oracle_vsi(f, rec["rows"], rec["fields"])
        assert len(g) == rec["unique"]
        assert sha(g) == rec["global_ids_sha256"] and sha(v) == rec["virtual_ids_sha256"]
