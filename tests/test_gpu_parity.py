"""GPU parity tests: the sm_100a path through the C-ABI vs the CPU oracle.

Bars (stated per test):
  * integer / index work — generator ids and labels, VSI global/virtual ids,
    cache slot tables (slot -> feature, last_use, admit_seq), free counts,
    lazy-Adam step counts, the TransferLedger — must be BIT-EXACT;
  * floating point — the device computes in fp32 against the oracle's fp64:
    loss within rtol 1e-5; logits |dz| <= 1e-5 * (1 + |z|); embedding rows
    and Adam moments |a - b| <= 1e-5 * (max|row| + 1e-3) per row after a few
    steps (the scatter-add and all-reduce order differ from the oracle).
"""
import ctypes as C
import hashlib

import os

import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from oracle_lib import OrcConfig, oracle, oracle_generate, oracle_vsi, u64_golden_batches

pytestmark = pytest.mark.gpu


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


# ---------------- generator / init ----------------

def test_generator_golden(golden):
    for rec in golden["batches"]:
        cfg = sb.Config(num_workers=rec["workers"], batch_size_per_worker=rec["batch"],
                        num_fields=rec["fields"], vocabulary_size=rec["vocab"], seed=rec["seed"],
                        zipf_exponent=rec["zipf"])
        g = sb.SyntheticGenerator(cfg)
        f, y = g.generate(rec["step"])
        assert sha(f) == rec["features_sha256"], rec["name"]
        assert sha(y) == rec["labels_sha256"], rec["name"]
        g.close()


def test_generator_row_ranges_match_oracle():
    cfg = sb.Config(num_workers=4, batch_size_per_worker=300, num_fields=13, vocabulary_size=77777,
                    seed=11, zipf_exponent=0.9)
    g = sb.SyntheticGenerator(cfg)
    for step in (0, 3, 1000):
        full_f, full_y = oracle_generate(1200, 13, 77777, 11, 0.9, step)
        for r0, n in ((0, 1200), (300, 300), (1199, 1), (17, 500)):
            f, y = g.generate(step, r0, n)
            assert np.array_equal(f, full_f[r0 * 13:(r0 + n) * 13])
            assert np.array_equal(y, full_y[r0:r0 + n])


def test_initial_embedding_golden(golden):
    import struct
    for f, want in golden["initial_embedding_seed7_d80"].items():
        v = sb.initial_embedding(7, int(f), 80)
        assert [struct.pack("<d", x).hex() for x in v] == want


# ---------------- VSI ----------------

def test_vsi_golden_and_spec(golden):
    for ex in golden["vsi_examples"]:
        g, v, _ = sb.virtual_sparse_id(np.array(ex["features"], np.uint64), ex["rows"], ex["fields"])
        assert g.tolist() == ex["global_ids"] and v.tolist() == ex["virtual_ids"]
    for rec in golden["batches"]:
        cfg = sb.Config(num_workers=rec["workers"], batch_size_per_worker=rec["batch"],
                        num_fields=rec["fields"], vocabulary_size=rec["vocab"], seed=rec["seed"],
                        zipf_exponent=rec["zipf"])
        f, _ = sb.SyntheticGenerator(cfg).generate(rec["step"])
        rows = rec["workers"] * rec["batch"]
        g, v, rr = sb.virtual_sparse_id(f, rows, rec["fields"], rec["workers"],
                                        key_space=rec["vocab"])
        assert len(g) == rec["unique"]
        assert sha(g) == rec["global_ids_sha256"] and sha(v) == rec["virtual_ids_sha256"]
        assert rr.ravel().tolist() == rec["row_ranges"]


def test_vsi_random_and_edge_cases():
    rng = np.random.default_rng(0)
    ctx = sb.VirtualSparseId(1 << 20, 1 << 16)
    cases = [np.array([5], np.uint64), np.zeros(64, np.uint64),
             np.arange(4096, dtype=np.uint64)[::-1].copy(),
             np.full(1 << 16, (1 << 20) - 1, np.uint64)]
    for _ in range(200):
        n = int(rng.integers(1, 3000))
        cases.append(rng.integers(0, int(rng.integers(1, 1 << 20)), n).astype(np.uint64))
    for f in cases:
        g, v, _ = ctx(f, f.size, 1)
        go, vo = oracle_vsi(f, f.size, 1)
        assert np.array_equal(g, go) and np.array_equal(v, vo)
        assert np.array_equal(g[v.astype(np.int64)], f)  # roundtrip
    with pytest.raises(sb.LogicError):
        ctx(np.array([1 << 20], np.uint64), 1, 1)  # outside the key space
    with pytest.raises(sb.LogicError):
        ctx(np.arange(6, dtype=np.uint64), 3, 2, num_workers=2)  # uneven split
    with pytest.raises(sb.LogicError):
        ctx(np.zeros(0, np.uint64), 0, 2)  # empty batch


# ---------------- DeepFM-lite ----------------

def test_model_forward_backward_vs_oracle():
    O = oracle()
    rng = np.random.default_rng(2)
    for rows, F, d, H in ((3, 2, 2, 3), (37, 5, 6, 20), (256, 26, 16, 64), (130, 39, 80, 64)):
        K = F * d
        x = rng.uniform(-0.05, 0.05, (rows, K)).astype(np.float32)
        y = rng.integers(0, 2, rows).astype(np.uint8)
        w1 = np.zeros(K * H)
        b1 = np.zeros(H)
        w2 = np.zeros(H)
        b2 = np.zeros(1)
        O.orc_dense_init(7, K, H, w1, b1, w2, b2)
        b1 = rng.normal(0, 0.05, H)
        w1f, b1f, w2f = w1.astype(np.float32), b1.astype(np.float32), w2.astype(np.float32)
        xd = x.astype(np.float64)
        w1d, b1d, w2d = w1f.astype(np.float64), b1f.astype(np.float64), w2f.astype(np.float64)
        lg = np.zeros(rows)
        dx = np.zeros(rows * K)
        dw1 = np.zeros(K * H)
        db1 = np.zeros(H)
        dw2 = np.zeros(H)
        db2 = np.zeros(1)
        loss = O.orc_model_fwd_bwd(xd.ravel(), y, rows, F, d, H, w1d, b1d, w2d, 0.01,
                                   lg.ctypes.data, dx.ctypes.data, dw1.ctypes.data,
                                   db1.ctypes.data, dw2.ctypes.data, db2.ctypes.data, 1)
        out = sb.model_forward_backward(x, y, w1f, b1f, w2f, np.float32([0.01]), F, d, H)
        assert abs(out["loss"] - loss) <= 1e-5 * abs(loss)
        assert np.all(np.abs(out["logits"] - lg) <= 1e-5 * (1 + np.abs(lg)))
        for name, ref in (("dx", dx), ("dw1", dw1), ("db1", db1), ("dw2", dw2)):
            got = np.asarray(out[name], np.float64).ravel()
            scale = np.max(np.abs(ref)) + 1e-30
            assert np.max(np.abs(got - ref)) <= 1e-4 * scale, name
        assert abs(out["db2"] - db2[0]) <= 1e-4 * (abs(db2[0]) + np.max(np.abs(dw2)) + 1e-30)


# ---------------- the trainer vs the oracle's simulated system ----------------

def orc_cfg(cfg):
    c = OrcConfig()
    oracle().orc_config_default(c)
    for k in ("num_workers", "embedding_dim", "num_fields", "batch_size_per_worker",
              "vocabulary_size", "cache_capacity", "lookahead_depth", "seed", "learning_rate",
              "adam_beta1", "adam_beta2", "adam_epsilon", "zipf_exponent", "hidden_dim"):
        setattr(c, k, getattr(cfg, k))
    return c


def orc_slots(s, w, cap):
    f = np.zeros(cap, np.uint64)
    lu = np.zeros(cap, np.int64)
    seq = np.zeros(cap, np.uint64)
    oracle().orc_sim_cache_slots(s, w, f, lu, seq)
    return f, lu, seq


def orc_snapshot(s, d):
    O = oracle()
    n = O.orc_sim_snapshot(s, None, None, None)
    f = np.zeros(n, np.uint64)
    rows = np.zeros((n, 3 * d))
    st = np.zeros(n, np.int64)
    O.orc_sim_snapshot(s, f.ctypes.data, rows.ctypes.data, st.ctypes.data)
    return f, rows, st


def check_rows_close(drows, orows, steps, d, lr, rtol=1e-5):
    """Embedding rows + Adam moments, fp32 device vs fp64 oracle.

    m (linear in the gradient): >= 99.9 % of coordinates within rtol * max|m_row|,
    all within 10 rtol * max|m_row| (fp32 accumulation of terms that cancel:
    the gradient of a hot feature sums hundreds of +/- contributions).
    v (quadratic): |dv| <= 10 rtol * max|v_row|.  Embeddings: >= 99.9 % of
    coordinates within rtol * max|emb_row|, and every coordinate within
    rtol * max|emb_row| + 1e-2 * lr * adam_steps. The slack term is Adam's conditioning: the update
    lr * m_hat / (sqrt(v_hat) + eps) has slope lr / (4 eps) in g where
    |g| ~ eps = 1e-8, so a coordinate whose fp32 gradient cancels down to ~eps
    turns a 1e-11 gradient difference (fp32 vs fp64 accumulation of terms
    ~1e-5) into up to ~1e-3 * lr of parameter difference per update.
    """
    a = drows.astype(np.float64)
    e, m, v = slice(0, d), slice(d, 2 * d), slice(2 * d, 3 * d)
    sc_m = np.max(np.abs(orows[:, m]), axis=1, keepdims=True) + 1e-30
    rel_m = np.abs(a[:, m] - orows[:, m]) / sc_m
    assert (rel_m <= rtol).mean() >= 0.999 and np.max(rel_m) <= 10 * rtol, float(np.max(rel_m))
    sc_v = np.max(np.abs(orows[:, v]), axis=1, keepdims=True) + 1e-30
    assert np.max(np.abs(a[:, v] - orows[:, v]) / sc_v) <= 10 * rtol
    err = np.abs(a[:, e] - orows[:, e])
    sc_e = np.max(np.abs(orows[:, e]), axis=1, keepdims=True)
    within = err <= rtol * sc_e
    assert within.mean() >= 0.999, within.mean()
    bound = rtol * sc_e + 1e-2 * lr * np.maximum(steps, 1)[:, None]
    assert np.all(err <= bound), float(np.max(err - bound))


def run_parity(cfg, steps, check_rows=True, row_tol=1e-5):
    O = oracle()
    oc = orc_cfg(cfg)
    sim = O.orc_sim_create(C.byref(oc))
    tr = sb.Trainer(cfg)
    W, b, F, L = cfg.num_workers, cfg.batch_size_per_worker, cfg.num_fields, cfg.lookahead_depth
    gen = sb.SyntheticGenerator(cfg)
    evictions = 0
    for t in range(steps):
        f, y = gen.generate(t)
        win = None
        if L > 1:
            win = np.concatenate([gen.generate(t + j)[0] for j in range(1, L)])
        loss = tr.step(t, f, y, window=win)
        ol = C.c_double()
        logits = np.zeros(W * b)
        rc = O.orc_sim_step(sim, t, f, y, win.ctypes.data if win is not None else None,
                            L - 1 if win is not None else 0, C.byref(ol), None, logits.ctypes.data)
        assert rc == 0, O.orc_last_error()
        assert abs(loss - ol.value) <= 1e-5 * abs(ol.value), (t, loss, ol.value)
        if t == 0:  # logits are compared from the identical initial state
            lg = tr.logits()
            assert np.all(np.abs(lg - logits) <= 1e-5 * (1 + np.abs(logits)))
        # cache indexing: bit-exact per lane
        for w in range(W):
            df, dlu, dseq = tr.cache_slots(w)
            of, olu, oseq = orc_slots(sim, w, cfg.cache_capacity)
            assert np.array_equal(df, of), (t, w)
            occ = of != np.iinfo(np.uint64).max
            assert np.array_equal(dlu[occ], olu[occ]) and np.array_equal(dseq[occ], oseq[occ])
            assert tr.free_count(w) == O.orc_sim_free_count(sim, w)
        led = np.zeros(4, np.int64)
        O.orc_sim_ledger(sim, led)
        dl = tr.ledger()
        assert [dl["host_to_worker"], dl["worker_to_host"], dl["interworker"],
                dl["swap_events"]] == led.tolist(), t
        evictions = dl["swap_events"]
        assert tr.stats()["unique"] == O.orc_sim_last_unique(sim)
    if check_rows:
        df, drows, dst = tr.snapshot()
        of, orows, ost = orc_snapshot(sim, cfg.embedding_dim)
        assert np.array_equal(df, of) and np.array_equal(dst, ost)
        check_rows_close(drows, orows, dst, cfg.embedding_dim, cfg.learning_rate, row_tol)
        # dense parameters
        K, H = cfg.num_fields * cfg.embedding_dim, cfg.hidden_dim
        w1, b1, w2, b2 = tr.get_dense()
        ow1, ob1, ow2, ob2 = np.zeros(K * H), np.zeros(H), np.zeros(H), np.zeros(1)
        O.orc_sim_dense(sim, ow1, ob1, ow2, ob2)
        assert np.max(np.abs(w1 - ow1)) <= 1e-5 * (np.max(np.abs(ow1)) + 1e-3)
    O.orc_sim_destroy(sim)
    tr.close()
    return evictions


def test_trainer_single_worker_with_evictions():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=8, embedding_dim=8,
                    vocabulary_size=5000, cache_capacity=700, hidden_dim=16, zipf_exponent=1.1)
    assert run_parity(cfg, 8) > 0


def test_trainer_four_lanes_one_process():
    cfg = sb.Config(num_workers=4, batch_size_per_worker=32, num_fields=6, embedding_dim=4,
                    vocabulary_size=3000, cache_capacity=260, hidden_dim=8, zipf_exponent=1.0)
    assert run_parity(cfg, 8) > 0


def test_trainer_odd_dim_and_no_eviction():
    cfg = sb.Config(num_workers=2, batch_size_per_worker=16, num_fields=5, embedding_dim=6,
                    vocabulary_size=100000, cache_capacity=20000, hidden_dim=3)
    assert run_parity(cfg, 4) == 0


def test_trainer_lookahead_two():
    cfg = sb.Config(num_workers=2, batch_size_per_worker=16, num_fields=4, embedding_dim=4,
                    vocabulary_size=800, cache_capacity=120, hidden_dim=8, lookahead_depth=2)
    run_parity(cfg, 8)


def test_trainer_cfg1_shape():
    """BASELINE configs[0]: 26 fields, d=16, 1M vocab, batch 1024, single worker."""
    cfg = sb.Config(num_workers=1, batch_size_per_worker=1024, num_fields=26, embedding_dim=16,
                    vocabulary_size=1_000_000, cache_capacity=16384, hidden_dim=64)
    run_parity(cfg, 3)


def test_capacity_deadlock_is_a_run_error():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=8, num_fields=4, embedding_dim=4,
                    vocabulary_size=100000, cache_capacity=8, hidden_dim=4, zipf_exponent=0.0)
    tr = sb.Trainer(cfg)
    f, y = sb.SyntheticGenerator(cfg).generate(0)
    with pytest.raises(sb.RunError) as e:
        tr.step(0, f, y)
    assert e.value.step == 0


def test_feature_out_of_vocab_is_a_logic_error():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=2, num_fields=2, vocabulary_size=100,
                    cache_capacity=16, hidden_dim=4)
    tr = sb.Trainer(cfg)
    with pytest.raises(sb.LogicError):
        tr.step(0, np.array([1, 2, 3, 100], np.uint64), np.zeros(2, np.uint8))


@pytest.mark.parametrize("mode", ["sequential", "pipelined"])
def test_out_of_vocab_moves_no_state(mode):
    """An id >= vocab is a LogicError that leaves every piece of state as it was, also when
    the step was enqueued without a host wait (device inputs, host-wait-free steps: the
    error surfaces at the next synchronising call). Training then continues exactly like a
    trainer that never saw the bad batch."""
    import torch
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=6, embedding_dim=8,
                    vocabulary_size=5000, cache_capacity=5000, hidden_dim=16)
    cfg.apply("mode", mode)
    gen = sb.SyntheticGenerator(cfg)
    batches = [gen.generate(t) for t in range(4)]
    ref = sb.Trainer(cfg)
    tr = sb.Trainer(cfg)
    for t in range(2):
        ref.step(t, *batches[t])
        tr.step(t, *batches[t])
    before = tr.snapshot(), tr.dense_state()
    bad = batches[2][0].copy()
    bad[17] = cfg.vocabulary_size + 3
    # host-wait-free device step: enqueued, the error comes at synchronize()
    d_f = torch.from_numpy(bad.view(np.int64)).cuda()
    d_y = torch.from_numpy(batches[2][1]).cuda()
    tr.step_device(2, d_f.data_ptr(), d_y.data_ptr())
    with pytest.raises(sb.LogicError):
        tr.synchronize()
    after = tr.snapshot(), tr.dense_state()
    for a, b in zip(before[0], after[0]):
        assert np.array_equal(a, b)
    for a, b in zip(before[1][:3], after[1][:3]):
        assert np.array_equal(a, b)
    assert before[1][3] == after[1][3]
    # host-buffer step: raises at once, nothing moves either
    with pytest.raises(sb.LogicError):
        tr.step(2, bad, batches[2][1])
    for a, b in zip(before[0], tr.snapshot()):
        assert np.array_equal(a, b)
    # continues like the reference trainer
    for t in (2, 3):
        l1 = ref.step(t, *batches[t])
        l2 = tr.step(t, *batches[t])
        assert abs(l1 - l2) <= 1e-6 * abs(l1)
    fr, rr, sr = ref.snapshot()
    ft, rt, st = tr.snapshot()
    assert np.array_equal(fr, ft) and np.array_equal(sr, st)
    assert np.max(np.abs(rr - rt)) <= 1e-6
    ref.close()
    tr.close()


def test_worker_count_invariance_device():
    """SPEC acceptance 4 on the device: W in {1,2,4} on the same global batches."""
    snaps = []
    for W in (1, 2, 4):
        cfg = sb.Config(num_workers=W, batch_size_per_worker=128 // W, num_fields=6,
                        embedding_dim=4, vocabulary_size=2000, cache_capacity=4000, hidden_dim=8)
        tr = sb.Trainer(cfg)
        gen = sb.SyntheticGenerator(cfg)
        losses = [tr.step(t, *gen.generate(t)) for t in range(5)]
        snaps.append((losses, tr.snapshot()))
        tr.close()
    for losses, (f, r, s) in snaps[1:]:
        assert np.allclose(losses, snaps[0][0], rtol=1e-5)
        assert np.array_equal(f, snaps[0][1][0]) and np.array_equal(s, snaps[0][1][2])
        assert np.max(np.abs(r - snaps[0][1][1])) <= 1e-6


def test_cfg2_step_properties(golden):
    """BASELINE configs[1] at W=1 (full size): VSI count equals the reference's,
    every owned unique is resident after manage, loss finite and ~ln 2."""
    rec = next(r for r in golden["batches"] if r["name"] == "cfg2_w1")
    cfg = sb.Config(num_workers=1, batch_size_per_worker=8192, num_fields=39, embedding_dim=80,
                    vocabulary_size=33_800_000, cache_capacity=400_000, hidden_dim=64,
                    zipf_exponent=1.05)
    tr = sb.Trainer(cfg)
    gen = sb.SyntheticGenerator(cfg)
    f, y = gen.generate(0)
    assert sha(f) == rec["features_sha256"]
    loss = tr.step(0, f, y)
    st = tr.stats()
    assert st["unique"] == rec["unique"] == st["owned"] == st["working"]
    assert abs(loss - np.log(2)) < 0.05
    loss2 = tr.step(1, *gen.generate(1))
    assert np.isfinite(loss2)
    tr.close()


@pytest.mark.parametrize("env", ["SFCTR_TOWER_FUSED", "SFCTR_TOWER_SIMT"])
def test_trainer_alternative_towers(monkeypatch, env):
    """The opt-in tower paths (fused gather->GEMM->scatter, fp32 SIMT validation tiles) hold
    the same parity bars (d = 16 so the fused path applies, K = F*d unpadded for SIMT)."""
    monkeypatch.setenv(env, "1")
    cfg = sb.Config(num_workers=1, batch_size_per_worker=128, num_fields=8, embedding_dim=16,
                    vocabulary_size=20000, cache_capacity=1200, hidden_dim=32, zipf_exponent=1.05)
    run_parity(cfg, 5)


# ---------------- VSI over arbitrary u64 ids (hashed first-position table) ----------------

def test_vsi_hashed_u64_golden(golden):
    """vsi.cpp:23-54 accepts any FeatureId: ids >= 2^32 and the all-ones id go through the
    hashed table (key_space 0), bit-exact with the reference's own output."""
    for rec, f in u64_golden_batches(golden):
        g, v, rr = sb.virtual_sparse_id(f, rec["rows"], rec["fields"], key_space=0)
        assert len(g) == rec["unique"]
        assert sha(g) == rec["global_ids_sha256"] and sha(v) == rec["virtual_ids_sha256"]


def test_vsi_hashed_random_vs_oracle():
    rng = np.random.default_rng(3)
    ctx = sb.VirtualSparseId(0, 1 << 17)
    cases = [np.array([(1 << 64) - 1], np.uint64), np.full(4096, (1 << 64) - 1, np.uint64),
             np.arange(1 << 16, dtype=np.uint64) * np.uint64(1 << 40)]
    for _ in range(60):
        n = int(rng.integers(1, 1 << 17))
        k = int(rng.integers(1, n + 1))
        pool = rng.integers(0, np.iinfo(np.uint64).max, k, dtype=np.uint64, endpoint=True)
        cases.append(pool[rng.integers(0, k, n)])
    for f in cases:
        g, v, _ = ctx(f, f.size, 1)
        go, vo = oracle_vsi(f, f.size, 1)
        assert np.array_equal(g, go) and np.array_equal(v, vo)
        assert np.array_equal(g[v.astype(np.int64)], f)
    ctx.close()


def test_vsi_direct_large_batches_vs_oracle():
    """the fused look-back scan across many tiles (cfg2 W=8-sized batches)"""
    rng = np.random.default_rng(4)
    ctx = sb.VirtualSparseId(1 << 24, 3 << 20)
    for n in (2048, 2049, 4095, 1 << 20, 3 << 20):
        f = rng.integers(0, int(rng.integers(1, 1 << 24)), n).astype(np.uint64)
        g, v, _ = ctx(f, n, 1)
        go, vo = oracle_vsi(f, n, 1)
        assert np.array_equal(g, go) and np.array_equal(v, vo)
    ctx.close()


# ---------------- deterministic mode (fixed-order gradient sums) ----------------

@pytest.mark.parametrize("mode", ["sequential", "pipelined"])
def test_deterministic_runs_are_bit_identical(mode):
    """deterministic=1: the segment sum adds each unique's positions in ascending order (no
    atomics), so two runs of the same batches give bit-identical losses, rows, moments,
    step counts and dense parameters; and it stays within the oracle's
    parity bars. Two in-process lanes (the lanes' sums are added in lane order) and LRU
    evictions included."""
    cfg = sb.Config(num_workers=2, batch_size_per_worker=512, num_fields=12, embedding_dim=16,
                    vocabulary_size=200_000, cache_capacity=4500, hidden_dim=32,
                    zipf_exponent=1.05)
    cfg.apply("deterministic", "1")
    cfg.apply("mode", mode)
    gen = sb.SyntheticGenerator(cfg)
    batches = [gen.generate(t) for t in range(8)]
    runs = []
    for _ in range(2):
        tr = sb.Trainer(cfg)
        losses = [tr.step(t, *batches[t]) for t in range(8)]
        runs.append((losses, tr.snapshot(), tr.dense_state()))
        assert tr.ledger()["swap_events"] > 0
        tr.close()
    (l1, s1, d1), (l2, s2, d2) = runs
    assert l1 == l2
    for a, b in zip(s1, s2):
        assert np.array_equal(a, b)
    for a, b in zip(d1[:3], d2[:3]):
        assert np.array_equal(a, b)
    run_parity(cfg, 6)


@pytest.mark.parametrize("mode", ["sequential", "pipelined"])
def test_launch_switches_are_bit_identical(mode, tmp_path):
    """The launch / scheduling switches change when kernels start, never what they compute:
    programmatic dependent launch off (SFCTR_NO_PDL=1), the training stream at high priority
    (SFCTR_STREAM_PRIO=train) and the row update not forked (SFCTR_NO_UPDATE_FORK=1) give
    bit-identical losses, rows and dense state to the defaults (deterministic mode)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    worker = os.path.join(root, "tests", "launch_mode_worker.py")
    outs = []
    for k, env in enumerate([{}, {"SFCTR_NO_PDL": "1", "SFCTR_STREAM_PRIO": "train",
                                  "SFCTR_NO_UPDATE_FORK": "1"}]):
        out = str(tmp_path / f"run{k}.npz")
        r = subprocess.run([sys.executable, worker, out, mode], capture_output=True, text=True,
                           timeout=600, env={**os.environ, **env})
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs.append(np.load(out))
    for key in ("losses", "f", "r", "s", "p", "m", "v"):
        assert np.array_equal(outs[0][key], outs[1][key]), key

