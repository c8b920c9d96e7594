"""BASELINE configs[1] (cfg2) parity in the bench's exact configuration.

d=80, F=39, b=8192, vocab 33.8M, Zipf 1.05, hidden 64, the whole owned shard as the HBM
cache (no evictions, rows lazily initialised on first touch), pipelined mode, owner-routed
sync: the configuration `bench.py` times (bench.py run_ours). Every step is compared with
the oracle FROM IDENTICAL STATE (tests/parity_util.py): after each step the device rows
of the step's features and the dense state are loaded into the oracle, so every bar
measures one step's fp32-vs-fp64 error. Bars: loss 1e-5 relative, logits 1e-5 (1+|z|)
at every step, the summed gradient within 1e-5 of its condition scale, rows / moments
1e-5 of the row scale plus that gradient tolerance carried through Adam (the explicit
exceptions: coordinates whose gradient is within tolerance of zero, and the gradient mass
behind ReLU units whose pre-activation is within fp32 error of zero), slot tables, step
counts and the ledger bit-exact.

The oracle runs with a 1M-slot cache: with no eviction on either side the LIFO free list
(cache_buffer.cpp:27-28) hands out slots 0, 1, 2, ... in admission order, so the device's
first 1M slots must equal the oracle's table and the rest stay empty.
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from oracle_lib import OrcConfig, oracle, oracle_vsi
from parity_util import (check_dense_one_step, check_logits, check_rows_one_step, load_dense,
                         load_rows, oracle_dense, oracle_rows, Grads)

pytestmark = pytest.mark.gpu

STEPS = int(os.environ.get("SFCTR_CFG2_PARITY_STEPS", "6"))
ORACLE_SLOTS = 1_000_000


def bench_config():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=8192, num_fields=39, embedding_dim=80,
                    vocabulary_size=33_800_000, cache_capacity=33_800_000, hidden_dim=64,
                    zipf_exponent=1.05, seed=7)
    cfg.apply("sync", "alltoall")
    cfg.apply("mode", "pipelined")
    return cfg


def per_step_parity(cfg, oracle_slots, steps, golden_rec=None):
    """Runs `steps` steps of `cfg` on the device and the oracle from identical state per step
    and checks every bar; oracle_slots: the oracle's cache capacity (== the device's when
    evictions happen; smaller is fine while neither side evicts). Returns per-step stats."""
    O = oracle()
    oc = OrcConfig()
    O.orc_config_default(oc)
    for k in ("num_workers", "embedding_dim", "num_fields", "batch_size_per_worker",
              "vocabulary_size", "lookahead_depth", "seed", "learning_rate", "adam_beta1",
              "adam_beta2", "adam_epsilon", "zipf_exponent", "hidden_dim"):
        setattr(oc, k, getattr(cfg, k))
    oc.cache_capacity = oracle_slots
    oc.num_threads = os.cpu_count() or 1
    sim = O.orc_sim_create(C.byref(oc))
    O.orc_sim_keep_grads(sim, 1)
    tr = sb.Trainer(cfg)
    gen = sb.SyntheticGenerator(cfg)
    d, F, H, b = cfg.embedding_dim, cfg.num_fields, cfg.hidden_dim, cfg.batch_size_per_worker
    K = F * d
    P = K * H + 2 * H + 1
    # identical dense start (both are the same function of the seed; load the fp32 values)
    p, m, v, ds = tr.dense_state()
    load_dense(O, sim, p, m, v, ds)
    report = []
    for t in range(steps):
        f, y = gen.generate(t)
        if t == 0 and golden_rec is not None:
            import hashlib
            assert hashlib.sha256(f.tobytes()).hexdigest() == golden_rec["features_sha256"]
        gids, _ = oracle_vsi(f, b, F, 1)
        old, old_st = oracle_rows(O, sim, gids, d)  # == device state before the step
        old_dense = oracle_dense(O, sim, P)[:3]
        loss = tr.step(t, f, y)
        ol = C.c_double()
        logits = np.zeros(b)
        rc = O.orc_sim_step(sim, t, f, y, None, 0, C.byref(ol), None, logits.ctypes.data)
        assert rc == 0, O.orc_last_error()
        assert abs(loss - ol.value) <= 1e-5 * abs(ol.value), (t, loss, ol.value)
        lg_rel = check_logits(tr.logits(), logits, f"step {t}")
        st = tr.stats()
        assert st["unique"] == O.orc_sim_last_unique(sim) == gids.size
        if t == 0 and golden_rec is not None:
            assert st["unique"] == golden_rec["unique"]
        # cache indexing, bit-exact: the device's first oracle_slots slots, the rest empty
        df, dlu, dseq = tr.cache_slots(0, 0, oracle_slots)
        of = np.zeros(oracle_slots, np.uint64)
        olu = np.zeros(oracle_slots, np.int64)
        oseq = np.zeros(oracle_slots, np.uint64)
        O.orc_sim_cache_slots(sim, 0, of, olu, oseq)
        assert np.array_equal(df, of), t
        occ = of != np.iinfo(np.uint64).max
        assert np.array_equal(dlu[occ], olu[occ]) and np.array_equal(dseq[occ], oseq[occ]), t
        assert (tr.free_count(0) - (cfg.cache_capacity - oracle_slots)
                == O.orc_sim_free_count(sim, 0)), t
        led = np.zeros(4, np.int64)
        O.orc_sim_ledger(sim, led)
        dl = tr.ledger()
        assert [dl["host_to_worker"], dl["worker_to_host"], dl["interworker"],
                dl["swap_events"]] == led.tolist(), t
        # rows of this step's features (emb | m | v) and step counts, one step from the
        # same state (wherever they live: cache slot or host pool)
        drows, dst = tr.peek_rows(gids)
        orows, ost = oracle_rows(O, sim, gids, d)
        gr = Grads(O, sim, gids.size, d, P)
        stats = check_rows_one_step(gids, old, drows, dst, orows, ost, gr, d, cfg, f"step {t}")
        stats["relu_undetermined_units"] = gr.n_amb
        pd, md, vd, dsd = tr.dense_state()
        po, mo, vo, dso = oracle_dense(O, sim, P)
        assert dsd == dso == t + 1
        stats["dense"] = check_dense_one_step(old_dense, (pd, md, vd), (po, mo, vo), gr, dsd, cfg,
                                              f"step {t}")
        stats["logit_max_rel"] = lg_rel
        stats["loss_rel"] = abs(loss - ol.value) / abs(ol.value)
        stats["evictions_total"] = dl["swap_events"]
        report.append(stats)
        # identical state for the next step: the device's rows and dense state
        load_rows(O, sim, gids, drows, dst)
        load_dense(O, sim, pd, md, vd, dsd)
    for t, r in enumerate(report):  # compact per-step summary (pytest -s)
        print(f"step {t}: loss_rel {r['loss_rel']:.2e} logit {r['logit_max_rel']:.2e} "
              f"rows {r['rows']} theta {r['theta_max_rel']:.2e} m {r['m_max_rel']:.2e} "
              f"v {r['v_max_rel']:.2e} |g|<=tol coords {r['sensitive_coords']} "
              f"relu-undetermined units {r['relu_undetermined_units']} "
              f"(coords using it {r['relu_ambiguous_coords']}) "
              f"theta beyond plain 1e-5 (propagated-tolerance) {r['theta_outside_plain_1e-5']} "
              f"dense w1 theta {r['dense']['w1']['theta_max_rel']:.2e} "
              f"evictions so far {r['evictions_total']}")
    O.orc_sim_destroy(sim)
    tr.close()
    return report


def test_cfg2_bench_config_per_step_parity(golden):
    rec = next(r for r in golden["batches"] if r["name"] == "cfg2_w1")
    per_step_parity(bench_config(), ORACLE_SLOTS, STEPS, rec)


def test_cfg4_shape_with_evictions_per_step_parity():
    """BASELINE configs[3] shapes (d=32, F=26, b=8192, Zipf 1.05) at a shrunk vocabulary
    (4M rows instead of 1B, so the fp64 oracle holds the table) with a 200k-slot cache: LRU
    evictions into the host pool and refills from it every step after the first few. Same
    per-step bars; slot tables equal the oracle's in full (same capacity)."""
    cfg = sb.Config(num_workers=1, batch_size_per_worker=8192, num_fields=26, embedding_dim=32,
                    vocabulary_size=4_000_000, cache_capacity=200_000, hidden_dim=64,
                    zipf_exponent=1.05, seed=7)
    cfg.apply("mode", "pipelined")
    rep = per_step_parity(cfg, 200_000, 8)
    assert rep[-1]["evictions_total"] > 100_000
