"""Pipelined mode (RunMode::kPipelined, config.hpp:30) on the device:
the manager stage of step t+1 (ids, VSI, MixCache probe / eviction / admission) runs on
its own stream while step t trains. SPEC.md:378-380 requires the loss traces and ledgers
of pipelined and sequential runs to be identical, and the pipelined run must still match
the CPU oracle. Bars: cache slot tables, free counts, Adam step counts and the ledger
BIT-EXACT between modes and against the oracle; losses and rows within the fp32 bars of
tests/test_gpu_parity.py (the scatter-add's atomics make fp32 sums order-dependent, so
two device runs agree to rounding, not bitwise)."""
import ctypes as C

import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from oracle_lib import oracle, oracle_vsi
from test_gpu_parity import check_rows_close, orc_cfg, orc_slots, orc_snapshot

pytestmark = pytest.mark.gpu


def _batches(cfg, steps):
    gen = sb.SyntheticGenerator(cfg)
    L = cfg.lookahead_depth
    out = []
    for t in range(steps):
        f, y = gen.generate(t)
        win = None
        if L > 1:
            win = np.concatenate([gen.generate(t + j)[0] for j in range(1, L)])
        out.append((f, y, win))
    return out


def _run(cfg, batches, mode, inflight=2):
    cfg.apply("mode", mode)
    tr = sb.Trainer(cfg)
    assert tr.config.run_mode == (1 if mode == "pipelined" else 0)
    losses = []
    if mode == "pipelined":  # keep `inflight` steps outstanding (the host runs ahead)
        for t, (f, y, w) in enumerate(batches):
            tr.submit(t, f, y, w)
            if t >= inflight:
                losses.append(tr.loss(t - inflight))
        for t in range(max(0, len(batches) - inflight), len(batches)):
            losses.append(tr.loss(t))
    else:
        for t, (f, y, w) in enumerate(batches):
            losses.append(tr.step(t, f, y, window=w))
    W = cfg.num_workers
    out = {"losses": np.array(losses), "snap": tr.snapshot(), "ledger": tr.ledger(),
           "slots": [tr.cache_slots(w) for w in range(W)],
           "free": [tr.free_count(w) for w in range(W)], "stats": tr.stats(),
           "dense": tr.get_dense()}
    tr.close()
    return out


def _oracle(cfg, batches):
    O = oracle()
    sim = O.orc_sim_create(C.byref(orc_cfg(cfg)))
    L = cfg.lookahead_depth
    losses = []
    for t, (f, y, w) in enumerate(batches):
        ol = C.c_double()
        rc = O.orc_sim_step(sim, t, f, y, w.ctypes.data if w is not None else None,
                            L - 1 if w is not None else 0, C.byref(ol), None, None)
        assert rc == 0, O.orc_last_error()
        losses.append(ol.value)
    return O, sim, np.array(losses)


def check_modes(cfg, steps, inflight=2):
    batches = _batches(cfg, steps)
    seq = _run(cfg, batches, "sequential")
    pip = _run(cfg, batches, "pipelined", inflight)
    # pipelined == sequential (semantic transparency)
    assert np.allclose(pip["losses"], seq["losses"], rtol=1e-6, atol=0)
    assert pip["ledger"] == seq["ledger"]
    assert pip["free"] == seq["free"]
    for a, b in zip(pip["slots"], seq["slots"]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    (pf, pr, ps), (sf, sr, ss) = pip["snap"], seq["snap"]
    assert np.array_equal(pf, sf) and np.array_equal(ps, ss)
    check_rows_close(pr, sr.astype(np.float64), ps, cfg.embedding_dim, cfg.learning_rate)
    # ... and both equal the oracle
    O, sim, ol = _oracle(cfg, batches)
    assert np.all(np.abs(pip["losses"] - ol) <= 1e-5 * np.abs(ol))
    for w in range(cfg.num_workers):
        of, olu, oseq = orc_slots(sim, w, cfg.cache_capacity)
        df, dlu, dseq = pip["slots"][w]
        assert np.array_equal(df, of)
        occ = of != np.iinfo(np.uint64).max
        assert np.array_equal(dlu[occ], olu[occ]) and np.array_equal(dseq[occ], oseq[occ])
        assert pip["free"][w] == O.orc_sim_free_count(sim, w)
    led = np.zeros(4, np.int64)
    O.orc_sim_ledger(sim, led)
    dl = pip["ledger"]
    assert [dl["host_to_worker"], dl["worker_to_host"], dl["interworker"],
            dl["swap_events"]] == led.tolist()
    of, orows, ost = orc_snapshot(sim, cfg.embedding_dim)
    assert np.array_equal(pf, of) and np.array_equal(ps, ost)
    check_rows_close(pr, orows, ps, cfg.embedding_dim, cfg.learning_rate)
    O.orc_sim_destroy(sim)
    return pip["stats"]


def test_pipelined_single_worker_with_evictions():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=8, embedding_dim=8,
                    vocabulary_size=5000, cache_capacity=700, hidden_dim=16, zipf_exponent=1.1)
    st = check_modes(cfg, 12)
    assert st["total_evicted"] > 0


def test_pipelined_four_lanes_one_process():
    cfg = sb.Config(num_workers=4, batch_size_per_worker=32, num_fields=6, embedding_dim=4,
                    vocabulary_size=3000, cache_capacity=260, hidden_dim=8, zipf_exponent=1.0)
    st = check_modes(cfg, 10)
    assert st["total_evicted"] > 0


def test_pipelined_lookahead_two():
    cfg = sb.Config(num_workers=2, batch_size_per_worker=16, num_fields=4, embedding_dim=4,
                    vocabulary_size=800, cache_capacity=120, hidden_dim=8, lookahead_depth=2)
    check_modes(cfg, 10)


def test_pipelined_tight_cache_waits_for_pinned_rows():
    """Capacity just above the largest batch: evictions must take rows the previous
    (still training) batch used, so the manager waits for it — and results still match."""
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=8, embedding_dim=8,
                    vocabulary_size=20000, cache_capacity=600, hidden_dim=16, zipf_exponent=0.6)
    gen = sb.SyntheticGenerator(cfg)
    umax = max(len(oracle_vsi(gen.generate(t)[0], 64, 8)[0]) for t in range(10))
    cfg.cache_capacity = umax + 4
    st = check_modes(cfg, 10)
    assert st["total_evicted"] > 0 and st["total_pinned_waits"] > 0


def test_pipelined_whole_shard_free_steps():
    """No eviction possible: every step runs without a host wait and the manager of
    step t+1 overlaps step t entirely."""
    cfg = sb.Config(num_workers=1, batch_size_per_worker=512, num_fields=13, embedding_dim=16,
                    vocabulary_size=200_000, cache_capacity=200_000, hidden_dim=32,
                    zipf_exponent=1.05)
    st = check_modes(cfg, 6)
    assert st["total_free_steps"] == 6


@pytest.mark.parametrize("inflight", [1, 3])
def test_pipelined_host_queue_depths(inflight):
    """Besides the step it submits, the host leaves 1 or 3 steps unread (3 = the loss ring's
    depth), so the two device buffer sets are reused while earlier steps are still queued
    and each loss lands in its mapped host slot: results must not change."""
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=8, embedding_dim=8,
                    vocabulary_size=5000, cache_capacity=700, hidden_dim=16, zipf_exponent=1.1)
    st = check_modes(cfg, 12, inflight)
    assert st["total_evicted"] > 0
    cfg = sb.Config(num_workers=1, batch_size_per_worker=512, num_fields=13, embedding_dim=16,
                    vocabulary_size=200_000, cache_capacity=200_000, hidden_dim=32,
                    zipf_exponent=1.05)
    st = check_modes(cfg, 8, inflight)
    assert st["total_free_steps"] == 8


def test_submit_protocol_errors():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=8, num_fields=4, embedding_dim=4,
                    vocabulary_size=1000, cache_capacity=200, hidden_dim=4)
    cfg.apply("mode", "pipelined")
    tr = sb.Trainer(cfg)
    gen = sb.SyntheticGenerator(cfg)
    b = [gen.generate(t) for t in range(5)]
    for t in range(4):  # up to four steps may be outstanding
        tr.submit(t, *b[t])
    with pytest.raises(sb.LogicError):  # loss of step 0 not read yet
        tr.submit(4, *b[4])
    with pytest.raises(sb.LogicError):  # never submitted
        tr.loss(9)
    assert all(np.isfinite(tr.loss(t)) for t in range(4))
    tr.close()


def test_prepare_train_split_matches_step():
    """sfctr_trainer_prepare + sfctr_trainer_train (the Host-Manager / GPU-Worker stages)
    give the same run as sfctr_trainer_step_device, and misuse is a LogicError."""
    import torch
    cfg = sb.Config(num_workers=1, batch_size_per_worker=64, num_fields=8, embedding_dim=8,
                    vocabulary_size=5000, cache_capacity=700, hidden_dim=16, zipf_exponent=1.1)
    cfg.apply("mode", "pipelined")
    batches = _batches(cfg, 8)
    feats = [torch.from_numpy(f.view(np.int64)).cuda() for f, _, _ in batches]
    labs = [torch.from_numpy(y).cuda() for _, y, _ in batches]
    outs = []
    for split in (False, True):
        tr = sb.Trainer(cfg)
        loss = torch.zeros(len(batches), dtype=torch.float32, device="cuda")
        for t in range(len(batches)):
            lp = loss[t:t + 1].data_ptr()
            if split:
                tr.prepare_device(t, feats[t].data_ptr())
                tr.train_device(t, labs[t].data_ptr(), lp)
            else:
                tr.step_device(t, feats[t].data_ptr(), labs[t].data_ptr(), None, lp)
        tr.synchronize()
        outs.append((loss.cpu().numpy(), tr.snapshot(), tr.ledger(), tr.cache_slots(0)))
        if split:
            tr.prepare_device(len(batches), feats[0].data_ptr())
            with pytest.raises(sb.LogicError):  # prepared but not trained
                tr.prepare_device(len(batches) + 1, feats[1].data_ptr())
            with pytest.raises(sb.LogicError):  # train of a step that was not prepared
                tr.train_device(len(batches) + 5, labs[0].data_ptr())
        tr.close()
    (l0, s0, g0, c0), (l1, s1, g1, c1) = outs
    assert np.allclose(l0, l1, rtol=1e-6)
    assert g0 == g1 and all(np.array_equal(a, b) for a, b in zip(c0, c1))
    assert np.array_equal(s0[0], s1[0]) and np.array_equal(s0[2], s1[2])
    check_rows_close(s1[1], s0[1].astype(np.float64), s1[2], cfg.embedding_dim, cfg.learning_rate)


@pytest.mark.parametrize("lanes,slack", [(1, 8), (1, 200), (4, 4), (4, 60)])
def test_pipelined_long_run_stress(lanes, slack):
    """40 pipelined steps with steady evictions (and pinned waits when the cache is tight):
    every step's slot table stays bit-exact with the oracle's — a cross-stream race in the
    double-buffered state would show up as a diverging slot table or ledger."""
    cfg = sb.Config(num_workers=lanes, batch_size_per_worker=256 // lanes, num_fields=6,
                    embedding_dim=8, vocabulary_size=8000, cache_capacity=1, hidden_dim=16,
                    zipf_exponent=0.9)
    cfg.apply("mode", "pipelined")
    batches = _batches(cfg, 40)
    owned = max(int(np.sum(oracle_vsi(f, 256, 6)[0] % lanes == w))
                for f, _, _ in batches for w in range(lanes))
    cap = owned + slack  # tight: evictions reach into the previous (in-flight) batch's rows
    cfg.cache_capacity = cap
    O, sim, ol = _oracle(cfg, batches)
    tr = sb.Trainer(cfg)
    losses = []
    for t, (f, y, w) in enumerate(batches):
        tr.submit(t, f, y, w)
        if t > 0:
            losses.append(tr.loss(t - 1))
    losses.append(tr.loss(len(batches) - 1))
    assert np.all(np.abs(np.array(losses) - ol) <= 1e-5 * np.abs(ol))
    for w in range(lanes):
        of, olu, oseq = orc_slots(sim, w, cap)
        df, dlu, dseq = tr.cache_slots(w)
        assert np.array_equal(df, of)
        occ = of != np.iinfo(np.uint64).max
        assert np.array_equal(dlu[occ], olu[occ]) and np.array_equal(dseq[occ], oseq[occ])
    led = np.zeros(4, np.int64)
    O.orc_sim_ledger(sim, led)
    dl = tr.ledger()
    assert [dl["host_to_worker"], dl["worker_to_host"], dl["interworker"],
            dl["swap_events"]] == led.tolist()
    assert dl["swap_events"] > 0
    of, orows, ost = orc_snapshot(sim, cfg.embedding_dim)
    df, drows, dst = tr.snapshot()
    assert np.array_equal(df, of) and np.array_equal(dst, ost)
    check_rows_close(drows, orows, dst, cfg.embedding_dim, cfg.learning_rate)
    O.orc_sim_destroy(sim)
    tr.close()
