"""One rank of the multi-GPU per-step parity check at cfg2 dimensions (launched by
tests/test_gpu_multi.py through torch.distributed.run).

d = 80, F = 39, b = 1024 rows per GPU, vocab 33.8M, Zipf 1.05 (BASELINE configs[1]
shapes at a batch the fp64 oracle steps in well under a second), W = the number of
ranks, one worker per GPU. Every rank trains its rows of the same global batches; after
each step the ranks send rank 0 their loss, logits, slot table, ledger, dense state and
the rows of the step's features they own, and rank 0 compares them with the oracle's
W-worker step FROM IDENTICAL STATE, then loads the device state into the oracle
(tests/parity_util.py: loss / logits 1e-5, the summed gradient within 1e-5 of its
condition scale, rows and moments 1e-5 + that tolerance through Adam, slot tables /
steps / ledger bit-exact). The dense parameters must also be bit-identical across ranks
(same all-reduced gradient, same update). Exit code 0 = parity.

--cache: slots per worker (40000: LRU evictions from step 3 on; 200000: no eviction,
the whole-shard regime of the bench).
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sync", default="alltoall")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--mode", default="pipelined")
    ap.add_argument("--cache", type=int, default=40000)
    ap.add_argument("--batch", type=int, default=1024)
    args = ap.parse_args()
    import torch
    import torch.distributed as td

    import paper_2104_08542_b200 as sb
    from paper_2104_08542_b200 import dist

    D = dist.from_env()
    torch.cuda.set_device(D.local_rank)
    W = D.world
    d, F, H = 80, 39, 64
    cfg = sb.Config(num_workers=W, batch_size_per_worker=args.batch, num_fields=F,
                    embedding_dim=d, vocabulary_size=33_800_000, cache_capacity=args.cache,
                    hidden_dim=H, zipf_exponent=1.05, seed=7)
    cfg.apply("sync", args.sync)
    cfg.apply("mode", args.mode)
    nid = dist.nccl_id_for(D, sb.nccl_unique_id)
    tr = sb.Trainer(cfg, rank=D.rank, world=W, nccl_id=nid, device=D.local_rank)
    gen = sb.SyntheticGenerator(cfg, device=D.local_rank)
    r0, n = dist.rows_of(D.rank, tr.lanes, cfg.batch_size_per_worker)
    P = F * d * H + 2 * H + 1
    from oracle_lib import OrcConfig, oracle, oracle_vsi
    from parity_util import (Grads, check_dense_one_step, check_logits, check_rows_one_step,
                             load_dense, load_rows, oracle_dense, oracle_rows)
    O = sim = None
    if D.rank == 0:
        O = oracle()
        oc = OrcConfig()
        O.orc_config_default(oc)
        for k in ("num_workers", "embedding_dim", "num_fields", "batch_size_per_worker",
                  "vocabulary_size", "cache_capacity", "hidden_dim", "zipf_exponent", "seed"):
            setattr(oc, k, getattr(cfg, k))
        oc.num_threads = os.cpu_count() or 1
        sim = O.orc_sim_create(C.byref(oc))
        O.orc_sim_keep_grads(sim, 1)
        p, m, v, ds = tr.dense_state()
        load_dense(O, sim, p, m, v, ds)
    ok = True
    msg = ""
    evictions = 0
    for t in range(args.steps):
        f, y = gen.generate(t)  # the global batch (each rank trains its rows)
        fl, yl = f[r0 * F:(r0 + n) * F].copy(), y[r0:r0 + n].copy()
        gids, _ = oracle_vsi(f, W * args.batch, F, W)
        mine = gids[gids % W == D.rank]
        if D.rank == 0:
            old, _ = oracle_rows(O, sim, gids, d)
            old_dense = oracle_dense(O, sim, P)[:3]
        loss = tr.step(t, fl, yl)
        drows, dst = tr.peek_rows(mine)
        slots, lus, seqs = tr.cache_slots(0)
        payload = (D.rank, loss, tr.logits(), slots, lus, seqs, tr.free_count(0), tr.ledger(),
                   tr.stats()["unique"], mine, drows, dst, tr.dense_state())
        got = [None] * W
        td.all_gather_object(got, payload)
        if D.rank == 0 and ok:
            try:
                ol = C.c_double()
                logits = np.zeros(W * args.batch)
                assert O.orc_sim_step(sim, t, f, y, None, 0, C.byref(ol), None,
                                      logits.ctypes.data) == 0, O.orc_last_error()
                got.sort(key=lambda g: g[0])
                for g in got:
                    assert abs(g[1] - ol.value) <= 1e-5 * abs(ol.value), (t, g[0], g[1], ol.value)
                    check_logits(g[2], logits[g[0] * args.batch:(g[0] + 1) * args.batch],
                                 f"step {t} rank {g[0]}")
                    of = np.zeros(cfg.cache_capacity, np.uint64)
                    olu = np.zeros(cfg.cache_capacity, np.int64)
                    oseq = np.zeros(cfg.cache_capacity, np.uint64)
                    O.orc_sim_cache_slots(sim, g[0], of, olu, oseq)
                    assert np.array_equal(g[3], of), ("slots", t, g[0])
                    occ = of != np.iinfo(np.uint64).max
                    assert np.array_equal(g[4][occ], olu[occ]), ("last_use", t, g[0])
                    assert np.array_equal(g[5][occ], oseq[occ]), ("admit_seq", t, g[0])
                    assert g[6] == O.orc_sim_free_count(sim, g[0]), ("free", t, g[0])
                    assert g[8] == gids.size == O.orc_sim_last_unique(sim), ("unique", t)
                led_o = np.zeros(4, np.int64)
                O.orc_sim_ledger(sim, led_o)
                keys = ("host_to_worker", "worker_to_host", "interworker", "swap_events")
                led_d = [sum(g[7][k] for g in got) for k in keys]
                assert led_d == led_o.tolist(), ("ledger", t, led_d, led_o.tolist())
                evictions = led_d[3]
                # rows of the step's features, assembled in global_ids order from their owners
                pos = {int(x): i for i, x in enumerate(gids)}
                drows_all = np.zeros((gids.size, 3 * d), np.float32)
                dst_all = np.zeros(gids.size, np.int64)
                for g in got:
                    idx = np.array([pos[int(x)] for x in g[9]], np.int64)
                    drows_all[idx] = g[10]
                    dst_all[idx] = g[11]
                orows, ost = oracle_rows(O, sim, gids, d)
                gr = Grads(O, sim, gids.size, d, P)
                st = check_rows_one_step(gids, old, drows_all, dst_all, orows, ost, gr, d, cfg,
                                         f"step {t}")
                pd, md, vd, dsd = got[0][12]
                for g in got[1:]:  # replicated dense state: bit-identical on every rank
                    assert all(np.array_equal(a, b) for a, b in zip(g[12][:3], (pd, md, vd))), t
                po, mo, vo, dso = oracle_dense(O, sim, P)
                assert dsd == dso == t + 1
                dn = check_dense_one_step(old_dense, (pd, md, vd), (po, mo, vo), gr, dsd, cfg,
                                          f"step {t}")
                print(f"step {t}: U {gids.size} theta {st['theta_max_rel']:.2e} m "
                      f"{st['m_max_rel']:.2e} v {st['v_max_rel']:.2e} |g|<=tol "
                      f"{st['sensitive_coords']} relu-undetermined {gr.n_amb} dense-w1 "
                      f"{dn['w1']['theta_max_rel']:.2e} evictions {evictions}", flush=True)
                load_rows(O, sim, gids, drows_all, dst_all)
                load_dense(O, sim, pd, md, vd, dsd)
            except AssertionError as e:
                ok = False
                msg = repr(e)[:2000]
                print("PARITY FAILURE:", msg, flush=True)
    if D.rank == 0:
        print(f"sync={args.sync} mode={args.mode} W={W} cache={args.cache} steps={args.steps} "
              f"evictions={evictions} parity {'ok' if ok else 'FAILED'}", flush=True)
    flag = torch.tensor([1 if ok else 0])
    td.broadcast(flag, 0)
    tr.close()
    D.close()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
