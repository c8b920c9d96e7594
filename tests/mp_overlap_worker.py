"""One rank of the multi-GPU in-flight check (launched by tests/test_gpu_multi.py
through torch.distributed.run). Every rank trains its rows of the same global
batches with up to three steps in flight (pipelined mode: the manager stage of step
t+1 overlaps step t's training, and a faster peer's pushes of step t+1 race this
rank's step t); rank 0 compares the merged final state with the CPU oracle running
the same W-worker system (multi-step trajectory: tests/test_gpu_parity.py bars; the
per-step identical-state bars are tests/mp_parity_worker.py's). Exit code 0 = parity."""
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
    ap.add_argument("--sync", default="allreduce")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--mode", default="sequential")
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--dump", default="", help="rank 0 saves the merged final state (npz)")
    args = ap.parse_args()
    import torch
    import torch.distributed as td

    import paper_2104_08542_b200 as sb
    from paper_2104_08542_b200 import dist

    D = dist.from_env()
    torch.cuda.set_device(D.local_rank)
    W = D.world
    cfg = sb.Config(num_workers=W, batch_size_per_worker=256, num_fields=12, embedding_dim=16,
                    vocabulary_size=200_000, cache_capacity=2500, hidden_dim=32,
                    zipf_exponent=1.05)
    cfg.apply("sync", args.sync)
    cfg.apply("mode", args.mode)
    if args.deterministic:
        cfg.apply("deterministic", "1")
    nid = dist.nccl_id_for(D, sb.nccl_unique_id)
    tr = sb.Trainer(cfg, rank=D.rank, world=W, nccl_id=nid, device=D.local_rank)
    gen = sb.SyntheticGenerator(cfg, device=D.local_rank)
    r0, n = dist.rows_of(D.rank, tr.lanes, cfg.batch_size_per_worker)
    F = cfg.num_fields
    losses = []
    if args.mode == "pipelined":  # three steps in flight: submit t, then read the loss of t-2
        batches = [gen.generate(t, r0, n) for t in range(args.steps)]
        for t in range(args.steps):
            tr.submit(t, *batches[t])
            if t >= 2:
                losses.append(tr.loss(t - 2))
        for t in range(max(0, args.steps - 2), args.steps):
            losses.append(tr.loss(t))
    else:
        for t in range(args.steps):
            f, y = gen.generate(t, r0, n)
            losses.append(tr.step(t, f, y))
    feats, rows, steps = tr.snapshot()
    slots = tr.cache_slots(0)[0]
    led = tr.ledger()
    stats = tr.stats()
    # gather everything on rank 0 through gloo (object lists)
    payload = (D.rank, losses, feats, rows, steps, slots, led, stats)
    gathered = [None] * W
    td.all_gather_object(gathered, payload)
    ok = True
    if D.rank == 0:
        from oracle_lib import OrcConfig, oracle
        from test_gpu_parity import check_rows_close
        O = oracle()
        oc = OrcConfig()
        O.orc_config_default(oc)
        for k in ("num_workers", "embedding_dim", "num_fields", "batch_size_per_worker",
                  "vocabulary_size", "cache_capacity", "hidden_dim", "zipf_exponent", "seed"):
            setattr(oc, k, getattr(cfg, k))
        sim = O.orc_sim_create(C.byref(oc))
        full = sb.SyntheticGenerator(cfg, device=0)
        for t in range(args.steps):
            f, y = full.generate(t)
            ol = C.c_double()
            assert O.orc_sim_step(sim, t, f, y, None, 0, C.byref(ol), None, None) == 0
            for g in gathered:
                if abs(g[1][t] - ol.value) > 1e-5 * abs(ol.value):
                    print(f"loss mismatch rank {g[0]} step {t}: {g[1][t]} vs {ol.value}")
                    ok = False
        for g in gathered:  # per-worker cache slot tables: bit-exact
            of = np.zeros(cfg.cache_capacity, np.uint64)
            O.orc_sim_cache_slots(sim, g[0], of, np.zeros(cfg.cache_capacity, np.int64),
                                  np.zeros(cfg.cache_capacity, np.uint64))
            if not np.array_equal(g[5], of):
                print(f"cache slots differ on worker {g[0]}")
                ok = False
        order = np.argsort(np.concatenate([g[2] for g in gathered]), kind="stable")
        df = np.concatenate([g[2] for g in gathered])[order]
        dr = np.concatenate([g[3] for g in gathered])[order]
        ds = np.concatenate([g[4] for g in gathered])[order]
        if args.dump:
            np.savez(args.dump, features=df, rows=dr, steps=ds,
                     losses=np.array([g[1] for g in gathered]))
        n_orc = O.orc_sim_snapshot(sim, None, None, None)
        of = np.zeros(n_orc, np.uint64)
        orows = np.zeros((n_orc, 3 * cfg.embedding_dim))
        ost = np.zeros(n_orc, np.int64)
        O.orc_sim_snapshot(sim, of.ctypes.data, orows.ctypes.data, ost.ctypes.data)
        if not (np.array_equal(df, of) and np.array_equal(ds, ost)):
            print("snapshot features/steps differ")
            ok = False
        else:
            try:
                check_rows_close(dr, orows, ds, cfg.embedding_dim, cfg.learning_rate)
            except AssertionError as e:
                print("rows differ:", e)
                ok = False
        led_o = np.zeros(4, np.int64)
        O.orc_sim_ledger(sim, led_o)
        led_d = [sum(g[6][k] for g in gathered) for k in
                 ("host_to_worker", "worker_to_host", "interworker", "swap_events")]
        if led_d != led_o.tolist():
            print("ledger differs", led_d, led_o.tolist())
            ok = False
        print(f"sync={args.sync} mode={args.mode} W={W} parity {'ok' if ok else 'FAILED'}; nvlink bytes/step "
              f"{[g[7]['nvlink_bytes'] for g in gathered]}", flush=True)
    flag = torch.tensor([1 if ok else 0])
    td.broadcast(flag, 0)
    D.close()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
