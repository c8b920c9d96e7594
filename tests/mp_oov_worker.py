"""One rank of the multi-GPU out-of-vocabulary check (launched by tests/test_gpu_multi.py
through torch.distributed.run). Rank 1's batch of step 2 carries an id >= vocab: every rank's
step must fail with LogicError (the bad-id bit travels with the manager stage's first
barrier, or with the id all-gather's), no rank's rows, moments, step counts, slot tables or
dense state may move, and training then continues exactly like a run that never saw the bad
batch (bit-identical final state; same bars as tests/test_gpu_parity.py's single-GPU
test_out_of_vocab_moves_no_state). Exit code 0 = pass."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sync", default="alltoall")
    ap.add_argument("--mode", default="pipelined")
    args = ap.parse_args()
    import torch

    import paper_2104_08542_b200 as sb
    from paper_2104_08542_b200 import dist

    D = dist.from_env()
    torch.cuda.set_device(D.local_rank)
    W = D.world
    cfg = sb.Config(num_workers=W, batch_size_per_worker=128, num_fields=8, embedding_dim=16,
                    vocabulary_size=50_000, cache_capacity=4000, hidden_dim=16)
    cfg.apply("sync", args.sync)
    cfg.apply("mode", args.mode)
    gen = sb.SyntheticGenerator(cfg, device=D.local_rank)
    r0, n = dist.rows_of(D.rank, 1, cfg.batch_size_per_worker)
    batches = [gen.generate(t, r0, n) for t in range(4)]

    def state(tr):
        return tr.snapshot(), tr.cache_slots(0), tr.dense_state()

    def same(a, b, what, tol=0.0):
        """Bit-identical indices and tables; float state within tol (0: bit-identical). The
        continued run is compared with tol = 1e-6: float atomics in the default
        (non-deterministic) mode reorder sums between any two runs."""
        for nm, x, y in zip(("features", "rows", "steps"), a[0], b[0]):
            if nm == "rows" and tol:
                assert np.max(np.abs(x - y)) <= tol, (what, nm, float(np.max(np.abs(x - y))))
            else:
                assert np.array_equal(x, y), (what, nm, np.argwhere(x != y)[:4].tolist())
        for nm, x, y in zip(("slots", "last_use", "admit_seq"), a[1], b[1]):
            assert np.array_equal(x, y), (what, nm, np.argwhere(x != y)[:4].tolist())
        for nm, x, y in zip(("dense", "m", "v"), a[2][:3], b[2][:3]):
            err = float(np.max(np.abs(x - y) / (np.abs(y) + 1e-3)))
            assert err <= tol, (what, nm, err)
        assert a[2][3] == b[2][3], (what, "dense step")

    ok = True
    try:
        tr = sb.Trainer(cfg, rank=D.rank, world=W, nccl_id=dist.nccl_id_for(D, sb.nccl_unique_id),
                        device=D.local_rank)
        for t in range(2):
            tr.step(t, *batches[t])
        before = state(tr)
        bad = batches[2][0].copy()
        if D.rank == 1:
            bad[5] = cfg.vocabulary_size + 7
        raised = False
        try:
            tr.step(2, bad, batches[2][1])
        except sb.LogicError:
            raised = True
        assert raised, f"rank {D.rank}: no LogicError for the gated step"
        same(before, state(tr), "gated step")
        losses = [tr.step(t, *batches[t]) for t in (2, 3)]
        got = state(tr)
        tr.close()
        ref = sb.Trainer(cfg, rank=D.rank, world=W,
                         nccl_id=dist.nccl_id_for(D, sb.nccl_unique_id), device=D.local_rank)
        ref_losses = [ref.step(t, *batches[t]) for t in range(4)][2:]
        same(state(ref), got, "continued", tol=1e-6)
        assert all(abs(a - b) <= 1e-6 * abs(b) for a, b in zip(losses, ref_losses)), \
            (losses, ref_losses)
        ref.close()
    except AssertionError as e:
        ok = False
        print(f"rank {D.rank} OOV FAILURE: {e!r}"[:2000], flush=True)
    import torch.distributed as td
    flags = [None] * W
    td.all_gather_object(flags, ok)
    if D.rank == 0:
        print(f"sync={args.sync} mode={args.mode} W={W} oov {'ok' if all(flags) else 'FAILED'}",
              flush=True)
    D.close()
    sys.exit(0 if all(flags) else 1)


if __name__ == "__main__":
    main()
