#!/usr/bin/env python
"""BASELINE configs[2]: Virtual Sparse Id + embedding-sync microbenchmark.

Sweeps batch 1K-64K per GPU and the unique-id ratio (set by vocabulary and Zipf
exponent, measured, not assumed) at N GPUs (torchrun, one process per GPU), on the
device path's own phases: ids all-gather (NCCL), VSI over the global batch, and the
embedding / gradient synchronisation — the owner-routed exchange over NVLink peer
stores (sync=alltoall, default) or the reference's NCCL all-reduce of the zero-padded
common embedding (sync=allreduce). Each point runs full training steps in sequential
mode (phases do not overlap, so each phase's CUDA-event time is its own) and reports
per-phase device time (max over ranks) with the rates the phases achieve:

  vsi        ids/s and algorithmic HBM GB/s (8 N_g + 12 U bytes)
  allgather  bytes received per GPU ((W-1) x 4 n) / time
  sync       alltoall: rows pushed per GPU per direction x 4d / time of the row moves;
             allreduce: NCCL bus bytes 2(W-1)/W x 4 d U per all-reduce / time

One JSON line per point on rank 0. Synthetic data (the reference generator, seed 7).
  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 bench_cfg3.py
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (vocab, zipf) -> unique ratio from ~1 % to ~99 % (measured at b=8192, W=8)
RATIO_POINTS = [(1_000_000, 2.0), (1_000_000, 1.2), (1_000_000, 0.8), (33_800_000, 0.5),
                (33_800_000, 0.0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1024,4096,16384,65536")
    ap.add_argument("--fields", type=int, default=26)
    ap.add_argument("--dim", type=int, default=80)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sync", default="alltoall", choices=["alltoall", "allreduce"])
    ap.add_argument("--points", default="", help="vocab:zipf,... (default: the ratio sweep)")
    args = ap.parse_args()
    import torch

    import paper_2104_08542_b200 as sb
    from paper_2104_08542_b200 import dist as sdist

    D = sdist.from_env()
    dev = D.local_rank
    torch.cuda.set_device(dev)
    W = D.world
    points = RATIO_POINTS
    if args.points:
        points = [(int(p.split(":")[0]), float(p.split(":")[1])) for p in args.points.split(",")]
    nid_cache = {}
    for b in [int(x) for x in args.batches.split(",")]:
        for vocab, zipf in points:
            cfg = sb.Config(num_workers=W, batch_size_per_worker=b, num_fields=args.fields,
                            embedding_dim=args.dim, vocabulary_size=vocab,
                            cache_capacity=(vocab + W - 1) // W, hidden_dim=64,
                            zipf_exponent=zipf, seed=7)
            cfg.apply("sync", args.sync)
            cfg.apply("mode", "sequential")
            nid = sdist.nccl_id_for(D, sb.nccl_unique_id) if W > 1 else None
            tr = sb.Trainer(cfg, rank=D.rank, world=W, nccl_id=nid, device=dev)
            gen = sb.SyntheticGenerator(cfg, device=dev)
            r0, nrows = sdist.rows_of(D.rank, tr.lanes, b)
            F = args.fields
            nb = args.warmup + args.steps
            d_feat = torch.empty((nb, nrows * F), dtype=torch.int64, device=f"cuda:{dev}")
            d_lab = torch.empty((nb, nrows), dtype=torch.uint8, device=f"cuda:{dev}")
            for s in range(nb):
                gen.generate_device(s, r0, nrows, d_feat[s].data_ptr(), d_lab[s].data_ptr())
            torch.cuda.synchronize()
            for s in range(args.warmup):
                tr.step_device(s, d_feat[s].data_ptr(), d_lab[s].data_ptr())
            tr.synchronize()
            st0 = tr.stats()
            tr.set_timing(True)
            D.barrier()
            t0 = time.perf_counter()
            for i in range(args.steps):
                s = args.warmup + i
                tr.step_device(s, d_feat[s].data_ptr(), d_lab[s].data_ptr())
            tr.synchronize()
            wall = D.max(time.perf_counter() - t0) / args.steps
            ph = {k: D.max(v / args.steps) for k, v in tr.phase_times()}
            st1 = tr.stats()
            K = args.steps
            U = (st1["total_unique"] - st0["total_unique"]) / K
            nv = (st1["total_nvlink_bytes"] - st0["total_nvlink_bytes"]) / K
            tr.close()
            n = b * F
            Ng = W * n
            out = {"bench": "cfg3 vsi+sync", "n_gpus": W, "batch_per_gpu": b, "fields": F,
                   "dim": args.dim, "vocab": vocab, "zipf": zipf, "sync": args.sync,
                   "global_ids": Ng, "unique": round(U, 1), "unique_ratio": round(U / Ng, 4),
                   "step_ms_wall": round(wall * 1e3, 4)}
            vms = ph.get("vsi", 0)
            if vms > 0:
                out["vsi"] = {"ms": round(vms, 4), "gids_per_s": round(Ng / vms / 1e6, 3),
                              "hbm_gbs": round((8 * Ng + 12 * U) / vms / 1e6, 1)}
            if W > 1:
                ag = ph.get("ids_allgather", 0)
                out["allgather"] = {"ms": round(ag, 4),
                                    "gbs": round((W - 1) * 4 * n / ag / 1e6, 1) if ag else None}
                if args.sync == "alltoall":
                    # rows pushed + received in the forward exchange (counted once; the
                    # backward moves the same rows the other way)
                    rows_b = nv - 4 * n - 4 * (F * args.dim * 64 + 2 * 64 + 2)
                    per_dir = rows_b / 2
                    fwd = ph.get("exchange_embed", 0)
                    bwd = ph.get("exchange_grad_send", 0)
                    plan = ph.get("exchange_plan", 0)
                    out["sync"] = {
                        "plan_ms": round(plan, 4), "fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
                        "reduce_ms": round(ph.get("exchange_grad", 0), 4),
                        "barrier_ms": round(ph.get("exchange_barrier", 0)
                                            + ph.get("exchange_grad_barrier", 0), 4),
                        "bytes_per_dir": int(per_dir),
                        "fwd_gbs": round(per_dir / fwd / 1e6, 1) if fwd else None,
                        "bwd_gbs": round(per_dir / bwd / 1e6, 1) if bwd else None,
                        "peak_gbs": 770.0, "peak_source": "B200_PROFILING.md measured peer copy"}
                else:
                    pay = 4 * args.dim * U
                    bus = 2 * (W - 1) / W * pay
                    a1, a2 = ph.get("allreduce_embed", 0), ph.get("allreduce_grad", 0)
                    out["sync"] = {"allreduce_embed_ms": round(a1, 4),
                                   "allreduce_grad_ms": round(a2, 4),
                                   "payload_bytes": int(pay),
                                   "busbw_embed_gbs": round(bus / a1 / 1e6, 1) if a1 else None,
                                   "busbw_grad_gbs": round(bus / a2 / 1e6, 1) if a2 else None,
                                   "peak_gbs": 770.0,
                                   "peak_source": "B200_PROFILING.md measured peer copy"}
            if D.rank == 0:
                print(json.dumps(out), flush=True)
            D.barrier()
    D.close()


if __name__ == "__main__":
    main()
