#!/usr/bin/env python
"""Benchmark: DeepFM training samples/s on the ScaleFreeCTR embedding hot path.

Workload (BASELINE.json configs[1]): Criteo-shaped DeepFM-lite, 39 sparse
fields, 33.8M-row table, d=80, hidden 64, batch 8192 per GPU, Zipf 1.05,
lazy Adam. MixCache sized for the B200: by default (--cache 0) the whole owned
shard of the table (33.8M/W rows x emb+m+v = 32 GB at W=1) is the HBM cache, so
rows are lazily initialised on first touch and never leave HBM; --cache N runs
the paper's small-cache regime (e.g. 2^19 slots = 0.48 GiB) over the pinned host
table with LRU eviction over PCIe. One process per GPU (torchrun), weak scaling.

Arms
  ours       : `value` = samples/s with each step's batch already resident in
               HBM (device-resident API, CUDA events on the trainer stream,
               max over ranks); `e2e` = the same through the public host-buffer
               API (pinned host batch -> H2D -> step -> loss into mapped
               host memory, read every step; `--inflight` steps left unread). Also `roofline` of the dominant kernel (per-phase CUDA
               events over the timed region), per-kernel rows, `cpu_baseline`.
  reference  : the CPU path (the oracle port of the reference in fp64; the
               reference's own TUs cover only VSI/generator/cache primitives)
               on the host cores, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

os.environ.setdefault("SFCTR_PHASE_GATE_US", "1500")  # read by the trainer in its phase pass

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = ("cfg2: DeepFM-lite Criteo-shaped, 39 sparse fields, 33.8M-row table, d=80, hidden 64, "
            "batch 8192/GPU, Zipf 1.05, lazy Adam, MixCache")
METRIC = "training samples/sec"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--batch", type=int, default=8192)
    p.add_argument("--fields", type=int, default=39)
    p.add_argument("--dim", type=int, default=80)
    p.add_argument("--vocab", type=int, default=33_800_000)
    p.add_argument("--zipf", type=float, default=1.05)
    p.add_argument("--hidden", type=int, default=64)
    p.add_argument("--cache", type=int, default=0,
                   help="HBM cache slots per GPU; 0 = the whole owned shard")
    # alltoall = owner-routed exchange of only the touched rows (default); allreduce = the
    # reference's all-reduce of the zero-padded common embedding / gradients
    p.add_argument("--sync", default="alltoall", choices=["allreduce", "alltoall"])
    # pipelined = the manager stage of step t+1 overlaps step t's training (identical results)
    p.add_argument("--mode", default="pipelined", choices=["pipelined", "sequential"])
    p.add_argument("--inflight", type=int, default=3, choices=[1, 2, 3],
                   help="e2e arm (pipelined): submitted steps whose loss is not yet read")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-mixcache", action="store_true",
                   help="skip the MixCache-over-PCIe sub-lines (mixcache_small, cfg4)")
    p.add_argument("--only-mixcache", action="store_true",
                   help="run the MixCache sub-lines only (development)")
    p.add_argument("--cfg4-cache-frac", type=float, default=0.10,
                   help="cfg4 hot cache as a fraction of HBM (BASELINE configs[3]: 10-50 %%)")
    p.add_argument("--cpu-rows", type=int, default=8192,
                   help="rows per CPU-baseline step (default: the full cfg2 batch per GPU)")
    p.add_argument("--cpu-steps", type=int, default=3)
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
hs = [pynvml.nvmlDeviceGetHandleByIndex(int(i)) for i in sys.argv[1].split(",")]
mx = [pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) for h in hs]
print("max", *mx, flush=True)
period = float(sys.argv[2])
while True:
    for i, h in enumerate(hs):
        print(i, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)
    time.sleep(period)
"""


class Clocks:
    """SM clock / throttle-reason sampler for the timed region (B200_PROFILING.md clocks line):
    NVML polled every 5 ms for every GPU of the job from ONE separate process started by
    rank 0 (no GIL or driver-lock contention inside the ranks that issue the steps)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, indices, period_s=None):
        if period_s is None:  # BENCH_CLOCK_MS: sampler period (default 1 ms)
            period_s = float(os.environ.get("BENCH_CLOCK_MS", "1")) / 1e3
        self.indices, self.period = list(indices), period_s
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                [sys.executable, "-c", _SAMPLER, ",".join(map(str, self.indices)), str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()  # "max ..." once NVML is up
            self.mx = [int(x) for x in first[1:]] if first and first[0] == "max" else []
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampler not started"]}
        self.proc.terminate()
        out_txt, _ = self.proc.communicate(timeout=10)
        sm, reasons = [], set()
        for line in out_txt.splitlines():
            f = line.split()
            if len(f) != 3:
                continue
            sm.append(int(f[1]))
            for n, bit in self.REASONS.items():
                if int(f[2]) & bit:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "gpus": len(self.indices),
                "sampler": "nvml every 1 ms in a separate process, from the start of the value "
                           "region through the phase pass and the e2e region"}


def phase_bytes(name, U, Uw, n, b, d, F, H, Ntot, fused_scatter=False, xrecv=0):
    """Algorithmic bytes (or FLOPs for the tower) per step for each phase.
    fused_scatter: the segment sum runs in the dX GEMM's epilogue (one worker)."""
    if name == "vsi":
        return 8 * Ntot + 12 * U, "B"
    if name == "gather_cache":  # + the fused zeroing of dG / the FM coefficients (W = 1)
        return 8 * Uw + 8 * d * Uw + (4 * d * U + 4 * U if Ntot == n else 0), "B"
    if name == "zero_grads":  # one worker: dG[0:U) and the FM coefficients cleared
        return 4 * d * U + 4 * U, "B"
    if name == "gather_instances":
        return 4 * n + 8 * d * n + 4 * b * d + b * d, "B"
    if name == "segment_sum":
        return 4 * n + 4 * d * n + 4 * d * U, "B"
    if name == "sparse_adam":  # (owner-routed: + the owner's read of the pushed gradient rows)
        return 28 * d * Uw + 12 * Uw + xrecv, "B"
    if name in ("tower_gemm1", "tower_gemm3"):  # X [b x F*d] streamed once (W1 / dh from L2)
        return 4 * b * F * d, "B"
    if name == "tower_gemm2":  # dX [b x F*d] written once, or (fused) scattered into dG
        if fused_scatter:
            return 4 * n + 4 * d * n + 4 * d * U, "B"
        return 4 * b * F * d, "B"
    if name == "tower":  # SIMT validation tiles (SFCTR_TOWER_SIMT=1)
        return 6 * b * F * d * H, "FLOP"
    return None, None


def run_ours(args, D):
    import torch

    import paper_2104_08542_b200 as sb
    from paper_2104_08542_b200 import dist as sdist

    rank, world = D.rank, D.world
    dev = D.local_rank
    torch.cuda.set_device(dev)
    if args.cache <= 0:  # the whole owned shard resident in HBM
        args.cache = (args.vocab + world - 1) // world
    cfg = sb.Config(num_workers=world, batch_size_per_worker=args.batch, num_fields=args.fields,
                    embedding_dim=args.dim, vocabulary_size=args.vocab, cache_capacity=args.cache,
                    hidden_dim=args.hidden, zipf_exponent=args.zipf, seed=7)
    cfg.apply("sync", args.sync)
    cfg.apply("mode", args.mode)
    nid = sdist.nccl_id_for(D, sb.nccl_unique_id)
    t0 = time.time()
    tr = sb.Trainer(cfg, rank=rank, world=world, nccl_id=nid, device=dev)
    setup_s = time.time() - t0
    gen = sb.SyntheticGenerator(cfg, device=dev)
    r0, nrows = sdist.rows_of(rank, tr.lanes, args.batch)
    F = args.fields
    W, K = args.warmup, args.steps
    nb = W + 3 * K  # warm-up | value | phase breakdown | e2e
    # device-resident batches (value arm) and pinned host copies (e2e arm)
    d_feat = torch.empty((nb, nrows * F), dtype=torch.int64, device=f"cuda:{dev}")
    d_lab = torch.empty((nb, nrows), dtype=torch.uint8, device=f"cuda:{dev}")
    for s in range(nb):
        gen.generate_device(s, r0, nrows, d_feat[s].data_ptr(), d_lab[s].data_ptr())
    torch.cuda.synchronize()
    h_feat = d_feat.cpu().pin_memory()
    h_lab = d_lab.cpu().pin_memory()
    hf = h_feat.numpy().view(np.uint64)
    hl = h_lab.numpy()

    for s in range(W):  # warm-up through the public host API
        tr.step(s, hf[s], hl[s])
    stream = torch.cuda.ExternalStream(tr.stream, device=f"cuda:{dev}")
    d_loss = torch.zeros(1, dtype=torch.float32, device=f"cuda:{dev}")

    # ---- value: device-resident inputs, CUDA events on the trainer stream (no
    # per-phase events inside this region; the breakdown is a separate pass below)
    phases = {}
    stats_acc = {}
    clocks = Clocks(range(world)) if rank == 0 else None
    launches = 0
    if clocks:
        clocks.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    st0 = tr.stats()  # running totals before the timed region (waits for the stream)
    ev0.record(stream)
    h0 = time.perf_counter()
    for i in range(K):
        s = W + i
        tr.step_device(s, d_feat[s].data_ptr(), d_lab[s].data_ptr(), None, d_loss.data_ptr())
    host_issue_ms = (time.perf_counter() - h0) * 1e3 / K
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    dev_ms = ev0.elapsed_time(ev1)
    tr.synchronize()  # deferred device counters
    st1 = tr.stats()
    tot = {k2: st1[k2] - st0[k2] for k2 in st1 if k2.startswith("total")}
    launches = tot["total_kernel_launches"]
    filled = tot["total_filled_from_host"]
    stats_acc = {"unique": tot["total_unique"], "owned": tot["total_owned"],
                 "working": tot["total_working"], "evicted": tot["total_evicted"],
                 "filled_from_host": filled, "pcie_h2d_bytes": filled * (3 * args.dim + 1) * 4,
                 "pcie_d2h_bytes": tot["total_evicted"] * (3 * args.dim + 1) * 4,
                 "nvlink_bytes": tot["total_nvlink_bytes"], "kernel_launches": launches,
                 "host_wait_free_steps": tot["total_free_steps"],
                 "pinned_waits": tot["total_pinned_waits"]}
    D.barrier()
    ms_step = D.max(dev_ms) / K
    loss_dev = float(d_loss.item())

    # ---- per-phase breakdown: K more device-resident steps with phase events (the trainer
    # issues both stages on one stream while timing, so each phase time is its own; a
    # SFCTR_PHASE_GATE_US hold at the head of every step lets the host enqueue the whole
    # step first, so a phase's time is device time, not the host's issue time)
    tr.set_timing(True)
    D.barrier()
    for i in range(K):
        s = W + K + i
        tr.step_device(s, d_feat[s].data_ptr(), d_lab[s].data_ptr(), None, d_loss.data_ptr())
    tr.synchronize()
    phases = dict(tr.phase_times())
    tr.set_timing(False)
    D.barrier()

    # ---- e2e: host batch -> H2D -> step -> D2H loss, through the public API
    D.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    losses = []
    t_sub = t_wait = 0.0
    if args.mode == "pipelined":  # D steps in flight: submit step s, read the loss of s-D
        D_in = args.inflight
        for i in range(K):
            s = W + 2 * K + i
            a0 = time.perf_counter()
            tr.submit(s, hf[s], hl[s])
            a1 = time.perf_counter()
            if i >= D_in:
                losses.append(tr.loss(s - D_in))
            t_sub += a1 - a0
            t_wait += time.perf_counter() - a1
        for s in range(W + 3 * K - min(D_in, K), W + 3 * K):
            losses.append(tr.loss(s))
    else:
        for i in range(K):
            s = W + 2 * K + i
            losses.append(tr.step(s, hf[s], hl[s]))
    torch.cuda.synchronize()
    e2e_s = D.max(time.perf_counter() - w0)
    # the sampler ran from the start of the `value` region through the phase pass and the
    # e2e region (the value region alone is a few ms, shorter than NVML's update period)
    clk = clocks.stop() if clocks else None
    D.barrier()

    rows_global = world * args.batch
    value = rows_global / (ms_step / 1e3)
    e2e_value = rows_global * K / e2e_s
    per_step = {k2: v / K for k2, v in stats_acc.items()}
    phase_ms = {k2: v / K for k2, v in phases.items()}
    peaks, peak_kind = measured_peaks()
    U = per_step.get("unique", 0)
    Uw = per_step.get("owned", 0)
    n = args.batch * F
    Ntot = world * n
    d, H = args.dim, args.hidden
    # owner-routed exchange: nvlink_bytes counts the forward rows pushed + received once;
    # per direction each GPU moves about half of it each way, forward and backward alike
    xrecv = per_step.get("nvlink_bytes", 0) / 2 if (world > 1 and args.sync == "alltoall") else 0
    kernels = {}
    for nm, ms in phase_ms.items():
        amount, unit = phase_bytes(nm, U, Uw, n, args.batch, d, F, H, Ntot,
                                   fused_scatter="segment_sum" not in phase_ms,
                                   xrecv=xrecv)
        row = {"ms": round(ms, 4)}
        if amount is not None and ms > 0:
            if unit == "B":
                gbs = amount / (ms / 1e3) / 1e9
                row.update(bytes=int(amount), gbs=round(gbs, 1),
                           frac_hbm=round(gbs / peaks["hbm_gbs"], 3))
            else:
                tf = amount / (ms / 1e3) / 1e12
                row.update(flops=int(amount), tflops=round(tf, 2),
                           frac_bf16_sustained=round(tf / peaks["bf16_tflops_sustained"], 4))
        kernels[nm] = row
    tower_ms = sum(v["ms"] for k2, v in kernels.items() if k2.startswith("tower"))
    if tower_ms > 0:  # the tower as a whole, for reference: 3 GEMMs (3xTF32) + head + reductions
        fl = 3 * 6 * args.batch * F * d * H
        kernels["tower_total"] = {"ms": round(tower_ms, 4), "tf32_flops": fl,
                                  "tflops": round(fl / (tower_ms / 1e3) / 1e12, 2)}
    traffic = {}
    try:  # DRAM bytes per launch from the committed ncu --set full capture (profiles/): a
        # one-GPU capture (ncu never wraps a multi-rank command), so it describes N = 1 only;
        # at N > 1 the dominant kernel is the fused owner reduction + Adam, never captured
        if world == 1:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch", {})
    except Exception:
        pass
    # dominant kernel = the largest single-kernel phase with an algorithmic model
    cand = [(v["ms"], k2) for k2, v in kernels.items() if "bytes" in v or "flops" in v]
    dom = max(cand)[1] if cand else None
    roofline = None
    if dom:
        r = kernels[dom]
        if "bytes" in r:
            roofline = {"kernel": dom if world == 1 or dom != "sparse_adam"
                        else "owner_reduce_adam (fused owner reduction + sparse Adam)",
                        "bound": "hbm", "achieved": r["gbs"], "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": r["frac_hbm"], "traffic": traffic.get(dom),
                        "algorithmic_bytes": r["bytes"],
                        "peak_source": peak_kind + " (copy GB/s, MEASURED_PEAKS.json)"}
            if world > 1:
                roofline["traffic_note"] = ("null: ncu never wraps a multi-rank command; the "
                                            "committed capture is N = 1 (profiles/ncu_traffic.json)")
        else:
            roofline = {"kernel": dom, "bound": "tensor", "achieved": r["tflops"],
                        "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                        "frac": r["frac_bf16_sustained"], "traffic": None,
                        "peak_source": peak_kind + " (bf16 sustained; tower runs fp32)"}
    # NVLink sync rate (world > 1): bytes this rank handed to NCCL per step / time of the sync phases
    sync = None
    if world > 1:
        sync_ms = sum(v for k2, v in phase_ms.items()
                      if k2.startswith(("allreduce", "exchange", "shard_")) or k2 == "ids_allgather")
        nv = per_step.get("nvlink_bytes", 0)
        # all-reduce: NCCL bus bytes = 2(W-1)/W x payload; all-to-all: every byte
        # this rank sends crosses NVLink once
        busbytes = nv if args.sync == "alltoall" else 2 * (world - 1) / world * nv
        sync = {"ms": round(sync_ms, 4), "bytes_per_step": int(nv), "scheme": args.sync,
                "busbw_gbs": round(busbytes / (sync_ms / 1e3) / 1e9, 1) if sync_ms else None,
                "peak_gbs": 770.0, "peak_source": "B200_PROFILING.md measured peer copy",
                "note": "busbw over every sync phase (id all-gather, plan, barriers included)"}
        if args.sync == "alltoall":  # the row moves alone: bytes per direction / push time
            per_dir = nv / 2
            fwd, bwd = phase_ms.get("exchange_embed", 0), phase_ms.get("exchange_grad_send", 0)
            sync["rows"] = {"bytes_per_direction": int(per_dir),
                            "fwd_push_ms": round(fwd, 4), "bwd_push_ms": round(bwd, 4),
                            "fwd_gbs": round(per_dir / (fwd / 1e3) / 1e9, 1) if fwd else None,
                            "bwd_gbs": round(per_dir / (bwd / 1e3) / 1e9, 1) if bwd else None,
                            "frac_fwd": round(per_dir / (fwd / 1e3) / 1e9 / 770.0, 3) if fwd else None,
                            "frac_bwd": round(per_dir / (bwd / 1e3) / 1e9 / 770.0, 3) if bwd else None}
    fill_ms = phase_ms.get("manage_evict_admit", 0.0)
    mix = {"cache_slots_per_gpu": args.cache, "owned_uniques_per_step": round(Uw, 1),
           "misses_per_step": round(per_step.get("working", 0), 1),
           "evictions_per_step": round(per_step.get("evicted", 0), 1),
           "pcie_h2d_bytes_per_step": int(per_step.get("pcie_h2d_bytes", 0)),
           "pcie_d2h_bytes_per_step": int(per_step.get("pcie_d2h_bytes", 0)),
           "evict_admit_ms": round(fill_ms, 4)}
    if fill_ms > 0:
        pc = (per_step.get("pcie_h2d_bytes", 0) + per_step.get("pcie_d2h_bytes", 0))
        mix["pcie_gbs"] = round(pc / (fill_ms / 1e3) / 1e9, 2)
        mix["pcie_peak_gbs"] = 64.0
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (device Zipf generator, bit-exact with the reference SyntheticGenerator)",
        "config": {"workload": WORKLOAD, "global_batch": rows_global, "fields": F, "dim": d,
                   "vocab": args.vocab, "hidden": H, "zipf": args.zipf,
                   "cache_slots_per_gpu": args.cache, "sync": args.sync, "mode": args.mode,
                   "parallelism": f"dp{world} (embedding rows owned f mod {world})",
                   "l2": "no flush: per-step working set > L2 (X alone is 102 MB/GPU)",
                   "setup_s": round(setup_s, 2)},
        "e2e": {"value": round(e2e_value, 1), "unit": "samples/s", "inflight": args.inflight if args.mode == "pipelined" else 1,
                "host_submit_ms_per_step": round(t_sub * 1e3 / K, 4),
                "host_loss_wait_ms_per_step": round(t_wait * 1e3 / K, 4),
                "h2d_bytes_per_step": int(nrows * F * 8 + nrows),
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches),
        "host_issue_ms_per_step": round(D.max(host_issue_ms), 4),
        "roofline": roofline,
        "kernels": kernels,
        "mixcache": mix,
        "sync": sync,
        "clocks": clk,
        "loss": {"device_last": loss_dev, "e2e_last": losses[-1] if losses else None},
        "per_step": {k2: round(v, 1) for k2, v in per_step.items()},
    }
    tr.close()
    return out


def run_cache_line(name, vocab, dim, fields, batch, zipf, cache, host_reserve, steps, max_fill,
                   dev=0):
    """MixCache over the pinned host pool (PCIe): one GPU, a cache smaller than the touched
    table, so every step evicts LRU rows to the host and refills the ones that come back.
    Fills the cache first (device-resident batches until steps evict), then times `steps`
    steps on the trainer stream (CUDA events) and a second pass with per-phase events for
    the eviction + admission time: fill / write-back GB/s against PCIe Gen5 x16."""
    import torch

    import paper_2104_08542_b200 as sb
    cfg = sb.Config(num_workers=1, batch_size_per_worker=batch, num_fields=fields,
                    embedding_dim=dim, vocabulary_size=vocab, cache_capacity=cache,
                    hidden_dim=64, zipf_exponent=zipf, seed=7)
    cfg.apply("mode", "pipelined")
    cfg.apply("host_rows", str(host_reserve))
    t0 = time.time()
    tr = sb.Trainer(cfg, device=dev)
    gen = sb.SyntheticGenerator(cfg, device=dev)
    setup_s = time.time() - t0
    n = batch * fields
    ring = 64
    d_feat = torch.empty((ring, n), dtype=torch.int64, device=f"cuda:{dev}")
    d_lab = torch.empty((ring, batch), dtype=torch.uint8, device=f"cuda:{dev}")

    def fill_ring(s0):
        for i in range(ring):
            gen.generate_device(s0 + i, 0, batch, d_feat[i].data_ptr(), d_lab[i].data_ptr())
        torch.cuda.synchronize()

    # fill: until steps evict (the cache is full) for a few steps in a row
    s = 0
    t0 = time.time()
    evicting = 0
    while s < max_fill and evicting < 3:
        fill_ring(s)
        for i in range(ring):
            tr.step_device(s + i, d_feat[i].data_ptr(), d_lab[i].data_ptr())
        tr.synchronize()
        s += ring
        evicting = evicting + 1 if tr.stats()["evicted"] > 0 else 0
    fill_s = time.time() - t0
    stream = torch.cuda.ExternalStream(tr.stream, device=f"cuda:{dev}")
    fill_ring(s)
    K = min(steps, ring // 2)
    st0 = tr.stats()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(K):
        tr.step_device(s + i, d_feat[i].data_ptr(), d_lab[i].data_ptr())
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / K
    tr.synchronize()
    st1 = tr.stats()
    tot = {k: st1[k] - st0[k] for k in st1 if k.startswith("total")}
    tr.set_timing(True)
    for i in range(K, 2 * K):
        tr.step_device(s + i, d_feat[i].data_ptr(), d_lab[i].data_ptr())
    tr.synchronize()
    ph = {k: v / K for k, v in tr.phase_times()}
    tr.set_timing(False)
    st2 = tr.stats()
    tot2 = {k: st2[k] - st1[k] for k in st2 if k.startswith("total")}
    ev = tot["total_evicted"] / K
    fh = tot["total_filled_from_host"] / K
    row_b = (3 * dim + 1) * 4
    d2h, h2d = ev * row_b, fh * row_b
    # eviction + admission: LRU select (histogram) + candidate sort + the fused write-back /
    # refill / lazy-init kernel (the rest of manage_evict_admit)
    ea = sum(ph.get(k, 0.0) for k in ("evict_select", "evict_sort", "manage_evict_admit"))
    ev2 = tot2["total_evicted"] / K
    fh2 = tot2["total_filled_from_host"] / K
    pcie_ea = (ev2 + fh2) * row_b
    tr.close()
    return {"name": name, "value": round(batch / (ms / 1e3), 1), "unit": "samples/s",
            "ms_per_step": round(ms, 4), "steps": K,
            "config": {"vocab": vocab, "dim": dim, "fields": fields, "batch": batch, "zipf": zipf,
                       "cache_slots": cache, "cache_gb": round(cache * (12 * dim + 32) / 1e9, 2),
                       "host_pool_reserved_rows": host_reserve, "mode": "pipelined"},
            "fill": {"steps": s, "seconds": round(fill_s, 1)},
            "per_step": {"unique": round(tot["total_unique"] / K, 1),
                         "misses": round(tot["total_working"] / K, 1),
                         "evictions": round(ev, 1), "refills_from_host": round(fh, 1),
                         "pcie_d2h_bytes": int(d2h), "pcie_h2d_bytes": int(h2d)},
            "pcie": {"evict_admit_ms": round(ea, 4),
                     "gbs": round(pcie_ea / (ea / 1e3) / 1e9, 2) if ea else None,
                     "writeback_gbs": round(ev2 * row_b / (ea / 1e3) / 1e9, 2) if ea else None,
                     "fill_gbs": round(fh2 * row_b / (ea / 1e3) / 1e9, 2) if ea else None,
                     "step_gbs": round((d2h + h2d) / (ms / 1e3) / 1e9, 2),
                     "peak_gbs": 64.0,
                     "peak_source": "PCIe Gen5 x16 nominal per direction; 44-56 GB/s measured "
                                    "(profiles/r01s2_pcie_microbench.txt)"},
            "phases_ms": {k: round(v, 4) for k, v in ph.items()}}


def cpu_sample(args, workers, rows_total, steps, threads):
    """The oracle port (fp64 reference semantics) on host cores: rows_total rows/step."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import OrcConfig, oracle, oracle_generate
    O = oracle()
    c = OrcConfig()
    O.orc_config_default(c)
    c.num_workers = workers
    c.batch_size_per_worker = rows_total // workers
    c.num_fields = args.fields
    c.embedding_dim = args.dim
    c.vocabulary_size = args.vocab
    # per-worker cache: the arm's own size, capped at what the sample can touch (every
    # id of every step) — with no evictions possible the computation is identical, and
    # the fp64 port does not allocate a 33.8M-slot table for a 2048-row sample
    shard = (args.vocab + workers - 1) // workers
    cap = args.cache if 0 < args.cache < shard else shard
    c.cache_capacity = min(cap, rows_total * args.fields * steps + 1)
    c.hidden_dim = args.hidden
    c.zipf_exponent = args.zipf
    c.num_threads = threads
    sim = O.orc_sim_create(C.byref(c))
    if not sim:
        raise RuntimeError("oracle: " + str(O.orc_last_error()))
    rows = c.batch_size_per_worker * workers
    batches = [oracle_generate(rows, args.fields, args.vocab, 7, args.zipf, s) for s in range(steps)]
    times = []
    for s, (f, y) in enumerate(batches):
        loss = C.c_double()
        t0 = time.perf_counter()
        rc = O.orc_sim_step(sim, s, f, y, None, 0, C.byref(loss), None, None)
        times.append(time.perf_counter() - t0)
        assert rc == 0, O.orc_last_error()
    O.orc_sim_destroy(sim)
    return rows, times


def run_reference(args, D):
    if D.rank != 0:
        return None
    threads = os.cpu_count() or 1
    rows = min(args.cpu_rows, args.batch * D.world)
    rows -= rows % D.world
    rows_step, times = cpu_sample(args, D.world, rows, args.warmup + args.steps, threads)
    t = times[args.warmup:]
    ms = 1e3 * sum(t) / len(t)
    val = rows_step / (ms / 1e3)
    return {"metric": METRIC, "value": round(val, 1), "unit": "samples/s", "n_gpus": D.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (oracle port of the reference SyntheticGenerator)",
            "config": {"workload": WORKLOAD, "global_batch": args.batch * D.world,
                       "sample_rows_per_step": rows_step,
                       "cache_slots_per_gpu": args.cache if args.cache > 0
                       else (args.vocab + D.world - 1) // D.world},
            "impl": "reference",
            "cpu_baseline": {"value": round(val, 1), "unit": "samples/s", "cores": threads,
                             "kind": "port",
                             "sample": f"{rows_step} rows/step of the same workload, "
                                       f"{D.world} simulated workers, {args.steps} timed steps"},
            "e2e": {"value": round(val, 1), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    from paper_2104_08542_b200 import dist as sdist
    D = sdist.from_env()
    if D.world > 1 and args.gpus != D.world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {D.world}")
    if args.impl == "reference":
        out = run_reference(args, D)
        if out is not None:
            print(json.dumps(out), flush=True)
        D.close()
        return
    out = run_ours(args, D) if not args.only_mixcache else {}
    if D.world == 1 and not args.no_mixcache:
        # MixCache regimes over PCIe (north_star (2)): the paper's 0.5 GB cache at cfg2, and
        # BASELINE configs[3] (1B rows x d=32) with a hot cache of a fraction of HBM
        import torch
        sub = {}
        try:
            sub["mixcache_small"] = run_cache_line(
                "mixcache_small: cfg2 with a 2^19-slot (0.5 GB) cache", args.vocab, args.dim,
                args.fields, args.batch, args.zipf, 524288, 16_000_000, 20, 64 * 4)
        except Exception as e:  # noqa: BLE001
            sub["mixcache_small"] = {"error": str(e)[:300]}
        try:
            hbm = torch.cuda.get_device_properties(0).total_memory
            slots = int(args.cfg4_cache_frac * hbm / (12 * 32 + 32))
            sub["cfg4"] = run_cache_line(
                f"cfg4 (BASELINE configs[3]): 1B rows x d=32, F=26, b=8192, hot cache "
                f"{args.cfg4_cache_frac:.0%} of HBM", 1_000_000_000, 32, 26, 8192, 1.05, slots,
                12_000_000, 20, 64 * 40)
        except Exception as e:  # noqa: BLE001
            sub["cfg4"] = {"error": str(e)[:300]}
        out["mixcache_lines"] = sub
    if D.rank == 0:
        if D.world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            rows_step, times = cpu_sample(args, 1, args.cpu_rows, args.cpu_steps, threads)
            t = times[1:] if len(times) > 1 else times
            v = rows_step / (sum(t) / len(t))
            out["cpu_baseline"] = {"value": round(v, 1), "unit": "samples/s", "cores": threads,
                                   "kind": "port",
                                   "sample": f"{rows_step} rows/step x {len(t)} steps of the same "
                                             f"cfg2 workload, oracle port (fp64), "
                                             f"{threads} threads"}
        print(json.dumps(out), flush=True)
    D.close()


if __name__ == "__main__":
    main()
