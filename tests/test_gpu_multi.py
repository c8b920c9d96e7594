"""Multi-GPU parity (NCCL / NVLink path): W ranks, one per GPU, vs the CPU oracle running
the same W-worker system.

* test_multi_rank_parity (tests/mp_parity_worker.py): cfg2 dimensions (d = 80, F = 39,
  b = 1024 per GPU, 33.8M vocab), 10 steps, both sync schemes (the reference's all-reduce
  and the owner-routed exchange), both run modes, with and without LRU evictions, at
  W = 2 and 4; every step compared from identical state (tests/parity_util.py bars).
* test_multi_rank_overlap (tests/mp_overlap_worker.py): steps kept in flight (the
  pipelined manager of step t+1 overlapping step t's training across ranks), the
  fallback transports, final state against the oracle's multi-step trajectory.
* The owner-routed exchange runs the owner-sharded manager stage by default;
  test_multi_rank_parity_replicated_manager keeps the replicated one covered, and
  test_multi_rank_out_of_vocab (tests/mp_oov_worker.py) checks the bad-id gate across ranks
  for the sharded, replicated and all-reduce paths.
Skipped with fewer GPUs than ranks."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2104_08542_b200 as sb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("sync,mode,cache", [("allreduce", "sequential", 40000),
                                             ("alltoall", "sequential", 40000),
                                             ("allreduce", "pipelined", 40000),
                                             ("alltoall", "pipelined", 40000),
                                             ("alltoall", "pipelined", 200000)])
def test_multi_rank_parity(n, sync, mode, cache):
    if sb.device_count() < n:
        pytest.skip(f"needs >= {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "--sync", sync, "--mode", mode,
           "--cache", str(cache)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(out.stdout[-6000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "parity ok" in out.stdout


@pytest.mark.skipif(sb.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["allreduce", "alltoall"])
def test_multi_rank_overlap(sync):
    """Three steps in flight per rank: step t+1's manager stage overlaps step t's training
    (and the peers' pushes of step t+1 race this rank's step-t reduction)."""
    n = min(sb.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_overlap_worker.py"), "--sync", sync, "--mode",
           "pipelined"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "parity ok" in out.stdout


@pytest.mark.parametrize("n", [2, 4])
def test_multi_rank_parity_replicated_manager(n):
    """The owner-routed exchange with the replicated manager stage (every rank all-gathers
    the ids and runs VSI + the plan over the global batch; SFCTR_SHARD_MANAGER=0) instead
    of the owner-sharded one (the default): same per-step parity bars."""
    if sb.device_count() < n:
        pytest.skip(f"needs >= {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "--sync", "alltoall", "--mode",
           "pipelined", "--cache", "40000"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env={**os.environ, "SFCTR_SHARD_MANAGER": "0"})
    print(out.stdout[-6000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "parity ok" in out.stdout


@pytest.mark.skipif(sb.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("env", [{"SFCTR_NO_P2P": "1", "SFCTR_NCCL_IDS": "1"},
                                 {"SFCTR_NCCL_BARRIER": "1"},
                                 {"SFCTR_P2P_COPY_ENGINE": "1"}])
def test_two_rank_parity_fallback_transports(env):
    """The transports a box without full peer access (or a debugging run) falls back to:
    NCCL send/recv rows with the NCCL id all-gather, the NCCL all-reduce barrier, and
    copy-engine peer copies — same parity bars, pipelined mode."""
    n = min(sb.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_overlap_worker.py"), "--sync", "alltoall",
           "--mode", "pipelined"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, **env})
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "parity ok" in out.stdout


@pytest.mark.skipif(sb.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync,env", [("alltoall", {}), ("alltoall", {"SFCTR_SHARD_MANAGER": "0"}),
                                      ("allreduce", {})])
def test_multi_rank_out_of_vocab(sync, env):
    """An id >= vocab on one rank gates the step on every rank (sharded manager: the bad-id
    bit rides the routing barrier; replicated: the id all-gather's reduction): LogicError
    everywhere, no state moves, training continues like a run that never saw the batch."""
    n = min(sb.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_oov_worker.py"), "--sync", sync]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, **env})
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "oov ok" in out.stdout


@pytest.mark.skipif(sb.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync", ["allreduce", "alltoall"])
def test_multi_rank_deterministic(sync, tmp_path):
    """deterministic=1 across ranks: two launches of the same in-flight run give
    bit-identical final rows, moments, step counts and losses (fixed-order segment sums,
    fixed source order in the owner reduction, NCCL's fixed reduction order)."""
    n = min(sb.device_count(), 4)
    dumps = []
    for k in range(2):
        dump = str(tmp_path / f"run{k}.npz")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
               str(_port()), os.path.join(ROOT, "tests", "mp_overlap_worker.py"), "--sync", sync,
               "--mode", "pipelined", "--deterministic", "--dump", dump]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
        dumps.append(np.load(dump))
    for key in ("features", "rows", "steps", "losses"):
        assert np.array_equal(dumps[0][key], dumps[1][key]), key
