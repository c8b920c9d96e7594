"""Multi-GPU parity (NCCL path): W ranks, one per GPU, vs the CPU oracle running
the same W-worker system. Both sync schemes — the reference's all-reduce of
the common embedding / gradients and the owner-routed all-to-all — must give
bit-exact cache slot tables, Adam step counts and ledger, and fp32-tolerance
losses and rows (same bars as tests/test_gpu_parity.py). Skipped with < 2 GPUs."""
import os
import socket
import subprocess
import sys

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


@pytest.mark.skipif(sb.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("sync,mode", [("allreduce", "sequential"), ("alltoall", "sequential"),
                                       ("allreduce", "pipelined"), ("alltoall", "pipelined")])
def test_two_rank_parity(sync, mode):
    n = min(sb.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "--sync", sync, "--mode", mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(out.stdout[-3000:], out.stderr[-3000:])
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
           os.path.join(ROOT, "tests", "mp_parity_worker.py"), "--sync", "alltoall",
           "--mode", "pipelined"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, **env})
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "parity ok" in out.stdout
