"""Process-group plumbing for one-process-per-GPU runs.

torch.distributed (gloo, host side only) is used for the rendezvous: it
broadcasts rank 0's ncclUniqueId so the library can build its own NCCL
communicator (the data path never goes through torch), and it provides the
barrier and the max-over-ranks reduction the benchmark timing needs.
"""
import os
from dataclasses import dataclass

import numpy as np


@dataclass
class Dist:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    initialized: bool = False

    def barrier(self):
        if self.initialized:
            import torch.distributed as td
            td.barrier()

    def max(self, x: float) -> float:
        if not self.initialized:
            return float(x)
        import torch
        import torch.distributed as td
        t = torch.tensor([float(x)], dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.initialized:
            return float(x)
        import torch
        import torch.distributed as td
        t = torch.tensor([float(x)], dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.SUM)
        return float(t.item())

    def broadcast_bytes(self, data: bytes, src: int = 0, size: int = 128) -> bytes:
        if not self.initialized:
            return data
        import torch
        import torch.distributed as td
        buf = torch.zeros(size, dtype=torch.uint8)
        if self.rank == src:
            buf[:len(data)] = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy())
        td.broadcast(buf, src=src)
        return bytes(buf.numpy().tobytes())

    def close(self):
        if self.initialized:
            import torch.distributed as td
            td.destroy_process_group()
            self.initialized = False


def from_env() -> Dist:
    """Reads RANK/WORLD_SIZE/LOCAL_RANK (torchrun) and joins a gloo group when world > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    d = Dist(rank=rank, world=world, local_rank=local)
    if world > 1:
        import torch.distributed as td
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        td.init_process_group("gloo", rank=rank, world_size=world)
        d.initialized = True
    return d


def nccl_id_for(d: Dist, make_id) -> bytes:
    """Rank 0 creates the ncclUniqueId (make_id()), everyone receives it."""
    if d.world == 1:
        return None
    data = make_id() if d.rank == 0 else b"\0" * 128
    return d.broadcast_bytes(data, src=0, size=128)


def rows_of(rank: int, lanes: int, batch_per_worker: int):
    """This process's contiguous row range of the global batch (vsi.cpp:48-52)."""
    r0 = rank * lanes * batch_per_worker
    return r0, lanes * batch_per_worker
