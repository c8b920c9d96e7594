"""Multi-process host logic on CPU (gloo, world_size 2): the rendezvous that
hands rank 0's NCCL id to every rank, the max-over-ranks timing reduction and
the per-rank row split the benchmark and the NCCL trainer rely on."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2104_08542_b200 import dist
    d = dist.from_env()
    nid = dist.nccl_id_for(d, lambda: bytes(range(128)))
    mx = d.max(float(rank * 10 + 1))
    sm = d.sum(1.0)
    d.barrier()
    r0, n = dist.rows_of(d.rank, 1, 8192)
    q.put((rank, nid, mx, sm, r0, n))
    d.close()


def test_gloo_rendezvous_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, nid, mx, sm, r0, n in out:
        assert nid == bytes(range(128))  # every rank holds rank 0's id
        assert mx == 11.0 and sm == 2.0
        assert (r0, n) == (rank * 8192, 8192)


def test_rows_split_matches_reference_ranges():
    from paper_2104_08542_b200 import dist
    W, b = 8, 8192
    # vsi.cpp:48-52: worker w owns rows [w*b, (w+1)*b)
    assert [dist.rows_of(w, 1, b) for w in range(W)] == [(w * b, b) for w in range(W)]
    # two lanes per process
    assert dist.rows_of(1, 2, b) == (2 * b, 2 * b)
    assert np.all(np.diff([dist.rows_of(r, 2, b)[0] for r in range(4)]) == 2 * b)
