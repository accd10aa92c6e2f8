"""Multi-process host logic on CPU (gloo, world_size 2): the handle exchange
that maps peer buffers, barriers, and max-over-ranks timing used by bench.py
and the multi-GPU C3 sessions."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2412_14335_b200 import _capi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    from paper_2412_14335_b200.dist import Dist, join_handles
    d = Dist()
    blob = bytes([rank + 1]) * _capi.SESSION_HANDLE_BYTES
    blobs = d.allgather_bytes(blob)
    joined = join_handles(blobs, _capi.SESSION_HANDLE_BYTES)
    d.barrier()
    m = d.max_list([float(rank), 10.0 - rank, 3.5])
    q.put((rank, [b[0] for b in blobs], len(joined), m))
    d.close()


def test_two_rank_exchange_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (order, n, m)) for r, order, n, m in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        order, n, m = out[r]
        assert order == [1, 2]  # rank order
        assert n == world * _capi.SESSION_HANDLE_BYTES
        assert m == [1.0, 10.0, 3.5]


def test_join_handles_rejects_bad_blob():
    from paper_2412_14335_b200.dist import join_handles
    with pytest.raises(ValueError):
        join_handles([b"x" * 3], _capi.SESSION_HANDLE_BYTES)
