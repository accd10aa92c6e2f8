"""The copy-engine (ConCCL) path measured on one GPU: the host-staged proxy
(c3_session_set_ce_proxy) puts every peer's buffers in pinned host memory, so
this GPU's share of the plan -- its n-1 outgoing transfers (D2H) and the n-1
incoming ones (H2D) -- runs on the copy engines (a same-device copy would run
on SMs).

  * parity: after a proxy step, rank 0's result equals the oracle (all-gather,
    all-to-all, reduce-scatter incl. the local reduce) and every peer's host
    buffer holds exactly what rank 0's plan sends it;
  * no SM: with every SM held by a spinning kernel (c3_sm_hog), the proxy
    collective still completes, while the same collective as same-device
    copies waits for the hog.
"""
import ctypes as C
import time

import numpy as np
import pytest

from tests import _oracle as orc

pytestmark = pytest.mark.gpu
SEED = 20241217


@pytest.fixture(scope="module")
def c3():
    import paper_2412_14335_b200 as c3
    return c3


def _d2h(c3, ptr, nbytes):
    out = np.empty(nbytes, np.uint8)
    c3.check(c3.lib().c3_memcpy(out.ctypes.data, ptr, nbytes, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    return out


def _host(ptr, nbytes):
    return np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr)).copy()


def _proxy_bufs(c3, s, q):
    snd, rcv = C.c_void_p(), C.c_void_p()
    c3.check(c3.lib().c3_session_proxy_buffers(s.h, q, C.byref(snd), C.byref(rcv)))
    return snd.value, rcv.value


@pytest.mark.parametrize("coll", [0, 1, 2], ids=["all-gather", "all-to-all", "reduce-scatter"])
@pytest.mark.parametrize("n", [2, 8])
@pytest.mark.parametrize("strategy", ["COMM_ONLY_DMA", "CONCCL", "CONCCL_RP"])
def test_proxy_parity(c3, coll, n, strategy):
    w = c3.World(0, n, 0, loopback=True)
    chunk = (1 << 20) + 4096
    M, N, K = 512, 1024, 256
    s = c3.Session(w, M, N, K, coll, n * chunk)
    c3.check(c3.lib().c3_session_set_ce_proxy(s.h, 1))
    s.fill(SEED)
    t = s.run(getattr(c3, strategy))
    assert t.total_ms > 0 and t.comm_ctas == 0
    p = s.pointers(0)
    if coll == 0:
        got = _d2h(c3, p.recv, n * chunk)
        assert np.array_equal(got, orc.expected_allgather(n, chunk, SEED, 2))
        mine = got[:chunk]
        for q in range(1, n):
            assert np.array_equal(_host(_proxy_bufs(c3, s, q)[1], chunk), mine), q
    elif coll == 1:
        got = _d2h(c3, p.recv, n * chunk)
        assert np.array_equal(got, orc.expected_alltoall(n, 0, chunk, SEED, 4))
        send = _d2h(c3, p.send, n * chunk)
        for q in range(1, n):
            assert np.array_equal(_host(_proxy_bufs(c3, s, q)[1], chunk), send[q * chunk:(q + 1) * chunk]), q
    else:
        count = chunk // 2
        host_in = [orc.bf16(n * count, SEED, g, 3) for g in range(n)]
        got = _d2h(c3, p.recv, chunk).view(np.uint16)
        assert np.array_equal(got, orc.reduce_scatter(host_in, 0, count))
        for q in range(1, n):  # rank 0's slot q went to peer q
            assert np.array_equal(_host(_proxy_bufs(c3, s, q)[1], chunk).view(np.uint16),
                                  host_in[0][q * count:(q + 1) * count]), q
    s.close()
    w.close()


def test_copy_engines_need_no_sm(c3):
    """Every SM held by a spinning kernel: the proxy all-gather (copy engines)
    completes long before the hog ends; the same plan as same-device copies
    (SM copy kernels) cannot start until it ends."""
    import torch
    n, chunk = 8, 16 << 20
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, 256, 256, 256, c3.ALL_GATHER, n * chunk)
    c3.check(c3.lib().c3_session_set_ce_proxy(s.h, 1))
    s.fill(SEED)  # also fills the proxy peers' host buffers
    s.run(c3.COMM_ONLY_DMA)  # warm: streams, batches
    hog_ms = 400.0
    side = torch.cuda.Stream()
    done = torch.cuda.Event()
    torch.cuda.synchronize()
    c3.check(c3.lib().c3_sm_hog(w.h, hog_ms, C.c_void_p(side.cuda_stream)))
    done.record(side)
    time.sleep(0.02)  # the hog is resident on every SM
    t0 = time.perf_counter()
    t = s.run(c3.COMM_ONLY_DMA)
    ce_wall = (time.perf_counter() - t0) * 1e3
    hog_running = not done.query()
    torch.cuda.synchronize()
    assert hog_running, "the hog ended before the copy-engine collective"
    assert ce_wall < hog_ms / 2, ce_wall
    assert np.array_equal(_d2h(c3, s.pointers(0).recv, n * chunk), orc.expected_allgather(n, chunk, SEED, 2))
    # control: the same collective as same-device copies waits for the SMs
    c3.check(c3.lib().c3_session_set_ce_proxy(s.h, 0))
    s.run(c3.COMM_ONLY_DMA)
    torch.cuda.synchronize()
    c3.check(c3.lib().c3_sm_hog(w.h, hog_ms, C.c_void_p(side.cuda_stream)))
    time.sleep(0.02)
    t0 = time.perf_counter()
    s.run(c3.COMM_ONLY_DMA)
    sm_wall = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    assert sm_wall > hog_ms / 2, sm_wall
    s.close()
    w.close()
