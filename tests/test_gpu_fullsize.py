"""GPU parity at BASELINE.json's full collective sizes: the
896 MiB all-gather / all-to-all / reduce-scatter of cfg2 / cfg3 across 8
ranks (loopback world, every virtual rank's share), checked against the CPU
oracle with size-independent properties:
  * all-gather: rank 0's whole receive buffer bit-equal to the oracle's
    expected buffer, and every other rank's buffer bit-equal to rank 0's;
  * all-to-all: every (destination, source) slot's words at sampled offsets
    equal the oracle's label words of the source rank's send slot;
  * reduce-scatter: sampled output elements bit-equal to the fixed-order fp32
    sum of the oracle's bf16 inputs with one RNE rounding.
The all-gather runs as the co-resident C3 step beside the cfg2 GEMM, whose
output is checked at sampled entries within the stated bf16 tolerance."""
import ctypes as C

import numpy as np
import pytest

from tests import _oracle as orc

pytestmark = pytest.mark.gpu

SEED = 20241217
N = 8
PAYLOAD = 896 << 20


@pytest.fixture(scope="module")
def c3():
    import paper_2412_14335_b200 as c3
    return c3


def _d2h(c3, ptr, nbytes):
    out = np.empty(nbytes, np.uint8)
    c3.check(c3.lib().c3_memcpy(out.ctypes.data, ptr, nbytes, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    return out


def _dev_equal(c3, a_ptr, b_ptr, nbytes):
    """Bit equality of two device buffers, compared on the device through torch
    views of the raw pointers (no host copy)."""
    import torch
    return bool(torch.equal(_view(a_ptr, nbytes), _view(b_ptr, nbytes)))


def _view(ptr, nbytes):
    import torch

    class _A:  # __cuda_array_interface__ wrapper
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False),
                                             "version": 3}
    return torch.as_tensor(_A(ptr, nbytes), device="cuda")


@pytest.mark.parametrize("M,Nn,K,payload,pace", [(8192, 28672, 8192, PAYLOAD, 0.0),
                                                   (8192, 53248, 16384, 1664 << 20, 250.0)],
                         ids=["cfg2", "cfg4-paced"])
def test_allgather_full_size_coresident_with_gemm(c3, M, Nn, K, payload, pace):
    """cfg2 (896 MiB) and cfg4 (LLaMA-405B, 1664 MiB, the collective paced
    below the link rate) all-gathers, co-resident beside their GEMMs."""
    w = c3.World(0, N, 0, loopback=True)
    s = c3.Session(w, M, Nn, K, c3.ALL_GATHER, payload)
    s.fill(SEED)
    a = s.default_alloc(c3.C3_BASE)
    a.cus_gemm, a.cus_comm, a.comm_pace_gbps = w.info.sm_count, 24, pace
    s.run(c3.C3_BASE, a, all_ranks=True)
    chunk = payload // N
    got0 = _d2h(c3, s.pointers(0).recv, payload)
    assert np.array_equal(got0, orc.expected_allgather(N, chunk, SEED, 2))
    for v in range(1, N):
        assert _dev_equal(c3, s.pointers(v).recv, s.pointers(0).recv, payload), f"rank {v}"
    # the GEMM that ran beside it: sampled entries against the fp64 definition
    rng = np.random.default_rng(7)
    rows = rng.integers(0, M, 2048)
    cols = rng.integers(0, Nn, 2048)
    A, B = orc.bf16(M * K, SEED, 0, 0), orc.bf16(Nn * K, SEED, 0, 1)
    ref, mag = orc.gemm_samples(A, B, M, Nn, K, rows, cols)
    cbits = np.empty(M * Nn, np.uint16)
    c3.check(c3.lib().c3_memcpy(cbits.ctypes.data, s.pointers(0).c, M * Nn * 2, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    orc.check_bf16_gemm(cbits[rows * Nn + cols], ref, mag)
    s.close()
    w.close()


@pytest.mark.parametrize("strategy", ["conccl", "c3_fused"])
def test_allgather_896mib_copy_engine_plan_and_fused(c3, strategy):
    """The same 896 MiB all-gather through the reference's transfer plan
    (56 batched copies) and through the fused pair GEMM's copy warp."""
    w = c3.World(0, N, 0, loopback=True)
    s = c3.Session(w, 8192, 8192, 1024, c3.ALL_GATHER, PAYLOAD)
    s.fill(SEED)
    st = c3.CONCCL if strategy == "conccl" else c3.FUSED
    s.run(st, s.default_alloc(st), all_ranks=True)
    chunk = PAYLOAD // N
    got0 = _d2h(c3, s.pointers(0).recv, PAYLOAD)
    assert np.array_equal(got0, orc.expected_allgather(N, chunk, SEED, 2))
    for v in range(1, N):
        assert _dev_equal(c3, s.pointers(v).recv, s.pointers(0).recv, PAYLOAD), f"rank {v}"
    s.close()
    w.close()


def test_alltoall_896mib_sampled_slots(c3):
    w = c3.World(0, N, 0, loopback=True)
    s = c3.Session(w, 256, 256, 256, c3.ALL_TO_ALL, PAYLOAD)
    s.fill(SEED)
    a = s.default_alloc(c3.COMM_ONLY_CU)
    a.cus_comm = 148
    s.run(c3.COMM_ONLY_CU, a, all_ranks=True)
    slot = PAYLOAD // N
    rng = np.random.default_rng(11)
    words = np.unique(rng.integers(0, slot // 8, 512))
    L = orc.lib()
    for v in range(N):  # destination rank v, slot q holds rank q's send slot v
        recv = _d2h(c3, s.pointers(v).recv, PAYLOAD).view(np.uint64)
        for q in range(N):
            want = np.array([L.c3o_label_word(SEED, q, 4, int(v * slot // 8 + wd)) for wd in words],
                            np.uint64)
            assert np.array_equal(recv[q * slot // 8 + words], want), (v, q)
    s.close()
    w.close()


@pytest.mark.parametrize("mode", ["sm_pull", "copy_engine", "conccl_cfg3"])
def test_reduce_scatter_896mib_sampled_elements(c3, mode):
    """cfg3's 896 MiB reduce-scatter: the SM pull, the copy-engine plan
    (plan_reduce_scatter transpose into staging + local reduce), and the whole
    conccl C3 step beside the cfg3 weight-grad GEMM."""
    w = c3.World(0, N, 0, loopback=True)
    mnk = (8192, 28672, 8192) if mode == "conccl_cfg3" else (256, 256, 256)
    s = c3.Session(w, *mnk, c3.REDUCE_SCATTER, PAYLOAD)
    s.fill(SEED)
    if mode == "sm_pull":
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = 148
        s.run(c3.COMM_ONLY_CU, a, all_ranks=True)
    elif mode == "copy_engine":
        s.run(c3.COMM_ONLY_DMA, s.default_alloc(c3.COMM_ONLY_DMA), all_ranks=True)
    else:
        t = s.run(c3.CONCCL, s.default_alloc(c3.CONCCL), all_ranks=True)
        assert t.gemm_ctas == 148 and t.comm_ctas == 0
    count = PAYLOAD // N // 2
    rng = np.random.default_rng(13)
    idx = np.unique(rng.integers(0, count, 256))
    L = orc.lib()
    for v in (0, 3, 7):
        out = _d2h(c3, s.pointers(v).recv, count * 2).view(np.uint16)
        for i in idx:
            acc = np.float32(0.0)
            for g in range(N):  # fixed rank order, fp32, one RNE rounding
                acc = np.float32(acc + orc.bf16_to_f32(np.array([L.c3o_bf16_value(SEED, g, 3, int(v * count + i))],
                                                                  np.uint16))[0])
            assert out[i] == L.c3o_f32_to_bf16_rne(C.c_float(acc)), (v, i)
    s.close()
    w.close()
