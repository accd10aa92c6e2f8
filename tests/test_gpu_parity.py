"""GPU parity: the sm_100a kernels, called through the C ABI (libc3cuda.so),
against the CPU oracle (oracle/c3oracle.c) on identical seeded inputs.

Bars (BASELINE.json north_star):
  * data movement (all-gather push, copy-engine plans, reduce-scatter copy
    phase): bit-exact;
  * reduce-scatter sums: bit-exact (same fp32 rank order 0..n-1, one bf16 RNE
    rounding) — the stated fallback tolerance of 1 bf16 ulp is never needed;
  * GEMM (bf16 in, fp32 accumulate, bf16 out) per element:
        |C - C_ref| <= 2^-8 |C_ref| + K 2^-23 sum_k |A_ik B_jk|
    plus a statistical bar: RMS(C - C_ref) / RMS(C_ref) <= 2^-8.
"""
import ctypes as C

import numpy as np
import pytest

from tests import _oracle as orc

pytestmark = pytest.mark.gpu

SEED = 20241217


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    return torch


@pytest.fixture(scope="module")
def c3():
    import paper_2412_14335_b200 as c3
    return c3


def dev_bytes(torch, nbytes):
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")


def to_host_u8(t, nbytes):
    return t[:nbytes].cpu().numpy()


def gemm_check(c_bits, A, B, M, N, K, rows, cols):
    """The stated bf16 tolerance (tests/_oracle.py check_bf16_gemm) on the
    sampled entries, and the relative RMS error."""
    ref, mag = orc.gemm_samples(A, B, M, N, K, rows, cols)
    err, _ = orc.check_bf16_gemm(c_bits[rows * N + cols], ref, mag)
    rel_rms = np.sqrt(np.mean(err ** 2)) / max(np.sqrt(np.mean(ref ** 2)), 1e-30)
    assert rel_rms <= 2.0 ** -8, rel_rms
    return rel_rms


def test_fill_matches_oracle(torch_mod, c3):
    torch = torch_mod
    w = c3.World()
    for count in (1, 7, 4096, 1 << 20):
        t = torch.empty(count, dtype=torch.int16, device="cuda")
        c3.check(c3.lib().c3_fill_bf16(t.data_ptr(), count, SEED, 3, 1, None))
        got = t.cpu().numpy().view(np.uint16)
        assert np.array_equal(got, orc.bf16(count, SEED, 3, 1))
    for nbytes in (1, 13, 4096, 1 << 20):
        t = dev_bytes(torch, nbytes)
        c3.check(c3.lib().c3_fill_labels(t.data_ptr(), nbytes, SEED, 5, 2, None))
        assert np.array_equal(to_host_u8(t, nbytes), orc.labels(nbytes, SEED, 5, 2))
    w.close()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (384, 768, 320),
                                   (100, 264, 72), (64, 1024, 512), (1000, 2056, 136)])
def test_gemm_small_full(torch_mod, c3, M, N, K):
    torch = torch_mod
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    Cm = torch.zeros(M * N, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K)
    torch.cuda.synchronize()
    Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
    rows, cols = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    gemm_check(Cm.cpu().numpy().view(np.uint16), Ah, Bh, M, N, K, rows.ravel(), cols.ravel())
    w.close()


@pytest.mark.parametrize("kernel", ["pair", "pair512", "wide", "narrow"])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (512, 768, 1024), (1000, 2056, 136),
                                   (300, 520, 200), (768, 1536, 512), (512, 1024, 320), (512, 1024, 448)])
def test_gemm_kernel_variants_full(torch_mod, c3, monkeypatch, kernel, M, N, K):
    """Each GEMM kernel variant (CTA-pair 256x256 and 256x512, single-CTA
    128x256 and 128x128 tiles), forced, on full outputs including ragged M/N/K
    tails."""
    monkeypatch.setenv("C3_GEMM_KERNEL", kernel)
    torch = torch_mod
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    Cm = torch.zeros(M * N, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    for cap in (0, 6):
        Cm.zero_()
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, cap)
        torch.cuda.synchronize()
        Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
        rows, cols = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
        gemm_check(Cm.cpu().numpy().view(np.uint16), Ah, Bh, M, N, K, rows.ravel(), cols.ravel())
    w.close()


@pytest.mark.parametrize("M,N,K,kernel", [(256, 4096, 2048, None), (512, 2048, 1024, "narrow"),
                                          (1024, 8192, 1024, "wide"), (128, 53248, 512, None)])
def test_gemm_stream_k_tail(torch_mod, c3, monkeypatch, M, N, K, kernel):
    """Compute-bound single-CTA GEMMs whose last wave on the full GPU is partly
    empty (64 128x128 tiles; 64 forced-narrow; 256 forced-wide 128x256 tiles):
    that wave's k-blocks are spread over one segment per SM, a tile cut into
    up to four pieces finished by the piece that arrives last (fp32 partials
    summed in piece order, one bf16 rounding). The memory-bound M = 128 shape
    keeps whole tiles. Every output checked; bit-identical across runs and
    across CTA caps (the decomposition depends on the SM count only)."""
    if kernel:
        monkeypatch.setenv("C3_GEMM_KERNEL", kernel)
    torch = torch_mod
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
    rows, cols = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    outs = []
    for cap in (0, 0, 140, 37):
        Cm = torch.zeros(M * N, dtype=torch.int16, device="cuda")
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, cap)
        outs.append(Cm)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    gemm_check(outs[0].cpu().numpy().view(np.uint16), Ah, Bh, M, N, K, rows.ravel(), cols.ravel())
    w.close()


@pytest.mark.parametrize("max_ctas", [1, 7, 148])
def test_gemm_cta_cap_same_result(torch_mod, c3, max_ctas):
    """The CTA cap (SM allocation) must not change a single output bit."""
    torch = torch_mod
    w = c3.World()
    M, N, K = 512, 1024, 512
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    C1 = torch.zeros(M * N, dtype=torch.int16, device="cuda")
    C2 = torch.zeros(M * N, dtype=torch.int16, device="cuda")
    w.gemm(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, 0)
    w.gemm(A.data_ptr(), B.data_ptr(), C2.data_ptr(), M, N, K, max_ctas)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    w.close()


@pytest.mark.parametrize("M,N,K", [(8192, 28672, 8192), (128, 53248, 16384), (64, 53248, 16384)])
def test_gemm_llama_shapes_sampled(torch_mod, c3, M, N, K):
    """BASELINE configs[1]/[3] shapes: sampled entries + full tile-boundary rows/cols."""
    torch = torch_mod
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    Cm = torch.zeros(M * N, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K)
    torch.cuda.synchronize()
    Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
    rng = np.random.default_rng(7)
    rows = list(rng.integers(0, M, 4096))
    cols = list(rng.integers(0, N, 4096))
    for r in (0, 127, 128, M - 1):  # tile-boundary rows, sampled columns
        if r < M:
            rows += [r] * 256
            cols += list(rng.integers(0, N, 256))
    for c in (0, 255, 256, N - 1):
        rows += list(rng.integers(0, M, 128))
        cols += [c] * 128
    Ch = Cm.cpu().numpy().view(np.uint16)
    gemm_check(Ch, Ah, Bh, M, N, K, np.array(rows), np.array(cols))
    w.close()


def _ag_buffers(torch, n, chunk):
    bufs = [dev_bytes(torch, n * chunk) for _ in range(n)]
    for g, b in enumerate(bufs):
        b.zero_()
        own = orc.labels(chunk, SEED, g, 2)
        b[g * chunk:(g + 1) * chunk] = torch.from_numpy(own).cuda()
    return bufs


@pytest.mark.parametrize("n", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("chunk", [1, 3, 16, 4096, 1000 * 16 + 7, 8 << 20])
def test_allgather_p2p_bit_exact(torch_mod, c3, n, chunk):
    torch = torch_mod
    w = c3.World(0, n, 0, loopback=True)
    bufs = _ag_buffers(torch, n, chunk)
    ptrs = [b.data_ptr() for b in bufs]
    for g in range(n):  # every virtual rank pushes its chunk (in place)
        w.allgather_p2p(g, ptrs[g] + g * chunk, ptrs, chunk, n_ctas=16)
    torch.cuda.synchronize()
    want = orc.expected_allgather(n, chunk, SEED, 2)
    for g in range(n):
        assert np.array_equal(to_host_u8(bufs[g], n * chunk), want), f"rank {g}"
    w.close()


@pytest.mark.parametrize("n", [2, 3, 4, 7, 8])
@pytest.mark.parametrize("chunk", [1, 3, 4096, 8 << 20])
def test_allgather_ce_plan_bit_exact(torch_mod, c3, n, chunk):
    """Copy-engine executor runs the product's validated plan_all_gather."""
    torch = torch_mod
    w = c3.World(0, n, 0, loopback=True)
    plan, cnt = c3.plan_transfers(c3.ALL_GATHER, n, chunk, max(1, w.info.async_engines))
    assert cnt == n * (n - 1)
    bufs = _ag_buffers(torch, n, chunk)
    dst = [b.data_ptr() for b in bufs]
    src = [b.data_ptr() + g * chunk for g, b in enumerate(bufs)]
    w.ce_execute(plan, cnt, src, dst)
    torch.cuda.synchronize()
    want = orc.expected_allgather(n, chunk, SEED, 2)
    for g in range(n):
        assert np.array_equal(to_host_u8(bufs[g], n * chunk), want), f"rank {g}"
    w.close()


@pytest.mark.parametrize("n", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("count", [1, 5, 8, 4096, 123456, 1 << 22])
def test_reduce_scatter_p2p_bit_exact(torch_mod, c3, n, count):
    torch = torch_mod
    w = c3.World(0, n, 0, loopback=True)
    host_in = [orc.bf16(n * count, SEED, g, 3) for g in range(n)]
    dev_in = [torch.from_numpy(h.view(np.int16)).cuda() for h in host_in]
    outs = [torch.zeros(max(count, 8), dtype=torch.int16, device="cuda") for _ in range(n)]
    for r in range(n):
        w.reduce_scatter_p2p(r, [t.data_ptr() for t in dev_in], outs[r].data_ptr(), count, 32)
    torch.cuda.synchronize()
    for r in range(n):
        want = orc.reduce_scatter(host_in, r, count)
        got = outs[r][:count].cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want), f"rank {r}: {np.count_nonzero(got != want)} differ"
    w.close()


def test_ce_execute_rejects_out_of_range(c3):
    w = c3.World(0, 2, 0, loopback=True)
    bad = (c3._capi.Transfer * 1)()
    bad[0] = c3._capi.Transfer(0, 5, 0, 0, 16, 0, 0)
    with pytest.raises(c3.C3Error) as e:
        w.ce_execute(bad, 1, [0, 0], [0, 0])
    assert e.value.code == 4
    w.close()


SESSION_STRATS = list(range(7)) + [100, 101, 102]


@pytest.mark.parametrize("collective", [0, 2])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_session_all_strategies_loopback(torch_mod, c3, collective, n):
    """Every strategy executes the full C3 pair; the collective's output is
    bit-exact for every virtual rank and the GEMM is within tolerance."""
    torch = torch_mod
    w = c3.World(0, n, 0, loopback=True)
    M, N, K = 256, 512, 256
    payload = n * (64 << 10)
    s = c3.Session(w, M, N, K, collective, payload)
    chunk = payload // n
    Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
    for strat in SESSION_STRATS:
        s.fill(SEED)
        t = s.run(strat, all_ranks=True)
        torch.cuda.synchronize()
        assert t.total_ms > 0
        if strat in (c3.C3_RP, c3.C3_SP_RP):
            # the SM partition really is a green-context split (no CTA-cap fallback)
            assert t.partition == 1 and t.comm_ctas % w.info.sm_grain == 0, (t.partition, t.comm_ctas)
        if strat != c3.COMM_ONLY_CU and strat != c3.COMM_ONLY_DMA:
            p = s.pointers(0)
            Cbits = np.empty(M * N, np.uint16)
            c3.check(c3.lib().c3_memcpy(Cbits.ctypes.data, p.c, M * N * 2, 2, None))
            c3.check(c3.lib().c3_stream_sync(None))
            rng = np.random.default_rng(strat)
            gemm_check(Cbits, Ah, Bh, M, N, K, rng.integers(0, M, 512), rng.integers(0, N, 512))
        if strat == c3.GEMM_ONLY:
            continue
        if collective == 0:
            want = orc.expected_allgather(n, chunk, SEED, 2)
            for v in range(n):
                p = s.pointers(v)
                got = np.empty(payload, np.uint8)
                c3.check(c3.lib().c3_memcpy(got.ctypes.data, p.recv, payload, 2, None))
                c3.check(c3.lib().c3_stream_sync(None))
                assert np.array_equal(got, want), f"strategy {strat} rank {v}"
        else:
            count = chunk // 2
            host_in = [orc.bf16(n * count, SEED, g, 3) for g in range(n)]
            for v in range(n):
                p = s.pointers(v)
                got = np.empty(count, np.uint16)
                c3.check(c3.lib().c3_memcpy(got.ctypes.data, p.recv, count * 2, 2, None))
                c3.check(c3.lib().c3_stream_sync(None))
                assert np.array_equal(got, orc.reduce_scatter(host_in, v, count)), \
                    f"strategy {strat} rank {v}"
    s.close()
    w.close()


@pytest.mark.parametrize("n", [2, 3, 4, 7, 8])
@pytest.mark.parametrize("slot", [1, 5, 4096, 1 << 20])
def test_alltoall_p2p_and_ce_bit_exact(torch_mod, c3, n, slot):
    """All-to-all (reference plan_all_to_all semantics, §8(f) F1): P2P push and
    the copy-engine executor running the product's validated plan."""
    torch = torch_mod
    w = c3.World(0, n, 0, loopback=True)
    send = [torch.from_numpy(orc.labels(n * slot, SEED, g, 4)).cuda() for g in range(n)]
    for path in ("p2p", "ce"):
        recv = [dev_bytes(torch, n * slot) for _ in range(n)]
        for r in recv:
            r.zero_()
        rptr = [r.data_ptr() for r in recv]
        if path == "p2p":
            for g in range(n):
                w.alltoall_p2p(g, send[g].data_ptr(), rptr, slot, n_ctas=8)
        else:
            plan, cnt = c3.plan_transfers(c3.ALL_TO_ALL, n, slot, max(1, w.info.async_engines))
            w.ce_execute(plan, cnt, [s.data_ptr() for s in send], rptr)
            for g in range(n):  # the self slot is local, not part of the plan
                recv[g][g * slot:(g + 1) * slot] = send[g][g * slot:(g + 1) * slot]
        torch.cuda.synchronize()
        for r in range(n):
            assert np.array_equal(to_host_u8(recv[r], n * slot),
                                  orc.expected_alltoall(n, r, slot, SEED, 4)), f"{path} rank {r}"
    w.close()


@pytest.mark.parametrize("n", [2, 8])
def test_session_alltoall_all_strategies(torch_mod, c3, n):
    w = c3.World(0, n, 0, loopback=True)
    payload = n * (32 << 10)
    s = c3.Session(w, 256, 256, 128, c3.ALL_TO_ALL, payload)
    for strat in SESSION_STRATS:
        s.fill(SEED)
        s.run(strat, all_ranks=True)
        if strat == c3.GEMM_ONLY:
            continue
        for v in range(n):
            got = np.empty(payload, np.uint8)
            c3.check(c3.lib().c3_memcpy(got.ctypes.data, s.pointers(v).recv, payload, 2, None))
            c3.check(c3.lib().c3_stream_sync(None))
            assert np.array_equal(got, orc.expected_alltoall(n, v, payload // n, SEED, 4)), \
                f"strategy {strat} rank {v}"
    s.close()
    w.close()


@pytest.mark.parametrize("collective", [0, 1], ids=["all-gather", "all-to-all"])
@pytest.mark.parametrize("n", [2, 8])
@pytest.mark.parametrize("pace,piece", [(0.0, 4096), (0.8, 16384), (0.0, 0), (0.0, 2048), (0.5, 1040)])
@pytest.mark.parametrize("kernel", ["pair", "pair512"])
def test_fused_c3_bit_exact(torch_mod, c3, monkeypatch, collective, n, pace, piece, kernel):
    """C3_FUSED: the collective moved inside the CTA-pair GEMM by its copy warp
    (TMA bulk copies). Every virtual rank's output bit-exact; GEMM in tolerance."""
    monkeypatch.setenv("C3_GEMM_KERNEL", kernel)
    w = c3.World(0, n, 0, loopback=True)
    M, N, K = 512, 1024, 512
    payload = n * ((3 << 16) + 48)  # slots not a multiple of the 16 KiB piece
    s = c3.Session(w, M, N, K, collective, payload)
    s.set_fused_pace(pace, piece)
    s.fill(SEED)
    t = s.run(c3.FUSED, all_ranks=True)
    assert t.launches == 1
    chunk = payload // n
    for v in range(n):
        got = np.empty(payload, np.uint8)
        c3.check(c3.lib().c3_memcpy(got.ctypes.data, s.pointers(v).recv, payload, 2, None))
        c3.check(c3.lib().c3_stream_sync(None))
        want = (orc.expected_allgather(n, chunk, SEED, 2) if collective == 0
                else orc.expected_alltoall(n, v, chunk, SEED, 4))
        assert np.array_equal(got, want), f"rank {v}"
    Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
    Cbits = np.empty(M * N, np.uint16)
    c3.check(c3.lib().c3_memcpy(Cbits.ctypes.data, s.pointers(0).c, M * N * 2, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    rows, cols = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    gemm_check(Cbits, Ah, Bh, M, N, K, rows.ravel(), cols.ravel())
    s.close()
    w.close()


def test_fused_rejects_reduce_scatter(c3):
    w = c3.World(0, 2, 0, loopback=True)
    s = c3.Session(w, 2048, 2048, 256, c3.REDUCE_SCATTER, 2 << 20)
    with pytest.raises(c3.C3Error) as e:
        s.run(c3.FUSED)
    assert e.value.code == 102
    s.close()
    w.close()


def test_green_partition_rejects_unrealisable_split(c3):
    """c3_rp with an SM split the green-context grain cannot realise is an
    error, not a silent rounding (the driver grants multiples of the grain)."""
    w = c3.World(0, 2, 0, loopback=True)
    assert w.info.green_ctx == 1 and w.info.sm_grain >= 1
    s = c3.Session(w, 256, 256, 64, 0, 2 * 4096)
    a = s.default_alloc(c3.C3_RP)
    assert a.cus_comm % w.info.sm_grain == 0
    if w.info.sm_grain > 1:
        a.cus_comm = w.info.sm_grain + 1
        a.cus_gemm = w.info.sm_count - a.cus_comm
        with pytest.raises(c3.C3Error) as e:
            s.run(c3.C3_RP, a)
        assert e.value.code == 4
    s.close()
    w.close()


@pytest.mark.parametrize("collective", [0, 1, 2])
def test_degenerate_worlds(c3, collective):
    """A 1-rank collective is an empty plan (conccl.hpp:30-32) and a zero-byte
    payload moves nothing; every strategy still runs and the GEMM still runs."""
    w1 = c3.World(0, 1, 0, loopback=False)
    s = c3.Session(w1, 256, 256, 64, collective, 4096)
    for strat in list(range(7)) + [100, 101, 102]:
        t = s.run(strat)
        assert t.total_ms >= 0
    s.close()
    w1.close()
    w = c3.World(0, 4, 0, loopback=True)
    s = c3.Session(w, 256, 256, 64, collective, 0)
    for strat in (c3.SERIAL, c3.C3_SP, c3.CONCCL, c3.COMM_ONLY_CU, c3.COMM_ONLY_DMA):
        s.run(strat, all_ranks=True)
    s.close()
    w.close()


@pytest.mark.parametrize("collective", [0, 1, 2], ids=["all-gather", "all-to-all", "reduce-scatter"])
@pytest.mark.parametrize("kernel", ["pair", "pair512"])
def test_link_rate_emulation_exact_and_paced(torch_mod, c3, monkeypatch, collective, kernel):
    """c3_session_set_link_rate: the paced SM collective (and the paced fused
    copies) deliver bit-identical data, and the isolated collective takes the
    link time (n-1)/n * P / rate, independent of the CTA count."""
    monkeypatch.setenv("C3_GEMM_KERNEL", kernel)  # the fused path needs a CTA-pair GEMM
    n, rate = 8, 200.0  # GB/s: slow enough that pacing, not HBM, sets the time
    payload = n * (8 << 20)  # enough 32 KiB iterations per CTA for the pace to be smooth
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, 512, 1024, 512, collective, payload)
    chunk = payload // n
    target_ms = (n - 1) / n * payload / (rate * 1e9) * 1e3
    s.set_link_rate(rate)
    for ctas in (16, 64):
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = ctas
        ms = sorted(_comm_ms(s.run(c3.COMM_ONLY_CU, a)) for _ in range(3))[1]
        assert 0.95 * target_ms <= ms <= 1.25 * target_ms, (ctas, ms, target_ms)
    strats = [c3.C3_SP] + ([c3.FUSED] if collective != 2 else [])
    for strat in strats:
        s.fill(SEED)
        t = s.run(strat, all_ranks=True)
        assert t.total_ms > 0
        for v in range(n):
            p = s.pointers(v)
            if collective == 2:
                count = chunk // 2
                host_in = [orc.bf16(n * count, SEED, g, 3) for g in range(n)]
                got = np.empty(count, np.uint16)
                c3.check(c3.lib().c3_memcpy(got.ctypes.data, p.recv, count * 2, 2, None))
                c3.check(c3.lib().c3_stream_sync(None))
                assert np.array_equal(got, orc.reduce_scatter(host_in, v, count))
                continue
            got = np.empty(payload, np.uint8)
            c3.check(c3.lib().c3_memcpy(got.ctypes.data, p.recv, payload, 2, None))
            c3.check(c3.lib().c3_stream_sync(None))
            want = (orc.expected_allgather(n, chunk, SEED, 2) if collective == 0
                    else orc.expected_alltoall(n, v, chunk, SEED, 4))
            assert np.array_equal(got, want), f"strategy {strat} rank {v}"
    s.set_link_rate(0.0)
    a = s.default_alloc(c3.COMM_ONLY_CU)
    a.cus_comm = 32
    fast = min(_comm_ms(s.run(c3.COMM_ONLY_CU, a)) for _ in range(3))
    assert fast < 0.5 * target_ms  # unpaced is much faster: the pacing is what set the time
    with pytest.raises(c3.C3Error):
        s.set_link_rate(-1.0)
    s.close()
    w.close()


def _comm_ms(t):
    return t.comm_end_ms - t.comm_start_ms


@pytest.mark.parametrize("collective", [0, 2], ids=["all-gather", "reduce-scatter"])
def test_comm_pace_in_concurrent_runs(torch_mod, c3, collective):
    """c3_alloc.comm_pace_gbps: a concurrent run paces its collective to the
    given rate (bit-identical data, the collective stretched to the paced
    time); the isolated collective with the same allocation ignores it."""
    n, rate = 8, 100.0
    payload = n * (4 << 20)
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, 512, 1024, 512, collective, payload)
    target_ms = (n - 1) / n * payload / (rate * 1e9) * 1e3
    a = s.default_alloc(c3.C3_BASE)
    a.cus_gemm, a.cus_comm, a.comm_pace_gbps = w.info.sm_count, 16, rate
    t = s.run(c3.C3_BASE, a)  # this rank's share: (n-1)/n * payload of peer traffic
    comm_ms = t.comm_end_ms - t.comm_start_ms
    assert 0.95 * target_ms <= comm_ms <= 1.5 * target_ms, (comm_ms, target_ms)
    s.fill(SEED)
    s.run(c3.C3_BASE, a, all_ranks=True)  # every virtual rank's share, for the data check
    chunk = payload // n
    got = np.empty(payload if collective == 0 else chunk // 2 * 2, np.uint8)
    c3.check(c3.lib().c3_memcpy(got.ctypes.data, s.pointers(0).recv, got.size, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    if collective == 0:
        assert np.array_equal(got, orc.expected_allgather(n, chunk, SEED, 2))
    else:
        count = chunk // 2
        host_in = [orc.bf16(n * count, SEED, g, 3) for g in range(n)]
        assert np.array_equal(got.view(np.uint16), orc.reduce_scatter(host_in, 0, count))
    iso = s.default_alloc(c3.COMM_ONLY_CU)
    iso.cus_comm, iso.comm_pace_gbps = 16, rate
    fast = min(_comm_ms(s.run(c3.COMM_ONLY_CU, iso)) for _ in range(3))
    assert fast < 0.5 * target_ms
    s.close()
    w.close()


def test_pair512_tail_split_matches_256_wide(torch_mod, c3, monkeypatch):
    """cfg2's GEMM on the 512-wide pair kernel claims its underfilled last
    wave as 256-column halves (1792 tiles on 74 pairs: 16 tiles split); the
    result is bit-identical to the 256-wide pair kernel (same per-element K
    order), and within the bf16 bar at sampled entries."""
    torch = torch_mod
    M, N, K = 8192, 28672, 8192
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
    out = {}
    for kernel in ("pair512", "pair"):
        monkeypatch.setenv("C3_GEMM_KERNEL", kernel)
        C_ = torch.zeros(M * N, dtype=torch.int16, device="cuda")
        w.gemm(A.data_ptr(), B.data_ptr(), C_.data_ptr(), M, N, K, 0)
        torch.cuda.synchronize()
        out[kernel] = C_
    assert torch.equal(out["pair512"], out["pair"])
    # the split tiles are the last 16 of the raster: check their columns' region
    rng = np.random.default_rng(5)
    rows = rng.integers(0, M, 1024)
    cols = rng.integers(N - 4096, N, 1024)
    gemm_check(out["pair512"].cpu().numpy().view(np.uint16), orc.bf16(M * K, SEED, 0, 0),
               orc.bf16(N * K, SEED, 0, 1), M, N, K, rows, cols)
    w.close()


def _h2d(c3, ptr, host):
    c3.check(c3.lib().c3_memcpy(ptr, host.ctypes.data, host.nbytes, 1, None))
    c3.check(c3.lib().c3_stream_sync(None))


def _d2h_np(c3, ptr, nbytes):
    out = np.empty(nbytes, np.uint8)
    c3.check(c3.lib().c3_memcpy(out.ctypes.data, ptr, nbytes, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    return out


@pytest.mark.parametrize("collective", [0, 1, 2], ids=["all-gather", "all-to-all", "reduce-scatter"])
@pytest.mark.parametrize("strategy", ["SERIAL", "C3_BASE", "C3_SP", "CONCCL", "FUSED"])
@pytest.mark.parametrize("slot_mib", [1, 5, "5odd"])
def test_run_host_matches_device_run(torch_mod, c3, monkeypatch, collective, strategy, slot_mib):
    """c3_session_run_host: A and this rank's collective input copied in from
    pinned host memory, C read back inside the step. The device state after
    it (C, every virtual rank's receive buffer) and the returned bytes are
    bit-identical to the device-resident run of the same strategy. 5 MiB
    slots take the pipelined form (the input in 4 pieces, one collective per
    piece, the last piece carrying the remainder)."""
    torch = torch_mod
    if strategy == "FUSED" and collective == 2:
        pytest.skip("fused C3 moves all-gather / all-to-all data only")
    if strategy == "FUSED" and slot_mib == "5odd":
        pytest.skip("fused C3 needs 16-byte slots")
    if strategy == "FUSED":
        monkeypatch.setenv("C3_GEMM_KERNEL", "pair")  # fused needs the CTA-pair GEMM
    st = getattr(c3, strategy)
    n, M, N, K = 8, 512, 1024, 512
    if slot_mib == "5odd":  # slots not 16-byte aligned (the all-to-all keeps one piece)
        payload = n * ((5 << 20) + 4096 * 3 + 2 * 5)
    else:
        payload = n * ((slot_mib << 20) + 4096 * 3 + 16 * 5)  # pieces of 4 KiB multiples + a remainder
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, M, N, K, collective, payload)
    s.fill(SEED)
    p0 = s.pointers(0)
    a_h = _d2h_np(c3, p0.a, p0.a_bytes)
    send_h = _d2h_np(c3, p0.send, p0.send_bytes)
    c_bytes = M * N * 2

    def reset():
        for v in range(n):
            pv = s.pointers(v)
            _h2d(c3, pv.recv, np.zeros(pv.recv_bytes, np.uint8))
        _h2d(c3, p0.c, np.zeros(c_bytes, np.uint8))

    reset()
    _h2d(c3, p0.send, send_h)
    s.run(st, None)
    c_ref = _d2h_np(c3, p0.c, c_bytes)
    recv_ref = [_d2h_np(c3, s.pointers(v).recv, s.pointers(v).recv_bytes) for v in range(n)]
    assert c_ref.any()

    reset()
    _h2d(c3, p0.a, np.zeros(p0.a_bytes, np.uint8))
    _h2d(c3, p0.send, np.zeros(p0.send_bytes, np.uint8))
    pin_a = torch.from_numpy(a_h).pin_memory()
    pin_s = torch.from_numpy(send_h).pin_memory()
    pin_o = torch.zeros(c_bytes, dtype=torch.uint8).pin_memory()
    t = s.run_host(st, None, pin_a.data_ptr(), pin_s.data_ptr(), pin_o.data_ptr(), c_bytes)
    assert t.total_ms > 0
    assert np.array_equal(pin_o.numpy(), c_ref)
    assert np.array_equal(_d2h_np(c3, p0.c, c_bytes), c_ref)
    for v in range(n):
        assert np.array_equal(_d2h_np(c3, s.pointers(v).recv, s.pointers(v).recv_bytes), recv_ref[v]), v
    with pytest.raises(c3.C3Error):
        s.run_host(st, None, None, None, pin_o.data_ptr(), c_bytes + 2)
    s.close()
    w.close()


# ---------------------------------------------------------------- fp32 / TF32
# configs[0] is an fp32 GEMM. The product runs it at fp32
# accuracy on the TF32 tensor cores: split-TF32 (c3_gemm_f32, c3cuda.h), each
# operand x ~ hi + lo with hi the TF32 rounding of x and lo that of the
# remainder, three kind::tf32 MMAs per K step A_lo B_hi + A_hi B_lo + A_hi B_hi,
# fp32 accumulate. Stated tolerances:
#   * inputs representable in bf16 (the synthetic fill): lo = 0 and every
#     product is exact in fp32, so only the fp32 accumulation differs from the
#     fp64 definition:
#         |C - C_ref| <= 2^-19 |C_ref| + 2^-17 (|A||B|)[i,j]
#   (split inside the SM by converter warps, gemm_f32.cu; split-K with a
#   fixed-order sum of the partials when the tiles are fewer than the SMs)
#   * general fp32 inputs: |x - hi| <= 2^-11 |x|, |x - hi - lo| <= 2^-22 |x|,
#     so the dropped A_lo B_lo and the remainders cost at most 2^-20 |a b| per
#     product (unbiased):
#         |C - C_ref| <= 2^-18 (|A||B|)[i,j]
#     and an RMS error (normalised by (|A||B|)) <= 2^-20. Measured on B200
#     (tools/dev/gemm_err_probe.py, 512x768x4096, normalised by (|A||B|)):
#     split-TF32 RMS 2^-22.0, max 2^-19.5; plain TF32 (cuBLAS) RMS 2^-17.1,
#     max 2^-14.8; host fp32 (numpy) RMS 2^-26.7. The gap to the host is the
#     tensor core's own fp32 accumulation (the bf16 kernels show the same
#     2^-22 accumulation excess).

def _f32_check(got, A64, B64, K, exact_inputs):
    ref = A64 @ B64.T
    mag = np.abs(A64) @ np.abs(B64).T
    tol = 2.0 ** -19 * np.abs(ref) + 2.0 ** -17 * mag if exact_inputs else 2.0 ** -18 * mag
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= tol), (float(err.max()), float((err / np.maximum(mag, 1e-30)).max()))
    if not exact_inputs:  # split-TF32 accuracy, not TF32's (2^-17 RMS)
        rms = float(np.sqrt(np.mean((err / mag) ** 2)))
        assert rms <= 2.0 ** -20, rms


def test_fill_f32_matches_oracle(torch_mod, c3):
    torch = torch_mod
    w = c3.World()
    for count in (1, 7, 4096, 1 << 20):
        t = torch.empty(count, dtype=torch.float32, device="cuda")
        c3.check(c3.lib().c3_fill_f32(t.data_ptr(), count, SEED, 3, 1, None))
        assert np.array_equal(t.cpu().numpy(), orc.bf16_to_f32(orc.bf16(count, SEED, 3, 1)))
    w.close()


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 1024), (128, 256, 32), (300, 520, 200), (1000, 2056, 136),
                                   (64, 1024, 512), (2048, 4096, 1024)])
def test_gemm_f32_tf32_full(torch_mod, c3, M, N, K):
    """c3_gemm_f32 on the synthetic (bf16-valued) fp32 inputs, every entry."""
    torch = torch_mod
    w = c3.World()
    A = torch.empty(M * K, dtype=torch.float32, device="cuda")
    B = torch.empty(N * K, dtype=torch.float32, device="cuda")
    Cm = torch.full((M * N,), float("nan"), dtype=torch.float32, device="cuda")
    c3.check(c3.lib().c3_fill_f32(A.data_ptr(), M * K, SEED, 0, 0, None))
    c3.check(c3.lib().c3_fill_f32(B.data_ptr(), N * K, SEED, 0, 1, None))
    w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    A64 = orc.bf16_to_f32(orc.bf16(M * K, SEED, 0, 0)).astype(np.float64).reshape(M, K)
    B64 = orc.bf16_to_f32(orc.bf16(N * K, SEED, 0, 1)).astype(np.float64).reshape(N, K)
    _f32_check(Cm.cpu().numpy().reshape(M, N), A64, B64, K, True)
    w.close()


@pytest.mark.parametrize("M,N,K", [(512, 768, 1000), (300, 520, 204), (1024, 1024, 1024)])
def test_gemm_f32_general_inputs(torch_mod, c3, M, N, K):
    """General fp32 inputs (normal, wide exponent range): the split-TF32
    bound, 32x below plain TF32's error."""
    torch = torch_mod
    w = c3.World()
    g = torch.Generator().manual_seed(3)
    Ah = torch.randn(M, K, generator=g) * torch.exp2(torch.randint(-6, 7, (M, 1), generator=g).float())
    Bh = torch.randn(N, K, generator=g)
    A, B = Ah.cuda(), Bh.cuda()
    Cm = torch.empty(M, N, dtype=torch.float32, device="cuda")
    w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    _f32_check(Cm.cpu().numpy(), Ah.double().numpy(), Bh.double().numpy(), K, False)
    w.close()


def test_gemm_f32_stream_ordered_back_to_back(torch_mod, c3):
    """c3_gemm_f32 on a side stream, several calls back to back with no host
    sync between them: each call's workspace is stream-ordered
    (cudaMallocAsync / cudaFreeAsync), so no call sees another's partials."""
    torch = torch_mod
    w = c3.World()
    M, N, K = 256, 384, 512
    g = torch.Generator().manual_seed(11)
    As = [torch.randn(M, K, generator=g) for _ in range(4)]
    Bs = [torch.randn(N, K, generator=g) for _ in range(4)]
    Ad, Bd = [a.cuda() for a in As], [b.cuda() for b in Bs]
    Cs = [torch.empty(M, N, dtype=torch.float32, device="cuda") for _ in range(4)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    for i in range(4):
        w.gemm(Ad[i].data_ptr(), Bd[i].data_ptr(), Cs[i].data_ptr(), M, N, K, dtype_bytes=4,
               stream=side.cuda_stream)
    side.synchronize()
    for i in range(4):
        _f32_check(Cs[i].cpu().numpy(), As[i].double().numpy(), Bs[i].double().numpy(), K, False)
    w.close()


@pytest.mark.parametrize("K", [64, 128, 192, 256])  # split-K 1, 2 (TMA adds), 3 and 4 (workspace) parts
def test_gemm_f32_propagates_inf_and_nan(torch_mod, c3, K):
    """Infinities and NaNs follow IEEE fp32 GEMM semantics: every product
    a*b is formed once (inf * finite = inf, inf * 0 = NaN, inf * inf = inf,
    -inf + inf = NaN), and a finite input next to FLT_MAX stays finite."""
    torch = torch_mod
    w = c3.World()
    M, N = 128, 128
    A = torch.ones(M, K)
    B = torch.ones(N, K) * 0.5
    A[3, 5] = float("inf")
    A[7, 9] = float("nan")
    A.view(torch.int32)[11, 2] = 0x7FFFFFFF  # NaN with every payload bit set
    A[13, 20] = float("inf")
    B[4, 20] = float("inf")  # inf * inf in C[13, 4]; 1 * inf down column 4
    A[17, 1] = -float("inf")  # -inf row, NaN at column 4 (-inf + inf)
    A[21, 30] = float("inf")
    B[9, 30] = 0.0  # inf * 0 = NaN at C[21, 9]
    A[25, 0] = 3.4e38  # finite: its TF32 rounding would overflow
    Ad, Bd = A.cuda(), B.cuda()
    Cm = torch.empty(M, N, dtype=torch.float32, device="cuda")
    w.gemm(Ad.data_ptr(), Bd.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    C = Cm.cpu().double().numpy()
    with np.errstate(invalid="ignore", over="ignore"):
        ref = A.double().numpy() @ B.double().numpy().T
    assert np.array_equal(np.isnan(C), np.isnan(ref))
    assert np.array_equal(np.isposinf(C), np.isposinf(ref)) and np.array_equal(np.isneginf(C), np.isneginf(ref))
    fin = np.isfinite(ref)
    assert np.all(np.abs(C[fin] - ref[fin]) <= 2.0 ** -20 * np.abs(ref[fin]))
    assert np.isposinf(C[13, 4]) and np.isnan(C[17, 4]) and np.isnan(C[21, 9]) and np.isfinite(C[25, 0])
    w.close()


def test_gemm_f32_split_k_is_bit_reproducible(torch_mod, c3):
    """configs[0]'s shape runs split-K (the last-arriving part sums the
    partials in fixed order), so repeated calls are bitwise identical."""
    torch = torch_mod
    w = c3.World()
    M = N = K = 1024
    g = torch.Generator().manual_seed(5)
    A, B = torch.randn(M, K, generator=g).cuda(), torch.randn(N, K, generator=g).cuda()
    outs = []
    for _ in range(4):
        Cm = torch.empty(M, N, dtype=torch.float32, device="cuda")
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
        outs.append(Cm)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32))
    _f32_check(outs[0].cpu().numpy(), A.cpu().double().numpy(), B.cpu().double().numpy(), K, False)
    w.close()


def test_gemm_f32_rejects_unaligned(c3, torch_mod):
    w = c3.World()
    t = torch_mod.empty(64 * 64, dtype=torch_mod.float32, device="cuda")
    with pytest.raises(c3.C3Error):
        w.gemm(t.data_ptr(), t.data_ptr(), t.data_ptr(), 8, 8, 6, dtype_bytes=4)  # K rows of 24 bytes
    w.close()


@pytest.mark.parametrize("strategy", ["SERIAL", "C3_BASE", "C3_SP", "CONCCL"])
def test_cfg1_fp32_session(torch_mod, c3, strategy):
    """configs[0] end to end: fp32 GEMM 1024^3 (split-TF32) with a
    16 MiB all-gather at world 2: the all-gather bit-exact, every GEMM entry
    within the stated bound, through the host-buffer call as well."""
    torch = torch_mod
    n, M, N, K, payload = 2, 1024, 1024, 1024, 16 << 20
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, M, N, K, c3.ALL_GATHER, payload, dtype_bytes=4)
    s.fill(SEED)
    p = s.pointers(0)
    assert p.a_bytes == M * K * 4 and p.c_bytes == M * N * 4
    s.run(getattr(c3, strategy), None, all_ranks=True)
    got = np.empty(payload, np.uint8)
    c3.check(c3.lib().c3_memcpy(got.ctypes.data, p.recv, payload, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    assert np.array_equal(got, orc.expected_allgather(n, payload // n, SEED, 2))
    A64 = orc.bf16_to_f32(orc.bf16(M * K, SEED, 0, 0)).astype(np.float64).reshape(M, K)
    B64 = orc.bf16_to_f32(orc.bf16(N * K, SEED, 0, 1)).astype(np.float64).reshape(N, K)
    cm = np.empty(M * N, np.float32)
    c3.check(c3.lib().c3_memcpy(cm.ctypes.data, p.c, M * N * 4, 2, None))
    c3.check(c3.lib().c3_stream_sync(None))
    _f32_check(cm.reshape(M, N), A64, B64, K, True)
    # host buffers: A in from pinned memory, all of C back
    a_h = torch.from_numpy(A64.astype(np.float32).ravel().view(np.uint8).copy()).pin_memory()
    out = torch.zeros(M * N * 4, dtype=torch.uint8).pin_memory()
    s.run_host(getattr(c3, strategy), None, a_h.data_ptr(), None, out.data_ptr(), M * N * 4)
    assert np.array_equal(out.numpy().view(np.float32), cm)
    s.close()
    w.close()


@pytest.mark.parametrize("kernel", ["pair", "pair512"])
@pytest.mark.parametrize("strategy", ["C3_BASE", "C3_SP", "GEMM_ONLY"])
@pytest.mark.parametrize("M,a_pieces", [(1024, "4"), (1000, "3"), (2048, "8")])
def test_run_host_row_gated_gemm(torch_mod, c3, monkeypatch, kernel, strategy, M, a_pieces):
    """c3_session_run_host with the CTA-pair GEMM: A lands in row bands, each
    published by a stream-memop flag the GEMM's TMA producers wait on, so the
    GEMM starts on the first band. C must be bit-identical to the
    device-resident run (ragged last band included)."""
    torch = torch_mod
    monkeypatch.setenv("C3_GEMM_KERNEL", kernel)
    monkeypatch.setenv("C3_H2D_A_PIECES", a_pieces)  # read per call (a_row_bands)
    st = getattr(c3, strategy)
    n, N, K = 8, 1536, 512
    payload = n * (5 << 20)
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, M, N, K, c3.ALL_GATHER, payload)
    s.fill(SEED)
    p0 = s.pointers(0)
    a_h = _d2h_np(c3, p0.a, p0.a_bytes)
    send_h = _d2h_np(c3, p0.send, p0.send_bytes)
    c_bytes = M * N * 2
    s.run(st, None)
    c_ref = _d2h_np(c3, p0.c, c_bytes)
    for rep in range(3):  # repeated steps: the flags' epochs advance
        _h2d(c3, p0.c, np.zeros(c_bytes, np.uint8))
        _h2d(c3, p0.a, np.zeros(p0.a_bytes, np.uint8))
        pin_a = torch.from_numpy(a_h).pin_memory()
        pin_s = torch.from_numpy(send_h).pin_memory()
        pin_o = torch.zeros(c_bytes, dtype=torch.uint8).pin_memory()
        s.run_host(st, None, pin_a.data_ptr(), pin_s.data_ptr(), pin_o.data_ptr(), c_bytes)
        assert np.array_equal(pin_o.numpy(), c_ref), rep
    s.close()
    w.close()
