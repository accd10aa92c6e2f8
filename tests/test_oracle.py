"""Pin the CPU oracle (oracle/c3oracle.c) before trusting it.

* ByteOracle restatement vs the REFERENCE's own plans (tests/golden/plans/*.json,
  emitted by the reference planner via oracle/_ref, tests/golden/make_golden.py):
  every reference plan passes; every mutation the reference tests apply
  (drop / duplicate / retarget, acceptance.cpp:141-170; test_conccl.cpp:142-179)
  is rejected.
* Plan replay of byte labels == the collective's definition (expected_allgather).
* bf16 helpers and the reduce-scatter / GEMM references on small hand cases.
* The reference's own golden constants that pin the metric arithmetic
  (test_taxonomy.cpp:68-74, test_workload.cpp:14-22).
"""
import glob
import json
import os

import numpy as np
import pytest

from tests import _oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PLANS = sorted(glob.glob(os.path.join(GOLD, "plans", "*.json")))
# the byte-level replay holds 8 bytes of label per destination byte; like the
# reference's ByteOracle tests (sizes <= 4096) keep it to small plans
SMALL = [p for p in PLANS if "117440512" not in p]


def load(path):
    with open(path) as f:
        return json.load(f)


def test_golden_plans_exist():
    assert len(PLANS) == 14 and len(SMALL) == 12


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
def test_byte_oracle_accepts_reference_plans(path):
    p = load(path)
    kind = 0 if p["kind"] == "all-gather" else 1
    ts = orc.to_transfers(p["transfers"])
    rc, why = orc.byte_oracle(kind, p["n_ranks"], p["chunk_bytes"], p["src_buffer_bytes"],
                              p["dst_buffer_bytes"], ts, len(p["transfers"]))
    assert rc == 0, why


@pytest.mark.parametrize("path", [p for p in SMALL if "_n1_" not in p],
                         ids=[os.path.basename(p) for p in SMALL if "_n1_" not in p])
def test_byte_oracle_rejects_mutations(path):
    p = load(path)
    kind = 0 if p["kind"] == "all-gather" else 1
    T = p["transfers"]
    rng = np.random.default_rng(20240814)
    args = (kind, p["n_ranks"], p["chunk_bytes"], p["src_buffer_bytes"], p["dst_buffer_bytes"])
    for _ in range(4):
        i = int(rng.integers(0, len(T)))
        dropped = T[:i] + T[i + 1:]
        assert orc.byte_oracle(*args, orc.to_transfers(dropped), len(dropped))[0] != 0
        dup = T + [T[i]]
        assert orc.byte_oracle(*args, orc.to_transfers(dup), len(dup))[0] != 0
        moved = [dict(t) for t in T]
        moved[i]["dst_off"] = (moved[i]["dst_off"] + 1) % (p["dst_buffer_bytes"] - moved[i]["len"] + 1)
        assert orc.byte_oracle(*args, orc.to_transfers(moved), len(moved))[0] != 0


@pytest.mark.parametrize("path", [p for p in PLANS if "all-gather" in p and "117440512" not in p])
def test_replay_of_reference_allgather_plan_gives_definition(path):
    """memcpy replay of the reference plan over labelled buffers == oracle's
    expected all-gather (this is the check applied to GPU outputs)."""
    import ctypes as C
    p = load(path)
    n, chunk = p["n_ranks"], p["chunk_bytes"]
    seed = 99
    src = [orc.labels(chunk, seed, g, 2) for g in range(n)]
    dst = [np.zeros(n * chunk, np.uint8) for _ in range(n)]
    for g in range(n):
        dst[g][g * chunk:(g + 1) * chunk] = src[g]  # resident slot
    sp = (C.c_void_p * n)(*[a.ctypes.data for a in src])
    dp = (C.c_void_p * n)(*[a.ctypes.data for a in dst])
    rc = orc.lib().c3o_replay_plan(orc.to_transfers(p["transfers"]), len(p["transfers"]), n, sp,
                                   chunk, dp, n * chunk)
    assert rc == 0
    want = orc.expected_allgather(n, chunk, seed, 2)
    for g in range(n):
        assert np.array_equal(dst[g], want)


def test_bf16_rne_and_values():
    L = orc.lib()
    assert L.c3o_f32_to_bf16_rne(1.0) == 0x3F80
    assert L.c3o_f32_to_bf16_rne(1.0 + 2 ** -8) == 0x3F80      # tie -> even
    assert L.c3o_f32_to_bf16_rne(1.0 + 3 * 2 ** -8) == 0x3F82  # tie -> even (up)
    assert L.c3o_f32_to_bf16_rne(-2.5) == 0xC020
    v = orc.bf16_to_f32(orc.bf16(100000, 1, 0, 0))
    assert np.all(np.abs(v) <= 0.125) and abs(float(v.mean())) < 2e-3


def test_labels_distinct_per_rank_and_tensor():
    a = orc.labels(4096, 7, 0, 2)
    assert not np.array_equal(a, orc.labels(4096, 7, 1, 2))
    assert not np.array_equal(a, orc.labels(4096, 7, 0, 3))
    assert np.array_equal(orc.labels(13, 7, 0, 2), a[:13])


def test_reduce_scatter_reference_small():
    n, count = 3, 4
    ins = [orc.bf16(n * count, 5, g, 3) for g in range(n)]
    for r in range(n):
        out = orc.reduce_scatter(ins, r, count)
        f = [orc.bf16_to_f32(x) for x in ins]
        for i in range(count):
            acc = np.float32(0)
            for g in range(n):
                acc = np.float32(acc + f[g][r * count + i])
            assert out[i] == orc.lib().c3o_f32_to_bf16_rne(float(acc))


def test_f64_to_bf16_rounding_matches_oracle():
    """The vectorised bf16 rounding the GEMM tolerance uses (tests/_oracle.py)
    against the oracle's scalar RNE."""
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(2000) * np.exp2(rng.integers(-20, 20, 2000)),
                        [1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 0.0]])
    want = np.array([orc.lib().c3o_f32_to_bf16_rne(float(np.float32(v))) for v in x], np.uint16)
    assert np.array_equal(orc.f64_to_bf16_bits(x), want)


def test_gemm_reference_small():
    M, N, K = 3, 5, 7
    A, B = orc.bf16(M * K, 1, 0, 0), orc.bf16(N * K, 1, 0, 1)
    fa = orc.bf16_to_f32(A).astype(np.float64).reshape(M, K)
    fb = orc.bf16_to_f32(B).astype(np.float64).reshape(N, K)
    rows, cols = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ref, mag = orc.gemm_samples(A, B, M, N, K, rows.ravel(), cols.ravel())
    assert np.allclose(ref, (fa @ fb.T).ravel(), rtol=0, atol=1e-15)
    assert np.allclose(mag, (np.abs(fa) @ np.abs(fb).T).ravel())


def test_metric_golden_constants():
    import paper_2412_14335_b200 as c3
    assert abs(c3.fraction_of_ideal(1.13, 1.60) - 0.2167) <= 0.0005  # test_taxonomy.cpp:68-74
    assert c3.ideal_speedup(1.0, 1.0) == 2.0
    assert c3.fraction_of_ideal(0.9, 1.5) == 0.0
    assert c3.fraction_of_ideal(1.9, 1.5) > 1.0  # not capped (Appendix A.1)
