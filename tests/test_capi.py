"""The C-ABI boundary without a GPU: libc3cuda.so loads, exports every symbol
include/c3cuda.h declares, returns status codes (never crashes) when there is
no device, and its model-layer entry point (c3_plan_transfers) matches the
reference planner's golden plans.
"""
import ctypes as C
import glob
import json
import os
import re

import pytest

import paper_2412_14335_b200 as c3
from paper_2412_14335_b200 import _capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "c3cuda.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(c3_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "c3_session_run" in names and "c3_gemm_bf16" in names and len(names) >= 30


def test_library_exports_every_declared_symbol():
    L = c3.lib()
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared()) <= set(_capi.SIGNATURES)


def test_no_gpu_returns_status_not_crash():
    if _has_gpu():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = c3.lib().c3_world_create(0, 1, 0, 0, C.byref(h))
    assert rc >= 100
    assert c3.lib().c3_last_error()


def test_bad_arguments_are_validation_errors():
    h = C.c_void_p()
    assert c3.lib().c3_world_create(0, 9, 0, 0, C.byref(h)) == 4
    assert c3.lib().c3_world_create(3, 2, 0, 0, C.byref(h)) == 4
    n = C.c_int()
    assert c3.lib().c3_plan_transfers(7, 2, 64, 4, None, 0, C.byref(n)) == 3
    assert c3.lib().c3_plan_transfers(0, 2, 0, 4, None, 0, C.byref(n)) == 4


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(REPO, "tests", "golden", "plans",
                                                               "*.json"))))
def test_plan_transfers_match_reference(path):
    p = json.load(open(path))
    kind = c3.ALL_GATHER if p["kind"] == "all-gather" else c3.ALL_TO_ALL
    engines = 14  # the machine file the golden plans were generated with
    arr, cnt = c3.plan_transfers(kind, p["n_ranks"], p["chunk_bytes"], engines)
    got = [{"src": t.src_gpu, "dst": t.dst_gpu, "src_off": t.src_offset, "dst_off": t.dst_offset,
            "len": t.length, "engine": t.engine_id, "seq": t.seq} for t in arr[:cnt]]
    assert got == p["transfers"]


def test_reduce_scatter_plan_is_transpose():
    arr, cnt = c3.plan_transfers(c3.REDUCE_SCATTER, 8, 1024, 4)
    assert cnt == 56
    for t in arr[:cnt]:
        assert t.src_offset == t.dst_gpu * 1024 and t.dst_offset == t.src_gpu * 1024
        assert 0 <= t.engine_id < 4


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_ingest_model_llama70b_layer():
    """ingest_model (workload.cpp:217-251 semantics) through the C ABI."""
    layer = c3.ingest_model(8192, 28672, 8192, 2, 8)
    assert [(m, n, k) for m, n, k, _ in layer] == [
        (8192, 3 * 8192, 8192), (8192, 8192, 8192), (8192, 2 * 28672, 8192), (8192, 8192, 28672)]
    assert [p for *_, p in layer] == [3 * 8192 * 8192 * 2, 8192 * 8192 * 2, 2 * 28672 * 8192 * 2,
                                      28672 * 8192 * 2]
    assert all(p % 8 == 0 for *_, p in layer)
    assert all(p == 0 for *_, p in c3.ingest_model(4096, 11008, 2048, 2, 1))
