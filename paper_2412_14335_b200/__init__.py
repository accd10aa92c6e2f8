"""c3-b200: B200-native execution of the C3 hot path of arXiv 2412.14335 —
a GEMM concurrent with an all-gather / reduce-scatter across one node's GPUs,
under the paper's strategies (serial, c3_base, c3_sp, c3_rp, c3_sp_rp, conccl,
conccl_rp).

The product is native: ``lib/libc3sim.so`` (the reference's c3sim C++ API,
``include/c3sim/*.hpp``) and ``lib/libc3cuda.so`` (sm_100a kernels + runtime
behind the C ABI ``include/c3cuda.h``). This package is the thin Python host
mirror used by bench.py and the tests; it owns no compute.
"""
import ctypes as C

from . import _capi
from ._capi import (ALL_GATHER, ALL_TO_ALL, REDUCE_SCATTER, SERIAL, C3_BASE, C3_SP, C3_RP,
                    C3_SP_RP, CONCCL, CONCCL_RP, FUSED, GEMM_ONLY, COMM_ONLY_CU, COMM_ONLY_DMA,
                    SERIAL_OVERLAP_IO,
                    STRATEGY_NAMES, BACKEND_CU, BACKEND_DMA, BACKEND_TMA, C3Error, check, lib,
                    ptr_array)

__all__ = ["World", "Session", "plan_transfers", "ideal_speedup", "fraction_of_ideal",
           "STRATEGY_NAMES", "C3Error"]


def ideal_speedup(t_gemm, t_comm):
    """(t_g + t_c) / max(t_g, t_c) — reference taxonomy.cpp:23-27."""
    if not (t_gemm > 0 and t_comm > 0):
        raise ValueError("ideal_speedup: times must be positive")
    return (t_gemm + t_comm) / max(t_gemm, t_comm)


def fraction_of_ideal(speedup, ideal):
    """(speedup - 1) / (ideal - 1), 0 for a slowdown, not capped — taxonomy.cpp:29-33."""
    if not ideal > 1:
        raise ValueError("fraction_of_ideal: ideal must be > 1")
    return 0.0 if speedup < 1.0 else (speedup - 1.0) / (ideal - 1.0)


def plan_transfers(kind, n_ranks, chunk_bytes, dma_engines):
    """The validated ConCCL plan from the product model layer (libc3sim)."""
    L = lib()
    n = C.c_int(0)
    check(L.c3_plan_transfers(kind, n_ranks, chunk_bytes, dma_engines, None, 0, C.byref(n)))
    arr = (_capi.Transfer * max(1, n.value))()
    check(L.c3_plan_transfers(kind, n_ranks, chunk_bytes, dma_engines, arr, n.value, C.byref(n)))
    return arr, n.value


def ingest_model(hidden, ffn, tokens, dtype_bytes=2, shards=8):
    """The layer's C3 scenarios (model layer ingest_model): list of
    (m, n, k, all-gather payload bytes of that GEMM's weight)."""
    L = lib()
    n = C.c_int(0)
    check(L.c3_ingest_model(hidden, ffn, tokens, dtype_bytes, shards, None, 0, C.byref(n)))
    arr = (_capi.ScenarioDesc * max(1, n.value))()
    check(L.c3_ingest_model(hidden, ffn, tokens, dtype_bytes, shards, arr, n.value, C.byref(n)))
    return [(d.m, d.n, d.k, d.payload_bytes) for d in arr[:n.value]]


class World:
    """One device; `loopback=True` hosts all n ranks virtually on it."""

    def __init__(self, rank=0, n_ranks=1, device=0, loopback=False):
        self.h = C.c_void_p()
        check(lib().c3_world_create(rank, n_ranks, device, int(bool(loopback)), C.byref(self.h)))
        info = _capi.WorldInfo()
        check(lib().c3_world_get_info(self.h, C.byref(info)))
        self.info = info
        self.rank, self.n_ranks = info.rank, info.n_ranks

    def close(self):
        if self.h:
            check(lib().c3_world_destroy(self.h))
            self.h = C.c_void_p()

    def gemm(self, a, b, c, m, n, k, max_ctas=0, stream=None, dtype_bytes=2):
        """C = A B^T: bf16 (dtype_bytes 2) or fp32 (4: split-TF32 on the tensor cores, see c3cuda.h)."""
        fn = lib().c3_gemm_f32 if dtype_bytes == 4 else lib().c3_gemm_bf16
        check(fn(self.h, a, b, c, m, n, k, max_ctas, stream))

    def allgather_p2p(self, self_rank, send, recv_ptrs, chunk_bytes, n_ctas=32, stream=None):
        check(lib().c3_allgather_p2p(self.h, self_rank, send, ptr_array(recv_ptrs), chunk_bytes,
                                     n_ctas, stream))

    def alltoall_p2p(self, self_rank, send, recv_ptrs, per_peer_bytes, n_ctas=32, stream=None):
        check(lib().c3_alltoall_p2p(self.h, self_rank, send, ptr_array(recv_ptrs), per_peer_bytes,
                                    n_ctas, stream))

    def reduce_scatter_p2p(self, self_rank, in_ptrs, out, count, n_ctas=32, stream=None):
        check(lib().c3_reduce_scatter_p2p(self.h, self_rank, ptr_array(in_ptrs), out, count,
                                          n_ctas, stream))

    def ce_execute(self, transfers, n_transfers, src_ptrs, dst_ptrs, src_filter=-1, stream=None):
        check(lib().c3_ce_execute(self.h, transfers, n_transfers, ptr_array(src_ptrs),
                                  ptr_array(dst_ptrs), src_filter, stream))


class Session:
    """One C3 scenario's operands, executed under a strategy (c3_session_*)."""

    def __init__(self, world, m, n, k, collective, payload_bytes, dtype_bytes=2):
        self.world = world
        d = _capi.ScenarioDesc(m, n, k, collective, world.n_ranks, payload_bytes, dtype_bytes)
        self.desc = d
        self.h = C.c_void_p()
        check(lib().c3_session_create(world.h, C.byref(d), C.byref(self.h)))

    def close(self):
        if self.h:
            check(lib().c3_session_destroy(self.h))
            self.h = C.c_void_p()

    def pointers(self, virtual_rank=0):
        p = _capi.SessionPtrs()
        check(lib().c3_session_pointers(self.h, virtual_rank, C.byref(p)))
        return p

    def fill(self, seed=20241217):
        check(lib().c3_session_fill(self.h, seed))

    def export_handles(self):
        buf = C.create_string_buffer(_capi.SESSION_HANDLE_BYTES)
        check(lib().c3_session_export(self.h, buf))
        return buf.raw

    def import_handles(self, blobs):
        joined = b"".join(blobs)
        check(lib().c3_session_import(self.h, C.create_string_buffer(joined, len(joined))))

    def set_barrier(self, fn):
        """Kept for source compatibility: cross-rank completion of every
        backend is device-side now and the callback is not called."""
        def _cb(_ctx):
            try:
                fn()
                return 0
            except Exception:
                return 1
        self._barrier_cb = _capi.BARRIER_FN(_cb)  # keep alive
        check(lib().c3_session_set_barrier(self.h, C.cast(self._barrier_cb, C.c_void_p), None))

    def set_ce_proxy(self, on=True):
        """Host-staged copy-engine proxy (loopback): the DMA backend's peers
        become pinned host buffers, so this GPU's share of the plan runs on
        the copy engines over PCIe. Call before fill()."""
        check(lib().c3_session_set_ce_proxy(self.h, int(bool(on))))

    def set_wait_timeout(self, ms):
        """Bound (ms) of every device-side cross-rank wait; an expired wait
        fails the step with C3Error code 103 (Timeout)."""
        check(lib().c3_session_set_wait_timeout(self.h, float(ms)))

    def load_tables(self, csv_path):
        check(lib().c3_session_load_tables(self.h, csv_path.encode()))

    def set_fused_pace(self, pace=0.0, piece_bytes=4096):
        check(lib().c3_session_set_fused_pace(self.h, pace, piece_bytes))

    def set_link_rate(self, gbps):
        """Link-rate emulation (loopback): pace the collective's peer traffic
        to `gbps` GB/s per direction (0 = off)."""
        check(lib().c3_session_set_link_rate(self.h, float(gbps)))

    def load_machine(self, json_path):
        """Reference-format machine descriptor for the predictor (e.g.
        data/b200-node-n8.json)."""
        check(lib().c3_session_load_machine(self.h, json_path.encode()))

    def load_params(self, json_path):
        check(lib().c3_session_load_params(self.h, json_path.encode()))

    def choose(self, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms=0.0, allow_dma=True):
        """Runtime heuristic: (strategy, alloc, predicted_ms)."""
        st, a, pred = C.c_int(), _capi.Alloc(), C.c_double()
        check(lib().c3_session_choose(self.h, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms,
                                      int(bool(allow_dma)), C.byref(st), C.byref(a), C.byref(pred)))
        return st.value, a, pred.value

    def predict(self, strategy, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms=0.0):
        """Model-layer predicted makespan (ms) of one strategy."""
        ms = C.c_double()
        check(lib().c3_session_predict(self.h, strategy, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms,
                                       C.byref(ms)))
        return ms.value

    def set_comm_curve(self, points):
        """Measured collective time vs CTA count [(ctas, ms), ...] under this
        world's link rate; replaces the comm slowdown table in predictions
        ([] restores it)."""
        pts = sorted(points)
        n = len(pts)
        ct = (C.c_int * max(n, 1))(*[int(c) for c, _ in pts])
        ms = (C.c_double * max(n, 1))(*[float(t) for _, t in pts])
        check(lib().c3_session_set_comm_curve(self.h, ct, ms, n))

    def load_coresident(self, json_path):
        """Co-residency penalties (B200 model extension); None disables."""
        check(lib().c3_session_load_coresident(self.h, json_path.encode() if json_path else None))

    def predict_alloc(self, strategy, alloc, t_gemm_ms, t_comm_cu_ms, t_comm_dma_ms=0.0):
        """Predicted makespan (ms) of (strategy, alloc); co-resident allocations
        use the co-resident model."""
        ms = C.c_double()
        check(lib().c3_session_predict_alloc(self.h, strategy, C.byref(alloc), t_gemm_ms, t_comm_cu_ms,
                                             t_comm_dma_ms, C.byref(ms)))
        return ms.value

    def autotune(self, candidates, rounds=3, reduce_max=None, medians=None):
        """candidates: [(strategy, Alloc)] -> (best index, median ms). With
        several ranks pass reduce_max (elementwise max over ranks of a list) so
        every rank picks the same candidate. `medians` (a list) receives every
        candidate's median step time."""
        n = len(candidates)
        sts = (C.c_int * n)(*[c[0] for c in candidates])
        als = (_capi.Alloc * n)(*[c[1] for c in candidates])
        med = (C.c_double * n)()
        best, ms = C.c_int(), C.c_double()
        check(lib().c3_session_autotune(self.h, sts, als, n, rounds, med, C.byref(best),
                                        C.byref(ms)))
        meds = list(med)
        if reduce_max is not None:
            meds = reduce_max(meds)
        if medians is not None:
            medians[:] = meds
        i = min(range(n), key=lambda j: meds[j])
        return i, meds[i]

    def default_alloc(self, strategy):
        a = _capi.Alloc()
        check(lib().c3_session_default_alloc(self.h, strategy, C.byref(a)))
        return a

    def run(self, strategy, alloc=None, all_ranks=False):
        t = _capi.Timing()
        fn = lib().c3_session_run_all_ranks if all_ranks else lib().c3_session_run
        check(fn(self.h, strategy, C.byref(alloc) if alloc is not None else None, C.byref(t)))
        return t

    def run_host(self, strategy, alloc, host_a, host_send, host_out=None, out_bytes=0):
        """One step on host buffers (c3_session_run_host): raw host addresses
        (ints, pinned memory for overlap) or None for A / the collective input /
        the result read-back."""
        t = _capi.Timing()
        check(lib().c3_session_run_host(self.h, strategy, C.byref(alloc) if alloc is not None else None,
                                        host_a, host_send, host_out, out_bytes, C.byref(t)))
        return t
