"""ctypes binding of libc3cuda.so (include/c3cuda.h) — the C ABI a reference-side
maintainer binds. No torch types cross this boundary.

Loading is strict: if the in-tree library is missing, import fails with a
build hint. There is no CPU fallback anywhere on the product path.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
CUDA_LIB = os.path.join(LIB_DIR, "libc3cuda.so")
MODEL_LIB = os.path.join(LIB_DIR, "libc3sim.so")
CLI = os.path.join(_HERE, "bin", "c3sim")

C3_OK = 0
ERR_NAMES = {2: "IoError", 3: "UnknownEntityError", 4: "ValidationError", 5: "FitError",
             100: "CudaError", 101: "DriverError", 102: "Unsupported", 103: "Timeout"}

ALL_GATHER, ALL_TO_ALL, REDUCE_SCATTER = 0, 1, 2
SERIAL, C3_BASE, C3_SP, C3_RP, C3_SP_RP, CONCCL, CONCCL_RP = range(7)
FUSED = 7  # B200 extension: collective moved inside the GEMM kernel by its TMA unit
GEMM_ONLY, COMM_ONLY_CU, COMM_ONLY_DMA, SERIAL_OVERLAP_IO = 100, 101, 102, 103
STRATEGY_NAMES = ["serial", "c3_base", "c3_sp", "c3_rp", "c3_sp_rp", "conccl", "conccl_rp",
                  "c3_fused"]
BACKEND_CU, BACKEND_DMA, BACKEND_TMA = 0, 1, 2
IPC_HANDLE_BYTES = 64
SESSION_HANDLE_BYTES = 4 * IPC_HANDLE_BYTES
MAX_RANKS = 8
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class Transfer(C.Structure):
    _fields_ = [("src_gpu", C.c_int32), ("dst_gpu", C.c_int32), ("src_offset", C.c_int64),
                ("dst_offset", C.c_int64), ("length", C.c_int64), ("engine_id", C.c_int32),
                ("seq", C.c_int32)]


class WorldInfo(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("rank", "n_ranks", "device", "loopback", "sm_count",
                                       "async_engines", "l2_bytes", "cc_major", "cc_minor",
                                       "green_ctx", "sm_grain", "stream_prio_lo",
                                       "stream_prio_hi")]


class ScenarioDesc(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("collective", C.c_int32),
                ("n_ranks", C.c_int32), ("payload_bytes", C.c_int64), ("dtype_bytes", C.c_int32)]


class Alloc(C.Structure):
    _fields_ = [("cus_gemm", C.c_int32), ("cus_comm", C.c_int32), ("cus_idle", C.c_int32),
                ("backend", C.c_int32), ("comm_first", C.c_int32), ("comm_pace_gbps", C.c_float)]


class Timing(C.Structure):
    _fields_ = [("gemm_start_ms", C.c_double), ("gemm_end_ms", C.c_double),
                ("comm_start_ms", C.c_double), ("comm_end_ms", C.c_double),
                ("total_ms", C.c_double), ("gemm_ctas", C.c_int32), ("comm_ctas", C.c_int32),
                ("partition", C.c_int32), ("launches", C.c_int32)]


class SessionPtrs(C.Structure):
    _fields_ = [("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p), ("send", C.c_void_p),
                ("recv", C.c_void_p), ("staging", C.c_void_p), ("a_bytes", C.c_int64),
                ("b_bytes", C.c_int64), ("c_bytes", C.c_int64), ("send_bytes", C.c_int64),
                ("recv_bytes", C.c_int64), ("staging_bytes", C.c_int64),
                ("virtual_ranks", C.c_int32)]


# name -> (restype, argtypes); every entry point include/c3cuda.h declares.
P, I, I64, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
PP = C.POINTER(C.c_void_p)
SIGNATURES = {
    "c3_last_error": (C.c_char_p, []),
    "c3_version": (I, []),
    "c3_world_create": (I, [I, I, I, I, PP]),
    "c3_world_destroy": (I, [P]),
    "c3_world_get_info": (I, [P, C.POINTER(WorldInfo)]),
    "c3_malloc": (I, [P, I64, PP]),
    "c3_free": (I, [P, P]),
    "c3_memcpy": (I, [P, P, I64, I, P]),
    "c3_stream_sync": (I, [P]),
    "c3_device_sync": (I, []),
    "c3_ipc_export": (I, [P, P, P]),
    "c3_ipc_import": (I, [P, P, PP]),
    "c3_ipc_close": (I, [P, P]),
    "c3_fill_bf16": (I, [P, I64, U64, I, I, P]),
    "c3_fill_f32": (I, [P, I64, U64, I, I, P]),
    "c3_fill_labels": (I, [P, I64, U64, I, I, P]),
    "c3_gemm_bf16": (I, [P, P, P, P, I64, I64, I64, I, P]),
    "c3_gemm_f32": (I, [P, P, P, P, I64, I64, I64, I, P]),
    "c3_allgather_p2p": (I, [P, I, P, PP, I64, I, P]),
    "c3_alltoall_p2p": (I, [P, I, P, PP, I64, I, P]),
    "c3_reduce_scatter_p2p": (I, [P, I, PP, P, I64, I, P]),
    "c3_reduce_local_bf16": (I, [PP, I, P, I64, I, P]),
    "c3_ce_execute": (I, [P, C.POINTER(Transfer), I, PP, PP, I, P]),
    "c3_plan_transfers": (I, [I, I, I64, I, C.POINTER(Transfer), I, C.POINTER(C.c_int)]),
    "c3_ingest_model": (I, [I64, I64, I64, I, I, C.POINTER(ScenarioDesc), I, C.POINTER(C.c_int)]),
    "c3_session_create": (I, [P, C.POINTER(ScenarioDesc), PP]),
    "c3_session_destroy": (I, [P]),
    "c3_session_pointers": (I, [P, I, C.POINTER(SessionPtrs)]),
    "c3_session_fill": (I, [P, U64]),
    "c3_session_export": (I, [P, P]),
    "c3_session_import": (I, [P, P]),
    "c3_session_run": (I, [P, I, C.POINTER(Alloc), C.POINTER(Timing)]),
    "c3_session_run_all_ranks": (I, [P, I, C.POINTER(Alloc), C.POINTER(Timing)]),
    "c3_session_run_host": (I, [P, I, C.POINTER(Alloc), P, P, P, I64, C.POINTER(Timing)]),
    "c3_session_default_alloc": (I, [P, I, C.POINTER(Alloc)]),
    "c3_session_set_barrier": (I, [P, C.c_void_p, P]),
    "c3_session_set_wait_timeout": (I, [P, C.c_double]),
    "c3_session_set_ce_proxy": (I, [P, I]),
    "c3_session_proxy_buffers": (I, [P, I, PP, PP]),
    "c3_sm_hog": (I, [P, C.c_double, P]),
    "c3_session_set_fused_pace": (I, [P, C.c_float, I]),
    "c3_session_set_link_rate": (I, [P, C.c_double]),
    "c3_session_load_tables": (I, [P, C.c_char_p]),
    "c3_session_load_params": (I, [P, C.c_char_p]),
    "c3_session_load_machine": (I, [P, C.c_char_p]),
    "c3_session_predict": (I, [P, I, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "c3_session_autotune": (I, [P, C.POINTER(C.c_int), C.POINTER(Alloc), I, I,
                                C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "c3_session_choose": (I, [P, C.c_double, C.c_double, C.c_double, I, C.POINTER(C.c_int),
                              C.POINTER(Alloc), C.POINTER(C.c_double)]),
    "c3_session_set_comm_curve": (I, [P, C.POINTER(C.c_int), C.POINTER(C.c_double), I]),
    "c3_session_load_coresident": (I, [P, C.c_char_p]),
    "c3_session_predict_alloc": (I, [P, I, C.POINTER(Alloc), C.c_double, C.c_double, C.c_double,
                                     C.POINTER(C.c_double)]),
}


class C3Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libc3cuda.so (in-tree). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(CUDA_LIB):
            raise ImportError(f"{CUDA_LIB} missing: run `make -C {os.path.dirname(_HERE)}` "
                              "(or __graft_entry__.build()) — there is no fallback path")
        L = C.CDLL(CUDA_LIB, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != C3_OK:
        raise C3Error(rc, lib().c3_last_error().decode(errors="replace"))
    return rc


def ptr_array(ptrs):
    arr = (C.c_void_p * MAX_RANKS)()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
