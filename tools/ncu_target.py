"""One small, profiler-friendly invocation per kernel family for ncu:
GEMM (cfg2 shape by default), loopback all-gather push and reduce-scatter
pull, and the fused C3 pair GEMM next to the plain pair GEMM (cfg2 + 896 MiB
all-gather, loopback), all through the C ABI.
cublas: torch.matmul (cuBLAS) on the same shape, for a side-by-side capture.
f32: the split-TF32 fp32 GEMM (configs[0]: 1024^3 by default with this mode).
Usage: python tools/ncu_target.py [gemm|cublas|ag|rs|fused|f32|all] [M N K]"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
M, N, K = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (8192, 28672, 8192)
if what in ("gemm", "all"):
    w = c3.World()
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K)
    torch.cuda.synchronize()
    w.close()
if what == "f32":
    if len(sys.argv) < 5:
        M = N = K = 1024
    w = c3.World()
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    Cm = torch.empty(M, N, device="cuda")
    for _ in range(3):
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    w.close()
if what == "cublas":
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        torch.matmul(A, B.t(), out=Cm)
    torch.cuda.synchronize()
if what in ("ag", "rs", "all"):
    n = 8
    wl = c3.World(0, n, 0, loopback=True)
    for coll in ([c3.ALL_GATHER] if what == "ag" else [c3.REDUCE_SCATTER] if what == "rs"
                 else [c3.ALL_GATHER, c3.REDUCE_SCATTER]):
        s = c3.Session(wl, 256, 256, 256, coll, 896 << 20)
        s.fill()
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = 148
        for _ in range(2):
            s.run(c3.COMM_ONLY_CU, a)
        s.close()
    wl.close()
if what == "fused":
    n = 8
    wl = c3.World(0, n, 0, loopback=True)
    s = c3.Session(wl, M, N, K, c3.ALL_GATHER, 896 << 20)
    s.fill()
    for _ in range(2):
        s.run(c3.GEMM_ONLY)
        s.run(c3.FUSED)
    s.close()
    wl.close()
