"""Small invocations of every kernel family for compute-sanitizer (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("C3_GEMM_KERNEL", "pair")
import paper_2412_14335_b200 as c3
for coll in (c3.ALL_GATHER, c3.ALL_TO_ALL, c3.REDUCE_SCATTER):
    w = c3.World(0, 4, 0, loopback=True)
    s = c3.Session(w, 512, 1024, 256, coll, 4 * (64 << 10))
    s.fill()
    strats = [c3.SERIAL, c3.C3_SP, c3.CONCCL, c3.COMM_ONLY_CU]
    if coll != c3.REDUCE_SCATTER:
        strats.append(c3.FUSED)
    for st in strats:
        s.run(st, all_ranks=True)
    s.close()
    w.close()
print("sanitize target done")
if os.environ.get("C3_SANITIZE_F32", "1") == "1":
    # the fp32 split-TF32 kernel: split-K S = 4 and 3 (workspace), S = 1, S = 2 (TMA add), a non-finite stage
    import torch
    w = c3.World()
    for (M, N, K) in ((256, 256, 256), (300, 520, 200), (512, 1024, 64), (1024, 1024, 128)):
        A = torch.randn(M, K, device="cuda")
        B = torch.randn(N, K, device="cuda")
        A[1, 3] = float("inf")
        C = torch.empty(M, N, device="cuda")
        w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    w.close()
    print("sanitize f32 done")
