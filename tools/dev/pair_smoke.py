"""Hang-guarded first run of the CTA-pair GEMM: one small and one cfg2 launch,
checked against cuBLAS (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["C3_GEMM_KERNEL"] = sys.argv[1] if len(sys.argv) > 1 else "pair"
import torch
import paper_2412_14335_b200 as c3
w = c3.World()
for (M, N, K) in ((256, 256, 64), (512, 1024, 512), (8192, 28672, 8192)):
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch.matmul(A, B.t())
    print(M, N, K, "max abs diff vs cuBLAS", float((C.float() - ref.float()).abs().max()),
          "equal", bool(torch.equal(C, ref)), flush=True)
