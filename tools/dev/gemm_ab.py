"""A/B GEMM timing in one process (dev aid): python tools/dev/gemm_ab.py M N K [reps]."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2412_14335_b200 as c3
M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
w = c3.World()
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t_ours():
    w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, st)
def t_cublas():
    torch.matmul(A, B.t(), out=C)
res = {"ours": [], "cublas": []}
for _ in range(3):
    t_ours(); t_cublas()
for i in range(reps):  # interleaved so clocks affect both alike
    for name, fn in (("ours", t_ours), ("cublas", t_cublas)):
        s.record(); fn(); e.record(); e.synchronize(); res[name].append(s.elapsed_time(e))
f = 2 * M * N * K
print({k: (round(statistics.median(v), 4), round(f / statistics.median(v) / 1e9, 1)) for k, v in res.items()},
      os.environ.get("C3_GEMM_SCHED", "dynamic"))
