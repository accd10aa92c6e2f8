"""GEMM kernel variants A/B in one process (dev aid): our CTA-pair 256x256 and
256x512 kernels and cuBLAS (torch.matmul), in two regimes:
  burst      one launch per variant, interleaved, 20 rounds (cool GPU);
  sustained  each variant back to back for ~0.4 s, alternating, 3 rounds
             (the 1 kW power cap engages, as in bench.py's timed region).
usage: python tools/dev/gemm_variant_ab.py M N K [variants=pair,pair512,cublas]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
variants = sys.argv[4].split(",") if len(sys.argv) > 4 else ["pair", "pair512", "cublas"]
w = c3.World()
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
ref = torch.matmul(A, B.t())


def launch(v):
    if v == "cublas":
        torch.matmul(A, B.t(), out=C)
    else:
        os.environ["C3_GEMM_KERNEL"] = v
        w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, st)


for v in variants:  # warm-up + a correctness spot check
    launch(v)
    torch.cuda.synchronize()
    err = (C.float() - ref.float()).abs().max().item() / ref.float().abs().max().item()
    assert err < 1e-2, (v, err)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(400)]
f = 2.0 * M * N * K
burst = {v: [] for v in variants}
for r in range(20):
    for v in variants[r % len(variants):] + variants[:r % len(variants)]:
        s, e = ev[0]
        s.record()
        launch(v)
        e.record()
        e.synchronize()
        burst[v].append(s.elapsed_time(e))
sus = {v: [] for v in variants}
for r in range(3):
    for v in variants[r % len(variants):] + variants[:r % len(variants)]:
        n = max(20, int(400 / max(statistics.median(burst[v]), 0.05)))
        n = min(n, len(ev))
        for i in range(n):
            ev[i][0].record()
            launch(v)
            ev[i][1].record()
        torch.cuda.synchronize()
        ts = [ev[i][0].elapsed_time(ev[i][1]) for i in range(n)]
        sus[v] += ts[n // 2:]  # the settled second half
for v in variants:
    b, s_ = statistics.median(burst[v]), statistics.median(sus[v])
    print(f"{M}x{N}x{K} {v:8s} burst {b:.4f} ms {f / b / 1e9:7.1f} TF/s   sustained {s_:.4f} ms {f / s_ / 1e9:7.1f} TF/s")
w.close()
