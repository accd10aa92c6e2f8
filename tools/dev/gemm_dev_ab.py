#!/usr/bin/env python3
"""What would the pair GEMM gain without its DRAM re-reads or its exposed TMEM
drain? (dev A/B). Each mode runs in its own process
(C3_GEMM_DEV is read once): 0 = the product kernel, 1 = every tile loads the
operands of tile (0, 0) (L2-resident operands: no DRAM re-reads), 2 = the
epilogue releases the accumulator undrained (no TMEM drain), 3 = both,
4 = half 0 released as soon as the tile is done (drained after: the half-0
drain hidden), 8 = both halves released early (the whole drain hidden, its
work kept); cuBLAS
beside mode 0. Two regimes: `burst` (one launch after 20 ms idle, median of
15) and `sustained` (300 back-to-back launches, median of the last 150).
Results are invalid outputs for modes 1-3; only the time matters.

usage: python tools/dev/gemm_dev_ab.py [M N K]
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r"""
import json, os, statistics, sys, time
sys.path.insert(0, {repo!r})
import torch
import paper_2412_14335_b200 as c3
M, N, K = {m}, {n}, {k}
w = c3.World()
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
cublas = {cublas}
def run():
    if cublas:
        torch.matmul(A, B.t(), out=C)
    else:
        w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0, st)
for _ in range(5):
    run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
burst = []
for _ in range(15):
    time.sleep(0.02)
    s.record(); run(); e.record(); e.synchronize(); burst.append(s.elapsed_time(e))
evs = [torch.cuda.Event(enable_timing=True) for _ in range(301)]
evs[0].record()
for i in range(300):
    run(); evs[i + 1].record()
torch.cuda.synchronize()
sus = [evs[i].elapsed_time(evs[i + 1]) for i in range(150, 300)]
f = 2.0 * M * N * K
print(json.dumps({{"burst_ms": statistics.median(burst), "sustained_ms": statistics.median(sus),
                  "burst_tflops": f / statistics.median(burst) / 1e9,
                  "sustained_tflops": f / statistics.median(sus) / 1e9}}))
"""


def main():
    m, n, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 28672, 8192)
    out = {}
    modes = (("product", 0, False), ("cublas", 0, False), ("l2_resident", 1, False),
             ("no_drain", 2, False), ("both", 3, False), ("h0_early", 4, False),
             ("all_early", 8, False), ("product_again", 0, False))
    if os.environ.get("C3_DEV_MODES"):  # subset, e.g. "product,h0_early,all_early"
        keep = os.environ["C3_DEV_MODES"].split(",")
        modes = tuple(x for x in modes if x[0] in keep)
    for name, dev, cublas in modes:
        cublas = name == "cublas"
        env = dict(os.environ, C3_GEMM_DEV=str(dev))
        code = CHILD.format(repo=REPO, m=m, n=n, k=k, cublas=cublas)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        out[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-500:]}
        print(name, out[name], flush=True)
    print(json.dumps({"mnk": [m, n, k], "modes": out}))


if __name__ == "__main__":
    main()
