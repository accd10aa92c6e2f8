#!/usr/bin/env python3
"""fp32 split-TF32 GEMM timing (dev aid): CUDA-event time per launch over
many back-to-back launches, per shape; run under different C3_F32_DEV values
(subprocesses, since the knob is read once per process).

usage: python tools/dev/f32_ab.py [dev values, comma-separated]"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import json, sys, torch
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3
w = c3.World()
out = {}
for (M, N, K) in [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096)]:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(N, K, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(5):
        w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, dtype_bytes=4)
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, dtype_bytes=4)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    ct = torch.empty(M, N, device="cuda")
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(3): torch.matmul(A, B.t(), out=ct)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): torch.matmul(A, B.t(), out=ct)
    e1.record(); torch.cuda.synchronize()
    tf32_us = e0.elapsed_time(e1) / reps * 1e3
    out[f"{M}x{N}x{K}"] = {"us": us, "tflops": 2 * M * N * K / us / 1e6, "cublas_tf32_us": tf32_us}
print(json.dumps(out))
'''.replace("REPO", repr(REPO))

devs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"]
for d in devs:
    env = dict(os.environ, C3_F32_DEV=d)
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env)
    print(json.dumps({"C3_F32_DEV": d, "res": json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]}))
