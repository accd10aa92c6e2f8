#!/usr/bin/env python3
"""fp32 split-TF32 GEMM per-CTA timeline (dev aid; needs a build with
NVCC_EXTRA=-DC3_F32_TIMELINE, e.g. `make cuda NVCC_EXTRA=-DC3_F32_TIMELINE`): globaltimer stamps the
kernel writes when C3_F32_DBG holds a device address (gemm_f32.cu):
0 entry, 1 setup done, 2 first stage converted (MMA side), 3 first unit's
MMAs issued, 4 its accumulator ready (epilogue), 5 (last part) the other partials ready,
6 C written (last arriver), 7 CTA done. Printed relative to the earliest
entry, as medians / max over CTAs."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = c3.World()
A, B = torch.randn(M, K, device="cuda"), torch.randn(N, K, device="cuda")
C = torch.empty(M, N, device="cuda")
dbg = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
for it in range(4):
    os.environ["C3_F32_DBG"] = str(dbg.data_ptr()) if it == 3 else ""
    if it < 3:
        os.environ.pop("C3_F32_DBG")
    dbg.zero_()
    torch.cuda.synchronize()
    w.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
t = dbg.view(148, 8).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0).double() / 1e3
names = ["entry", "setup", "first_conv", "mma_issued", "acc_ready", "parts_ready", "c_written", "done"]
for j, nm in enumerate(names):
    col = rel[:, j][t[:, j] > 0]
    if len(col):
        print(f"{nm:16s} n={len(col):3d} min {col.min():7.2f} med {col.median():7.2f} max {col.max():7.2f} us")
w.close()
