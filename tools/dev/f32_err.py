#!/usr/bin/env python3
"""fp32 GEMM error vs the fp64 definition, normalised by |A||B| (dev aid)."""
import json, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import numpy as np, torch  # noqa: E402
import paper_2412_14335_b200 as c3  # noqa: E402
M, N, K = 512, 768, 1024
g = torch.Generator().manual_seed(3)
A = torch.randn(M, K, generator=g) * torch.exp2(torch.randint(-6, 7, (M, 1), generator=g).float())
B = torch.randn(N, K, generator=g)
w = c3.World()
C = torch.empty(M, N, device="cuda")
Ad, Bd = A.cuda(), B.cuda()
w.gemm(Ad.data_ptr(), Bd.data_ptr(), C.data_ptr(), M, N, K, dtype_bytes=4)
torch.cuda.synchronize()
ref = A.double().numpy() @ B.double().numpy().T
mag = np.abs(A.double().numpy()) @ np.abs(B.double().numpy()).T
e = np.abs(C.cpu().double().numpy() - ref) / mag
print(json.dumps({"dev": os.environ.get("C3_F32_DEV", "0"), "rms_log2": float(np.log2(np.sqrt(np.mean(e ** 2)))),
                  "max_log2": float(np.log2(e.max())), "mean_signed_log2": float(np.log2(abs(np.mean((C.cpu().double().numpy() - ref) / mag)) + 1e-300))}))
