#!/usr/bin/env python3
"""Observed GEMM error against the fp64 definition, normalised by sum |a||b|
(the accumulation term of the stated tolerances): bf16 kernels (every
variant) and the fp32 split-TF32 kernel, plus the fraction of bf16 outputs
equal to the correctly rounded value. Sets the margin of the tolerances in
tests/_oracle.py and tests/test_gpu_parity.py.

usage: python tools/dev/gemm_err_probe.py
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402
from tests import _oracle as orc  # noqa: E402

SEED = 20241217
out = {}
w = c3.World()
rng = np.random.default_rng(1)
for kern in ("pair512", "pair", "wide", "narrow"):
    os.environ["C3_GEMM_KERNEL"] = kern
    for (M, N, K) in ((1024, 2048, 8192), (512, 1024, 16384)):
        A = torch.empty(M * K, dtype=torch.int16, device="cuda")
        B = torch.empty(N * K, dtype=torch.int16, device="cuda")
        Cm = torch.zeros(M * N, dtype=torch.int16, device="cuda")
        c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, SEED, 0, 0, None))
        c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, SEED, 0, 1, None))
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K)
        torch.cuda.synchronize()
        rows, cols = rng.integers(0, M, 20000), rng.integers(0, N, 20000)
        Ah, Bh = orc.bf16(M * K, SEED, 0, 0), orc.bf16(N * K, SEED, 0, 1)
        ref, mag = orc.gemm_samples(Ah, Bh, M, N, K, rows, cols)
        bits = Cm.cpu().numpy().view(np.uint16)[rows * N + cols]
        got = orc.bf16_to_f32(bits).astype(np.float64)
        exact = float(np.mean(bits == orc.f64_to_bf16_bits(ref)))
        excess = np.maximum(np.abs(got - ref) - 2.0 ** -8 * np.abs(ref), 0) / mag
        out[f"bf16 {kern} {M}x{N}x{K}"] = {"exact_frac": exact,
                                           "max_excess_over_mag_log2": float(np.log2(max(excess.max(), 1e-300))),
                                           "max_rel_err": float((np.abs(got - ref) / np.abs(ref)).max())}
        print(out[f"bf16 {kern} {M}x{N}x{K}"], kern, M, N, K, flush=True)
os.environ.pop("C3_GEMM_KERNEL")
g = torch.Generator().manual_seed(3)
for (M, N, K) in ((1024, 1024, 1024), (512, 768, 4096)):
    Ah = torch.randn(M, K, generator=g) * torch.exp2(torch.randint(-6, 7, (M, 1), generator=g).float())
    Bh = torch.randn(N, K, generator=g)
    Cm = torch.empty(M, N, dtype=torch.float32, device="cuda")
    Ad, Bd = Ah.cuda(), Bh.cuda()  # alive across the launch
    w.gemm(Ad.data_ptr(), Bd.data_ptr(), Cm.data_ptr(), M, N, K, dtype_bytes=4)
    torch.cuda.synchronize()
    A64, B64 = Ah.double().numpy(), Bh.double().numpy()
    ref = A64 @ B64.T
    mag = np.abs(A64) @ np.abs(B64).T
    e = np.abs(Cm.cpu().numpy().astype(np.float64) - ref) / mag
    f32 = (Ah.numpy() @ Bh.numpy().T).astype(np.float64)
    e32 = np.abs(f32 - ref) / mag
    torch.backends.cuda.matmul.allow_tf32 = True
    t32 = (Ah.cuda() @ Bh.cuda().T).cpu().numpy().astype(np.float64)
    torch.backends.cuda.matmul.allow_tf32 = False
    et = np.abs(t32 - ref) / mag
    r = {"split_tf32_max_log2": float(np.log2(e.max())), "split_tf32_rms_log2": float(np.log2(np.sqrt(np.mean(e ** 2)))),
         "host_fp32_max_log2": float(np.log2(e32.max())), "host_fp32_rms_log2": float(np.log2(np.sqrt(np.mean(e32 ** 2)))),
         "cublas_tf32_max_log2": float(np.log2(et.max())), "cublas_tf32_rms_log2": float(np.log2(np.sqrt(np.mean(et ** 2))))}
    out[f"fp32 {M}x{N}x{K}"] = r
    print(r, M, N, K, flush=True)
print(json.dumps(out))
