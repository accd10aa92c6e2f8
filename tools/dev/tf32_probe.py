"""fp32 GEMM on the TF32 tensor cores (c3_gemm_f32) against cuBLAS TF32
(torch.matmul with allow_tf32) on the same device buffers: interleaved,
event-timed medians. Dev probe: python tools/dev/tf32_probe.py [M N K]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402


def main():
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 8192)
    torch.backends.cuda.matmul.allow_tf32 = True
    w = c3.World()
    A = torch.empty(M, K, dtype=torch.float32, device="cuda")
    B = torch.empty(N, K, dtype=torch.float32, device="cuda")
    C1 = torch.empty(M, N, dtype=torch.float32, device="cuda")
    c3.check(c3.lib().c3_fill_f32(A.data_ptr(), M * K, 20241217, 0, 0, None))
    c3.check(c3.lib().c3_fill_f32(B.data_ptr(), N * K, 20241217, 0, 1, None))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def ours():
        w.gemm(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, 0, torch.cuda.current_stream().cuda_stream,
               dtype_bytes=4)

    def cublas():
        torch.matmul(A, B.t(), out=C1)

    t = {"c3_gemm_f32": [], "cublas_tf32": []}
    fns = {"c3_gemm_f32": ours, "cublas_tf32": cublas}
    for r in range(13):
        for k in (list(fns) if r % 2 == 0 else list(fns)[::-1]):
            torch.cuda.synchronize()
            ev[0].record()
            fns[k]()
            ev[1].record()
            ev[1].synchronize()
            if r >= 3:
                t[k].append(ev[0].elapsed_time(ev[1]))
    for k, v in t.items():
        ms = statistics.median(v)
        print(f"{k}: {M}x{N}x{K} {ms:.3f} ms {2.0 * M * N * K / ms / 1e9:.1f} TFLOP/s")
    w.close()


if __name__ == "__main__":
    main()
