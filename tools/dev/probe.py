"""Quick device probe: GEMM TFLOP/s (ours vs cuBLAS via torch), world info,
and loopback collective bandwidths. Development aid; numbers here are not
bench values."""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402


def time_fn(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    out = {}
    w = c3.World()
    info = w.info
    out["world"] = {f: getattr(info, f) for f, _ in info._fields_}
    shapes = [(8192, 28672, 8192), (8192, 8192, 8192), (128, 53248, 16384)]
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        shapes.append((8192, 53248, 16384))
    for (M, N, K) in shapes:
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16) * 0.1
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.1
        Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        flops = 2 * M * N * K
        res = {}
        for cap in (0, 132, 116):
            ms = time_fn(lambda: w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, cap,
                                        torch.cuda.current_stream().cuda_stream))
            res[f"ours_cap{cap}_ms"] = ms
            res[f"ours_cap{cap}_tflops"] = flops / ms / 1e9
        ms = time_fn(lambda: torch.matmul(A, B.t(), out=Cm))
        res["cublas_ms"] = ms
        res["cublas_tflops"] = flops / ms / 1e9
        ref = torch.matmul(A, B.t()).float()
        w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, 0,
               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        res["max_rel_err_vs_cublas"] = float(((Cm.float() - ref).abs().max() / ref.abs().max()))
        out[f"gemm_{M}x{N}x{K}"] = res
        del A, B, Cm
    w.close()
    # loopback collectives: rank 0's share (the per-GPU load) at n = 8
    n = 8
    wl = c3.World(0, n, 0, loopback=True)
    for mib in (16, 896):
        payload = mib << 20
        for coll in (c3.ALL_GATHER, c3.REDUCE_SCATTER):
            s = c3.Session(wl, 1024, 1024, 1024, coll, payload)
            s.fill()
            r = {}
            for strat in (c3.COMM_ONLY_CU, c3.COMM_ONLY_DMA):
                for ctas in (16, 32, 64, 148):
                    a = s.default_alloc(strat)
                    a.cus_comm = ctas
                    ts = []
                    for _ in range(8):
                        ts.append(s.run(strat, a).comm_end_ms)
                    ts.sort()
                    ms = ts[len(ts) // 2]
                    moved = (n - 1) / n * payload
                    r[f"{c3.STRATEGY_NAMES[0] if False else strat}_{ctas}"] = {
                        "ms": ms, "GBps_moved": moved / ms / 1e6}
                    if strat == c3.COMM_ONLY_DMA:
                        break
            out[f"loopback_{'ag' if coll == 0 else 'rs'}_{mib}MiB"] = r
            s.close()
    wl.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    t0 = time.time()
    main()
    print("probe wall", time.time() - t0, file=sys.stderr)
