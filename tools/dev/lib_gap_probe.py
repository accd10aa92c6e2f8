#!/usr/bin/env python3
"""Why does cuBLAS || torch copies sometimes finish its concurrent step before
ours at full local speed? Decomposes the comparison:
every job below runs in rotated rounds (same power states), device-event
timed, medians.

  ours_gemm / cublas_gemm           the GEMMs alone
  ours_comm / torch_copies          this GPU's share of the 8-rank all-gather alone
  ours_step:<variant>               our C3 step (full-speed candidates)
  lib_step                          cuBLAS || torch copies (the library baseline)
  ours_gemm+torch_copies            our GEMM beside the library's copies
  cublas+ours_comm:<units>          cuBLAS beside our collective

usage: python tools/dev/lib_gap_probe.py [cfg] [rounds]
"""
import ctypes as C
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def main():
    import torch

    import paper_2412_14335_b200 as c3
    from bench import CONFIGS
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    cfg = CONFIGS[name]
    n = 8
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, cfg["m"], cfg["n"], cfg["k"], c3.ALL_GATHER, cfg["payload"])
    s.fill()
    full = w.info.sm_count
    p = s.pointers(0)
    chunk = cfg["payload"] // n
    dev = torch.device("cuda", 0)
    A = torch.randn(cfg["m"], cfg["k"], device=dev, dtype=torch.bfloat16)
    B = torch.randn(cfg["n"], cfg["k"], device=dev, dtype=torch.bfloat16)
    Cc = torch.empty(cfg["m"], cfg["n"], device=dev, dtype=torch.bfloat16)
    src = torch.empty(chunk, dtype=torch.uint8, device=dev)
    dst = torch.empty(n * chunk, dtype=torch.uint8, device=dev)
    sg, sc = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    recv = [s.pointers(v).recv for v in range(n)]  # the 8 virtual ranks' buffers

    def copies():
        for q in range(1, n):
            dst[q * chunk:(q + 1) * chunk].copy_(src)

    def ours_gemm_on(stream):
        w.gemm(p.a, p.b, p.c, cfg["m"], cfg["n"], cfg["k"], 0, C.c_void_p(stream.cuda_stream))

    def ours_comm_on(stream, units):
        # rank 0's share: 7 chunk stores into stand-in peer slots of its own buffer
        w.allgather_p2p(0, p.recv, recv, chunk, units, C.c_void_p(stream.cuda_stream))

    def pair(g, c):
        torch.cuda.synchronize()
        ev[0].record()
        sg.wait_event(ev[0])
        sc.wait_event(ev[0])
        if g:
            g(sg)
        if c:
            c(sc)
        torch.cuda.current_stream().wait_stream(sg)
        torch.cuda.current_stream().wait_stream(sc)
        ev[1].record()
        ev[1].synchronize()
        return ev[0].elapsed_time(ev[1])

    def cublas(stream):
        with torch.cuda.stream(stream):
            torch.matmul(A, B.t(), out=Cc)

    def torch_copies(stream):
        with torch.cuda.stream(stream):
            copies()

    jobs = {
        "ours_gemm": lambda: pair(ours_gemm_on, None),
        "cublas_gemm": lambda: pair(cublas, None),
        "ours_comm148": lambda: pair(None, lambda st: ours_comm_on(st, full)),
        "torch_copies": lambda: pair(None, torch_copies),
        "lib_step": lambda: pair(cublas, torch_copies),
        "ours_gemm+torch_copies": lambda: pair(ours_gemm_on, torch_copies),
    }
    for units in (8, 16, 32):
        jobs[f"cublas+ours_comm{units}"] = (lambda u: lambda: pair(cublas, lambda st: ours_comm_on(st, u)))(units)
        jobs[f"ours_gemm+ours_comm{units}"] = (lambda u: lambda: pair(ours_gemm_on, lambda st: ours_comm_on(st, u)))(units)
    for st, units in ((c3.C3_BASE, 8), (c3.C3_BASE, 16), (c3.C3_BASE, 32), (c3.C3_SP, 16)):
        a = s.default_alloc(st)
        a.cus_gemm, a.cus_comm = full, units
        jobs[f"ours_step:{c3.STRATEGY_NAMES[st]}{units}"] = (lambda st_, a_: lambda: s.run(st_, a_).total_ms)(st, a)
    jobs["ours_step:fused"] = lambda: s.run(c3.FUSED).total_ms
    jobs["ours_step:serial"] = lambda: s.run(c3.SERIAL).total_ms
    t = {k: [] for k in jobs}
    names = list(jobs)
    for r in range(R + 2):
        for k in names[r % len(names):] + names[:r % len(names)]:
            v = jobs[k]()
            if r >= 2:
                t[k].append(v)
    out = {k: {"median": statistics.median(v), "min": min(v), "max": max(v)} for k, v in t.items()}
    print(json.dumps({"config": name, "rounds": R, "ms": out}, indent=1))


if __name__ == "__main__":
    main()
