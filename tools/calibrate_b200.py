"""Measure the B200 interference tables the runtime heuristic uses
(reference SlowdownTable, interference.hpp:18-28; CSV format of
proj/data/slowdown-tables.csv): isolated kernel time vs SMs available.

  gemm-compute-bound : 8192x28672x8192 GEMM, CTA cap c (= SMs it runs on)
  gemm-memory-bound  : 128x53248x16384 GEMM, CTA cap c
  all-gather         : loopback 8-rank push all-gather 896 MiB, c CTAs
  all-to-all         : loopback 8-rank pull reduce-scatter 896 MiB, c CTAs
                       (reduce-scatter maps to the all-to-all kernel class)

slowdown(c) = t(c) / t(148); points at grain-4 multiples, last point 1.0.
Writes data/b200-loopback-slowdown-tables.csv and a JSON of raw times.
usage: python tools/calibrate_b200.py [out_dir]
"""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402

CAPS = [4, 8, 12, 16, 24, 32, 48, 64, 80, 96, 112, 120, 128, 136, 140, 144, 148]


def ev_time(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def gemm_curve(w, M, N, K):
    A = torch.empty(M * K, dtype=torch.int16, device="cuda")
    B = torch.empty(N * K, dtype=torch.int16, device="cuda")
    Cm = torch.empty(M * N, dtype=torch.int16, device="cuda")
    c3.check(c3.lib().c3_fill_bf16(A.data_ptr(), M * K, 1, 0, 0, None))
    c3.check(c3.lib().c3_fill_bf16(B.data_ptr(), N * K, 1, 0, 1, None))
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    for cap in CAPS:
        out[cap] = ev_time(lambda: w.gemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), M, N, K, cap,
                                          st), reps=3 if cap < 32 else 5)
    return out


def comm_curve(coll):
    wl = c3.World(0, 8, 0, loopback=True)
    s = c3.Session(wl, 256, 256, 256, coll, 896 << 20)
    s.fill()
    out = {}
    for cap in CAPS:
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = cap
        ts = [s.run(c3.COMM_ONLY_CU, a).comm_end_ms for _ in range(6)]
        out[cap] = statistics.median(ts[1:])
    s.close()
    wl.close()
    return out


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "data")
    os.makedirs(out_dir, exist_ok=True)
    w = c3.World()
    raw = {"gemm-compute-bound": gemm_curve(w, 8192, 28672, 8192),
           "gemm-memory-bound": gemm_curve(w, 128, 53248, 16384)}
    w.close()
    raw["all-gather"] = comm_curve(c3.ALL_GATHER)
    raw["all-to-all"] = comm_curve(c3.REDUCE_SCATTER)
    lines = ["kernel_class,cus,slowdown"]
    for cls in ("gemm-compute-bound", "gemm-memory-bound", "all-gather", "all-to-all"):
        full = raw[cls][148]
        for cap in CAPS:
            slow = 1.0 if cap == 148 else raw[cls][cap] / full
            lines.append(f"{cls},{cap},{slow:.6g}")
    csv_path = os.path.join(out_dir, "b200-loopback-slowdown-tables.csv")
    with open(csv_path, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(out_dir, "b200-calibration-raw.json"), "w") as f:
        json.dump({k: {str(c): v for c, v in d.items()} for k, d in raw.items()}, f, indent=1)
    print(open(csv_path).read())


if __name__ == "__main__":
    main()
