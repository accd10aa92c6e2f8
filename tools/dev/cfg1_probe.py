#!/usr/bin/env python3
"""configs[0] step anatomy (dev aid): the fp32 1024^3 GEMM (split-TF32) and
the 16 MiB world-2 all-gather, isolated and as c3_base, interleaved; per run
the event times inside the step (GEMM start/end, collective start/end, total).

usage: python tools/dev/cfg1_probe.py [rounds]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 30
w = c3.World(0, 2, 0, loopback=True)
s = c3.Session(w, 1024, 1024, 1024, c3.ALL_GATHER, 16 << 20, dtype_bytes=4)
s.fill(20241217)
s.set_link_rate(770.0)
g = s.default_alloc(c3.GEMM_ONLY)
cu = s.default_alloc(c3.COMM_ONLY_CU)
cu.cus_comm = 16
jobs = {"gemm": (c3.GEMM_ONLY, g)}
jobs["comm16"] = (c3.COMM_ONLY_CU, cu)
for ctas, pace in ((8, 311.4), (16, 0.0), (32, 0.0)):
    a = s.default_alloc(c3.C3_BASE)
    a.cus_gemm, a.cus_comm, a.comm_pace_gbps = 148, ctas, pace
    jobs[f"c3_base{ctas}" + (f"p{pace:.0f}" if pace else "")] = (c3.C3_BASE, a)
rows = {k: [] for k in jobs}
for _ in range(5):
    for k, (st, a) in jobs.items():
        s.run(st, a)
for _ in range(R):
    for k, (st, a) in jobs.items():
        t = s.run(st, a)
        rows[k].append((t.total_ms, t.gemm_start_ms, t.gemm_end_ms, t.comm_start_ms, t.comm_end_ms, t.launches))
for k, rs in rows.items():
    tot = [r[0] for r in rs]
    print(f"{k:16s} total med {statistics.median(tot) * 1e3:7.1f} us  min {min(tot) * 1e3:7.1f}  max {max(tot) * 1e3:7.1f}"
          f"  gemm [{statistics.median([r[1] for r in rs]) * 1e3:.1f}, {statistics.median([r[2] for r in rs]) * 1e3:.1f}]"
          f"  comm [{statistics.median([r[3] for r in rs]) * 1e3:.1f}, {statistics.median([r[4] for r in rs]) * 1e3:.1f}]"
          f"  launches {rs[0][5]}")
    print("   totals:", " ".join(f"{x * 1e3:.0f}" for x in tot))
s.close()
w.close()
