"""Co-resident C3 (GEMM on all SMs + comm CTAs beside it) on the cfg2 loopback
session, interleaved rounds, for the collective implementation selected by the
environment (C3_COMM_IMPL etc.). Dev probe.
python tools/dev/coresident_ab.py [ag|a2a|rs] [link_gbps (0 = full speed)] [ctas,...]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ag"
link = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
ctas = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [16, 24, 32, 64, 148]
coll = {"ag": c3.ALL_GATHER, "a2a": c3.ALL_TO_ALL, "rs": c3.REDUCE_SCATTER}[kind]
w = c3.World(0, 8, 0, loopback=True)
s = c3.Session(w, 8192, 28672, 8192, coll, 896 << 20)
s.fill()
if link > 0:
    s.set_link_rate(link)
jobs = [("gemm", c3.GEMM_ONLY, None)]
for c in ctas:
    for name, strat in (("comm", c3.COMM_ONLY_CU), ("c3_base", c3.C3_BASE), ("c3_sp", c3.C3_SP)):
        a = s.default_alloc(strat)
        a.cus_gemm, a.cus_comm = 148, c
        jobs.append((f"{name}_c{c}", strat, a))
res = {}
for _ in range(2):
    for name, strat, a in jobs:
        s.run(strat, a)
for r in range(7):
    order = jobs[r % len(jobs):] + jobs[:r % len(jobs)]
    for name, strat, a in order:
        res.setdefault(name, []).append(s.run(strat, a).total_ms)
med = {k: statistics.median(v) for k, v in res.items()}
tg = med["gemm"]
impl = os.environ.get("C3_COMM_IMPL", "lsu") + " " + os.environ.get("C3_COMM_PIECE", "") + \
    " " + os.environ.get("C3_COMM_NBUF", "")
print(f"[{impl}] {kind} link={link} gemm {tg:.4f} ms")
for c in ctas:
    tc = med[f"comm_c{c}"]
    ideal = (tg + tc) / max(tg, tc)
    for name in ("c3_base", "c3_sp"):
        t = med[f"{name}_c{c}"]
        sp = (tg + tc) / t
        fr = (sp - 1) / (ideal - 1) if sp > 1 else 0.0
        print(f"  c{c:3d} comm {tc:.4f}  {name:7s} {t:.4f} ms  speedup {sp:.3f}  ideal {ideal:.3f}  frac {fr:.2f}")
s.close()
w.close()
