"""Does pacing the collective below the link rate (spreading it over the
GEMM) shorten the co-resident C3 step? cfg2 loopback, c3_base on all SMs +
c CTA units; serial reference at the link rate. Dev probe.
python tools/dev/pace_probe.py [ag|a2a|rs] [ctas] [rates,...]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ag"
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 24
rates = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [770, 600, 500, 400, 350]
coll = {"ag": c3.ALL_GATHER, "a2a": c3.ALL_TO_ALL, "rs": c3.REDUCE_SCATTER}[kind]
w = c3.World(0, 8, 0, loopback=True)
s = c3.Session(w, 8192, 28672, 8192, coll, 896 << 20)
s.fill()
g = s.default_alloc(c3.GEMM_ONLY)
cm = s.default_alloc(c3.COMM_ONLY_CU)
cm.cus_comm = ctas
b = s.default_alloc(c3.C3_BASE)
b.cus_gemm, b.cus_comm = 148, ctas
jobs = [("gemm", c3.GEMM_ONLY, g, 770.0), ("comm770", c3.COMM_ONLY_CU, cm, 770.0)]
jobs += [(f"c3_base@{r:.0f}", c3.C3_BASE, b, r) for r in rates]
res = {}
for r in range(9):
    for name, st, al, rate in jobs[r % len(jobs):] + jobs[:r % len(jobs)]:
        s.set_link_rate(rate)
        t = s.run(st, al).total_ms
        if r:
            res.setdefault(name, []).append(t)
tg, tc = statistics.median(res["gemm"]), statistics.median(res["comm770"])
ideal = (tg + tc) / max(tg, tc)
print(f"{kind} c{ctas} gemm {tg:.4f} comm@770 {tc:.4f} ideal {ideal:.3f}")
for name in res:
    if name.startswith("c3_base"):
        t = statistics.median(res[name])
        sp = (tg + tc) / t
        print(f"  {name:14s} {t:.4f} ms  speedup {sp:.3f}  frac {(sp - 1) / (ideal - 1):.2f}")
s.close()
w.close()
