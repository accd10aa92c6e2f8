"""C3_FUSED vs co-resident c3_base on the cfg2 loopback session at a link rate
(dev probe): python tools/dev/fused_probe.py [ag|a2a] [link_gbps] [pieces,...]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ag"
link = float(sys.argv[2]) if len(sys.argv) > 2 else 770.0
pieces = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2048, 4096, 8192]
coll = {"ag": c3.ALL_GATHER, "a2a": c3.ALL_TO_ALL}[kind]
w = c3.World(0, 8, 0, loopback=True)
s = c3.Session(w, 8192, 28672, 8192, coll, 896 << 20)
s.fill()
s.set_link_rate(link)
jobs = [("gemm", c3.GEMM_ONLY, None, None)]
a = s.default_alloc(c3.COMM_ONLY_CU)
a.cus_comm = 148
jobs.append(("comm", c3.COMM_ONLY_CU, a, None))
for c in (24, 48):
    b = s.default_alloc(c3.C3_BASE)
    b.cus_gemm, b.cus_comm = 148, c
    jobs.append((f"c3_base_c{c}", c3.C3_BASE, b, None))
for pc in pieces + [0]:
    jobs.append((f"fused_piece{pc}" if pc else "fused_lsu", c3.FUSED, s.default_alloc(c3.FUSED), pc))
res = {}
for r in range(8):
    for name, st, al, pc in jobs[r % len(jobs):] + jobs[:r % len(jobs)]:
        if pc is not None:
            s.set_fused_pace(0.0, pc)
        t = s.run(st, al).total_ms
        if r:
            res.setdefault(name, []).append(t)
tg, tc = statistics.median(res["gemm"]), statistics.median(res["comm"])
ideal = (tg + tc) / max(tg, tc)
print(f"{kind} link={link} gemm {tg:.4f} comm {tc:.4f} ideal {ideal:.3f}")
for name in res:
    if name in ("gemm", "comm"):
        continue
    t = statistics.median(res[name])
    sp = (tg + tc) / t
    print(f"  {name:16s} {t:.4f} ms  speedup {sp:.3f}  frac {max(0.0, (sp - 1) / (ideal - 1)):.2f}")
s.close()
w.close()
