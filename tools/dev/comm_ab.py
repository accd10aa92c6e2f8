"""Full-speed loopback collective throughput vs CTA count (dev aid).
python tools/dev/comm_ab.py [ag|a2a|rs] [payload_MiB] -> one line per CTA count:
median ms, per-GPU HBM bytes (read + write) / time, and fraction of the
measured HBM copy peak (MEASURED_PEAKS.json)."""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "ag"
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 896
ctas = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [24, 48, 74, 148, 296, 444, 592]
coll = {"ag": c3.ALL_GATHER, "a2a": c3.ALL_TO_ALL, "rs": c3.REDUCE_SCATTER}[kind]
n, P = 8, mib << 20
try:
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6550.0
# per-GPU HBM bytes of this rank's share: AG reads its chunk once and writes it n-1 times;
# A2A reads n-1 slots and writes n-1; RS reads n slots of P/n and writes one
hbm = {"ag": P / n * n, "a2a": 2 * P / n * (n - 1), "rs": P + P / n}[kind]
w = c3.World(0, n, 0, loopback=True)
s = c3.Session(w, 256, 256, 256, coll, P)
s.fill()
a = s.default_alloc(c3.COMM_ONLY_CU)
res = {}
for c in ctas:
    a.cus_comm = c
    for _ in range(3):
        s.run(c3.COMM_ONLY_CU, a)
for r in range(7):  # interleaved rounds
    for c in ctas:
        a.cus_comm = c
        res.setdefault(c, []).append(s.run(c3.COMM_ONLY_CU, a).total_ms)
for c in ctas:
    t = statistics.median(res[c])
    print(f"{kind} {mib}MiB ctas={c:4d} {t:.4f} ms  {hbm / t / 1e6:7.1f} GB/s  {hbm / t / 1e6 / peak:.3f} of HBM"
          f"  L2={os.environ.get('C3_COMM_L2', 'evict_first')}")
s.close()
w.close()
