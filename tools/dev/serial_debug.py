"""Raw per-step rows for isolated vs serial steps in different round orders (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2412_14335_b200 as c3
w = c3.World(0, 8, 0, loopback=True)
s = c3.Session(w, 8192, 28672, 8192, c3.ALL_GATHER, 896 << 20)
s.fill()
ga = s.default_alloc(c3.GEMM_ONLY)
ca = s.default_alloc(c3.COMM_ONLY_CU); ca.cus_comm = 148
sa = s.default_alloc(c3.SERIAL)
print("serial alloc", sa.cus_gemm, sa.cus_comm)
def row(st, a):
    t = s.run(st, a)
    return f"tot={t.total_ms:.3f} g={t.gemm_end_ms - t.gemm_start_ms:.3f} c={t.comm_end_ms - t.comm_start_ms:.3f} gs={t.gemm_start_ms:.3f} cs={t.comm_start_ms:.3f}"
for order in (["g", "c", "s"], ["s", "g", "c"], ["g", "s", "c"]):
    print("order", order)
    for r in range(6):
        out = []
        for k in order:
            st, a = {"g": (c3.GEMM_ONLY, ga), "c": (c3.COMM_ONLY_CU, ca), "s": (c3.SERIAL, sa)}[k]
            out.append(k + ":" + row(st, a))
        print("  ", " | ".join(out))
