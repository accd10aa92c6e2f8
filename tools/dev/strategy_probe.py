"""Grid of (strategy, GEMM CTA cap, comm CTAs) on the cfg2 loopback session:
measures whether comm CTAs co-resident with the persistent GEMM's CTAs beat
SM partitioning. Development probe; prints JSON."""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402


def main():
    coll = c3.REDUCE_SCATTER if len(sys.argv) > 1 and sys.argv[1] == "rs" else c3.ALL_GATHER
    payload = (int(sys.argv[2]) if len(sys.argv) > 2 else 896) << 20
    w = c3.World(0, 8, 0, loopback=True)
    s = c3.Session(w, 8192, 28672, 8192, coll, payload)
    s.fill()

    def med(strat, a, n=7):
        ts = [s.run(strat, a) for _ in range(n)]
        return (statistics.median(t.total_ms for t in ts[1:]),
                statistics.median(t.gemm_end_ms - t.gemm_start_ms for t in ts[1:]),
                statistics.median(t.comm_end_ms - t.comm_start_ms for t in ts[1:]))

    out = {}
    a = s.default_alloc(c3.GEMM_ONLY)
    out["gemm_only"] = med(c3.GEMM_ONLY, a)
    for ctas in (64, 148):
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = ctas
        out[f"comm_only_{ctas}"] = med(c3.COMM_ONLY_CU, a)
    for strat in (c3.C3_BASE,):
        for gemm in (148,):
            for ctas in (32, 64, 148):
                a = s.default_alloc(strat)
                a.cus_gemm, a.cus_comm = gemm, ctas
                out[f"{c3.STRATEGY_NAMES[strat]}_g{gemm}_c{ctas}"] = med(strat, a)
    for piece in (0, 2048, 4096, 8192):
        for pace in (0.0,):
            s.set_fused_pace(pace, piece)
            out[f"fused_piece{piece}_pace{pace}"] = med(c3.FUSED, s.default_alloc(c3.FUSED))
    for ctas in (8, 16, 32):
        a = s.default_alloc(c3.C3_RP)
        a.cus_gemm, a.cus_comm = 148 - ctas, ctas
        out[f"c3_rp_c{ctas}"] = med(c3.C3_RP, a)
    s.close()
    w.close()
    print(json.dumps({k: [round(x, 4) for x in v] for k, v in out.items()}, indent=0))


if __name__ == "__main__":
    main()
