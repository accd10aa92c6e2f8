#!/usr/bin/env python3
"""ConCCL strategies measured on ONE GPU through the host-staged copy-engine
proxy ("PCIe-rate CE proxy", c3_session_set_ce_proxy): conccl and conccl_rp
(the reference's DMA strategies, sim.cpp:40-100 / strategy.cpp:96-113) beside
a compute-bound and a memory-bound GEMM, with this GPU's share of an 8-rank
collective on the copy engines (7 transfers out D2H, 7 in H2D: the real
node's per-GPU HBM traffic, at PCIe's ~48 GB/s per direction instead of
NVLink's). Payloads are sized so the collective takes a fraction to a
multiple of the GEMM.

Reports, per scenario, the reference sweep schema plus measured columns:
  t_gemm_iso_ms, t_comm_dma_ms        isolated GEMM / proxy collective
  gemm_ms_in_step                     the GEMM inside the C3 step
  gemm_slowdown                       gemm_ms_in_step / t_gemm_iso_ms: the GEMM's
                                      co-run penalty beside copy-engine traffic
                                      (the DMA column of CoRunPenalty,
                                      interference.cpp:178-190)
  predicted_makespan_s                the model's prediction (c3_session_predict)
speedup = (t_gemm_iso + t_comm_dma) / makespan (the same backend's isolated
collective, north_star).

usage: python tools/ce_proxy_sweep.py OUT.csv [rounds]
"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

MIB = 1 << 20
KIND = {"all-gather": c3.ALL_GATHER, "all-to-all": c3.ALL_TO_ALL, "reduce-scatter": c3.REDUCE_SCATTER}
GEMMS = {"cb": (8192, 28672, 8192), "mb": (128, 53248, 16384)}
SCENARIOS = ([("cb", c, p) for c in ("all-gather", "all-to-all", "reduce-scatter") for p in (32, 64, 128, 256)] +
             [("mb", "all-gather", p) for p in (8, 16, 32, 64)])
WORLD = "loopback-8-ce-proxy-pcie"


def main():
    out_path = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    rows = ["scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal,"
            "t_gemm_iso_ms,t_comm_dma_ms,gemm_ms_in_step,gemm_slowdown,cus_gemm,cus_comm,cus_idle,backend,"
            "world,predicted_makespan_s"]
    for shape, coll, pmib in SCENARIOS:
        m, n, k = GEMMS[shape]
        w = c3.World(0, 8, 0, loopback=True)
        s = c3.Session(w, m, n, k, KIND[coll], pmib * MIB)
        s.set_ce_proxy(True)
        s.fill()
        s.load_tables(os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv"))
        jobs = {"gemm": (c3.GEMM_ONLY, s.default_alloc(c3.GEMM_ONLY)),
                "comm_dma": (c3.COMM_ONLY_DMA, s.default_alloc(c3.COMM_ONLY_DMA)),
                "conccl": (c3.CONCCL, s.default_alloc(c3.CONCCL)),
                "conccl_rp": (c3.CONCCL_RP, s.default_alloc(c3.CONCCL_RP))}
        t = {j: [] for j in jobs}
        names = list(jobs)
        for r in range(R + 1):
            for j in names[r % len(names):] + names[:r % len(names)]:
                tm = s.run(*jobs[j])
                if r:
                    t[j].append(tm)
        med = lambda j, f: statistics.median(f(x) for x in t[j])  # noqa: E731
        tg = med("gemm", lambda x: x.gemm_end_ms - x.gemm_start_ms)
        td = med("comm_dma", lambda x: x.comm_end_ms - x.comm_start_ms)
        ideal = c3.ideal_speedup(tg, td)
        tax = "G-long" if tg > 1.15 * td else "C-long" if td > 1.15 * tg else "GC-equal"
        sid = f"{shape}_{m}x{n}x{k}_{pmib}M"
        rows.append(f"{sid},{coll},{tax},serial,{(tg + td) / 1e3:.6g},1,{ideal:.6g},0,{tg:.4f},{td:.4f},"
                    f"{tg:.4f},1,{w.info.sm_count},0,0,DMA,{WORLD},{s.predict(c3.SERIAL, tg, td, td) / 1e3:.6g}")
        for j in ("conccl", "conccl_rp"):
            st, al = jobs[j]
            mk = med(j, lambda x: x.total_ms)
            gk = med(j, lambda x: x.gemm_end_ms - x.gemm_start_ms)
            sp = (tg + td) / mk
            pred = s.predict(st, tg, td, td) / 1e3
            rows.append(f"{sid},{coll},{tax},{j},{mk / 1e3:.6g},{sp:.6g},{ideal:.6g},"
                        f"{c3.fraction_of_ideal(sp, ideal):.6g},{tg:.4f},{td:.4f},{gk:.4f},{gk / tg:.4f},"
                        f"{al.cus_gemm},{al.cus_comm},{al.cus_idle},DMA,{WORLD},{pred:.6g}")
        s.close()
        w.close()
        print(f"{sid} {coll} done", file=sys.stderr, flush=True)
    with open(out_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
