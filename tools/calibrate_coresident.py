"""Fit the B200 co-residency penalties (include/c3sim/coresident.hpp) from a
measured sweep CSV (tools/c3_sweep.py): for every co-resident row (GEMM on
every SM, collective CTAs beside it) where the collective finished inside the
GEMM, solve the model for the GEMM penalty p_g (c3sim.fit_coresident_gemm_penalty,
p_c = 1) from the isolated GEMM time, the collective's isolated time at that
CTA count (column t_comm_ctas_ms when present, else rows whose CTA count
reaches the full-GPU collective time) and the measured makespan; the median
per GEMM class is written as the params JSON.

usage: python tools/calibrate_coresident.py SWEEP.csv [SWEEP2.csv ...] OUT.json"""
import csv
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "paper_2412_14335_b200", "python"))
import c3sim  # noqa: E402


def main():
    *ins, out = sys.argv[1:]
    fits = {"C-long": [], "G-long": [], "GC-equal": []}
    mb = {"cfg4_mb"}  # memory-bound GEMM scenarios (AI < machine op:byte)
    by_class = {"cb": [], "mb": []}
    for path in ins:
        for r in csv.DictReader(open(path)):
            if not r["strategy"].startswith("c3_base_coresident"):  # the runtime's co-resident mode
                continue
            tg = float(r["t_gemm_iso_ms"])
            tc = float(r.get("t_comm_ctas_ms") or "nan")
            if tc != tc:  # no per-CTA column: only CTA counts at the full-GPU collective time
                if int(r["cus_comm"]) < 32:
                    continue
                tc = float(r["t_comm_iso_ms"])
            mk = float(r["makespan_s"]) * 1e3
            if tc >= tg:  # the collective outlived the GEMM: p_g is not identifiable
                continue
            p = c3sim.fit_coresident_gemm_penalty(tg * 1e-3, tc * 1e-3, mk * 1e-3)
            cls = "mb" if any(r["scenario_id"].startswith(x) for x in mb) else "cb"
            by_class[cls].append(p)
            fits[r["taxonomy"]].append(p)
            print(f"{r['scenario_id']:16s} {r['collective']:15s} {r['strategy']:22s} p_g={p:.3f}")
    prm = c3sim.CoResidentParams()
    prm.gemm_compute_bound = statistics.median(by_class["cb"]) if by_class["cb"] else 1.0
    prm.gemm_memory_bound = statistics.median(by_class["mb"]) if by_class["mb"] else prm.gemm_compute_bound
    prm.comm = 1.0
    with open(out, "w") as f:
        f.write(c3sim.save_coresident_params(prm))
    print(f"fitted: compute-bound {prm.gemm_compute_bound:.3f} ({len(by_class['cb'])} rows), "
          f"memory-bound {prm.gemm_memory_bound:.3f} ({len(by_class['mb'])} rows) -> {out}")


if __name__ == "__main__":
    main()
