"""Fit the B200 co-residency parameters (include/c3sim/coresident.hpp) from
measured sweep CSVs (tools/c3_sweep.py, which carries t_comm_ctas_ms: the
isolated collective on each CTA count).

The runtime's co-resident mode is c3_base with the GEMM on every SM and c
collective CTAs beside it. Its model has two parameters:
  p_g  the GEMM's slowdown while the collective runs beside it;
  p_c  the collective CTA's cost factor: c co-resident CTAs move data like
       c / p_c isolated CTAs (t_comm = curve(c / p_c)).
Per scenario the curve is the measured (CTAs, time) points plus the
full-GPU time; (p_g, p_c) minimise the mean squared relative error of
c3sim.simulate_coresident against every c3_base_coresident row (grid search).
Memory-bound GEMM scenarios (cfg4_mb) fit their own p_g. Then the comm-pacing
exponent g (the penalty's excess scales with (paced rate / link rate)^g) is
fitted on the paced rows (c3_base_coresident{c}_pace{pct}, comm_pace_gbps).

usage: python tools/calibrate_coresident.py SWEEP.csv [SWEEP2.csv ...] OUT.json"""
import csv
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "paper_2412_14335_b200", "python"))
import c3sim  # noqa: E402

CB, MB = c3sim.KernelClass.GEMM_COMPUTE_BOUND, c3sim.KernelClass.GEMM_MEMORY_BOUND
SMS = 148


def load(paths):
    """-> {(path, scenario, collective): {"tg", "tc", "curve", "rows": [(c, makespan)]}}"""
    scen = {}
    for path in paths:
        for r in csv.DictReader(open(path)):
            if not r["strategy"].startswith("c3_base_coresident"):
                continue
            key = (path, r["scenario_id"], r["collective"])
            d = scen.setdefault(key, {"tg": float(r["t_gemm_iso_ms"]) * 1e-3,
                                      "tc": float(r["t_comm_iso_ms"]) * 1e-3, "pts": {}, "rows": [],
                                      "paced": [], "mib": float(r["scenario_id"].rsplit("_", 1)[1].rstrip("M"))})
            c = int(r["cus_comm"])
            pace = float(r.get("comm_pace_gbps") or 0.0)
            if pace > 0:
                d["paced"].append((c, pace, float(r["makespan_s"])))
                continue
            if not r.get("t_comm_ctas_ms"):
                continue
            d["pts"][c] = float(r["t_comm_ctas_ms"]) * 1e-3
            d["rows"].append((c, float(r["makespan_s"])))
    for d in scen.values():
        if not d["pts"]:
            continue
        pts = dict(d["pts"])
        pts[SMS] = min(d["tc"], min(pts.values()))
        cs = sorted(pts)
        d["curve"] = c3sim.CommCurve(cs, [pts[c] for c in cs])
    return scen


def error(scen, cls_of, pg, pc):
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound = p.gemm_memory_bound = pg
    p.comm = pc
    err, n = 0.0, 0
    for key, d in scen.items():
        cls = cls_of(key)
        for c, mk in d["rows"]:
            t_at = d["curve"].time_at(c3sim.coresident_comm_ctas(c, p))
            pred = c3sim.simulate_coresident(d["tg"], t_at, d["tc"], SMS, c, cls, p).makespan
            err += ((pred - mk) / mk) ** 2
            n += 1
    return err / max(n, 1), n


def fit(scen, cls_of):
    best = None
    for pc in [1.0 + 0.05 * i for i in range(41)]:        # 1.0 .. 3.0
        for pg in [1.0 + 0.01 * i for i in range(61)]:    # 1.0 .. 1.6
            e, n = error(scen, cls_of, pg, pc)
            if best is None or e < best[0]:
                best = (e, pg, pc, n)
    return best


def paced_error(scen, cls_of, pg, pc, gamma):
    """Mean squared relative error of the paced rows under (pg, pc, gamma)."""
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound = p.gemm_memory_bound = pg
    p.comm, p.rate_exponent = pc, gamma
    err, n = 0.0, 0
    for key, d in scen.items():
        peer = 7 / 8 * d["mib"] * 2 ** 20
        link = peer / d["tc"] / 1e9  # GB/s of the unpaced collective
        for c, pace, mk in d["paced"]:
            ratio = min(1.0, pace / link)
            t_at = max(d["curve"].time_at(c3sim.coresident_comm_ctas(c, p)), d["tc"] / ratio)
            pred = c3sim.simulate_coresident(d["tg"], t_at, d["tc"], SMS, c, cls_of(key), p, ratio).makespan
            err += ((pred - mk) / mk) ** 2
            n += 1
    return err / max(n, 1), n


def main():
    *ins, out = sys.argv[1:]
    scen = {k: v for k, v in load(ins).items() if "curve" in v}
    is_mb = lambda key: key[1].startswith("cfg4_mb")  # noqa: E731  M=128: memory-bound GEMM
    cb = {k: v for k, v in scen.items() if not is_mb(k)}
    mb = {k: v for k, v in scen.items() if is_mb(k)}
    e_cb, pg_cb, pc, n_cb = fit(cb, lambda k: CB)
    # memory-bound: p_c shared (a property of the collective CTA), p_g refit
    best_mb = min(((error(mb, lambda k: MB, pg, pc)[0], pg)
                   for pg in [1.0 + 0.01 * i for i in range(61)]), default=(0.0, pg_cb))
    gam, n_p = 1.0, 0
    if any(d["paced"] for d in cb.values()):
        best_g = min((paced_error(cb, lambda k: CB, pg_cb, pc, g)[0], g) for g in [0.5 + 0.25 * i for i in range(23)])
        gam, n_p = best_g[1], paced_error(cb, lambda k: CB, pg_cb, pc, best_g[1])[1]
        print(f"comm pacing: rate exponent {gam:.2f}, rms rel. error {best_g[0] ** 0.5:.3f} ({n_p} rows)")
    prm = c3sim.CoResidentParams()
    prm.gemm_compute_bound, prm.comm, prm.rate_exponent = pg_cb, pc, gam
    prm.gemm_memory_bound = best_mb[1] if mb else pg_cb
    with open(out, "w") as f:
        f.write(c3sim.save_coresident_params(prm))
    print(f"compute-bound: p_g {pg_cb:.2f}, p_c {pc:.2f}, rms rel. error {e_cb ** 0.5:.3f} ({n_cb} rows)")
    if mb:
        print(f"memory-bound:  p_g {best_mb[1]:.2f}, rms rel. error {best_mb[0] ** 0.5:.3f}")
    print(f"-> {out}")


if __name__ == "__main__":
    main()
