"""Measured C3 sweep on this GPU (loopback worlds): every BASELINE config x
collective x strategy, in the reference's sweep CSV schema
(scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal;
sim.cpp:319-334) plus measured columns. Isolated and concurrent runs are
interleaved round-robin.

usage: python tools/c3_sweep.py OUT.csv [rounds] [link_gbps]
link_gbps > 0 paces every SM collective (and the fused copies) to that NVLink
rate with the session's link governor (c3_session_set_link_rate), so the
loopback world has the real node's collective time; 0 = full local speed.

The co-resident rows also carry t_comm_ctas_ms, the isolated collective on
that many CTAs (the comm curve), and their model prediction uses the B200
co-residency extension (c3_session_set_comm_curve + data/b200-coresident.json).
OUT.picks.csv compares the runtime heuristic's pick (c3_session_choose) with
the measured best per scenario."""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402
from bench import CONFIGS  # noqa: E402

KIND = {"all-gather": c3.ALL_GATHER, "all-to-all": c3.ALL_TO_ALL,
        "reduce-scatter": c3.REDUCE_SCATTER}


def main():
    out_path = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    link = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    world = f"loopback-8-link{link:.0f}" if link > 0 else "loopback-8"
    rows = ["scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal,"
            "t_gemm_iso_ms,t_comm_iso_ms,gemm_tflops_in_step,cus_gemm,cus_comm,backend,world,"
            "predicted_makespan_s,t_comm_ctas_ms,comm_pace_gbps"]
    picks = ["scenario_id,collective,model_pick,model_cus_comm,model_pace_gbps,model_predicted_ms,"
             "model_pick_measured_ms,measured_best,measured_best_ms,pick_over_best"]
    CORES = (8, 16, 24, 32, 48, 64)
    cores_json = os.path.join(REPO, "data", "b200-coresident.json")
    for name in ("cfg2", "cfg2_448", "cfg3", "cfg4", "cfg4_mb"):
        cfg = CONFIGS[name]
        colls = [cfg["coll"]] + (["all-to-all"] if cfg["coll"] == "all-gather" else [])
        for coll in colls:
            w = c3.World(0, 8, 0, loopback=True)
            s = c3.Session(w, cfg["m"], cfg["n"], cfg["k"], KIND[coll], cfg["payload"])
            s.load_tables(os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv"))
            if os.path.exists(os.path.join(REPO, "data", "b200-loopback-params.json")):
                s.load_params(os.path.join(REPO, "data", "b200-loopback-params.json"))
            s.fill()
            s.set_link_rate(link)
            full = w.info.sm_count
            jobs = {"gemm": (c3.GEMM_ONLY, s.default_alloc(c3.GEMM_ONLY))}
            a = s.default_alloc(c3.COMM_ONLY_CU)
            a.cus_comm = full
            jobs["comm"] = (c3.COMM_ONLY_CU, a)
            jobs["comm_dma"] = (c3.COMM_ONLY_DMA, s.default_alloc(c3.COMM_ONLY_DMA))
            # copy-engine strategies are not paced (nothing to pace in a DMA
            # queue; in loopback they are SM copy kernels): full-speed sweep only
            for st in (range(1, 7) if link == 0 else range(1, 5)):
                jobs[c3.STRATEGY_NAMES[st]] = (st, s.default_alloc(st))
            # comm pacing (B200 extension): the co-resident collective spread
            # over 60% / 80% of the GEMM (rate from a quick GEMM probe)
            for _ in range(5):  # warm: the pace is set from the steady GEMM time, as the runtime's choice is
                s.run(c3.GEMM_ONLY)
            tg0 = statistics.median(s.run(c3.GEMM_ONLY).total_ms for _ in range(5))
            peer = (8 - 1) / 8 * cfg["payload"]
            for ctas in (8, 16, 24):
                for frac in (0.6, 0.8):
                    pace = peer / (frac * tg0 * 1e-3) / 1e9
                    if link > 0 and pace >= link:
                        continue
                    a = s.default_alloc(c3.C3_BASE)
                    a.cus_gemm, a.cus_comm, a.comm_pace_gbps = full, ctas, pace
                    jobs[f"c3_base_coresident{ctas}_pace{int(frac * 100)}"] = (c3.C3_BASE, a)
            for ctas in CORES:  # B200 co-resident SM variants + the comm curve
                a = s.default_alloc(c3.C3_BASE)
                a.cus_gemm, a.cus_comm = full, ctas
                jobs[f"c3_base_coresident{ctas}"] = (c3.C3_BASE, a)
                a = s.default_alloc(c3.C3_SP)
                a.cus_gemm, a.cus_comm = full, ctas
                jobs[f"c3_sp_coresident{ctas}"] = (c3.C3_SP, a)
                a = s.default_alloc(c3.COMM_ONLY_CU)
                a.cus_comm = ctas
                jobs[f"comm_c{ctas}"] = (c3.COMM_ONLY_CU, a)
            if KIND[coll] != c3.REDUCE_SCATTER:
                try:
                    s.run(c3.FUSED, s.default_alloc(c3.FUSED))
                    jobs["c3_fused"] = (c3.FUSED, s.default_alloc(c3.FUSED))
                except c3.C3Error:
                    pass  # shape not on the CTA-pair GEMM
            t = {k: [] for k in jobs}
            names = list(jobs)
            for r in range(R + 1):
                for k in names[r % len(names):] + names[:r % len(names)]:  # rotated order
                    st, al = jobs[k]
                    tm = s.run(st, al)
                    if r:
                        t[k].append(tm)
            med = lambda k, f: statistics.median(f(x) for x in t[k])  # noqa: E731
            tg = med("gemm", lambda x: x.gemm_end_ms - x.gemm_start_ms)
            tc = med("comm", lambda x: x.comm_end_ms - x.comm_start_ms)
            td = med("comm_dma", lambda x: x.comm_end_ms - x.comm_start_ms)
            curve = {c: med(f"comm_c{c}", lambda x: x.comm_end_ms - x.comm_start_ms) for c in CORES}
            s.set_comm_curve(sorted(curve.items()) + [(full, tc)])
            if os.path.exists(cores_json):
                s.load_coresident(cores_json)
            ideal = c3.ideal_speedup(tg, tc)
            tax = "G-long" if tg > 1.15 * tc else "C-long" if tc > 1.15 * tg else "GC-equal"
            sid = f"{name}_{cfg['payload'] >> 20}M"
            flops = 2.0 * cfg["m"] * cfg["n"] * cfg["k"]
            rows.append(f"{sid},{coll},{tax},serial,{(tg + tc) / 1e3:.6g},1,{ideal:.6g},0,{tg:.4f},"
                        f"{tc:.4f},{flops / tg / 1e9:.1f},{full},{full},CU,{world},"
                        f"{s.predict(c3.SERIAL, tg, tc, td) / 1e3:.6g},,0.0")
            measured = {}
            for k, (st, al) in jobs.items():
                if k in ("gemm", "comm", "comm_dma") or k.startswith("comm_c"):
                    continue
                try:
                    pred = s.predict_alloc(st, al, tg, tc, td) / 1e3 if st <= c3.CONCCL_RP else float("nan")
                except c3.C3Error:
                    pred = float("nan")
                mk = med(k, lambda x: x.total_ms)
                gk = med(k, lambda x: x.gemm_end_ms - x.gemm_start_ms)
                sp = (tg + tc) / mk
                rows.append(f"{sid},{coll},{tax},{k},{mk / 1e3:.6g},{sp:.6g},{ideal:.6g},"
                            f"{c3.fraction_of_ideal(sp, ideal):.6g},{tg:.4f},{tc:.4f},"
                            f"{flops / gk / 1e9:.1f},{al.cus_gemm},{al.cus_comm},"
                            f"{['CU', 'DMA', 'TMA'][al.backend]},{world},{pred:.6g},"
                            f"{curve.get(al.cus_comm, '') if 'coresident' in k else ''},{al.comm_pace_gbps:.1f}")
                measured[k] = (mk, st, al)
            # the runtime heuristic's pick vs the measured best
            st, al, pred = s.choose(tg, tc, td, allow_dma=False)
            def same_pace(x, y):
                return (x == 0 and y == 0) or (x > 0 and y > 0 and abs(x - y) <= 0.1 * max(x, y))
            key = next((k for k, (_, s2, a2) in measured.items()
                        if s2 == st and a2.cus_gemm == al.cus_gemm and a2.cus_comm == al.cus_comm
                        and same_pace(a2.comm_pace_gbps, al.comm_pace_gbps)), None)
            best = min(measured, key=lambda k: measured[k][0])
            bm = min(measured[best][0], tg + tc)
            if tg + tc < measured[best][0]:
                best = "serial"
            if st == c3.SERIAL:
                key, pk = "serial", tg + tc
            elif key:
                pk = measured[key][0]
            else:
                # the pick was not among the swept jobs: measure it head to head
                # against the measured best, alternating, and scale to the sweep
                if best == "serial":
                    pair = {"pick": (st, al), "best": None}
                else:
                    pair = {"pick": (st, al), "best": jobs[best]}
                hh = {"pick": [], "best": []}
                for r in range(R):
                    for k2 in (("pick", "best") if r % 2 == 0 else ("best", "pick")):
                        if pair[k2] is None:
                            tmg = s.run(c3.GEMM_ONLY, jobs["gemm"][1]).total_ms
                            tmc = s.run(*jobs["comm"]).total_ms
                            hh[k2].append(tmg + tmc)
                        else:
                            hh[k2].append(s.run(*pair[k2]).total_ms)
                pk = bm * statistics.median(hh["pick"]) / statistics.median(hh["best"])
                key = f"model_pick(c{al.cus_comm},pace{al.comm_pace_gbps:.0f})"
            picks.append(f"{sid},{coll},{key or c3.STRATEGY_NAMES[st]},{al.cus_comm},{al.comm_pace_gbps:.0f},"
                         f"{pred:.4f},{pk:.4f},"
                         f"{best},{bm:.4f},{pk / bm:.4f}")
            s.close()
            w.close()
            print(f"{sid} {coll} done", file=sys.stderr, flush=True)
    with open(out_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    with open(os.path.splitext(out_path)[0] + ".picks.csv", "w") as f:
        f.write("\n".join(picks) + "\n")
    print("\n".join(rows))
    print("\n".join(picks))


if __name__ == "__main__":
    main()
