"""BASELINE.json configs[4] on this GPU: GEMM shape (compute- vs memory-bound)
x all-gather size 1 MiB .. 2 GiB x world 2 / 4 / 8, comparing serial,
SM-concurrent and SM-partitioned execution and the runtime heuristic's pick.

Loopback worlds with the link governor at NVLink rate (c3_session_set_link_rate,
770 GB/s per direction by default): each rank's (n-1)/n * P of peer traffic
takes the time the node's links give it. Copy-engine strategies are left out:
in a loopback world same-device copies run as SM kernels, so
they would not measure the DMA offload.

Rows (one per shape x size x world x strategy) follow the reference sweep
schema (sim.cpp:319-334) plus measured columns; OUT.summary.csv holds, per
(shape, world), the mean fraction of ideal of the measured best strategy and
of the heuristic's pick (the paper's Fig. 8-style aggregate).

usage: python tools/size_sweep.py OUT.csv [rounds] [link_gbps] [worlds]"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

SHAPES = {
    "cb_8192": (8192, 8192, 8192),
    "cb_ffn": (8192, 28672, 8192),
    "mb_405b": (128, 53248, 16384),
}
SIZES_MIB = [1 << i for i in range(12)]  # 1 .. 2048 MiB
CORES = (16, 24, 48, 64)


def main():
    out_path = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    link = float(sys.argv[3]) if len(sys.argv) > 3 else 770.0
    worlds = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2, 4, 8]
    rows = ["scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal,"
            "shape,payload_mib,n_ranks,t_gemm_iso_ms,t_comm_iso_ms,cus_gemm,cus_comm,model_pick,"
            "t_comm_ctas_ms,comm_pace_gbps"]
    summary = {}
    tables = os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv")
    params = os.path.join(REPO, "data", "b200-loopback-params.json")
    cores_json = os.path.join(REPO, "data", "b200-coresident.json")
    for n in worlds:
        w = c3.World(0, n, 0, loopback=True)
        full = w.info.sm_count
        for shape, (m, nn, k) in SHAPES.items():
            for mib in SIZES_MIB:
                payload = (mib << 20) // n * n
                s = c3.Session(w, m, nn, k, c3.ALL_GATHER, payload)
                s.load_tables(tables)
                s.load_params(params)
                s.fill()
                s.set_link_rate(link)
                jobs = {"gemm": (c3.GEMM_ONLY, s.default_alloc(c3.GEMM_ONLY))}
                a = s.default_alloc(c3.COMM_ONLY_CU)
                a.cus_comm = full
                jobs["comm"] = (c3.COMM_ONLY_CU, a)
                for st in range(1, 5):  # c3_base, c3_sp, c3_rp, c3_sp_rp (the reference allocations)
                    jobs[c3.STRATEGY_NAMES[st]] = (st, s.default_alloc(st))
                for ctas in CORES:  # co-resident (GEMM on every SM) + the comm curve
                    a = s.default_alloc(c3.C3_BASE)
                    a.cus_gemm, a.cus_comm = full, ctas
                    jobs[f"c3_base_coresident{ctas}"] = (c3.C3_BASE, a)
                    a = s.default_alloc(c3.COMM_ONLY_CU)
                    a.cus_comm = ctas
                    jobs[f"comm_c{ctas}"] = (c3.COMM_ONLY_CU, a)
                t = {key: [] for key in jobs}
                names = list(jobs)
                for r in range(R + 1):
                    for key in names[r % len(names):] + names[:r % len(names)]:
                        st, al = jobs[key]
                        tm = s.run(st, al)
                        if r:
                            t[key].append(tm)
                med = lambda key, f: statistics.median(f(x) for x in t[key])  # noqa: E731
                tg = med("gemm", lambda x: x.gemm_end_ms - x.gemm_start_ms)
                tc = med("comm", lambda x: x.comm_end_ms - x.comm_start_ms)
                curve = {c: med(f"comm_c{c}", lambda x: x.comm_end_ms - x.comm_start_ms) for c in CORES}
                s.set_comm_curve(sorted(curve.items()) + [(full, tc)])
                s.load_coresident(cores_json)
                st_pick, al_pick, _ = s.choose(tg, tc, tc, allow_dma=False)
                ideal = c3.ideal_speedup(tg, tc)
                tax = "G-long" if tg > 1.15 * tc else "C-long" if tc > 1.15 * tg else "GC-equal"
                sid = f"n{n}_{shape}_{mib}M"
                measured = {"serial": tg + tc}
                pick_key = "serial" if st_pick == c3.SERIAL else None
                for key, (st, al) in jobs.items():
                    if key in ("gemm", "comm") or key.startswith("comm_c"):
                        continue
                    measured[key] = med(key, lambda x: x.total_ms)
                    if (pick_key is None and st == st_pick and al.cus_comm == al_pick.cus_comm
                            and al.cus_gemm == al_pick.cus_gemm and al_pick.comm_pace_gbps == 0):
                        pick_key = key
                if pick_key is None:  # the heuristic's allocation is not among the jobs: run it
                    ts = [s.run(st_pick, al_pick).total_ms for _ in range(R)]
                    pick_key = f"pick_{c3.STRATEGY_NAMES[st_pick]}{al_pick.cus_comm}"
                    measured[pick_key] = statistics.median(ts)
                for key, mk in measured.items():
                    sp = (tg + tc) / mk
                    st, al = jobs.get(key, (st_pick, al_pick)) if key != "serial" else (c3.SERIAL, None)
                    rows.append(f"{sid},all-gather,{tax},{key},{mk / 1e3:.6g},{sp:.6g},{ideal:.6g},"
                                f"{c3.fraction_of_ideal(sp, ideal):.6g},{shape},{mib},{n},{tg:.4f},{tc:.4f},"
                                f"{al.cus_gemm if al else full},{al.cus_comm if al else full},"
                                f"{int(key == pick_key)},"
                                f"{curve.get(al.cus_comm, '') if 'coresident' in key else ''},0.0")
                best = min(measured, key=measured.get)
                fb = c3.fraction_of_ideal((tg + tc) / measured[best], ideal)
                fp = c3.fraction_of_ideal((tg + tc) / measured[pick_key], ideal)
                summary.setdefault((shape, n), []).append((fb, fp, best, pick_key, mib, ideal))
                s.close()
                print(f"{sid}: ideal {ideal:.3f} best {best} {(tg + tc) / measured[best]:.3f}x "
                      f"pick {pick_key} {(tg + tc) / measured[pick_key]:.3f}x", file=sys.stderr, flush=True)
        w.close()
    with open(out_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    # fraction of ideal is (speedup - 1) / (ideal - 1) (taxonomy.cpp:29-33, not
    # capped): where the ideal is within a few % of 1 (tiny payloads) it is
    # timing noise over a near-zero denominator, so the summary also reports
    # the scenarios with ideal >= 1.1 on their own
    lines = ["shape,n_ranks,sizes,mean_fraction_of_ideal_best,mean_fraction_of_ideal_pick,"
             "sizes_ideal_ge_1.1,mean_fraction_best_ideal_ge_1.1,mean_fraction_pick_ideal_ge_1.1,best_strategies"]
    for (shape, n), v in summary.items():
        bests = sorted({b for _, _, b, _, _, _ in v})
        big = [x for x in v if x[5] >= 1.1]
        mb = f"{statistics.mean(x[0] for x in big):.4f}" if big else ""
        mp = f"{statistics.mean(x[1] for x in big):.4f}" if big else ""
        lines.append(f"{shape},{n},{len(v)},{statistics.mean(x[0] for x in v):.4f},"
                     f"{statistics.mean(x[1] for x in v):.4f},{len(big)},{mb},{mp},{'|'.join(bests)}")
    with open(os.path.splitext(out_path)[0] + ".summary.csv", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
