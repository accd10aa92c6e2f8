"""Model-level C3: one FSDP transformer layer as a pipeline
of C3 pairs on B200. The layer comes from the product model layer's
ingest_model (reference workload.cpp:217-251): forward GEMMs qkv, attn-out,
gate+up, down, each weight sharded over 8 ranks. Pair i = GEMM i concurrent
with the all-gather of weight i+1 (prefetch; the last GEMM prefetches the next
layer's first weight). Loopback world on one GPU, in two emulations: the
collective at full local speed, and paced to NVLink (770 GB/s per direction)
by the session's link governor (c3_session_set_link_rate, as in bench.py).
Isolated and concurrent runs interleaved in rotated order. Two layer totals:
the per-pair best of the measured candidates (an oracle choice, optimistic)
and the runtime heuristic's pick per pair (c3_session_choose on the measured
isolated times and comm curve with the co-residency model), measured after it.

usage: python tools/layer_pipeline.py OUT.csv [rounds]
"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

MODELS = {"llama70b": (8192, 28672), "llama405b": (16384, 53248)}
TAGS = ["attn_qkv", "attn_out", "ffn_in", "ffn_out"]
NVLINK_GBPS = 770.0


def link_ctas(s, payload, n):
    """Fewest CTAs with which the paced collective reaches the link time (+3%)."""
    target = (n - 1) / n * payload / (NVLINK_GBPS * 1e9) * 1e3
    s.set_link_rate(NVLINK_GBPS)
    for ctas in (8, 12, 16, 24, 32, 48, 64, 96, 148):
        a = s.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = ctas
        ms = statistics.median(s.run(c3.COMM_ONLY_CU, a).comm_end_ms for _ in range(3))
        if ms <= 1.03 * target:
            return ctas
    return 148


def main():
    out_path = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    n = 8
    rows = ["model,pair,gemm_mnk,ag_weight,payload_mib,emulation,comm_ctas,t_gemm_ms,t_comm_ms,"
            "serial_ms,best_strategy,concurrent_ms,speedup,ideal,fraction_of_ideal,"
            "model_pick,model_cus_comm,model_pace_gbps,model_pick_ms"]
    tables = os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv")
    params = os.path.join(REPO, "data", "b200-loopback-params.json")
    cores = os.path.join(REPO, "data", "b200-coresident.json")
    for model, (hidden, ffn) in MODELS.items():
        layer = c3.ingest_model(hidden, ffn, 8192, 2, n)
        totals = {}
        for i, (m, nn, kk, _) in enumerate(layer):
            j = (i + 1) % len(layer)
            payload = layer[j][3]
            w = c3.World(0, n, 0, loopback=True)
            s = c3.Session(w, m, nn, kk, c3.ALL_GATHER, payload)
            s.fill()
            s.load_tables(tables)
            s.load_params(params)
            s.load_coresident(cores)
            full = w.info.sm_count
            for emu in ("full-speed", "nvlink-rate"):
                s.set_link_rate(0.0)
                ctas = full if emu == "full-speed" else link_ctas(s, payload, n)
                comm = s.default_alloc(c3.COMM_ONLY_CU)
                comm.cus_comm = ctas  # isolated: whole GPU, or the link-rate CTA count
                jobs = {"gemm": (c3.GEMM_ONLY, s.default_alloc(c3.GEMM_ONLY)),
                        "comm": (c3.COMM_ONLY_CU, comm)}
                co = sorted({16, 32, 64} if emu == "full-speed" else {ctas, 2 * ctas})
                for st in (c3.C3_BASE, c3.C3_SP):
                    for cc in co:
                        a = s.default_alloc(st)
                        a.cus_gemm, a.cus_comm = full, cc
                        jobs[f"{c3.STRATEGY_NAMES[st]}_coresident{cc}"] = (st, a)
                for cc in co:  # the comm curve (co-residency model) at these CTA units
                    a = s.default_alloc(c3.COMM_ONLY_CU)
                    a.cus_comm = cc
                    jobs[f"comm_c{cc}"] = (c3.COMM_ONLY_CU, a)
                # comm pacing: the co-resident collective spread over 60% / 80% of the GEMM
                tg0 = statistics.median(s.run(c3.GEMM_ONLY).total_ms for _ in range(3))
                cap = NVLINK_GBPS if emu == "nvlink-rate" else 0.0
                for frac in (0.6, 0.8):
                    pace = (n - 1) / n * payload / (frac * tg0 * 1e-3) / 1e9
                    if cap and pace >= cap:
                        continue
                    a = s.default_alloc(c3.C3_BASE)
                    a.cus_gemm, a.cus_comm, a.comm_pace_gbps = full, co[-1] if emu == "full-speed" else 2 * ctas, pace
                    jobs[f"c3_base_pace{int(frac * 100)}"] = (c3.C3_BASE, a)
                try:
                    s.run(c3.FUSED, s.default_alloc(c3.FUSED))
                    jobs["c3_fused"] = (c3.FUSED, s.default_alloc(c3.FUSED))
                except c3.C3Error:
                    pass
                s.set_link_rate(NVLINK_GBPS if emu == "nvlink-rate" else 0.0)
                t = {k: [] for k in jobs}
                names = list(jobs)
                for r in range(R + 1):
                    for job in names[r % len(names):] + names[:r % len(names)]:
                        st, a = jobs[job]
                        tm = s.run(st, a)
                        if r:
                            t[job].append(tm)
                tg = statistics.median(x.gemm_end_ms - x.gemm_start_ms for x in t["gemm"])
                tc = statistics.median(x.comm_end_ms - x.comm_start_ms for x in t["comm"])
                conc = {name: statistics.median(x.total_ms for x in v) for name, v in t.items()
                        if name not in ("gemm", "comm") and not name.startswith("comm_c")}
                curve = {cc: statistics.median(x.comm_end_ms - x.comm_start_ms for x in t[f"comm_c{cc}"])
                         for cc in co}
                curve[full] = min(tc, min(curve.values()))
                s.set_comm_curve(sorted(curve.items()))
                st, al, _ = s.choose(tg, tc, 0.0, allow_dma=False)
                pick_ms = statistics.median(s.run(st, al).total_ms for _ in range(R))
                best = min(conc, key=conc.get)
                bc = min(conc[best], tg + tc)  # the runtime falls back to serial if nothing wins
                if bc == tg + tc:
                    best = "serial"
                ideal = c3.ideal_speedup(tg, tc)
                sp = (tg + tc) / bc
                rows.append(f"{model},{i},{m}x{nn}x{kk},{TAGS[j]},{payload / 2**20:.1f},{emu},{ctas},"
                            f"{tg:.4f},{tc:.4f},{tg + tc:.4f},{best},{bc:.4f},{sp:.4f},{ideal:.4f},"
                            f"{c3.fraction_of_ideal(sp, ideal):.4f},{c3.STRATEGY_NAMES[st]},{al.cus_comm},"
                            f"{al.comm_pace_gbps:.0f},{pick_ms:.4f}")
                acc = totals.setdefault(emu, [0.0, 0.0, 0.0, 0.0, 0.0])
                acc[0] += tg
                acc[1] += tc
                acc[2] += bc
                acc[3] += max(tg, tc)
                acc[4] += pick_ms
            s.close()
            w.close()
            print(f"{model} pair {i} done", file=sys.stderr, flush=True)
        for emu, (tg, tc, bc, ideal_ms, pk) in totals.items():
            ideal = (tg + tc) / ideal_ms
            sp = (tg + tc) / bc
            rows.append(f"{model},layer,all,all,,{emu},,{tg:.4f},{tc:.4f},{tg + tc:.4f},per-pair best,"
                        f"{bc:.4f},{sp:.4f},{ideal:.4f},{c3.fraction_of_ideal(sp, ideal):.4f},,,,")
            sp = (tg + tc) / pk
            rows.append(f"{model},layer,all,all,,{emu},,{tg:.4f},{tc:.4f},{tg + tc:.4f},model pick per pair,"
                        f"{pk:.4f},{sp:.4f},{ideal:.4f},{c3.fraction_of_ideal(sp, ideal):.4f},,,,")
    with open(out_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
