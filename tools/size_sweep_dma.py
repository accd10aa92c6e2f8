#!/usr/bin/env python3
"""BASELINE.json configs[4], the DMA-offloaded column: GEMM shape (compute- vs
memory-bound) x all-gather size 1 MiB .. 2 GiB x world 2 / 4 / 8 under the
copy-engine strategies (conccl, conccl_rp), through the host-staged
copy-engine proxy (c3_session_set_ce_proxy): this GPU's share
of the plan runs on its copy engines, peers in pinned host memory.

PCIe carries ~48 GB/s per direction where NVLink carries ~770, so each real
payload P runs as a proxy payload P * ce_gbs / 770 (ce_gbs measured here
first): the proxy collective lasts as long as the real one would at NVLink
rate, and the GEMM sees copy-engine traffic for the same time (at lower HBM
intensity than the real node). Rows follow tools/size_sweep.py's schema
(world = "ce-proxy-pcie") with the real and the proxy payload; speedup uses
the isolated proxy collective (the same backend, north_star). OUT.summary.csv
holds the mean fraction of ideal per (shape, world) for conccl and conccl_rp.

usage: python tools/size_sweep_dma.py OUT.csv [rounds] [worlds]
"""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2412_14335_b200 as c3  # noqa: E402

SHAPES = {"cb_8192": (8192, 8192, 8192), "cb_ffn": (8192, 28672, 8192), "mb_405b": (128, 53248, 16384)}
SIZES_MIB = [1 << i for i in range(12)]  # 1 .. 2048 MiB (real payloads)
NVLINK_GBPS = 770.0


def ce_gbs(n):
    """Measured proxy copy-engine rate per direction (GB/s) at this world size."""
    w = c3.World(0, n, 0, loopback=True)
    s = c3.Session(w, 256, 256, 256, c3.ALL_GATHER, n * (16 << 20))
    s.set_ce_proxy(True)
    s.fill()
    for _ in range(2):
        s.run(c3.COMM_ONLY_DMA)
    ms = statistics.median(s.run(c3.COMM_ONLY_DMA).total_ms for _ in range(5))
    s.close()
    w.close()
    return (n - 1) * (16 << 20) / (ms * 1e-3) / 1e9


def main():
    out_path = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    worlds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 4, 8]
    rows = ["scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal,"
            "shape,payload_mib,proxy_payload_bytes,n_ranks,t_gemm_iso_ms,t_comm_dma_ms,gemm_ms_in_step,"
            "cus_gemm,cus_idle,world"]
    summary = {}
    for n in worlds:
        rate = ce_gbs(n)
        print(f"world {n}: proxy copy engines {rate:.1f} GB/s per direction", file=sys.stderr, flush=True)
        w = c3.World(0, n, 0, loopback=True)
        for shape, (m, nn, k) in SHAPES.items():
            for mib in SIZES_MIB:
                step = 16 * n
                payload = max(step, int((mib << 20) * rate / NVLINK_GBPS) // step * step)
                s = c3.Session(w, m, nn, k, c3.ALL_GATHER, payload)
                s.set_ce_proxy(True)
                s.fill()
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
                sid = f"n{n}_{shape}_{mib}M"
                rows.append(f"{sid},all-gather,{tax},serial,{(tg + td) / 1e3:.6g},1,{ideal:.6g},0,{shape},{mib},"
                            f"{payload},{n},{tg:.4f},{td:.4f},{tg:.4f},{w.info.sm_count},0,ce-proxy-pcie")
                for j in ("conccl", "conccl_rp"):
                    st, al = jobs[j]
                    mk = med(j, lambda x: x.total_ms)
                    gk = med(j, lambda x: x.gemm_end_ms - x.gemm_start_ms)
                    sp = (tg + td) / mk
                    fr = c3.fraction_of_ideal(sp, ideal)
                    rows.append(f"{sid},all-gather,{tax},{j},{mk / 1e3:.6g},{sp:.6g},{ideal:.6g},{fr:.6g},{shape},"
                                f"{mib},{payload},{n},{tg:.4f},{td:.4f},{gk:.4f},{al.cus_gemm},{al.cus_idle},"
                                f"ce-proxy-pcie")
                    summary.setdefault((shape, n, j), []).append((fr, ideal))
                s.close()
                print(f"{sid}: ideal {ideal:.3f}", file=sys.stderr, flush=True)
        w.close()
    with open(out_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    lines = ["shape,n_ranks,strategy,sizes,mean_fraction_of_ideal,sizes_ideal_ge_1.1,mean_fraction_ideal_ge_1.1"]
    for (shape, n, j), v in summary.items():
        big = [x for x in v if x[1] >= 1.1]
        lines.append(f"{shape},{n},{j},{len(v)},{statistics.mean(x[0] for x in v):.4f},{len(big)},"
                     f"{statistics.mean(x[0] for x in big) if big else float('nan'):.4f}")
    with open(os.path.splitext(out_path)[0] + ".summary.csv", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
