"""B200 calibration loop: measured C3 sweep -> reference
formats -> the product's `c3sim calibrate` (fit_penalties, calibrate.cpp:95-238)
-> data/b200-loopback-params.json, which the runtime heuristic loads
(c3_session_load_params).

Inputs: a tools/c3_sweep.py CSV (measured). Outputs in data/:
  b200-loopback-node.json      machine descriptor (8 ranks, 148 SMs, grain 4)
  b200-loopback-dataset.json   the swept scenarios with measured isolated times
  b200-loopback-measured.csv   scenario_id,collective,strategy,measured_speedup
  b200-loopback-params.json    fitted co-run penalties (SM strategies)
usage: python tools/calibrate_penalties.py SWEEP.csv
"""
import csv
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from bench import CONFIGS  # noqa: E402

DATA = os.path.join(REPO, "data")
CLI = os.path.join(REPO, "paper_2412_14335_b200", "bin", "c3sim")
MACHINE = {
    "gpus_per_node": 8, "cus_per_gpu": 148, "xcds_per_gpu": 2, "cus_per_xcd": 74,
    "min_cu_grain": 4, "dma_engines_per_gpu": 4, "peak_compute_flops": 1.6097e15,
    "hbm_bandwidth": 6.5383e12, "llc_capacity": 132644864,
    "link_bandwidth_unidir": 900e9 / 7, "links_per_gpu": 7, "topology": "fully-connected",
    "cpu_launch_overhead": 2e-6, "dma_sync_overhead": 1e-5}
SM_STRATEGIES = ("c3_base", "c3_sp", "c3_rp", "c3_sp_rp")


def main():
    rows = list(csv.DictReader(open(sys.argv[1])))
    os.makedirs(DATA, exist_ok=True)
    with open(os.path.join(DATA, "b200-loopback-node.json"), "w") as f:
        json.dump(MACHINE, f, indent=2)
    scenarios, measured, seen = [], [], set()
    for r in rows:
        sid, coll = r["scenario_id"], r["collective"]
        cfg_name = sid.rsplit("_", 1)[0]
        cfg = CONFIGS[cfg_name]
        if (sid, coll) not in seen:
            seen.add((sid, coll))
            payload = cfg["payload"]
            scenarios.append({
                "id": sid, "source": "B200 loopback measurement",
                "gemm": {"tag": cfg_name, "m": cfg["m"], "n": cfg["n"], "k": cfg["k"],
                         "dtype_bytes": 2, "measured_time": float(r["t_gemm_iso_ms"]) * 1e-3},
                "collective": {"kind": coll, "payload_bytes": payload, "n_ranks": 8,
                               "measured_time": float(r["t_comm_iso_ms"]) * 1e-3}})
        if r["strategy"] in SM_STRATEGIES:
            measured.append((sid, coll, r["strategy"], float(r["speedup"])))
    ds = os.path.join(DATA, "b200-loopback-dataset.json")
    with open(ds, "w") as f:
        json.dump(scenarios, f, indent=2)
    mp = os.path.join(DATA, "b200-loopback-measured.csv")
    with open(mp, "w") as f:
        f.write("scenario_id,collective,strategy,measured_speedup\n")
        for m in measured:
            f.write("%s,%s,%s,%.9g\n" % m)
    start = os.path.join(DATA, "b200-start-params.json")
    with open(start, "w") as f:  # start from unit penalties (no prior about B200)
        json.dump({"efficiency": 1.0, "comm_launch_overhead_cu": 0.0,
                   "co_run_penalty": {c: {"cu": 1.0, "dma": 1.0} for c in
                                      ("gemm-compute-bound", "gemm-memory-bound", "all-gather",
                                       "all-to-all")},
                   "freeze_phase2_allocation": False}, f, indent=2)
    out = os.path.join(DATA, "b200-loopback-params.json")
    r = subprocess.run([CLI, "calibrate", "--machine", os.path.join(DATA, "b200-loopback-node.json"),
                        "--dataset", ds, "--tables",
                        os.path.join(DATA, "b200-loopback-slowdown-tables.csv"), "--params", start,
                        "--measured", mp, "--out", out], capture_output=True, text=True)
    os.remove(start)
    print(r.stdout)
    print(r.stderr, file=sys.stderr)
    sys.exit(r.returncode)


if __name__ == "__main__":
    main()
