"""Summarise an ncu report (ncu -i ... --page raw --csv) into the few numbers
the roofline needs; merge into profiles/ncu_gemm_summary.json (bench.py reads
`dram_bytes` from there as roofline.traffic).

usage: python tools/ncu_summary.py REPORT.ncu-rep KEY [OUT.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1,
         "Hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "nsecond": 1e-9}


def summarise(report):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for i, h in enumerate(hdr):
            if h in WANT:
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                rec[WANT[h]] = v * SCALE.get(units[i], 1)
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        out.append(rec)
    return out


def main():
    report, key = sys.argv[1], sys.argv[2]
    path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
        "ncu_gemm_summary.json")
    recs = summarise(report)
    data = {}
    if os.path.exists(path):
        data = json.load(open(path))
    data[key] = recs[-1] if recs else {}
    data[key]["report"] = os.path.basename(report)
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[key], indent=1))


if __name__ == "__main__":
    main()
