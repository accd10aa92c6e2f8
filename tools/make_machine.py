#!/usr/bin/env python3
"""B200 machine descriptors, one per world size: writes
data/b200-node-n{2,4,8}.json in the reference's machine format
(proj/include/c3sim/machine.hpp:13-28, proj/data/mi300x-node.json), which
c3_session_load_machine / c3sim --machine load.

Sources, all measured on this pool's B200s:
  peak_compute_flops, hbm_bandwidth   MEASURED_PEAKS.json (driver-written): the
                                      burst cuBLAS bf16 rate and the copy bandwidth
  cpu_launch_overhead                 data/b200-ce-overheads.json: host time per
                                      transfer of the copy-engine submit
  dma_sync_overhead                   same file: device time of a copy-engine
                                      collective of 4 KiB transfers (fixed cost)
  dma_engines_per_gpu                 asyncEngineCount (ce_overheads "async_engines")
  link_bandwidth_unidir               the measured 770 GB/s B200 peer copy per
                                      direction (B200_PROFILING.md), shared by the
                                      n-1 peers of a direct collective: 770e9/(n-1)
Fixed facts: 148 SMs in 2 dies of 74; L2 126.5 MiB; min_cu_grain 4. The
green-context split granularity is 8 SMs, but min_cu_grain must divide the SM
count (machine.cpp:37-38) and 148 = 8 * 18.5; the reference's partition
candidates {8, 16, 32, 64, 128} (strategy.cpp:35-46) are all multiples of 8,
so every split the model proposes is realisable, and the runtime rejects one
that is not (c3_session_run: C3_ERR_VALIDATION).

usage: python tools/make_machine.py [out_dir]
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEER_GBS = 770.0


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "data")
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
    with open(os.path.join(REPO, "data", "b200-ce-overheads.json")) as f:
        ce = json.load(f)
    for n in (2, 4, 8):
        md = {
            "gpus_per_node": n, "cus_per_gpu": 148, "xcds_per_gpu": 2, "cus_per_xcd": 74,
            "min_cu_grain": 4, "dma_engines_per_gpu": int(ce["async_engines"]),
            "peak_compute_flops": peaks["bf16_tflops"] * 1e12,
            "hbm_bandwidth": peaks["hbm_gbs"] * 1e9,
            "llc_capacity": 132644864,
            "link_bandwidth_unidir": PEER_GBS * 1e9 / (n - 1),
            "links_per_gpu": n - 1, "topology": "fully-connected",
            "cpu_launch_overhead": float(f"{ce['cpu_launch_overhead']:.3g}"),
            "dma_sync_overhead": float(f"{ce['dma_sync_overhead']:.3g}"),
        }
        path = os.path.join(out_dir, f"b200-node-n{n}.json")
        with open(path, "w") as f:
            json.dump(md, f, indent=2)
        print(path)


if __name__ == "__main__":
    main()
