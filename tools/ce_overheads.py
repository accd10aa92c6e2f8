#!/usr/bin/env python3
"""Copy-engine measurements on one B200: the host-staged
proxy's copy-engine bandwidth, and the two overheads the reference's
plan_cost charges (proj/src/conccl.cpp:200-229): cpu_launch_overhead (host
time to issue one transfer) and dma_sync_overhead (the fixed cost of one
copy-engine collective: fork, engine start, join).

    python tools/ce_overheads.py OUT.json

* bandwidth: loopback all-gather of 8 ranks with the proxy on (rank 0's 7
  outgoing transfers D2H into pinned host peers, the 7 incoming ones H2D),
  COMM_ONLY_DMA device time per chunk size; GB/s per direction.
* cpu_launch_overhead: host wall time of c3_ce_execute enqueueing the full
  56-transfer plan (D2H into pinned host buffers, one cudaMemcpyAsync per
  transfer), per transfer; it goes into the machine descriptor.
* dma_sync_overhead: device time of a proxy collective of 4 KiB transfers
  (bytes negligible): the fixed latency of a copy-engine collective.
"""
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def proxy_bandwidth(c3, sizes, reps=7):
    out = []
    for chunk in sizes:
        w = c3.World(0, 8, 0, loopback=True)
        s = c3.Session(w, 256, 256, 256, c3.ALL_GATHER, 8 * chunk)
        c3.check(c3.lib().c3_session_set_ce_proxy(s.h, 1))
        s.fill(20241217)
        for _ in range(2):
            s.run(c3.COMM_ONLY_DMA)
        ts = []
        for _ in range(reps):
            t = s.run(c3.COMM_ONLY_DMA)
            ts.append(t.comm_end_ms - t.comm_start_ms)
        ms = statistics.median(ts)
        per_dir = 7 * chunk
        out.append({"chunk_bytes": chunk, "device_ms": ms, "bytes_per_direction": per_dir,
                    "gbs_per_direction": per_dir / (ms * 1e-3) / 1e9,
                    "gbs_both_directions": 2 * per_dir / (ms * 1e-3) / 1e9})
        s.close()
        w.close()
    return out


def launch_overhead(reps=20):
    """Per-transfer host cost of enqueueing the 56-transfer plan (subprocess:
    a fresh process, no state from the bandwidth runs)."""
    code = f"""
import ctypes as C, json, sys, time, torch
sys.path.insert(0, {REPO!r})
import paper_2412_14335_b200 as c3
n, chunk = 8, 64 << 10
w = c3.World(0, n, 0, loopback=True)
plan, nt = c3.plan_transfers(c3.ALL_GATHER, n, chunk, w.info.async_engines)
src = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(n)]
dst = [torch.empty(n * chunk, dtype=torch.uint8).pin_memory() for _ in range(n)]
sp, dp = [t.data_ptr() for t in src], [t.data_ptr() for t in dst]
for _ in range(3):
    w.ce_execute(plan, nt, sp, dp)
torch.cuda.synchronize()
ts = []
for _ in range({reps}):
    t0 = time.perf_counter()
    w.ce_execute(plan, nt, sp, dp)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
ts.sort()
print(json.dumps({{"transfers": nt, "enqueue_s_median": ts[len(ts) // 2],
                   "per_transfer_s": ts[len(ts) // 2] / nt}}))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True)
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    import paper_2412_14335_b200 as c3
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "data", "b200-ce-overheads.json")
    bw = proxy_bandwidth(c3, [4 << 10, 64 << 10, 1 << 20, 16 << 20, 112 << 20])
    per = launch_overhead()
    w = c3.World(0, 8, 0, loopback=True)
    res = {
        "what": "copy-engine measurements on one B200 (tools/ce_overheads.py): host-staged proxy "
                "(pinned host peers, D2H out + H2D in) bandwidth; plan_cost overheads",
        "async_engines": w.info.async_engines,
        "proxy_bandwidth": bw,
        "enqueue_per_transfer_path": per,
        "cpu_launch_overhead": per["per_transfer_s"],
        "dma_sync_overhead": bw[0]["device_ms"] * 1e-3,
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    w.close()
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
