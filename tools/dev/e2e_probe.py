"""Timeline of one host-buffer C3 step (c3_session_run_host) on cfg2: the
device-event times of the GEMM and the collective and the call's wall time,
for the A row-band / collective-piece settings in the environment
(C3_H2D_A_PIECES, C3_H2D_PIECES). Dev probe: python tools/dev/e2e_probe.py [reps]"""
import os
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_2412_14335_b200 as c3  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    w = c3.World(0, 8, 0, loopback=True)
    m, n, k, mib = (int(x) for x in os.environ.get("PROBE_SHAPE", "8192,28672,8192,896").split(","))
    s = c3.Session(w, m, n, k, c3.ALL_GATHER, mib << 20)
    s.fill()
    s.set_link_rate(770.0)
    p = s.pointers(0)
    pin_a = torch.empty(p.a_bytes, dtype=torch.uint8, pin_memory=True)
    pin_s = torch.empty(p.send_bytes, dtype=torch.uint8, pin_memory=True)
    pin_o = torch.empty(4096, dtype=torch.uint8, pin_memory=True)
    a = s.default_alloc(c3.C3_BASE)
    a.cus_gemm, a.cus_comm = w.info.sm_count, 24
    rows = []
    for r in range(reps + 2):
        t0 = time.perf_counter()
        t = s.run_host(c3.C3_BASE, a, pin_a.data_ptr(), pin_s.data_ptr(), pin_o.data_ptr(), 4096)
        wall = (time.perf_counter() - t0) * 1e3
        if r >= 2:
            rows.append((wall, t.total_ms, t.gemm_start_ms, t.gemm_end_ms, t.comm_start_ms, t.comm_end_ms))
    med = [statistics.median(x[i] for x in rows) for i in range(6)]
    print(f"A_PIECES={os.environ.get('C3_H2D_A_PIECES', '-')} PIECES={os.environ.get('C3_H2D_PIECES', '-')}: "
          f"wall {med[0]:.3f} ms, device {med[1]:.3f}, gemm {med[2]:.3f}-{med[3]:.3f}, "
          f"comm {med[4]:.3f}-{med[5]:.3f}")
    s.close()
    w.close()


if __name__ == "__main__":
    main()
