#!/usr/bin/env python3
"""Pair-GEMM environment A/B (dev aid): for each setting (a string of
VAR=value pairs, e.g. "C3_GEMM_BAND=16 C3_GEMM_POL=113"), ncu DRAM bytes of one
launch plus burst / sustained timing (tools/dev/gemm_dev_ab.py's child, own
process per setting because the knobs are read once).

usage: python tools/dev/gemm_env_ab.py M N K "SETTING" ["SETTING" ...]
"""
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
from gemm_dev_ab import CHILD  # noqa: E402


def main():
    m, n, k = (int(x) for x in sys.argv[1:4])
    settings = sys.argv[4:]
    rows = []
    for rnd in range(2):  # two passes, so drift hits every setting alike
        for st in settings:
            env = dict(os.environ)
            for kv in st.split():
                key, val = kv.split("=", 1)
                env[key] = val
            row = {"setting": st, "pass": rnd}
            if rnd == 0:
                r = subprocess.run(
                    ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                     "lts__t_bytes.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "--clock-control", "none", "-k", "regex:gemm", "-s", "1", "-c", "1",
                     sys.executable, os.path.join(REPO, "tools", "ncu_target.py"), "gemm", str(m), str(n), str(k)],
                    env=env, capture_output=True, text=True)
                for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                             "lts__t_bytes.sum", "smsp__inst_executed.sum",
                             "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
                    mm = re.search(re.escape(name) + r"\s+(\S+)\s+([\d.,]+)", r.stdout)
                    if mm:
                        unit, val = mm.group(1), float(mm.group(2).replace(",", ""))
                        scale = {"inst": 1, "%": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                                 "ns": 1e-6, "us": 1e-3, "ms": 1.0, "msecond": 1.0, "usecond": 1e-3}.get(unit, 1)
                        row[name] = val * scale
            code = CHILD.format(repo=REPO, m=m, n=n, k=k, cublas=False)
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            row.update(json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0
                       else {"error": r.stderr[-300:]})
            print(json.dumps(row), flush=True)
            rows.append(row)


if __name__ == "__main__":
    main()
