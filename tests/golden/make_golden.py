#!/usr/bin/env python3
"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs /root/reference and the oracle build,
`make -C oracle`). The outputs are committed so the GPU box never reads
/root/reference:

* ``ref_data/*``          the reference's shipped model inputs (proj/data/*), the
                          exact files its acceptance suite loads (acceptance.cpp:49-55)
* ``sweep_mi300x.csv``    reference ``sweep_to_csv(sweep(all 30 scenarios x 7
                          strategies))`` — SURVEY.md §8(c): 22,351 bytes,
                          sha256 5b82de0b…159a
* ``sweep_mi300x_zero.csv`` the same under ``apply_zero_interference``
* ``plans/*.json``        reference ``to_json(plan_all_gather|plan_all_to_all)``
* ``plan_costs.json``     reference ``plan_cost`` totals for a size ladder
"""
import hashlib
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_DATA = "/root/reference/proj/data"
DRIVER = os.path.join(REPO, "oracle", "_ref", "c3sim_ref_driver")


def run(*args):
    return subprocess.run([DRIVER, *args], check=True, capture_output=True, text=True).stdout


def main():
    if not os.path.isdir(REF_DATA):
        sys.exit("reference data not present; run in the build container")
    subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "-s"], check=True)
    dst = os.path.join(HERE, "ref_data")
    os.makedirs(dst, exist_ok=True)
    for f in ("mi300x-node.json", "c3-dataset.json", "slowdown-tables.csv", "default-params.json"):
        shutil.copyfile(os.path.join(REF_DATA, f), os.path.join(dst, f))
    files = [os.path.join(dst, f) for f in
             ("mi300x-node.json", "c3-dataset.json", "slowdown-tables.csv", "default-params.json")]
    csv = run("sweep", *files)
    digest = hashlib.sha256(csv.encode()).hexdigest()
    assert len(csv) == 22351 and digest.startswith("5b82de0b"), (len(csv), digest)
    open(os.path.join(HERE, "sweep_mi300x.csv"), "w").write(csv)
    open(os.path.join(HERE, "sweep_mi300x_zero.csv"), "w").write(run("sweep", *files, "zero"))

    pdir = os.path.join(HERE, "plans")
    os.makedirs(pdir, exist_ok=True)
    machine = files[0]
    for kind in ("all-gather", "all-to-all"):
        for n, chunk in ((1, 64), (2, 8388608), (2, 1), (4, 4096), (8, 117440512), (8, 1024), (8, 3)):
            txt = run("plan", kind, str(n), str(chunk), machine)
            open(os.path.join(pdir, f"{kind}_n{n}_c{chunk}.json"), "w").write(txt)
    costs = {}
    for kind in ("all-gather", "all-to-all"):
        for mib in (1, 2, 4, 8, 16, 24, 31, 128, 256, 896):
            chunk = (mib << 20) // 8
            total, wire = run("cost", kind, "8", str(chunk), machine, files[3]).split()
            costs[f"{kind}:{chunk}"] = [float(total), float(wire)]
    json.dump(costs, open(os.path.join(HERE, "plan_costs.json"), "w"), indent=1, sort_keys=True)
    print("golden fixtures written; sweep sha256", digest)


if __name__ == "__main__":
    main()
