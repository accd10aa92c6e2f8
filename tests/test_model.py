"""The product's model layer (libc3sim behind include/c3sim/*.hpp) against the
reference: byte-identical sweep CSV (all 30 scenarios x 7 strategies, plus the
zero-interference reduction), identical plan JSON for the reference planner's
golden plans, plan costs, exit codes, and — when /root/reference is present
(build container) — the reference's own acceptance.cpp compiled against the
product library.
"""
import hashlib
import json
import os
import subprocess

import pytest

from paper_2412_14335_b200._capi import CLI

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(REPO, "tests", "golden")
DATA = os.path.join(GOLD, "ref_data")
FILES = {k: os.path.join(DATA, v) for k, v in (("machine", "mi300x-node.json"),
                                                ("dataset", "c3-dataset.json"),
                                                ("tables", "slowdown-tables.csv"),
                                                ("params", "default-params.json"))}


def cli(*args, check=True):
    r = subprocess.run([CLI, *args], capture_output=True, text=True)
    if check and r.returncode != 0:
        raise AssertionError(r.stderr)
    return r


def common():
    return ["--machine", FILES["machine"], "--dataset", FILES["dataset"], "--tables",
            FILES["tables"], "--params", FILES["params"]]


def test_sweep_byte_identical_to_reference():
    out = cli("sweep", *common(), "--strategy", "all").stdout
    gold = open(os.path.join(GOLD, "sweep_mi300x.csv")).read()
    assert len(out) == 22351
    assert hashlib.sha256(out.encode()).hexdigest() == \
        "5b82de0beac7015284e6007cf9cd710ab629dc6d8f1a0c9006b16c1c0c73159a"
    assert out == gold


def test_zero_interference_sweep_identical():
    out = cli("sweep", *common(), "--zero-interference").stdout
    assert out == open(os.path.join(GOLD, "sweep_mi300x_zero.csv")).read()


def test_sweep_deterministic_and_atomic(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    cli("sweep", *common(), "--out", str(a))
    cli("sweep", *common(), "--out", str(b))
    assert a.read_bytes() == b.read_bytes() and not (tmp_path / "a.csv.tmp").exists()


@pytest.mark.parametrize("name", sorted(os.listdir(os.path.join(GOLD, "plans"))))
def test_plan_json_identical(tmp_path, name):
    kind, n, c = name[:-5].split("_")
    n, chunk = int(n[1:]), int(c[1:])
    out = tmp_path / "p.json"
    cli("conccl-plan", "--machine", FILES["machine"], "--kind", kind, "--ranks", str(n),
        "--payload-bytes", str(n * chunk), "--out", str(out))
    if n == 1:  # the CLI pins a 1-rank zero payload to chunk 1; compare structure only
        got, want = json.loads(out.read_text()), json.load(open(os.path.join(GOLD, "plans", name)))
        assert got["transfers"] == want["transfers"] == []
        return
    assert out.read_text() == open(os.path.join(GOLD, "plans", name)).read()


def test_plan_costs_match_reference():
    gold = json.load(open(os.path.join(GOLD, "plan_costs.json")))
    for key, (total, wire) in gold.items():
        kind, chunk = key.split(":")
        r = cli("conccl-plan", "--machine", FILES["machine"], "--params", FILES["params"], "--kind",
                kind, "--ranks", "8", "--payload-bytes", str(8 * int(chunk)))
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("cost:")][0]
        got_total = float(line.split("total ")[1].split(" s")[0])
        got_wire = float(line.split("wire ")[1].split(" s")[0])
        assert abs(got_total - total) <= 1e-11 * total and abs(got_wire - wire) <= 1e-11 * wire


def test_reduce_scatter_plan_validates():
    r = cli("conccl-plan", "--machine", FILES["machine"], "--kind", "reduce-scatter", "--ranks",
            "8", "--payload-bytes", str(8 << 20))
    assert "56 transfers" in r.stdout and "validation: ok" in r.stdout


@pytest.mark.parametrize("args,code", [
    (["sweep", "--machine", "/nonexistent.json", "--dataset", "x", "--tables", "y"], 2),
    (["plan", "--scenario", "nope", "--strategy", "c3_rp"], 3),
    (["plan", "--scenario", "cb1_896M", "--strategy", "bogus"], 3),
    (["conccl-plan", "--kind", "all-gather", "--ranks", "16", "--payload-bytes", "64"], 4),
])
def test_exit_codes(args, code):
    full = list(args)
    if "--machine" not in full:
        full += ["--machine", FILES["machine"]]
    if full[0] == "plan":
        full += ["--dataset", FILES["dataset"], "--tables", FILES["tables"]]
    assert cli(*full, check=False).returncode == code


def test_partition_heuristic_picks_32_for_cb1():
    r = cli("plan", *common(), "--scenario", "cb1_896M", "--strategy", "c3_rp",
            "--filter-collective", "all-gather")
    assert '"cus_comm": 32' in r.stdout  # test_strategy.cpp:67-94


def test_calibrate_recovers_penalties(tmp_path):
    """Self-consistency (test_calibrate.cpp:66-97): simulate with perturbed
    penalties, fit from the defaults, recover them."""
    truth = json.load(open(FILES["params"]))
    truth["co_run_penalty"]["all-gather"] = {"cu": 1.55, "dma": 1.25}
    truth["co_run_penalty"]["gemm-compute-bound"] = {"cu": 1.06, "dma": 1.03}
    tp = tmp_path / "truth.json"
    tp.write_text(json.dumps(truth))
    rows = cli("sweep", "--machine", FILES["machine"], "--dataset", FILES["dataset"], "--tables",
               FILES["tables"], "--params", str(tp), "--filter-collective", "all-gather").stdout
    meas = tmp_path / "m.csv"
    with open(meas, "w") as f:
        f.write("scenario_id,collective,strategy,measured_speedup\n")
        for ln in rows.splitlines()[1:]:
            c = ln.split(",")
            if c[0] != "mean" and c[3] in ("c3_sp", "conccl", "c3_base"):
                f.write(f"{c[0]},{c[1]},{c[3]},{c[5]}\n")
    r = cli("calibrate", *common(), "--measured", str(meas))
    fit = json.loads(r.stdout)["co_run_penalty"]
    assert abs(fit["all-gather"]["cu"] - 1.55) < 0.02
    assert abs(fit["all-gather"]["dma"] - 1.25) < 0.02


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/tests/acceptance.cpp"),
                    reason="reference sources only in the build container")
def test_reference_acceptance_suite_against_product(tmp_path):
    """The reference's acceptance.cpp, unmodified, linked against libc3sim."""
    exe = tmp_path / "acceptance"
    lib = os.path.join(REPO, "paper_2412_14335_b200", "lib")
    subprocess.run(["g++-13", "-std=c++20", "-O1", f"-I{REPO}/include",
                    f'-DC3SIM_DATA_DIR="{DATA}"', f'-DC3SIM_CLI_PATH="{CLI}"',
                    "/root/reference/proj/tests/acceptance.cpp", f"-L{lib}", "-lc3sim",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 11
