"""_c3sim, the pybind11 module over the product model layer + execution API
(paper_2412_14335_b200/csrc/python/c3sim_module.cpp).

- The reference's OWN Python smoke test (proj/tests/python/test_smoke.py) runs
  unchanged through the reference's own `c3sim` package on top of our .so
  (needs /root/reference: this container only).
- The product `c3sim` package reproduces the golden sweep byte-for-byte, has
  the reduce-scatter extension, and refuses to execute without a B200.
- GPU: execute() / measure_isolated() on a loopback world, and `c3sim run`.
"""
import glob
import hashlib
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PYDIR = os.path.join(REPO, "paper_2412_14335_b200", "python")
REF_DATA = os.path.join(REPO, "tests", "golden", "ref_data")
REF_SMOKE = "/root/reference/proj/tests/python/test_smoke.py"
GOLDEN_SWEEP_SHA = "5b82de0beac7015284e6007cf9cd710ab629dc6d8f1a0c9006b16c1c0c73159a"

sys.path.insert(0, PYDIR)
import c3sim  # noqa: E402


def test_module_is_the_product_build():
    so = c3sim._c3sim.__file__
    assert so.startswith(PYDIR) and glob.glob(os.path.join(PYDIR, "c3sim", "_c3sim*.so"))


@pytest.mark.skipif(not os.path.exists(REF_SMOKE), reason="reference tree not mounted")
def test_reference_python_smoke_suite_against_product(tmp_path):
    env = dict(os.environ, PYTHONPATH=os.path.join(PYDIR, "c3sim") + ":/root/reference/proj/python",
               C3SIM_DATA_DIR=REF_DATA)
    probe = subprocess.run([sys.executable, "-c", "import c3sim; print(c3sim._impl.__file__)"],
                           env=env, cwd=tmp_path, capture_output=True, text=True)
    assert probe.returncode == 0 and probe.stdout.strip().startswith(PYDIR), probe.stderr
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-q", REF_SMOKE],
                       env=env, cwd=tmp_path, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "5 passed" in r.stdout, r.stdout + r.stderr


def test_golden_sweep_through_python():
    md = c3sim.load_machine_file(os.path.join(REF_DATA, "mi300x-node.json"))
    tables = c3sim.load_slowdown_tables(os.path.join(REF_DATA, "slowdown-tables.csv"), md.min_cu_grain)
    params = c3sim.load_params_file(os.path.join(REF_DATA, "default-params.json"))
    scen = c3sim.load_dataset(os.path.join(REF_DATA, "c3-dataset.json"))
    opt = c3sim.SimOptions()
    opt.freeze_phase2_allocation = params.freeze_phase2_allocation
    strategies = [getattr(c3sim.Strategy, n) for n in
                  ("SERIAL", "C3_BASE", "C3_SP", "C3_RP", "C3_SP_RP", "CONCCL", "CONCCL_RP")]
    res = c3sim.sweep(scen, strategies, md, tables, params.penalties, params.eff, opt)
    csv = c3sim.sweep_to_csv(res)
    assert hashlib.sha256(csv.encode()).hexdigest() == GOLDEN_SWEEP_SHA


def test_reduce_scatter_extension():
    md = c3sim.load_machine_file(os.path.join(REF_DATA, "mi300x-node.json"))
    plan = c3sim.plan_reduce_scatter(8, 1 << 20, md)
    assert plan.kind == c3sim.CollectiveKind.REDUCE_SCATTER and len(plan.transfers) == 56
    assert c3sim.validate_plan(plan, md).ok
    assert c3sim.collective_name(c3sim.CollectiveKind.REDUCE_SCATTER) == "reduce-scatter"


def test_errors_map_to_reference_types():
    with pytest.raises(c3sim.IoError):
        c3sim.load_machine_file("/nonexistent/machine.json")
    with pytest.raises(c3sim.ValidationError):
        c3sim.classify_c3(-1.0, 1.0)


def test_b200_machine_file_loads():
    md = c3sim.load_machine_file(c3sim.data_path("b200-loopback-node.json"))
    assert md.cus_per_gpu == 148


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_execute_without_gpu_is_a_device_error():
    if _has_gpu():
        pytest.skip("GPU present")
    with pytest.raises(c3sim.DeviceError):
        c3sim.World(0, 2, 0, True)


def _small_scenario(kind=None, n=2, m=2048, nn=2560):
    s = c3sim.C3Scenario()
    s.id = "small"
    s.gemm.m, s.gemm.n, s.gemm.k, s.gemm.dtype_bytes = m, nn, 1024, 2  # 80 pair tiles: c3_fused runs
    s.collective.kind = kind or c3sim.CollectiveKind.ALL_GATHER
    s.collective.n_ranks = n
    s.collective.payload_bytes = 16 << 20
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["serial", "c3_sp", "c3_rp", "conccl", "c3_fused"])
def test_execute_loopback(strategy):
    w = c3sim.World(0, 2, 0, True)
    r = c3sim.execute(_small_scenario(), strategy, w, warmup=2, reps=3)
    assert r.strategy == strategy and len(r.steps) == 3
    assert r.t_gemm > 0 and r.t_comm > 0 and r.makespan > 0
    assert r.serial_time == pytest.approx(r.t_gemm + r.t_comm)
    assert r.ideal == pytest.approx(c3sim.ideal_speedup(r.t_gemm, r.t_comm))
    assert r.fraction_of_ideal == pytest.approx(c3sim.fraction_of_ideal(r.speedup, r.ideal))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["serial", "c3_sp", "conccl"])
def test_execute_fp32_configs0(strategy):
    """configs[0] (fp32 GEMM 1024^3 || 16 MiB all-gather, world 2) through
    execute(): GemmKernel::dtype_bytes 4 runs on the TF32 tensor cores; fused
    C3 is bf16-only and refuses it."""
    s = _small_scenario(m=1024, nn=1024)
    s.gemm.dtype_bytes = 4
    w = c3sim.World(0, 2, 0, True)
    r = c3sim.execute(s, strategy, w, warmup=2, reps=3)
    assert r.t_gemm > 0 and r.t_comm > 0 and r.makespan > 0
    with pytest.raises(c3sim.UnsupportedError):
        c3sim.execute(s, "c3_fused", w, warmup=1, reps=1)
    s.gemm.dtype_bytes = 8
    with pytest.raises(c3sim.ValidationError):
        c3sim.execute(s, strategy, w, warmup=1, reps=1)


@pytest.mark.gpu
def test_fused_on_a_small_gemm_is_unsupported():
    w = c3sim.World(0, 2, 0, True)
    with pytest.raises(c3sim.UnsupportedError):
        c3sim.execute(_small_scenario(m=128, nn=1024), "c3_fused", w, warmup=1, reps=1)
    with pytest.raises(c3sim.ValidationError):  # UnsupportedError is a ValidationError
        c3sim.execute(_small_scenario(m=128, nn=1024), "c3_fused", w, warmup=1, reps=1)


@pytest.mark.gpu
def test_measure_isolated_feeds_the_model():
    w = c3sim.World(0, 2, 0, True)
    s = c3sim.measure_isolated(_small_scenario(c3sim.CollectiveKind.REDUCE_SCATTER), w, warmup=2, reps=3)
    assert s.gemm.measured_time > 0 and s.collective.measured_time > 0
    md = c3sim.load_machine_file(c3sim.data_path("b200-loopback-node.json"))
    eff = c3sim.EfficiencyParams()
    assert c3sim.roofline_gemm_time(s.gemm, md, eff) == s.gemm.measured_time


@pytest.mark.gpu
def test_execute_coresident_paced_at_link_rate():
    """B200 options of execute(): the co-resident allocation (all SMs + c
    collective units), comm pacing and NVLink-rate emulation."""
    w = c3sim.World(0, 8, 0, True)
    sc = _small_scenario(n=8)
    r = c3sim.execute(sc, "c3_base", w, warmup=2, reps=3, link_gbps=200.0, cus_gemm=w.sm_count,
                      cus_comm=16, comm_pace_gbps=100.0)
    assert r.gemm_ctas == w.sm_count and r.comm_ctas == 16
    assert r.t_comm == pytest.approx(7 / 8 * (16 << 20) / 200e9, rel=0.25)  # isolated at the link rate
    assert r.makespan > 0


@pytest.mark.gpu
def test_cli_run_executes_and_predicts(tmp_path):
    out = tmp_path / "run.json"
    exe = os.path.join(REPO, "paper_2412_14335_b200", "bin", "c3sim")
    r = subprocess.run([exe, "run", "--m", "2048", "--n", "2560", "--k", "1024", "--ranks", "2",
                        "--payload-bytes", str(16 << 20), "--strategy", "all", "--warmup", "2", "--reps",
                        "3", "--machine", os.path.join(REPO, "data", "b200-loopback-node.json"),
                        "--tables", os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv"),
                        "--format", "structured-text", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = json.loads(out.read_text())
    names = [x["strategy"] for x in rows]
    assert names == ["serial", "c3_base", "c3_sp", "c3_rp", "c3_sp_rp", "conccl", "conccl_rp", "c3_fused"]
    for x in rows:
        assert x["makespan_s"] > 0 and x["t_gemm_s"] > 0 and len(x["steps_s"]) == 3
        if x["strategy"] != "c3_fused":
            assert x["predicted_makespan_s"] > 0


@pytest.mark.gpu
def test_cli_run_auto_and_coresident(tmp_path):
    """`c3sim run --strategy auto`: the runtime heuristic (measured isolated
    times and comm curve -> c3_session_choose with the B200 co-residency
    model) picks and executes; an explicit co-resident, paced allocation runs
    too. Both at an emulated link rate."""
    exe = os.path.join(REPO, "paper_2412_14335_b200", "bin", "c3sim")
    base = [exe, "run", "--m", "2048", "--n", "4096", "--k", "2048", "--ranks", "8",
            "--payload-bytes", str(64 << 20), "--warmup", "2", "--reps", "3", "--link-gbps", "300",
            "--format", "structured-text"]
    out = tmp_path / "auto.json"
    r = subprocess.run(base + ["--strategy", "auto",
                               "--tables", os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv"),
                               "--params", os.path.join(REPO, "data", "b200-loopback-params.json"),
                               "--coresident", os.path.join(REPO, "data", "b200-coresident.json"),
                               "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "auto: picked" in r.stderr
    rows = json.loads(out.read_text())
    assert len(rows) == 1 and rows[0]["makespan_s"] > 0 and rows[0]["speedup"] > 0
    out = tmp_path / "co.json"
    r = subprocess.run(base + ["--strategy", "c3_base", "--cus-gemm", "148", "--cus-comm", "24",
                               "--comm-pace-gbps", "150", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    row = json.loads(out.read_text())[0]
    assert row["cus_gemm"] == 148 and row["cus_comm"] == 24 and row["comm_pace_gbps"] == pytest.approx(150)
    # serial = GEMM + the link-rate collective: (n-1)/n * P at 300 GB/s
    assert row["t_comm_s"] == pytest.approx(7 / 8 * (64 << 20) / 300e9, rel=0.25)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_b200_machine_files_validate(n):
    """data/b200-node-n{n}.json (tools/make_machine.py): measured B200 peaks
    and copy-engine overheads in the reference's machine format, one file per
    world size, accepted by the product's load_machine_file (validate,
    machine.cpp:26-49); every partition candidate is a multiple of the
    green-context grain (8)."""
    md = c3sim.load_machine_file(os.path.join(REPO, "data", f"b200-node-n{n}.json"))
    assert md.gpus_per_node == n and md.cus_per_gpu == 148 and md.links_per_gpu == n - 1
    assert md.peak_compute_flops > 1.5e15 and md.hbm_bandwidth > 6e12
    assert 0 < md.cpu_launch_overhead < 1e-5 and 0 < md.dma_sync_overhead < 1e-3
    with open(os.path.join(REPO, "data", "b200-ce-overheads.json")) as f:
        ce = json.load(f)
    assert md.cpu_launch_overhead == pytest.approx(ce["cpu_launch_overhead"], rel=1e-2)


def test_bounded_penalty_fit_is_physical(tmp_path):
    """tools/calibrate_penalties.py on the committed round-2 rows: every
    penalty in [1, 3], CU >= DMA per kernel class, the fitted rows' RMS under
    10%, and its output reloads as reference-format params."""
    import shutil
    root = tmp_path / "repo"
    for d in ("tools", "data", "profiles"):
        (root / d).mkdir(parents=True)
    shutil.copy(os.path.join(REPO, "tools", "calibrate_penalties.py"), root / "tools")
    shutil.copy(os.path.join(REPO, "bench.py"), root)
    for f in ("b200-node-n8.json", "b200-loopback-slowdown-tables.csv"):
        shutil.copy(os.path.join(REPO, "data", f), root / "data")
    for f in ("r02_c3_sweep_link770.csv", "r02_ce_proxy_sweep.csv"):
        shutil.copy(os.path.join(REPO, "profiles", f), root / "profiles")
    os.symlink(os.path.join(REPO, "paper_2412_14335_b200"), root / "paper_2412_14335_b200")
    r = subprocess.run([sys.executable, str(root / "tools" / "calibrate_penalties.py"),
                        str(root / "profiles" / "r02_c3_sweep_link770.csv"),
                        str(root / "profiles" / "r02_ce_proxy_sweep.csv")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rep = json.loads((root / "data" / "b200-loopback-params.fit.json").read_text())
    pen = rep["penalties"]
    assert all(1.0 <= v <= 3.0 for v in pen.values()), pen
    for cls in ("gemm-compute-bound", "gemm-memory-bound", "all-gather", "all-to-all"):
        assert pen[f"{cls}.cu"] >= pen[f"{cls}.dma"] - 1e-9
    assert rep["rms_rel_error"] < 0.10 and rep["rows_dma"] > 0
    rp = c3sim.load_params_file(str(root / "data" / "b200-loopback-params.json"))
    assert rp.freeze_phase2_allocation
