"""bench.py output contract (the driver parses one JSON line): required keys
and types, for the reference arm (CPU) and our arm (GPU), on the small cfg1."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["cores"] >= 1
    assert "workload" in d["config"]
    # the reference arm reports the steps it really ran and our arm's config
    assert d["steps"] == 2 and d["warmup"] == 3
    sys.path.insert(0, REPO)
    import bench
    from types import SimpleNamespace
    assert d["config"] == bench.bench_config(SimpleNamespace(config="cfg1"), 1)
    assert d["unit"] == d["e2e"]["unit"] == bench.UNIT


@pytest.mark.gpu
def test_our_arm_contract():
    d = run_bench("--config", "cfg1", "--steps", "3", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert roof["bound"] in ("hbm", "tensor") and roof["achieved"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb)
    from types import SimpleNamespace
    sys.path.insert(0, REPO)
    import bench
    assert d["config"] == bench.bench_config(SimpleNamespace(config="cfg1"), 1)
    assert d["e2e"]["unit"] == d["unit"]
    assert d["e2e"]["d2h_bytes_per_step"] == 1024 * 1024 * 4  # the whole fp32 C
    ks = d["kernel_span"]  # the metric with the step timed as a kernel span, beside the headline
    assert ks["t_concurrent_span_ms"] > 0 and ks["t_concurrent_span_ms"] <= d["ms_per_step_median"] + 1e-9
    assert ks["speedup"] >= d["value"] - 1e-9 and "power_w" in d["clocks"]
    assert d["details"]["strategy_choice"]["strategy"] in (
        "serial", "c3_base", "c3_sp", "c3_rp", "c3_sp_rp", "conccl", "conccl_rp", "c3_fused")


def test_bench_configs_static_and_l2_rule():
    """Every BASELINE config's static `config` (shared by both arms) names
    its workload, and says whether the timed steps flush the L2: only inputs
    that fit the 126 MB L2 (configs[0]) are flushed."""
    sys.path.insert(0, REPO)
    import bench
    from types import SimpleNamespace
    for name, cfg in bench.CONFIGS.items():
        c = bench.bench_config(SimpleNamespace(config=name), 1)
        assert c["workload"].startswith(name + ":") and c["gemm_mnk"] == [cfg["m"], cfg["n"], cfg["k"]]
        assert c["ranks"] == cfg.get("ranks", 8) and c["payload_bytes"] == cfg["payload"]
        assert ("flushed" in c["l2"]) == bench.l2_resident(cfg)
    assert bench.l2_resident(bench.CONFIGS["cfg1"]) and not bench.l2_resident(bench.CONFIGS["cfg2"])
