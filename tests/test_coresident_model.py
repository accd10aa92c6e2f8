"""B200 model extension: co-residency (include/c3sim/coresident.hpp) through
the product pybind module. CPU only: the fluid-model arithmetic, the measured
comm curve, the penalty fit (the inverse of the model) and the params file."""
import math
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "paper_2412_14335_b200", "python"))
import c3sim  # noqa: E402

CB = c3sim.KernelClass.GEMM_COMPUTE_BOUND
MB = c3sim.KernelClass.GEMM_MEMORY_BOUND


def test_comm_curve_interpolation_and_clamps():
    c = c3sim.CommCurve([8, 16, 24], [2.0e-3, 1.2e-3, 1.0e-3])
    assert c.time_at(16) == pytest.approx(1.2e-3)
    assert c.time_at(20) == pytest.approx(1.1e-3)
    assert c.time_at(4) == pytest.approx(4.0e-3)    # below the first point: 1/ctas
    assert c.time_at(148) == pytest.approx(1.0e-3)  # link-bound: flat above the last


def test_comm_curve_as_table_is_a_valid_slowdown_table():
    md = c3sim.load_machine_file(c3sim.data_path("b200-loopback-node.json"))
    c = c3sim.CommCurve([8, 16, 24], [2.0e-3, 1.2e-3, 1.0e-3])
    t = c.as_table(c3sim.KernelClass.ALL_GATHER, md)
    pts = [(p.cus, p.slowdown) for p in t.points]
    assert pts[-1] == (md.cus_per_gpu, 1.0)
    assert all(p[0] % md.min_cu_grain == 0 for p in pts)
    assert all(s >= 1.0 for _, s in pts)
    assert dict(pts)[8] == pytest.approx(2.0)


@pytest.mark.parametrize("bad", [([16, 8], [1e-3, 1e-3]), ([8], [0.0]), ([8, 16], [1e-3])])
def test_comm_curve_validation(bad):
    md = c3sim.load_machine_file(c3sim.data_path("b200-loopback-node.json"))
    with pytest.raises(Exception):
        c3sim.CommCurve(*bad).as_table(c3sim.KernelClass.ALL_GATHER, md)


def test_coresident_unit_penalties_hide_the_shorter_kernel():
    p = c3sim.CoResidentParams()
    tl = c3sim.simulate_coresident(2.5e-3, 1.1e-3, 1.1e-3, 148, 24, CB, p)
    assert tl.makespan == pytest.approx(2.5e-3)
    assert tl.speedup == pytest.approx(tl.ideal)
    assert tl.fraction_of_ideal == pytest.approx(1.0)
    tl = c3sim.simulate_coresident(0.3e-3, 2.0e-3, 2.0e-3, 148, 32, MB, p)  # C-long
    assert tl.makespan == pytest.approx(2.0e-3)


def test_coresident_penalty_closed_form():
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound = 1.2
    tg, tc = 2.4e-3, 1.0e-3
    tl = c3sim.simulate_coresident(tg, tc, tc, 148, 24, CB, p)
    # phase 1 ends with the collective at tc; the GEMM did tc/1.2 of its work
    assert tl.makespan == pytest.approx(tc + tg - tc / 1.2)
    assert len(tl.phases) == 2 and tl.phases[0].cus_gemm == 148 and tl.phases[0].cus_comm == 24
    # the memory-bound penalty is separate
    assert c3sim.simulate_coresident(tg, tc, tc, 148, 24, MB, p).makespan == pytest.approx(tg)


def test_coresident_slower_ctas_stretch_the_collective():
    p = c3sim.CoResidentParams()
    # 8 CTAs take 2x the full-GPU collective time; the collective outlives the GEMM
    tl = c3sim.simulate_coresident(1.0e-3, 2.4e-3, 1.2e-3, 148, 8, CB, p)
    assert tl.makespan == pytest.approx(2.4e-3)
    assert tl.serial_time == pytest.approx(2.2e-3)  # t_comm = the full-GPU time
    assert tl.speedup < 1.0 and tl.fraction_of_ideal == 0.0


@pytest.mark.parametrize("pen", [1.0, 1.07, 1.3, 2.0])
def test_fit_is_the_inverse_of_the_model(pen):
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound = pen
    tg, tc = 2.5e-3, 1.1e-3
    mk = c3sim.simulate_coresident(tg, tc, tc, 148, 24, CB, p).makespan
    assert c3sim.fit_coresident_gemm_penalty(tg, tc, mk) == pytest.approx(pen)


def test_fit_degenerate_cases():
    assert c3sim.fit_coresident_gemm_penalty(1e-3, 2e-3, 2e-3) == 1.0   # collective outlived the GEMM
    assert c3sim.fit_coresident_gemm_penalty(1e-3, 0.5e-3, 0.4e-3) == 1.0  # faster than possible
    assert c3sim.fit_coresident_gemm_penalty(1e-3, 0.5e-3, 5e-3) == 100.0


def test_params_roundtrip_and_validation(tmp_path):
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound, p.gemm_memory_bound, p.comm = 1.1, 1.3, 1.05
    f = tmp_path / "cores.json"
    f.write_text(c3sim.save_coresident_params(p))
    q = c3sim.load_coresident_params(str(f))
    assert (q.gemm_compute_bound, q.gemm_memory_bound, q.comm) == (1.1, 1.3, 1.05)
    f.write_text('{"gemm-compute-bound": 0.9, "gemm-memory-bound": 1.0}')
    with pytest.raises(Exception):
        c3sim.load_coresident_params(str(f))


def test_shipped_coresident_params_load():
    q = c3sim.load_coresident_params(c3sim.data_path("b200-coresident.json"))
    assert 1.0 <= q.gemm_compute_bound < 2.0 and 1.0 <= q.gemm_memory_bound and not math.isnan(q.comm)


def test_calibration_tool_recovers_known_parameters(tmp_path):
    """tools/calibrate_coresident.py on a sweep CSV synthesised with the
    runtime's arithmetic from known (p_g, p_c all-gather, p_c all-to-all,
    rate exponent) recovers them (values on the tool's grid: 0.04 / 0.2 / 0.2
    / {0.5, 1, 2, 3, 4, 6})."""
    import json
    import subprocess
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import calibrate_coresident as cal
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound = p.gemm_memory_bound = 1.12
    p.comm, p.comm_all_to_all, p.rate_exponent = 1.6, 2.0, 2.0
    p.all_gather_by_ranks = True  # as the tool fits
    hdr = ("scenario_id,collective,taxonomy,strategy,makespan_s,speedup,ideal,fraction_of_ideal,"
           "t_gemm_iso_ms,t_comm_iso_ms,gemm_tflops_in_step,cus_gemm,cus_comm,backend,world,"
           "predicted_makespan_s,t_comm_ctas_ms,comm_pace_gbps")
    rows = [hdr]
    for sid, coll, tg, tc in (("cfgA_896M", "all-gather", 2.4e-3, 1.1e-3), ("cfgB_1664M", "all-gather", 9.0e-3, 2.0e-3),
                              ("cfgC_896M", "all-to-all", 2.5e-3, 1.1e-3), ("cfgD_896M", "reduce-scatter", 2.4e-3, 1.0e-3)):
        # a link-bound collective: 1/ctas below 24 CTA units, flat from there
        pts = {c: tc * max(1.0, 24.0 / c) for c in (16, 24, 32, 48, 64)}
        d = {"tg": tg, "tc": tc, "mib": float(sid.rsplit("_", 1)[1].rstrip("M")), "n": 8,
             "kind": {"all-gather": c3sim.CollectiveKind.ALL_GATHER, "all-to-all": c3sim.CollectiveKind.ALL_TO_ALL,
                      "reduce-scatter": c3sim.CollectiveKind.REDUCE_SCATTER}[coll],
             "ccls": c3sim.KernelClass.ALL_GATHER if coll == "all-gather" else c3sim.KernelClass.ALL_TO_ALL,
             "curve": c3sim.CommCurve(sorted(pts) + [148], [pts[c] for c in sorted(pts)] + [tc])}
        peer = 7 / 8 * d["mib"] * 2 ** 20
        for c in (16, 24, 32, 48, 64):
            for pace in (0.0, peer / (0.8 * tg) / 1e9, peer / (0.6 * tg) / 1e9):
                mk = cal.predict(d, c, pace, CB, p)
                tag = "" if pace == 0 else f"_pace{int(pace)}"
                rows.append(f"{sid},{coll},G-long,c3_base_coresident{c}{tag},{mk},1,1,0,{tg * 1e3},{tc * 1e3},"
                            f"0,148,{c},CU,synthetic,nan,{pts[c] * 1e3 if pace == 0 else ''},{pace}")
    src = tmp_path / "sweep.csv"
    src.write_text("\n".join(rows) + "\n")
    out = tmp_path / "cores.json"
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "calibrate_coresident.py"), str(src),
                        str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    got = json.loads(out.read_text())
    assert got["gemm-compute-bound"] == pytest.approx(1.12, abs=0.011)
    assert got["comm"] == pytest.approx(1.6, abs=0.051)
    assert got["comm-all-to-all"] == pytest.approx(2.0, abs=0.051)
    assert got["rate-exponent"] == pytest.approx(2.0, abs=0.01)
    # the reduce-scatter rows were made with the all-to-all factor
    assert got.get("comm-reduce-scatter", 2.0) == pytest.approx(2.0, abs=0.21)
    assert got["all-gather-by-ranks"] is True
    assert got["comm-memory-bound"] == 1.0


def test_comm_factor_beside_memory_bound_gemm():
    """comm_memory_bound: beside a memory-bound GEMM every collective class
    uses that factor; 0 keeps the class factor."""
    p = c3sim.CoResidentParams()
    p.comm, p.comm_all_to_all = 1.0, 2.1
    A2A, MBc = c3sim.KernelClass.ALL_TO_ALL, c3sim.KernelClass.GEMM_MEMORY_BOUND
    assert c3sim.coresident_comm_ctas(42, p, A2A, 8, MBc) == 20
    p.comm_memory_bound = 1.0
    assert c3sim.coresident_comm_ctas(42, p, A2A, 8, MBc) == 42
    assert c3sim.coresident_comm_ctas(42, p, A2A, 8, CB) == 20
    p.comm_memory_bound = 0.5
    with pytest.raises(Exception):
        c3sim.coresident_comm_ctas(42, p, A2A, 8, MBc)


def test_all_gather_factor_by_ranks():
    """all_gather_by_ranks: beside a compute-bound GEMM the all-gather CTA's
    factor is comm + (comm_all_to_all - comm) / (n-1)^2 (n = 2: the all-to-all
    one); beside a memory-bound GEMM, and with the flag off, it is `comm`."""
    p = c3sim.CoResidentParams()
    p.comm, p.comm_all_to_all = 1.0, 2.1
    AG, A2A = c3sim.KernelClass.ALL_GATHER, c3sim.KernelClass.ALL_TO_ALL
    assert c3sim.coresident_comm_ctas(64, p, AG, 2, CB) == 64  # flag off
    p.all_gather_by_ranks = True
    assert c3sim.coresident_comm_ctas(63, p, AG, 2, CB) == 30   # 63 / 2.1
    assert c3sim.coresident_comm_ctas(64, p, AG, 4, CB) == round(64 / (1.0 + 1.1 / 9))
    assert c3sim.coresident_comm_ctas(64, p, AG, 8, CB) == round(64 / (1.0 + 1.1 / 49))
    assert c3sim.coresident_comm_ctas(64, p, AG, 2, c3sim.KernelClass.GEMM_MEMORY_BOUND) == 64
    assert c3sim.coresident_comm_ctas(63, p, A2A, 2, CB) == 30
    assert c3sim.coresident_comm_ctas(64, p, AG) == 64  # no world size: the class factor
    txt = c3sim.save_coresident_params(p)
    assert '"all-gather-by-ranks": true' in txt


def test_all_gather_two_rank_factor():
    """comm_all_gather_two_ranks replaces the all-to-all factor as the n = 2
    limit of the rank-dependent all-gather factor (the all-to-all class keeps
    its own); it round-trips through the params JSON and must be 0 or >= 1."""
    p = c3sim.CoResidentParams()
    p.comm, p.comm_all_to_all, p.all_gather_by_ranks = 1.0, 2.1, True
    p.comm_all_gather_two_ranks = 5.5
    AG, A2A = c3sim.KernelClass.ALL_GATHER, c3sim.KernelClass.ALL_TO_ALL
    assert c3sim.coresident_comm_ctas(55, p, AG, 2, CB) == 10            # 55 / 5.5
    assert c3sim.coresident_comm_ctas(64, p, AG, 4, CB) == round(64 / (1.0 + 4.5 / 9))
    assert c3sim.coresident_comm_ctas(64, p, AG, 8, CB) == round(64 / (1.0 + 4.5 / 49))
    assert c3sim.coresident_comm_ctas(63, p, A2A, 2, CB) == 30          # all-to-all: 63 / 2.1
    txt = c3sim.save_coresident_params(p)
    assert '"comm-all-gather-2": 5.5' in txt
    p.comm_all_gather_two_ranks = 0.5
    with pytest.raises(Exception):
        c3sim.coresident_comm_ctas(42, p, AG, 2, CB)


def test_shipped_coresident_params_load():
    prm = c3sim.load_coresident_params(os.path.join(REPO, "data", "b200-coresident.json"))
    assert prm.all_gather_by_ranks and prm.comm_all_gather_two_ranks >= 1.0


def test_paced_collective_scales_the_gemm_penalty():
    """rate_ratio r < 1 (comm pacing): the GEMM penalty's excess scales by
    r^rate_exponent; r = 1 is the unpaced model."""
    p = c3sim.CoResidentParams()
    p.gemm_compute_bound, p.rate_exponent = 1.2, 2.0
    tg, tc = 2.4e-3, 1.0e-3
    base = c3sim.simulate_coresident(tg, tc, tc, 148, 24, CB, p)
    assert c3sim.simulate_coresident(tg, tc, tc, 148, 24, CB, p, 1.0).makespan == pytest.approx(base.makespan)
    # paced to half the rate: the collective takes 2 tc, the penalty excess 0.2 * 0.25
    tl = c3sim.simulate_coresident(tg, 2 * tc, tc, 148, 24, CB, p, 0.5)
    pen = 1.0 + 0.2 * 0.25
    assert tl.makespan == pytest.approx(2 * tc + tg - 2 * tc / pen)
    assert tl.makespan < base.makespan  # exponent 2 > 1: spreading pays
    p.rate_exponent = 1.0  # linear: lost GEMM work ~ equal, no clear gain
    lin = c3sim.simulate_coresident(tg, 2 * tc, tc, 148, 24, CB, p, 0.5)
    assert lin.makespan == pytest.approx(2 * tc + tg - 2 * tc / 1.1)
    for bad in (0.0, 1.5):
        with pytest.raises(Exception):
            c3sim.simulate_coresident(tg, tc, tc, 148, 24, CB, p, bad)


def test_rate_exponent_roundtrip_and_default(tmp_path):
    p = c3sim.CoResidentParams()
    p.rate_exponent = 2.75
    f = tmp_path / "c.json"
    f.write_text(c3sim.save_coresident_params(p))
    assert c3sim.load_coresident_params(str(f)).rate_exponent == 2.75
    f.write_text('{"gemm-compute-bound": 1.1, "gemm-memory-bound": 1.0, "comm": 1.5}')
    assert c3sim.load_coresident_params(str(f)).rate_exponent == 1.0


def test_round2_extensions_cta_cost_phase2_and_reduce_scatter_factor(tmp_path):
    """cta_cost: every resident collective CTA unit slows the GEMM, paced or
    not; phase 2: once the GEMM is done the collective's CTAs run alone (the
    curve time, no co-residency factor); comm_reduce_scatter: the pull's own
    CTA factor, applied through for_kind."""
    p = c3sim.CoResidentParams()
    tg, tc = 2.4e-3, 1.0e-3
    base = c3sim.simulate_coresident(tg, tc, tc, 148, 16, CB, p).makespan
    p.cta_cost = 0.3
    m16 = c3sim.simulate_coresident(tg, tc, tc, 148, 16, CB, p).makespan
    m64 = c3sim.simulate_coresident(tg, tc, tc, 148, 64, CB, p).makespan
    assert base < m16 < m64
    # GEMM rate during phase 1: 1 / (1 + 0.3 * c / 148)
    assert m16 == pytest.approx(tc + tg - tc / (1 + 0.3 * 16 / 148))
    # C-long: the collective outlives the GEMM; after it, its CTAs run at the
    # alone-rate, not at the co-resident (derated) one
    q = c3sim.CoResidentParams()
    slow = c3sim.simulate_coresident(0.3e-3, 4.0e-3, 2.0e-3, 148, 8, MB, q).makespan
    fast = c3sim.simulate_coresident(0.3e-3, 4.0e-3, 2.0e-3, 148, 8, MB, q, 1.0, 2.0e-3).makespan
    assert fast == pytest.approx(0.3e-3 + (2.0e-3 - 0.3e-3 * 2.0e-3 / 4.0e-3) * 2.0e-3 / 2.0e-3)
    assert fast < slow
    # the reduce-scatter factor and its JSON round trip
    q.comm_all_to_all = 2.0
    q.comm_reduce_scatter = 3.5
    rs = q.for_kind(c3sim.CollectiveKind.REDUCE_SCATTER)
    a2a = q.for_kind(c3sim.CollectiveKind.ALL_TO_ALL)
    assert rs.comm_all_to_all == 3.5 and a2a.comm_all_to_all == 2.0
    assert c3sim.coresident_comm_ctas(24, rs, c3sim.KernelClass.ALL_TO_ALL) == 7
    q.cta_cost = 0.1
    path = tmp_path / "cores.json"
    path.write_text(c3sim.save_coresident_params(q))
    back = c3sim.load_coresident_params(str(path))
    assert back.comm_reduce_scatter == 3.5 and back.cta_cost == pytest.approx(0.1)


def test_shipped_coresident_params_are_the_fit():
    """data/b200-coresident.json: written by tools/calibrate_coresident.py from
    the r02 NVLink-rate sweeps; physically ordered factors."""
    p = c3sim.load_coresident_params(c3sim.data_path("b200-coresident.json"))
    assert 1.0 <= p.gemm_compute_bound <= 3.0 and 1.0 <= p.gemm_memory_bound <= 3.0
    assert 1.0 <= p.comm <= p.comm_all_to_all <= p.comm_reduce_scatter <= 6.0
