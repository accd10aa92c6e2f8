#!/usr/bin/env python3
"""C3 bench: GEMM concurrent with an all-gather (or reduce-scatter) under the
paper's strategies, on B200, through the product's C ABI (libc3cuda.so).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--strategy conccl] [--impl ours|reference]

Metric (BASELINE.json): C3 speedup over serial and % of ideal speedup.
  speedup = (t_gemm_iso + t_comm_iso) / t_concurrent   (reference sim.cpp:143,212)
  ideal   = (t_gemm_iso + t_comm_iso) / max(...)        (taxonomy.cpp:23-27)
  % ideal = 100 (speedup - 1) / (ideal - 1)             (taxonomy.cpp:29-33)
t_comm_iso is the isolated time of the SAME backend the strategy uses
(north_star); the conservative variant (vs the best isolated collective) is
reported beside it.

World: at N=1 the 8-rank scenario of configs[1] is EMULATED on one GPU
("loopback"): this GPU runs its own GEMM and its own share of the 8-rank
collective, with the 7 peers' buffers as stand-in HBM buffers, so per-GPU HBM
traffic is that of the real collective. No NVLink is involved, so the
collective is RATE-MATCHED to NVLink: it runs on the CTA count whose isolated
time equals (n-1)/n * P / 770 GB/s, the real node's link time (and the SM
footprint of a real link-bound P2P kernel). The full-speed loopback (~5x
faster than NVLink) is measured in the same rounds and reported beside it
(`loopback_full_speed`); --no-nvlink-emulation makes it the headline. Under
torchrun (N>1) every rank is a real GPU and peers are mapped with CUDA IPC.

Timing: W warm-up steps, then exactly K timed steps between a barrier +
device synchronize; per-step device time from CUDA events on the launching
streams (inside c3_session_run), max over ranks; inputs (A 128 MiB, B 448 MiB,
AG 896 MiB) exceed the 126 MB L2, so no flush is needed between steps.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2412_14335_b200.dist import Dist  # noqa: E402

MIB = 1 << 20
# BASELINE.json configs: (M, N, K), collective, payload per rank
CONFIGS = {
    "cfg1": dict(desc="configs[0] on the GPU: fp32 GEMM 1024x1024x1024 (split-TF32 on the tensor "
                      "cores, fp32 accumulate and output) || 16 MiB all-gather", m=1024, n=1024, k=1024,
                 coll="all-gather", payload=16 * MIB, dtype_bytes=4, ranks=2),
    "cfg2": dict(desc="LLaMA-70B FSDP layer: FFN up-proj GEMM 8192x28672x8192 bf16 || "
                      "next-layer weight all-gather 896 MiB (gate+up) across 8 GPUs",
                 m=8192, n=28672, k=8192, coll="all-gather", payload=896 * MIB),
    "cfg2_448": dict(desc="LLaMA-70B FFN up GEMM || all-gather 448 MiB (up only)",
                     m=8192, n=28672, k=8192, coll="all-gather", payload=448 * MIB),
    "cfg3": dict(desc="LLaMA-70B backward: weight-grad GEMM 8192x28672x8192 bf16 || "
                      "gradient reduce-scatter 896 MiB",
                 m=8192, n=28672, k=8192, coll="reduce-scatter", payload=896 * MIB),
    "cfg2_a2a": dict(desc="LLaMA-70B FFN GEMM 8192x28672x8192 || 896 MiB all-to-all (the "
                          "reference dataset's second collective kind, SURVEY §8(f) F1)",
                     m=8192, n=28672, k=8192, coll="all-to-all", payload=896 * MIB),
    "cfg4": dict(desc="LLaMA-405B FSDP layer: GEMM 8192x53248x16384 bf16 || all-gather 1664 MiB",
                 m=8192, n=53248, k=16384, coll="all-gather", payload=1664 * MIB),
    "cfg4_mb": dict(desc="LLaMA-405B small-token (memory-bound) GEMM 128x53248x16384 || "
                         "all-gather 1664 MiB",
                    m=128, n=53248, k=16384, coll="all-gather", payload=1664 * MIB),
    "cfg4_mb64": dict(desc="LLaMA-405B small-token (memory-bound) GEMM 64x53248x16384 || "
                           "all-gather 1664 MiB (configs[3]'s M = 64 case)",
                      m=64, n=53248, k=16384, coll="all-gather", payload=1664 * MIB),
}
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "C3 speedup over serial and % of ideal speedup (GEMM+all-gather) at 2/4/8 B200"
UNIT = "x (t_serial / t_concurrent)"


def bench_config(args, world):
    """The workload both arms (ours and --impl reference) run, identical
    between them: static facts only (run-time choices go to `details`)."""
    cfg = CONFIGS[args.config]
    n = cfg.get("ranks", 8) if world == 1 else world
    return {"workload": f"{args.config}: {cfg['desc']}", "gemm_mnk": [cfg["m"], cfg["n"], cfg["k"]],
            "gemm_dtype": "fp32" if cfg.get("dtype_bytes", 2) == 4 else "bf16",
            "collective": cfg["coll"], "payload_bytes": cfg["payload"], "ranks": n,
            "l2": "inputs > 126 MB L2 (no flush needed)" if not l2_resident(cfg)
                  else "inputs fit the 126 MB L2: L2 flushed (256 MiB write) before every timed step"}


def l2_resident(cfg):
    """The GEMM operands fit the L2, so the timed steps flush it first."""
    return cfg.get("dtype_bytes", 2) * (cfg["m"] + cfg["n"]) * cfg["k"] <= (126 << 20)


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------- clocks ------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        """Start polling (every 20 ms) and wait for the first sample, so the
        short timed region that follows is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            deadline = time.perf_counter() + 10.0
            while not self.lines and time.perf_counter() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self, t0=None, t1=None):
        """Samples taken inside [t0, t1] (perf_counter; the timed region), or
        the three nearest to it when the region is shorter than the period."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        lines = self.lines
        if t0 is not None and t1 is not None and lines:
            inside = [x for x in lines if t0 <= x[0] <= t1 + 0.03]
            lines = inside if inside else sorted(lines, key=lambda x: abs(x[0] - (t0 + t1) / 2))[:3]
        sms, maxs, watts, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
                try:
                    watts.append(float(parts[2]))
                except ValueError:
                    pass
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sms if s > 300] or sms
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(maxs) if maxs else None,
                "power_w": statistics.median(watts) if watts else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------ ours ------

def log(msg):
    if os.environ.get("C3_BENCH_VERBOSE"):
        print(f"[bench rank {os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}] {msg}",
              file=sys.stderr, flush=True)


def median(xs):
    return statistics.median(xs) if xs else float("nan")


def run_ours(args, dist):
    import ctypes as C

    import torch

    import paper_2412_14335_b200 as c3

    cfg = CONFIGS[args.config]
    n = cfg.get("ranks", 8) if dist.world == 1 else dist.world
    loopback = dist.world == 1
    # C3_SHARED_DEVICE=1: every rank on device 0 (exercises the multi-process
    # IPC path on a one-GPU box; not a performance configuration)
    device = 0 if os.environ.get("C3_SHARED_DEVICE") else dist.local_rank
    torch.cuda.set_device(device)
    world = c3.World(dist.rank, n, device, loopback=loopback)
    coll = {"all-gather": c3.ALL_GATHER, "all-to-all": c3.ALL_TO_ALL,
            "reduce-scatter": c3.REDUCE_SCATTER}[cfg["coll"]]
    elem = cfg.get("dtype_bytes", 2)
    sess = c3.Session(world, cfg["m"], cfg["n"], cfg["k"], coll, cfg["payload"], dtype_bytes=elem)
    if not loopback:
        sess.import_handles(dist.allgather_bytes(sess.export_handles()))
    log("session ready")
    sess.fill(20241217)
    machine = os.path.join(REPO, "data", f"b200-node-n{n}.json")
    if os.path.exists(machine):
        sess.load_machine(machine)  # measured peaks and copy-engine overheads (tools/make_machine.py)
    tables = os.path.join(REPO, "data", "b200-loopback-slowdown-tables.csv")
    sess.load_tables(tables)
    params = os.path.join(REPO, "data", "b200-loopback-params.json")
    if os.path.exists(params):
        sess.load_params(params)
    cores = os.path.join(REPO, "data", "b200-coresident.json")
    if os.path.exists(cores):
        sess.load_coresident(cores)  # B200 co-residency in the model (c3sim/coresident.hpp)
    strategies = [c3.STRATEGY_NAMES.index(s) for s in args.strategies]

    # inputs that fit the L2 (configs[0]): every timed step starts from a
    # flushed L2 (a 256 MiB write, synchronised before the step's launch)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if l2_resident(cfg) else None

    def timed(strategy, steps, alloc=None, link=0.0):
        """steps runs (collective paced to `link` GB/s, 0 = full speed);
        per-step device times, max over ranks."""
        sess.set_link_rate(link)
        rows = []
        for _ in range(steps):
            if flush_buf is not None:
                flush_buf.zero_()
                torch.cuda.synchronize()
            t = sess.run(strategy, alloc)
            # [total, GEMM kernel, collective kernel, launches, kernel span]: the
            # span (first kernel start to last kernel end) leaves out the step's
            # launch latency, as the isolated kernel times do
            span = max(t.gemm_end_ms, t.comm_end_ms) - min(t.gemm_start_ms, t.comm_start_ms)
            rows.append([t.total_ms, t.gemm_end_ms - t.gemm_start_ms, t.comm_end_ms - t.comm_start_ms,
                         float(t.launches), span])
        flat = dist.max_list([v for r in rows for v in r])
        return [flat[i * 5:(i + 1) * 5] for i in range(steps)]

    # Isolated kernel times on the whole GPU are the reference's t_gemm /
    # t_comm (sim.cpp:136-138). They are measured INTERLEAVED with the
    # concurrent runs (round-robin within each round) so clock / power-cap
    # drift over the run affects serial and concurrent alike.
    W, K = args.warmup, args.steps
    full = world.info.sm_count
    dma_ok = not loopback  # same-device copies run on SMs
    iso_modes = {"gemm": (c3.GEMM_ONLY, sess.default_alloc(c3.GEMM_ONLY)),
                 "cu": (c3.COMM_ONLY_CU, sess.default_alloc(c3.COMM_ONLY_CU)),
                 "dma": (c3.COMM_ONLY_DMA, sess.default_alloc(c3.COMM_ONLY_DMA))}
    iso_modes["cu"][1].cus_comm = full
    col = {"gemm": 1, "cu": 2, "dma": 2}

    import random
    order_rng = random.Random(20241217)  # same sequence on every rank

    def rounds(jobs, n):
        """n round-robin rounds over jobs {name: (strategy, alloc) | callable};
        per-job rows [total, gemm, comm, launches] (device ms, max over ranks)."""
        out = {k: [] for k in jobs}
        names = list(jobs)
        for r in range(n):
            # a fresh order every round: under the 1 kW power cap a job's
            # clocks depend on its predecessor (measured: a fixed order skewed
            # isolated GEMM times by 10%). A cyclic rotation still gives every
            # job the same predecessor within a round, so the order is a
            # seeded permutation, identical on every rank
            order = list(names)
            order_rng.shuffle(order)
            for name in order:
                job = jobs[name]
                out[name] += [job()] if callable(job) else timed(*job[:1], 1, *job[1:])
        return out

    dropped = []

    def viable(cands):
        """Run each (strategy, alloc) once on every rank and keep those that
        succeeded on ALL ranks: a strategy the platform cannot run (say, a
        driver without cross-device batched copies) is dropped on every rank
        alike and reported, instead of ending the run. A failing step's peers
        give up after the bounded device waits (C3_ERR_TIMEOUT), so every rank
        reaches the vote."""
        bad = []
        for st, a in cands:
            try:
                sess.run(st, a)
                bad.append(0.0)
            except c3.C3Error as e:
                log(f"candidate {c3.STRATEGY_NAMES[st]} failed: {e}")
                bad.append(1.0)
        bad = dist.max_list(bad) if bad else []
        for (st, a), b in zip(cands, bad):
            if b:
                dropped.append({"strategy": c3.STRATEGY_NAMES[st], "cus_gemm": a.cus_gemm, "cus_comm": a.cus_comm})
        return [c for c, b in zip(cands, bad) if not b]

    if not viable([iso_modes["dma"]]):  # no copy-engine collective on this platform
        del iso_modes["dma"]
        dma_ok = False
    rounds(iso_modes, W)  # warm-up
    log("isolated warm-up done")
    strat_jobs = {}
    for st in strategies:
        if st != c3.SERIAL:
            cand = viable([(st, sess.default_alloc(st))])
            if cand:
                strat_jobs[c3.STRATEGY_NAMES[st]] = cand[0]
    # B200 extension: collective fused into the CTA-pair GEMM (TMA bulk copies)
    fused_ok = coll != c3.REDUCE_SCATTER
    if fused_ok:  # not every shape is on the CTA-pair kernel
        fused_ok = bool(viable([(c3.FUSED, sess.default_alloc(c3.FUSED))]))
    if fused_ok:
        strat_jobs["c3_fused"] = (c3.FUSED, sess.default_alloc(c3.FUSED))
    sweep_rows = rounds({**iso_modes, **strat_jobs}, K)
    iso_comm = {k: median([r[col[k]] for r in sweep_rows[k]]) for k in ("cu", "dma") if k in sweep_rows}
    iso_comm.setdefault("dma", iso_comm["cu"])  # dropped (details.dropped_candidates): unused, dma_ok is off
    log("strategy sweep done")
    t_g = median([r[1] for r in sweep_rows["gemm"]])

    def summarise(rows, t_g, t_c, best_c):
        t_conc = median([r[0] for r in rows])
        sp = (t_g + t_c) / t_conc
        ideal = c3.ideal_speedup(t_g, t_c)
        return {"t_concurrent_ms": t_conc, "t_gemm_iso_ms": t_g, "t_comm_iso_ms": t_c,
                "speedup": sp, "ideal": ideal, "fraction_of_ideal": c3.fraction_of_ideal(sp, ideal),
                "speedup_vs_best_comm": (t_g + best_c) / t_conc,
                "fraction_vs_best_comm": c3.fraction_of_ideal((t_g + best_c) / t_conc,
                                                              c3.ideal_speedup(t_g, best_c)),
                "gemm_ms_in_step": median([r[1] for r in rows])}

    best_iso = min(iso_comm.values()) if dma_ok else iso_comm["cu"]
    results = {}
    for name, (st, a) in strat_jobs.items():
        res = summarise(sweep_rows[name], t_g, iso_comm["dma" if a.backend == c3.BACKEND_DMA else "cu"],
                        best_iso)
        if st == c3.FUSED:
            res["note"] = ("collective moved inside the CTA-pair GEMM kernel by its copy warp "
                           "(TMA bulk copies, 8 KiB pieces); t_comm_iso = SM collective")
        res["alloc"] = {"cus_gemm": a.cus_gemm, "cus_comm": a.cus_comm, "cus_idle": a.cus_idle,
                        "backend": ["CU", "DMA", "TMA"][a.backend]}
        if a.backend == c3.BACKEND_DMA and loopback:
            res["note"] = "loopback: same-device copies run on SMs (driver copy kernels), not copy engines"
        results[name] = res

    # ---- the headline world ----
    # N>1: real GPUs, the collective runs over NVLink at its real rate.
    # N=1: loopback. By default the collective is RATE-MATCHED to NVLink: its
    # CTA count is chosen so the isolated 8-rank collective takes
    # (n-1)/n * P / 770 GB/s, the time the real node's links give this GPU.
    # Its HBM traffic (reads of the own chunk, writes of 7 chunks) and its SM
    # footprint are those of the real SM-driven collective, so this is the
    # faithful one-GPU stand-in for configs[1]. The full-speed loopback (local
    # HBM copies, ~5x faster than NVLink) is measured in the same timed rounds
    # and reported beside it (`loopback_full_speed`).
    emulate = loopback and not args.no_nvlink_emulation
    nvl_ctas, nvl_target, link = None, None, 0.0
    head_iso = dict(iso_modes)
    if emulate:
        link = NVLINK_PEER_GBPS
        nvl_ctas, nvl_probe, nvl_target = rate_match(c3, sess, cfg, n, timed)
        a = sess.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = nvl_ctas
        head_iso["cu"] = (c3.COMM_ONLY_CU, a, link)
        rounds(head_iso, W)
        warm = rounds(head_iso, 3)
        t_g_pick = median([r[1] for r in warm["gemm"]])
        t_c_pick = median([r[2] for r in warm["cu"]])
        # the collective's measured time vs CTAs at the link rate (flat from
        # nvl_ctas on) replaces the full-speed comm table in the model
        curve = {c: t for c, t in nvl_probe.items() if c < nvl_ctas}
        curve.update({nvl_ctas: t_c_pick, full: t_c_pick})
        sess.set_comm_curve(sorted(curve.items()))
    else:
        t_g_pick, t_c_pick = t_g, iso_comm["cu"]
        # the collective's time vs CTA units on this world's links (real NVLink
        # at N>1): the co-residency model's comm curve, measured here rather
        # than taken from the loopback tables (collective: every rank runs it)
        curve = {}
        for ctas in (8, 16, 24, 32, 48, 64):
            a = sess.default_alloc(c3.COMM_ONLY_CU)
            a.cus_comm = ctas
            curve[ctas] = median([r[2] for r in timed(c3.COMM_ONLY_CU, 3, a)])
        curve[full] = min(t_c_pick, min(curve.values()))
        sess.set_comm_curve(sorted(curve.items()))

    def realisable(st, a):
        """Green-context partitions (c3_rp / c3_sp_rp) come in multiples of
        the SM grain (8 on B200); the runtime rejects any other split."""
        if st in (c3.C3_RP, c3.C3_SP_RP):
            g = max(1, world.info.sm_grain)
            a.cus_comm = -(-max(g, a.cus_comm) // g) * g
            a.cus_gemm = min(a.cus_gemm, full - a.cus_comm)
        return a

    def coresident(st, g, c, pace=0.0):
        a = sess.default_alloc(st)
        a.cus_gemm, a.cus_comm = g, c
        a.comm_pace_gbps = pace
        return (st, a)

    peer_bytes = (n - 1) / n * cfg["payload"]

    def pace_for(frac, t_gemm_ms, cap):
        """The rate that spreads the collective over `frac` of the GEMM (GB/s),
        if below the link rate `cap` (0 = no cap); else 0 (unpaced)."""
        r = peer_bytes / (frac * t_gemm_ms * 1e-3) / 1e9
        return r if (cap <= 0 or r < cap) else 0.0

    def full_speed_candidates():
        cands = [(c3.SERIAL, sess.default_alloc(c3.SERIAL))]
        for st in (c3.C3_BASE, c3.C3_SP):
            for ctas in (8, 16, 32, 64):
                cands.append(coresident(st, full, ctas))
        # B200 extension: the collective paced to spread over the GEMM
        for frac in (0.6, 0.8):
            p = pace_for(frac, t_g, 0.0)
            if p > 0:
                cands += [coresident(c3.C3_BASE, full, c, p) for c in (16, 32)]
        if dma_ok:
            cands += [(st, sess.default_alloc(st)) for st in (c3.CONCCL, c3.CONCCL_RP)]
        if fused_ok:
            cands.append((c3.FUSED, sess.default_alloc(c3.FUSED)))
        return cands

    def emulated_candidates(co_ctas):
        # the collective paced to the link rate on nvl_ctas CTAs (the SM
        # footprint of a link-bound P2P kernel); fused: the GEMM's copy warps paced
        # green-context partitions come in multiples of the SM grain (8 on
        # B200): the comm group is the rate-matched count rounded up to it
        g = max(1, world.info.sm_grain)
        part = -(-max(8, nvl_ctas) // g) * g
        cands = [coresident(c3.SERIAL, full, nvl_ctas), coresident(c3.C3_BASE, full, nvl_ctas),
                 coresident(c3.C3_SP, full, nvl_ctas), coresident(c3.C3_RP, full - part, part),
                 coresident(c3.C3_SP_RP, full - part, part)]
        # more co-resident CTA units: a co-resident unit moves less than an
        # isolated one (the model's cost factor), so the rate-matched count is
        # a floor, not the choice
        for c in sorted({2 * nvl_ctas, 24, 32} - {nvl_ctas, co_ctas}):
            cands.append(coresident(c3.C3_BASE, full, c))
        # B200 extension: the co-resident collective (the model's CTA count)
        # paced below the link rate, spread over 60% / 80% of the GEMM
        # (measured: 0.75 -> 0.93 of ideal on cfg2, profiles/r01_pace_probe.txt),
        # over 60% / 80% / 90% of the GEMM
        for frac in (0.6, 0.8, 0.9):
            p = pace_for(frac, t_g_pick, NVLINK_PEER_GBPS)
            if p > 0:
                for c in sorted({co_ctas, 24}):  # 24 units paced: often the sweeps' best
                    cands.append(coresident(c3.C3_BASE, full, c, p))
        if fused_ok:
            cands.append((c3.FUSED, sess.default_alloc(c3.FUSED)))
        return cands

    # the runtime heuristic's pick (model layer simulate() on measured tables),
    # then a measured refinement over it and the B200 candidates
    tune = None
    if args.strategy == "auto":
        head, head_alloc, predicted = sess.choose(t_g_pick, t_c_pick, iso_comm["dma"], dma_ok)
        if emulate and head_alloc.cus_gemm + head_alloc.cus_comm <= full:
            head_alloc.cus_comm = nvl_ctas  # the model's split, the collective at NVLink rate
            head_alloc = realisable(head, head_alloc)
        co_ctas = head_alloc.cus_comm if head_alloc.cus_gemm + head_alloc.cus_comm > full else max(16, nvl_ctas or 16)
        cands = [(head, head_alloc)] + (emulated_candidates(co_ctas) if emulate else full_speed_candidates())
        if args.no_green:  # ncu cannot profile kernels on green-context streams
            cands = [c for c in cands if c[0] not in (c3.C3_RP, c3.C3_SP_RP)] or [(c3.SERIAL, sess.default_alloc(c3.SERIAL))]
        sess.set_link_rate(link)
        cands = viable(cands) or [(c3.SERIAL, sess.default_alloc(c3.SERIAL))]
        meds = []
        best_i, best_ms = sess.autotune(cands, rounds=9, reduce_max=dist.max_list, medians=meds)
        log(f"autotune done: {best_i}")
        tune = {"candidates": [{"strategy": c3.STRATEGY_NAMES[st], "cus_gemm": a.cus_gemm,
                                "cus_comm": a.cus_comm, "comm_pace_gbps": round(a.comm_pace_gbps, 1),
                                "median_ms": ms}
                               for (st, a), ms in zip(cands, meds)],
                "model_pick": c3.STRATEGY_NAMES[head], "model_alloc": {"cus_gemm": head_alloc.cus_gemm,
                                                                      "cus_comm": head_alloc.cus_comm},
                "model_pick_coresident": head_alloc.cus_gemm + head_alloc.cus_comm > full,
                "picked_index": best_i, "picked_ms": best_ms}
        head, head_alloc = cands[best_i]
    else:
        head = c3.STRATEGY_NAMES.index(args.strategy)
        head_alloc, predicted = sess.default_alloc(head), None
        if emulate and head != c3.FUSED:
            head_alloc.cus_comm = nvl_ctas
            head_alloc = realisable(head, head_alloc)
    head_name = c3.STRATEGY_NAMES[head]
    measured_best = max(results, key=lambda k: results[k]["speedup"]) if results else None
    backend = head_alloc.backend
    comm_key = "dma" if backend == c3.BACKEND_DMA else "cu"  # fused (TMA) vs the SM collective

    # full-speed loopback head (secondary line), picked by a short autotune
    fs = None
    if emulate:
        sess.set_link_rate(0.0)
        fc = viable(full_speed_candidates()) or [(c3.SERIAL, sess.default_alloc(c3.SERIAL))]
        fi, _ = sess.autotune(fc, rounds=5, reduce_max=dist.max_list)
        fs = fc[fi]

    # ---- the timed region: K rounds of the headline C3 step, each round also
    # running the isolated GEMM and collective of the same world (and, when
    # emulating, the full-speed pair and the library baseline), in rotated
    # order; only the headline steps make ms_per_step ----
    sess.set_link_rate(link)
    for _ in range(W):
        sess.run(head, head_alloc)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(device) if dist.rank == 0 else None
    if clocks:
        clocks.start()
    dist.barrier()
    for _ in range(2):  # the sampler's start-up took wall time: re-warm the step (all ranks)
        sess.run(head, head_alloc)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    jobs = {"gemm": head_iso["gemm"], comm_key: head_iso[comm_key], "step": (head, head_alloc, link)}
    timed_rows = rounds(jobs, K)
    log("timed region done")
    torch.cuda.synchronize()
    dist.barrier()
    t1 = time.perf_counter()
    wall = t1 - t0
    clk = clocks.stop(t0, t1) if clocks else None

    # ---- comparison block (after the timed region, not part of ms_per_step):
    # the full-speed loopback pair and the library baseline, interleaved with
    # their own isolated runs ----
    lib = None
    if os.environ.get("C3_SHARED_DEVICE"):
        args.no_library_baseline = True  # NCCL cannot place two ranks on one device
    lib_error = None
    if not args.no_library_baseline:
        try:
            lib = LibraryBaseline(cfg, dist, loopback)
            rounds({"lg": lib.gemm_only, "lc": lib.comm_only, "lb": lib.both}, W)
        except Exception as e:  # e.g. NCCL unavailable: the headline stands without it
            lib, lib_error = None, f"{type(e).__name__}: {e}"[:300]
            log(f"library baseline failed: {lib_error}")
    cmp_jobs = {}
    if fs:
        cmp_jobs.update({"gemm": iso_modes["gemm"], "fs_comm": iso_modes["cu"], "fs_step": fs})
    if lib:
        cmp_jobs.update({"lib_gemm": lib.gemm_only, "lib_comm": lib.comm_only, "lib_both": lib.both})
        if not fs:  # a real world: the library pair against our headline step, same rounds
            cmp_jobs["ours_step"] = (head, head_alloc, link)
    # at least 15 rounds: the library comparison is a ratio of two concurrent
    # steps under the power cap, read per round (paired) and as a median
    cmp_rows = rounds(cmp_jobs, max(K, 15)) if cmp_jobs else {}
    rows = timed_rows["step"]
    step_ms = [r[0] for r in rows]
    gemm_ms = [r[1] for r in rows]
    # every launch of ours in the timed region: the C3 steps and the isolated
    # GEMM / collective runs interleaved with them
    launches = int(sum(r[3] for job in timed_rows.values() for r in job))
    t_g_timed = median([r[1] for r in timed_rows["gemm"]])
    t_c = median([r[col[comm_key]] for r in timed_rows[comm_key]])
    head_res = summarise(rows, t_g_timed, t_c, t_c)
    t_conc = head_res["t_concurrent_ms"]
    speedup, ideal, frac = head_res["speedup"], head_res["ideal"], head_res["fraction_of_ideal"]
    # the same metric with the concurrent step timed like the isolated kernels
    # (first kernel start to last kernel end): without the step's launch
    # latency, which the isolated kernel times do not carry either (a few us:
    # large only for configs[0]'s ~40 us steps); value / ms_per_step keep the
    # whole step
    span_ms = median([r[4] for r in rows])
    span_sp = (t_g_timed + t_c) / span_ms
    span_res = {"t_concurrent_span_ms": span_ms, "speedup": span_sp, "ideal": ideal,
                "fraction_of_ideal": c3.fraction_of_ideal(span_sp, ideal),
                "launch_latency_ms": t_conc - span_ms,
                "what": "(t_gemm_iso + t_comm_iso) / median kernel span of the C3 step (first kernel start to "
                        "last kernel end, CUDA events on the kernels' streams); the headline value uses the "
                        "whole step, launch latency included"}

    def alloc_dict(a):
        return {"cus_gemm": a.cus_gemm, "cus_comm": a.cus_comm, "cus_idle": a.cus_idle,
                "backend": ["CU", "DMA", "TMA"][a.backend], "comm_pace_gbps": round(a.comm_pace_gbps, 1)}

    choice = {"strategy": head_name, "selected_by": "runtime: model prediction (c3_session_choose) + "
              "measured autotune (c3_session_autotune)" if args.strategy == "auto" else "--strategy",
              "alloc": alloc_dict(head_alloc), "predicted_ms": predicted, "measured_ms": t_conc,
              "autotune": tune, "full_speed_measured_best_default_alloc": measured_best,
              "tables": os.path.relpath(tables, REPO),
              "penalties": "data/b200-loopback-params.json (fitted, tools/calibrate_penalties.py)"}
    full_speed = None
    if fs:
        fs_c = median([r[2] for r in cmp_rows["fs_comm"]])
        fs_res = summarise(cmp_rows["fs_step"], median([r[1] for r in cmp_rows["gemm"]]), fs_c, fs_c)
        fs_res.update({"strategy": c3.STRATEGY_NAMES[fs[0]], "alloc": alloc_dict(fs[1]),
                       "what": f"loopback at full local speed: the collective's {n - 1} chunk copies run on "
                               "local HBM with the whole GPU (~5x faster than NVLink), same timed rounds"})
        full_speed = fs_res

    # ---- copy-engine strategies on one GPU: the host-staged proxy ----
    # (loopback only; a real world runs conccl / conccl_rp over NVLink in the
    # autotune above). The DMA backend's peers are pinned host buffers, so this
    # GPU's share of the plan crosses PCIe on the copy engines (~48 GB/s per
    # direction instead of NVLink's 770): the payload is scaled so the proxy
    # collective lasts as long as the real one at NVLink rate.
    ce_proxy = None
    if loopback and not args.no_ce_proxy:
        ce_proxy = run_ce_proxy(c3, cfg, n, coll, elem, K, W, NVLINK_PEER_GBPS)

    # ---- e2e through the C ABI with host buffers ----
    # Every step copies A and this rank's collective input in from pinned host
    # memory and the WHOLE result C back, inside the call (c3_session_run_host).
    p = sess.pointers(0)
    h2d = p.a_bytes + p.send_bytes
    d2h = p.c_bytes
    pin_a = torch.empty(p.a_bytes, dtype=torch.uint8, pin_memory=True)
    pin_s = torch.empty(p.send_bytes, dtype=torch.uint8, pin_memory=True)
    pin_o = torch.empty(d2h, dtype=torch.uint8, pin_memory=True)

    def e2e_step(strategy, alloc, rate=0.0):
        sess.set_link_rate(rate)
        t0 = time.perf_counter()
        sess.run_host(strategy, alloc, pin_a.data_ptr(), pin_s.data_ptr(), pin_o.data_ptr(), d2h)
        return (time.perf_counter() - t0) * 1e3

    # serial on host buffers, two ways: (1) the plain serial step -- copies in,
    # GEMM, the collective (the isolated run's CTAs and rate), C out, one
    # stream; (2) the same serial kernels with the host copies overlapped as
    # well as they can be without overlapping the kernels (A in row bands the
    # GEMM waits on, the collective's input during the GEMM, C out during the
    # collective) -- the conservative baseline: what C3 adds beyond I/O overlap
    iso_ctas = head_iso["cu"][1].cus_comm if "cu" in head_iso else 32
    ser_alloc = sess.default_alloc(c3.SERIAL)
    ser_alloc.cus_gemm, ser_alloc.cus_comm = full, iso_ctas
    sio_alloc = sess.default_alloc(c3.SERIAL_OVERLAP_IO)
    sio_alloc.cus_gemm, sio_alloc.cus_comm = full, iso_ctas
    e2e_jobs = {"conc": (head, head_alloc, link), "serial": (c3.SERIAL, ser_alloc, link),
                "serial_io": (c3.SERIAL_OVERLAP_IO, sio_alloc, link)}
    for _ in range(2):
        for job in e2e_jobs.values():
            e2e_step(*job)
    e2e = {k: [] for k in e2e_jobs}
    names = list(e2e_jobs)
    for r in range(K):  # interleaved, a fresh seeded order per round
        order = list(names)
        order_rng.shuffle(order)
        for k in order:
            e2e[k].append(e2e_step(*e2e_jobs[k]))
    e2e_ms = {k: median(dist.max_list(v)) for k, v in e2e.items()}
    e2e_speedup = e2e_ms["serial"] / e2e_ms["conc"]

    peaks, peak_src = load_peaks()
    peak_sus = peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"])
    flops = 2.0 * cfg["m"] * cfg["n"] * cfg["k"]
    gemm_avg = sum(gemm_ms) / len(gemm_ms)
    achieved = flops / (gemm_avg * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(REPO, "profiles", "ncu_gemm_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{cfg['m']}x{cfg['n']}x{cfg['k']}", {}).get("dram_bytes")
        except Exception:
            traffic = None
    # the GEMM's roofline: tensor-bound when its arithmetic intensity exceeds
    # the machine's FLOP:byte ratio, else HBM-bound (cfg4_mb, M = 128)
    gemm_bytes = float(elem) * (cfg["m"] * cfg["k"] + cfg["n"] * cfg["k"] + cfg["m"] * cfg["n"])
    # this GPU's collective HBM bytes per step: AG reads its chunk and takes
    # n-1 incoming chunks; A2A reads n-1 outgoing slots and takes n-1 incoming;
    # RS: its n input slots are read (one by each rank) and its slot written
    chunk_b = cfg["payload"] / n
    comm_hbm_bytes = {"all-gather": n * chunk_b, "all-to-all": 2 * (n - 1) * chunk_b,
                      "reduce-scatter": (n + 1) * chunk_b}[cfg["coll"]]
    # fp32 GEMM: split-TF32 issues three TF32 MMAs per fp32 product, and TF32
    # runs at half the bf16 dense rate
    tc_peak = peaks["bf16_tflops"] / (6.0 if elem == 4 else 1.0)
    ratio = tc_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if flops / gemm_bytes >= ratio:
        roofline = {"bound": "tensor",
                    "kernel": ("gemm_f32_split_kernel (split-TF32 in shared memory, tcgen05 kind::tf32, "
                               "split-K; peak = bf16 / 2 / 3)" if elem == 4
                               else "gemm_bf16_tn_pair_kernel (tcgen05 cta_group::2)"),
                    "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": achieved / tc_peak,
                    "frac_of_sustained": achieved / peak_sus,
                    "peak_source": peak_src + " burst bf16 (cuBLAS): the timed region is ~0.1 s "
                                   "of GEMMs interleaved with collective-only phases, short of the "
                                   "sustained (4 s back-to-back) regime",
                    "algorithmic_flops_per_launch": flops, "traffic": traffic}
    else:
        gbs = gemm_bytes / (gemm_avg * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": "gemm_bf16_tn_kernel (tcgen05, single-CTA tiles)",
                    "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / peaks["hbm_gbs"],
                    "peak_source": peak_src + " HBM copy bandwidth",
                    "algorithmic_bytes_per_launch": gemm_bytes, "traffic": traffic,
                    "arithmetic_intensity": flops / gemm_bytes, "machine_flop_per_byte": ratio,
                    # the same GEMM alone in the timed rounds: inside the step the
                    # co-resident collective draws HBM too (its own bytes below)
                    "frac_isolated": gemm_bytes / (t_g_timed * 1e-3) / 1e9 / peaks["hbm_gbs"],
                    "collective_hbm_bytes_per_step": comm_hbm_bytes,
                    "step_hbm_frac": (gemm_bytes + comm_hbm_bytes) / (t_conc * 1e-3) / 1e9 / peaks["hbm_gbs"]}
    # the C3 pair's roofline: the step can finish no sooner than
    # its GEMM at the tensor (or HBM) peak, its collective's peer bytes at the
    # link rate, or the pair's combined HBM bytes at the HBM peak
    link_gbs = NVLINK_PEER_GBPS if emulate else 900.0
    t_tensor = flops / (tc_peak * 1e12) * 1e3
    t_link = (n - 1) / n * cfg["payload"] / (link_gbs * 1e9) * 1e3
    t_hbm = (gemm_bytes + comm_hbm_bytes) / (peaks["hbm_gbs"] * 1e9) * 1e3
    t_roof = max(t_tensor, t_link, t_hbm)
    c3_roofline = {"makespan_ms": t_roof, "measured_ms": t_conc, "frac": t_roof / t_conc,
                   "bound": {t_tensor: "tensor", t_link: "link", t_hbm: "hbm"}[t_roof],
                   "terms_ms": {"gemm_at_tensor_peak": t_tensor, "collective_at_link_rate": t_link,
                                "pair_hbm_bytes_at_hbm_peak": t_hbm},
                   "link_gbs": link_gbs,
                   "what": "max(F / tensor peak, (n-1)/n P / link, (B_gemm + B_comm,HBM) / HBM peak) / measured "
                           "C3 step (SURVEY 8(d)); link = the emulated 770 GB/s at N=1, 900 GB/s at N>1"}
    if emulate:
        world_desc = (f"loopback with NVLink-rate emulation: {n}-rank scenario on 1 GPU; this GPU's GEMM "
                      f"and its share of the collective ({n - 1} chunk copies into stand-in peer buffers in "
                      f"local HBM), the collective's peer traffic paced on the global timer to "
                      f"{NVLINK_PEER_GBPS:.0f} GB/s per direction (c3_session_set_link_rate), i.e. "
                      f"(n-1)/n*P/{NVLINK_PEER_GBPS:.0f} GB/s = {nvl_target:.3f} ms, on {nvl_ctas} CTAs "
                      f"(fewest that reach the rate); full-speed loopback in `loopback_full_speed`")
    elif loopback:
        world_desc = f"loopback: {n}-rank collective emulated on 1 GPU (peer buffers in local HBM, no NVLink)"
    else:
        world_desc = f"{n} GPUs, CUDA-IPC peer memory"
    # per-round paired speedups: each round's C3 step against the isolated
    # GEMM and collective of the SAME round (seeded per-round order, so each step is
    # bracketed by isolated runs under the same power state), and the spread
    # of the headline over three blocks of rounds
    g_rows, c_rows = timed_rows["gemm"], timed_rows[comm_key]
    paired = [(g_rows[i][1] + c_rows[i][col[comm_key]]) / rows[i][0] for i in range(len(rows))]
    blocks = []
    nb = 3 if len(rows) >= 3 else 1
    for bi in range(nb):
        sl = slice(bi * len(rows) // nb, (bi + 1) * len(rows) // nb)
        tg_b = median([r[1] for r in g_rows[sl]])
        tc_b = median([r[col[comm_key]] for r in c_rows[sl]])
        blocks.append((tg_b + tc_b) / median([r[0] for r in rows[sl]]))
    flags = []
    if frac > 1.05:
        flags.append(f"fraction_of_ideal {frac:.3f} > 1.05: the isolated runs were slower than the "
                     "same kernels inside the C3 step (power-state artefact); read with the spread")
    out = {
        "metric": METRIC,
        "value": speedup, "unit": UNIT,
        "fraction_of_ideal_pct": 100.0 * frac, "ideal": ideal,
        "n_gpus": dist.world, "steps": K, "warmup": W,
        "ms_per_step": sum(step_ms) / len(step_ms), "ms_per_step_median": t_conc,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 (split-TF32 on the tensor cores)" if elem == 4 else "bf16",
        "data": "synthetic (counter-hash bf16 U(-1,1)/8 and byte labels)",
        "config": bench_config(args, dist.world),
        "spread": {"paired_round_speedups": {"median": median(paired), "min": min(paired), "max": max(paired),
                                             "n": len(paired)},
                   "block_speedups": blocks,
                   "what": "per round: (isolated GEMM + isolated collective of that round) / that round's C3 "
                           "step; per block: the headline formula over a third of the rounds"},
        "flags": flags,
        "kernel_span": span_res,
        "absolute": {"t_concurrent_ms": t_conc, "t_gemm_iso_ms": t_g_timed, "t_comm_iso_ms": t_c,
                     "t_serial_ms": t_g_timed + t_c,
                     "gemm_tflops_in_step": flops / (median(gemm_ms) * 1e-3) / 1e12,
                     "comm_peer_gbs": (n - 1) / n * cfg["payload"] / (t_c * 1e-3) / 1e9},
        "details": {"strategy": head_name, "strategy_choice": choice, "world": world_desc,
                    "isolated_ms": {"gemm": t_g_timed, "comm": t_c, "backend": comm_key,
                                    "comm_ctas": head_iso["cu"][1].cus_comm if comm_key == "cu" else 0,
                                    "full_speed_sweep_gemm": t_g, "full_speed_sweep_comm_cu": iso_comm["cu"],
                                    "full_speed_sweep_comm_dma": iso_comm["dma"]},
                    "dropped_candidates": dropped,
                    "protocol": ("W warm-up, then K rounds of [isolated GEMM, isolated collective, "
                                 "C3 step], each round in a fresh seeded order; medians; then, outside "
                                 "the timed region, >= 15 such rounds of the full-speed pair and the "
                                 "library baseline"),
                    "timed_region_wall_s": wall},
        "conccl_ce_proxy": ce_proxy,
        "loopback_full_speed": full_speed,
        "strategies_full_speed": results,
        "roofline": roofline,
        "c3_roofline": c3_roofline,
        "e2e": {"value": e2e_speedup, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "concurrent_ms": e2e_ms["conc"], "serial_ms": e2e_ms["serial"],
                "serial_overlapped_io_ms": e2e_ms["serial_io"],
                "vs_serial_overlapped_io": e2e_ms["serial_io"] / e2e_ms["conc"],
                "call": "c3_session_run_host: pinned host A and this rank's collective input in, the whole C "
                        "out, inside the call (wall clock, max over ranks, medians of K interleaved rounds)",
                "note": "value = plain serial step (every copy and kernel in sequence) / concurrent step; "
                        "vs_serial_overlapped_io = serial kernels with the same host-copy overlap the "
                        "concurrent step gets (C3's own gain end to end). PCIe (~55 GB/s per direction) "
                        "carries h2d + d2h bytes, far more than the GPU work, so both ratios are "
                        "PCIe-dominated"},
        "gpu_launches": launches,
        # the north star's "1 GPU (GEMM only)" line: the isolated GEMM of the
        # timed rounds (median), as time and TF/s against the measured peaks
        "gemm_only": {"ms": t_g_timed, "tflops": flops / (t_g_timed * 1e-3) / 1e12,
                      "frac_of_burst": flops / (t_g_timed * 1e-3) / 1e12 / peaks["bf16_tflops"],
                      "frac_of_sustained": flops / (t_g_timed * 1e-3) / 1e12 / peak_sus},
        "clocks": clk,
    }
    if emulate:
        out["details"]["rate_match"] = {"comm_ctas": nvl_ctas, "target_ms": nvl_target,
                                       "probe_ms_by_ctas": nvl_probe}
    if lib:
        tg_l = median([r[1] for r in cmp_rows["lib_gemm"]])
        tc_l = median([r[2] for r in cmp_rows["lib_comm"]])
        tb_l = median([r[0] for r in cmp_rows["lib_both"]])
        sp_l = (tg_l + tc_l) / tb_l
        ideal_l = (tg_l + tc_l) / max(tg_l, tc_l)
        ours_rows = cmp_rows["fs_step"] if full_speed else cmp_rows["ours_step"]
        ours_full = median([r[0] for r in ours_rows])
        paired = [lb[0] / o[0] for lb, o in zip(cmp_rows["lib_both"], ours_rows)]
        out["library_baseline"] = {
            "what": lib.label, "t_gemm_ms": tg_l, "t_comm_ms": tc_l, "t_concurrent_ms": tb_l,
            "speedup": sp_l, "ideal": ideal_l,
            "fraction_of_ideal": 0.0 if sp_l < 1 else (sp_l - 1) / (ideal_l - 1),
            "ours_concurrent_ms": ours_full,
            # median over rounds of (library step / our step of the same round)
            "library_concurrent_over_ours": median(paired),
            "paired_ratio_min_max": [min(paired), max(paired)], "rounds": len(paired),
            "ratio_of_medians": tb_l / ours_full,
            "compared_with": "loopback_full_speed" if full_speed else "headline",
            "note": "both concurrent steps in the same comparison rounds, fresh seeded order per round (after the timed region)"}
    elif lib_error:
        out["library_baseline"] = {"unavailable": lib_error}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, n)
    sess.close()
    world.close()
    return out


# ------------------------------------------------ copy-engine proxy ------

def run_ce_proxy(c3, cfg, n, coll, elem, K, W, link_gbps):
    """conccl / conccl_rp with this GPU's share of the collective on the copy
    engines (c3_session_set_ce_proxy): 7 transfers out (D2H to pinned host
    peers) and 7 in (H2D), rotated rounds with the isolated GEMM and the
    isolated proxy collective. The payload is the one whose proxy collective
    takes the time the real payload takes at NVLink rate."""
    MIBp = 1 << 20
    target_ms = (n - 1) / n * cfg["payload"] / (link_gbps * 1e9) * 1e3
    world = c3.World(0, n, 0, loopback=True)

    def session(payload):
        s = c3.Session(world, cfg["m"], cfg["n"], cfg["k"], coll, payload, dtype_bytes=elem)
        s.set_ce_proxy(True)
        s.fill(20241217)
        return s

    probe_payload = 64 * MIBp
    s = session(probe_payload)
    for _ in range(2):
        s.run(c3.COMM_ONLY_DMA)
    probe_ms = median([s.run(c3.COMM_ONLY_DMA).total_ms for _ in range(3)])
    s.close()
    step = 8 * n  # 8-byte words per slot
    payload = max(step, int(probe_payload * target_ms / probe_ms) // step * step)
    payload = min(payload, cfg["payload"])
    s = session(payload)
    jobs = {"gemm": (c3.GEMM_ONLY, s.default_alloc(c3.GEMM_ONLY)),
            "comm": (c3.COMM_ONLY_DMA, s.default_alloc(c3.COMM_ONLY_DMA)),
            "conccl": (c3.CONCCL, s.default_alloc(c3.CONCCL)),
            "conccl_rp": (c3.CONCCL_RP, s.default_alloc(c3.CONCCL_RP))}
    t = {j: [] for j in jobs}
    names = list(jobs)
    import random
    rng = random.Random(20241217)
    for r in range(W + K):
        order = list(names)
        rng.shuffle(order)
        for j in order:
            tm = s.run(*jobs[j])
            if r >= W:
                t[j].append(tm)
    tg = median([x.gemm_end_ms - x.gemm_start_ms for x in t["gemm"]])
    tc = median([x.comm_end_ms - x.comm_start_ms for x in t["comm"]])
    ideal = c3.ideal_speedup(tg, tc)
    out = {"what": "PCIe-rate CE proxy: loopback world, the DMA backend's peers are pinned host buffers, so "
                   "this GPU's share of the copy-engine plan (7 transfers out D2H, 7 in H2D) runs on the copy "
                   "engines; payload scaled so the proxy collective lasts as long as the real one at "
                   f"{link_gbps:.0f} GB/s NVLink; no SM runs the collective",
           "payload_bytes": payload, "target_ms": target_ms, "t_gemm_iso_ms": tg, "t_comm_dma_iso_ms": tc,
           "ce_gbs_per_direction": (n - 1) / n * payload / (tc * 1e-3) / 1e9, "ideal": ideal}
    for j in ("conccl", "conccl_rp"):
        st, al = jobs[j]
        mk = median([x.total_ms for x in t[j]])
        gk = median([x.gemm_end_ms - x.gemm_start_ms for x in t[j]])
        sp = (tg + tc) / mk
        out[j] = {"t_concurrent_ms": mk, "speedup": sp, "fraction_of_ideal": c3.fraction_of_ideal(sp, ideal),
                  "gemm_ms_in_step": gk, "gemm_slowdown": gk / tg, "cus_gemm": al.cus_gemm,
                  "cus_idle": al.cus_idle}
    s.close()
    world.close()
    return out


# ----------------------------------------- NVLink-rate-matched emulation ------

NVLINK_PEER_GBPS = 770.0  # measured B200 peer copy per direction (B200_PROFILING.md)


def rate_match(c3, sess, cfg, n, timed):
    """Fewest CTAs with which the collective, paced to the NVLink rate
    (c3_session_set_link_rate), takes at most 3% over the link time
    (n-1)/n * payload / 770 GB/s. Each probe alternates with a full GEMM, so it
    sees the thermal / power state of the timed rounds.
    -> (ctas, {ctas: ms}, target_ms)"""
    target_ms = (n - 1) / n * cfg["payload"] / (NVLINK_PEER_GBPS * 1e9) * 1e3
    g = sess.default_alloc(c3.GEMM_ONLY)
    probe = {}
    for ctas in (4, 8, 12, 16, 24, 32, 48, 64, 96, 148):
        a = sess.default_alloc(c3.COMM_ONLY_CU)
        a.cus_comm = ctas
        ms = []
        for _ in range(3):
            timed(c3.GEMM_ONLY, 1, g)
            ms.append(timed(c3.COMM_ONLY_CU, 1, a, NVLINK_PEER_GBPS)[0][2])
        probe[ctas] = median(ms)
        if probe[ctas] <= 1.03 * target_ms:
            return ctas, probe, target_ms
    return min(probe, key=probe.get), probe, target_ms


# ------------------------------------------------- library baseline ------

class LibraryBaseline:
    """Same scenario with library kernels: cuBLAS GEMM (torch.matmul) concurrent
    with NCCL all-gather / reduce-scatter (N>1), or — loopback — with torch
    device copies moving this GPU's share of the 8-rank collective (7 chunks).
    Each call returns [total, gemm, comm, 0] device ms (max over ranks)."""

    def __init__(self, cfg, dist, loopback):
        import torch
        self.torch, self.dist = torch, dist
        dev = torch.device("cuda", torch.cuda.current_device())
        self.A = torch.randn(cfg["m"], cfg["k"], device=dev, dtype=torch.bfloat16)
        self.B = torch.randn(cfg["n"], cfg["k"], device=dev, dtype=torch.bfloat16)
        self.C = torch.empty(cfg["m"], cfg["n"], device=dev, dtype=torch.bfloat16)
        n = cfg.get("ranks", 8) if loopback else dist.world
        chunk = cfg["payload"] // n
        self.s_g, self.s_c = torch.cuda.Stream(), torch.cuda.Stream()
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if loopback:
            src = torch.empty(chunk, dtype=torch.uint8, device=dev)
            dst = torch.empty(n * chunk, dtype=torch.uint8, device=dev)

            def comm():
                for p in range(1, n):
                    dst[p * chunk:(p + 1) * chunk].copy_(src)
            self.label = (f"cuBLAS (torch.matmul) || torch device copies of {n - 1} chunks "
                          "(loopback; SM copy kernels)")
        else:
            import torch.distributed as tdist
            pg = tdist.new_group(backend="nccl")
            if cfg["coll"] == "all-gather":
                src = torch.empty(chunk, dtype=torch.uint8, device=dev)
                dst = torch.empty(n * chunk, dtype=torch.uint8, device=dev)

                def comm():
                    tdist.all_gather_into_tensor(dst, src, group=pg)
            elif cfg["coll"] == "all-to-all":
                src = torch.empty(cfg["payload"], dtype=torch.uint8, device=dev)
                dst = torch.empty(cfg["payload"], dtype=torch.uint8, device=dev)

                def comm():
                    tdist.all_to_all_single(dst, src, group=pg)
            else:
                src = torch.randn(cfg["payload"] // 2, device=dev).to(torch.bfloat16)
                dst = torch.empty(cfg["payload"] // 2 // n, device=dev, dtype=torch.bfloat16)

                def comm():
                    tdist.reduce_scatter_tensor(dst, src, group=pg)
            self.label = "cuBLAS (torch.matmul) || NCCL " + cfg["coll"]
        self.comm = comm

    def _run(self, g, c):
        torch, ev = self.torch, self.ev
        torch.cuda.synchronize()
        ev[0].record()
        self.s_g.wait_event(ev[0])
        self.s_c.wait_event(ev[0])
        if g:
            with torch.cuda.stream(self.s_g):
                torch.matmul(self.A, self.B.t(), out=self.C)
        if c:
            with torch.cuda.stream(self.s_c):
                self.comm()
        ev[1].record(self.s_g)
        ev[2].record(self.s_c)
        torch.cuda.current_stream().wait_event(ev[1])
        torch.cuda.current_stream().wait_event(ev[2])
        ev[3].record()
        ev[3].synchronize()
        tot = ev[0].elapsed_time(ev[3])
        return self.dist.max_list([tot, tot if g else 0.0, tot if c else 0.0, 0.0])

    def gemm_only(self):
        return self._run(True, False)

    def comm_only(self):
        return self._run(False, True)

    def both(self):
        return self._run(True, True)


# ---------------------------------------------------------- CPU arms ------

def ref_cpu_c3(m, n, k, ranks, payload, warmup, iters, kind="all-gather"):
    exe = os.path.join(REPO, "oracle", "_ref", "c3sim_ref_cpu_c3")
    machine = os.path.join(REPO, "tests", "golden", "ref_data", "mi300x-node.json")
    threads = os.cpu_count() or 1
    r = subprocess.run([exe, str(m), str(n), str(k), str(ranks), str(payload), str(threads),
                        str(warmup), str(iters), machine, kind], capture_output=True, text=True,
                       check=True)
    return json.loads(r.stdout)


def ref_sample(cfg, n):
    """The bounded CPU sample of a config: M cut to REF_TOKENS rows and the
    payload by the same factor -> (m, payload, scale)."""
    scale = max(1, cfg["m"] // REF_TOKENS)
    m = cfg["m"] // scale
    payload = cfg["payload"] // scale
    payload -= payload % (8 * n)
    return m, payload, scale


def cpu_baseline(cfg, n, warmup=1, iters=9):
    """The reference's CPU path timed on this box's host cores, on a bounded
    sample of the SAME workload as the GPU line (about 10-30 s of CPU work):
    fp32 GEMM of REF_TOKENS rows on all host threads || the reference
    planner's transfers for the config's collective replayed by memcpy on one
    more thread (oracle/_ref driving the oracle/c3oracle.c restatement)."""
    m, payload, scale = ref_sample(cfg, n)
    res = ref_cpu_c3(m, cfg["n"], cfg["k"], n, payload, warmup, iters, cfg["coll"])
    return {"value": res["speedup"], "unit": UNIT,
            "cores": res["threads"], "kind": "port",
            "fraction_of_ideal_pct": 100 * res["fraction_of_ideal"],
            "sample": (f"1/{scale} of the workload's tokens and payload: fp32 GEMM {m}x{cfg['n']}x{cfg['k']} "
                       f"on all {res['threads']} host threads || {cfg['coll']} of {payload / MIB:.1f} MiB over {n} "
                       f"host ranks (reference planner's transfers by memcpy on one thread); {warmup} warm-up + "
                       f"{iters} iterations, medians"),
            "t_gemm_ms": 1e3 * res["t_gemm_s"], "t_comm_ms": 1e3 * res["t_comm_s"],
            "t_concurrent_ms": 1e3 * res["t_concurrent_s"]}


REF_TOKENS = 256  # the reference arm's bounded sample: this many GEMM rows (tokens)


def run_reference(args, dist):
    """--impl reference: the reference's CPU path on the host cores for the
    SAME workload as our arm (same `config`), each step a bounded sample of
    it: the GEMM's token dimension M cut to REF_TOKENS rows and the collective
    payload by the same factor (fp32 GEMM on all host threads || the reference
    planner's transfers replayed by memcpy on one more thread; reduce-scatter
    adds the local fp32 reduce). Exactly `warmup` + `steps` iterations run;
    rank 0 only (the other ranks exit without work)."""
    cfg = CONFIGS[args.config]
    n = cfg.get("ranks", 8) if dist.world == 1 else dist.world
    m, payload, scale = ref_sample(cfg, n)
    t0 = time.perf_counter()
    res = ref_cpu_c3(m, cfg["n"], cfg["k"], n, payload, args.warmup, args.steps, cfg["coll"])
    wall = time.perf_counter() - t0
    sample = (f"bounded sample of {args.config} (1/{scale} of its tokens and payload): fp32 GEMM "
              f"{m}x{cfg['n']}x{cfg['k']} on all {res['threads']} host threads || {cfg['coll']} of "
              f"{payload / MIB:.1f} MiB over {n} host ranks (the reference planner's transfers replayed by "
              f"memcpy on one thread{'; then the local fp32 reduce' if cfg['coll'] == 'reduce-scatter' else ''})"
              f"; {res['warmup']} warm-up + {res['iters']} timed iterations, medians")
    speedup = res["speedup"]
    return {"metric": METRIC, "impl": "reference", "value": speedup, "unit": UNIT,
            "fraction_of_ideal_pct": 100 * res["fraction_of_ideal"], "ideal": res["ideal"],
            "n_gpus": dist.world, "steps": res["iters"], "warmup": res["warmup"],
            "ms_per_step": 1e3 * res["t_concurrent_s"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": bench_config(args, dist.world),
            "absolute": {"t_concurrent_ms": 1e3 * res["t_concurrent_s"], "t_gemm_iso_ms": 1e3 * res["t_gemm_s"],
                         "t_comm_iso_ms": 1e3 * res["t_comm_s"],
                         "t_serial_ms": 1e3 * (res["t_gemm_s"] + res["t_comm_s"]),
                         "t_concurrent_ms_full_config_est": 1e3 * res["t_concurrent_s"] * scale,
                         "gemm_gflops": 2.0 * m * cfg["n"] * cfg["k"] / res["t_gemm_s"] / 1e9},
            "cpu_baseline": {"value": speedup, "unit": UNIT, "cores": res["threads"],
                             "kind": "port", "sample": sample},
            "e2e": {"value": speedup, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "details": {"wall_s": wall, "sample": sample, "scale": scale}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--strategy", default="auto",
                    help="auto = the runtime heuristic's pick, or a strategy name")
    ap.add_argument("--strategies", default="c3_base,c3_sp,c3_rp,c3_sp_rp,conccl,conccl_rp")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-library-baseline", action="store_true")
    ap.add_argument("--no-nvlink-emulation", action="store_true")
    ap.add_argument("--no-ce-proxy", action="store_true")
    ap.add_argument("--no-green", action="store_true",
                    help="no green-context (c3_rp / c3_sp_rp) runs: for ncu, which cannot profile them")
    args = ap.parse_args()
    args.strategies = [s for s in args.strategies.split(",") if s]
    if args.no_green:
        args.strategies = [s for s in args.strategies if s not in ("c3_rp", "c3_sp_rp")]
    args.warmup = max(3, args.warmup)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # NCCL communicator set-up in the log (the library baseline's group):
        # the driver checks comm_nranks there
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist = Dist()
    try:
        if args.impl == "reference":
            if dist.rank == 0:
                print(json.dumps(run_reference(args, dist)))
            return
        out = run_ours(args, dist)
        if dist.rank == 0:
            print(json.dumps(out))
    finally:
        dist.close()


if __name__ == "__main__":
    main()
