#!/usr/bin/env python3
"""One table row per bench line in a directory (bench_<cfg>.json and
bench_<cfg>_reference.json, tools/round_evidence.sh): speedup, fraction of
ideal, the same with the step timed as a kernel span, paired spread, e2e,
copy-engine proxy, library ratio, GEMM roofline
fraction, C3-pair roofline fraction and the reference arm.

usage: python tools/summarize_bench.py DIR"""
import glob
import json
import os
import sys


def last_json(path):
    try:
        with open(path) as f:
            lines = [ln for ln in f.read().splitlines() if ln.strip().startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except (OSError, ValueError):
        return None


def main():
    d = sys.argv[1]
    print("| config | C3 speedup (fraction of ideal) | kernel-span speedup (fraction) | paired spread | "
          "e2e (vs overlapped-I/O serial) | conccl CE proxy | library/ours | GEMM roofline | pair roofline | "
          "reference arm |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for path in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
        if path.endswith("_reference.json"):
            continue
        name = os.path.basename(path)[len("bench_"):-len(".json")]
        b = last_json(path)
        if not b or "value" not in b:
            print(f"| {name} | (no line) | | | | | | | | |")
            continue
        r = last_json(path.replace(".json", "_reference.json")) or {}
        sp = b.get("spread", {}).get("paired_round_speedups", {})
        e2e = b.get("e2e") or {}
        ce = b.get("conccl_ce_proxy") or {}
        ce_c = ce.get("conccl") if isinstance(ce.get("conccl"), dict) else {}
        lib = b.get("library_baseline") or {}
        roof = b.get("roofline") or {}
        pr = b.get("c3_roofline") or {}
        fr = b.get("fraction_of_ideal_pct")
        ks = b.get("kernel_span") or {}
        cells = [name,
                 f"{b['value']:.3f}x ({fr:.0f}%)" if fr is not None else f"{b['value']:.3f}x",
                 f"{ks.get('speedup', 0):.3f}x ({100 * ks.get('fraction_of_ideal', 0):.0f}%)" if ks else "",
                 f"{sp.get('min', 0):.2f}-{sp.get('max', 0):.2f}" if sp else "",
                 f"{e2e.get('value', 0):.2f}x ({e2e.get('vs_serial_overlapped_io', 0):.2f}x)" if e2e else "",
                 (f"{ce_c.get('speedup', 0):.2f}x ({100 * ce_c.get('fraction_of_ideal', 0):.0f}%)" if ce_c else ""),
                 f"{lib.get('library_concurrent_over_ours', 0):.3f}" if "library_concurrent_over_ours" in lib else "",
                 f"{roof.get('frac', 0):.3f} {roof.get('bound', '')}" if roof else "",
                 f"{pr.get('frac', 0):.3f} {pr.get('bound', '')}" if pr else "",
                 f"{r.get('value', 0):.3f}x" if r.get("value") is not None else ""]
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
