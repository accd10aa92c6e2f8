#!/usr/bin/env python3
"""SASS op counts per kernel of the built CUDA library (cuobjdump -sass):
the evidence that the kernels use tcgen05 (UTCHMMA / UTCBAR / LDTM), TMA
(UTMALDG / UTMASTG / UBLKCP), system-scope flags and bounded waits.

usage: python tools/sass_summary.py [LIB.so] > profiles/<round>_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = re.compile(r"^(UTC|UTMA|UBLKCP|LDTM|STTM|SYNCS|LDG|STG|LD\.|ST\.|ATOM|RED|MEMBAR|FENCE|NANOSLEEP|CCTL|"
                  r"ERRBAR|CGAERRBAR|REDUX|HMMA|FFMA|FADD|F2FP)")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "paper_2412_14335_b200", "lib", "libc3cuda.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels, cur = collections.OrderedDict(), None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            kernels[cur]["__total__"] += 1
            op = m.group(1)
            if KEEP.match(op):
                kernels[cur][op] += 1
    print(f"# SASS op counts (cuobjdump -sass {os.path.relpath(lib, REPO)}); tools/sass_summary.py")
    print("# UTCHMMA(.2CTA) = tcgen05.mma (cta_group::2), UTCBAR = tcgen05.commit, LDTM = tcgen05.ld, UTMALDG / UTMASTG = TMA")
    print("# tensor load / store, UBLKCP = bulk copy; ST/LD .STRONG.SYS = st.release.sys / ld.acquire.sys flags, NANOSLEEP = bounded waits")
    for k, c in kernels.items():
        tot = c.pop("__total__", 0)
        print(f"== {k}\n   total SASS instructions: {tot}\n   " + ", ".join(f"{o}:{n}" for o, n in sorted(c.items())))


if __name__ == "__main__":
    main()
