#!/usr/bin/env python
"""Per-kernel SASS mnemonic summary of the shipped library (cuobjdump -sass): the evidence
that K3 moves bytes with the TMA engine (UBLKCP bulk copies, UTMALDG/UTMASTG tensor copies,
SYNCS mbarrier transactions) and K1/K2 with 16-byte vector LDG/STG.  Writes
profiles/sass_summary.json."""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2312_05181_b200", "libreshard_b200.so")
KEEP = re.compile(r"^(UBLKCP|UTMALDG|UTMASTG|UTMAPF|SYNCS|LDG|STG|LDGSTS|ATOMG|RED|ATOM|LDS|STS|SHFL|BAR|WARPSYNC|MEMBAR|FENCE|ELECT)")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m and KEEP.match(m.group(1)):
            kernels[cur][m.group(1)] += 1
    demangled = {}
    for k in kernels:
        d = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        demangled[d.replace("reshard::cuda::(anonymous namespace)::", "").replace("reshard::(anonymous namespace)::", "")] = dict(
            sorted(kernels[k].items()))
    path = os.path.join(ROOT, "profiles", "sass_summary.json")
    with open(path, "w") as f:
        json.dump({"library": "paper_2312_05181_b200/libreshard_b200.so (sm_100a)", "command": "cuobjdump -sass",
                   "kernels": dict(sorted(demangled.items()))}, f, indent=1)
    for k, v in sorted(demangled.items()):
        if "copy" in k:
            print(k[:90], {x: n for x, n in v.items() if x.startswith(("UBLK", "UTMA", "LDG", "STG"))})
    return 0


if __name__ == "__main__":
    sys.exit(main())
