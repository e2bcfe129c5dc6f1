#!/usr/bin/env python
"""Per-kernel counts of the SASS mnemonics that prove the Blackwell-native
paths (B200_PROFILING.md): UTC*MMA (tcgen05.mma), LDTM/STTM (tcgen05.ld/st),
UTMALDG/UTMASTG/UBLKCP (TMA), plus FFMA/DFMA/HMMA for context. Reads the
in-tree libmpir_gpu.so with cuobjdump and writes a table.

usage: python tools/sass_evidence.py [out.txt]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2311_14616_b200", "libmpir_gpu.so")
PAT = ["UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS",
       "UCGABAR", "FFMA", "DFMA", "HMMA", "REDUX", "LDGSTS"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                         check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True,
                                 text=True).stdout.strip()
            cur = cur.replace("(anonymous namespace)::", "")
            cur = re.sub(r"\(.*", "", cur)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for p in PAT:
            if re.search(r"\b" + p + r"[\w.]*", line):
                counts[cur][p] += 1
    rows = []
    for k, c in counts.items():
        if any(c[p] for p in PAT[:7]):
            rows.append((k, c))
    txt = ["# SASS evidence from paper_2311_14616_b200/libmpir_gpu.so (cuobjdump -sass)",
           "# kernels with tcgen05 / TMEM / TMA instructions; counts per kernel", ""]
    hdr = f"{'kernel':90s} " + " ".join(f"{p:>8s}" for p in PAT)
    txt.append(hdr)
    for k, c in rows:
        txt.append(f"{k[:90]:90s} " + " ".join(f"{c[p]:8d}" for p in PAT))
    s = "\n".join(txt) + "\n"
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s)
    else:
        print(s)


if __name__ == "__main__":
    main()
