"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"(\w+)(<[^(]*>)?\(", name)
    base = m.group(1) if m else name[:40]
    tm = re.search(r"<([^>]*)>", name)
    return base + ("<" + tm.group(1) + ">" if tm else "")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[short(r[ik])].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:60]:60s} n={len(v):4d} total={sum(v) / 1e3:9.1f}us "
              f"({sum(v) / tot * 100:5.1f}%) mean={sum(v) / len(v) / 1e3:8.2f}us")
    print(f"total {tot / 1e3:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
