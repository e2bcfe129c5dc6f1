"""Summarise an ncu --page source --csv --print-source sass dump: hottest SASS lines."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((float(r[iss] or 0), r[iex], r[ia], r[isrc]))
        except (ValueError, IndexError):
            continue
    tot = sum(d[0] for d in data) or 1
    print("total samples", tot, "instructions", len(data))
    for s, ex, a, src in sorted(data, key=lambda d: -d[0])[:top]:
        print(f"{s / tot * 100:5.1f}% ex={ex:>9} {a} {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
