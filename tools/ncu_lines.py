"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    fname = None
    agg = []
    hdr = None
    for r in csv.reader(open(path)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0]:
            continue
        try:
            ex = float(r[hdr.index("Instructions Executed")] or 0)
            smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        agg.append((ex, smp, f"{fname}:{r[0]}", r[1].strip()[:90]))
    tex = sum(a[0] for a in agg) or 1
    ts = sum(a[1] for a in agg) or 1
    print(f"total inst {tex:.0f} samples {ts:.0f}")
    for ex, smp, loc, src in sorted(agg, key=lambda a: -a[1])[:top]:
        print(f"{smp / ts * 100:5.1f}%smp {ex / tex * 100:5.1f}%inst {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
