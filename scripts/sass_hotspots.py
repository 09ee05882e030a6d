"""Top SASS instructions by warp-stall samples and by executed instructions
from `ncu -i X.ncu-rep --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[si] or 0), float(r[ii] or 0), r[0], r[1].strip()))
        except (ValueError, IndexError):
            pass
    ts = sum(d[0] for d in data) or 1
    ti = sum(d[1] for d in data) or 1
    print(f"samples {ts:.0f}  warp-instructions {ti:.3e}")
    print("-- by stall samples")
    for d in sorted(data, key=lambda x: -x[0])[:top]:
        print(f"{d[0] / ts * 100:5.1f}% st {d[1] / ti * 100:5.1f}% in  {d[2][-5:]} {d[3][:80]}")
    print("-- by instructions executed")
    for d in sorted(data, key=lambda x: -x[1])[:top]:
        print(f"{d[0] / ts * 100:5.1f}% st {d[1] / ti * 100:5.1f}% in  {d[2][-5:]} {d[3][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
