"""Aggregate warp-stall samples per CUDA source line from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    tot = defaultdict(float)
    reasons = defaultdict(lambda: defaultdict(float))
    src = {}
    fname = None
    hdr = None
    cur = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:  # a cuda source line row
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()
            continue
        if cur is None:
            continue
        try:
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        tot[cur] += s
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    reasons[cur][h[6:]] += float(r[i] or 0)
                except ValueError:
                    pass
    T = sum(tot.values()) or 1
    print(f"total samples {T:.0f}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        rs = sorted(reasons[k].items(), key=lambda x: -x[1])[:3]
        rs = " ".join(f"{a}:{b / v * 100:.0f}%" for a, b in rs if v)
        print(f"{v / T * 100:5.1f}% {k[0]}:{k[1]:<4} {src.get(k, '')[:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
