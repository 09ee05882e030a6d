"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':42s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:42s} {v[0]:8d} {v[1]:10.3f} {v[1] / v[0]:9.4f} {v[1] / tot * 100:5.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
