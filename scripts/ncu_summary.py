"""Summarise an `ncu --set full` report (one kernel) into the text format
kept under profiles/ncu/: key SOL / compute / memory / warp-state / launch /
occupancy lines, plus DRAM bytes, duration and FP64 tensor-pipe activity."""
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Warp State Statistics", "Launch Statistics", "Occupancy")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")


def ncu(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path):
    rows = ncu(path, "details")
    h = rows[0]
    ki, gi, bi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Block Size")
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    print(f"kernel: {rows[1][ki]} grid {rows[1][gi]} block {rows[1][bi]}")
    for r in rows[1:]:
        if r[si] in SECTIONS and r[mi]:
            print(f"{r[si]:32s} {r[mi]:45s} {r[vi]:>20s} {r[ui]}")
    raw = ncu(path, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    for k in RAW:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k} {vals[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
