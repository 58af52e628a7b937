"""Summarise an `ncu --set full` report into the profiles/ text format.

    python tools/ncu_summary.py <report.ncu-rep> <title> <kernel>[,<kernel>...] [top]

For each kernel (demangled short name, e.g. k_events, plan_loop_kernel) it
prints the speed-of-light / launch / occupancy metrics from the details page,
the raw DRAM and RED-sector counters, and the top warp-stall source lines
(via tools/ncu_lines.py against paper_2506_06472_b200/_lib/libtio.so).
"""

import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.environ.get("TIO_LIB_PATH") or os.path.join(ROOT, "paper_2506_06472_b200", "_lib", "libtio.so")
DETAILS = ["Memory Throughput", "DRAM Throughput", "Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput",
           "Compute (SM) Throughput", "Executed Ipc Active", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
           "Executed Instructions", "Block Size", "Grid Size", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
       "smsp__inst_executed.sum"]


def _rows(rep, page, kernel):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv", "-k", f"regex:^{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def _mangled(kernel):
    out = subprocess.run(["nm", "-C", SO], capture_output=True, text=True).stdout
    raw = subprocess.run(["nm", SO], capture_output=True, text=True).stdout.splitlines()
    for dem, man in zip(out.splitlines(), raw):
        if f"tio::{kernel}(" in dem:
            return man.split()[-1]
    return None


def summarise(rep, title, kernel, top):
    print(f"=== {kernel} ({title})")
    rows = _rows(rep, "details", kernel)
    if len(rows) > 1:
        h = rows[0]
        ni, ui, vi, idi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), h.index("ID")
        first = rows[1][idi]
        seen = {}
        for r in rows[1:]:
            if len(r) > vi and r[idi] == first and r[ni] in DETAILS and r[ni] not in seen:
                seen[r[ni]] = (r[ui], r[vi])
        for name in DETAILS:
            if name in seen:
                print(f"  {name:<40} {seen[name][0]:<12} {seen[name][1]}")
    rows = _rows(rep, "raw", kernel)
    if len(rows) > 2:
        h, units, vals = rows[0], rows[1], rows[2]
        for name in RAW:
            if name in h:
                i = h.index(name)
                print(f"  {name:<40} {units[i]:<12} {vals[i]}")
    man = _mangled(kernel)
    if man:
        print("  top warp-stall source lines:")
        samples = ncu_lines.sass_samples(rep, f"^{kernel}")
        lm = ncu_lines.line_map(SO, man)
        agg = {}
        for off, n in samples:
            k = lm.get(off, ("?", 0))
            agg[k] = agg.get(k, 0) + n
        tot = sum(agg.values()) or 1
        for (f, ln), n in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
            print(f"   {100 * n / tot:5.2f}%  {n:9d}  {f}:{ln}")


def main():
    rep, title, kernels = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    for k in kernels.split(","):
        summarise(rep, title, k, top)


if __name__ == "__main__":
    main()
