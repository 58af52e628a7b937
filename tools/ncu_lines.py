"""Attribute ncu warp-stall samples of a kernel to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <libtio.so> <mangled kernel> [top] [kernel regex]

ncu's SASS source page gives per-instruction stall samples with absolute
addresses; nvdisasm -g on the cubin extracted from libtio.so (compiled with
-lineinfo) gives offset -> file:line.  Offsets are aligned by instruction
order (the first listed instruction is offset 0).
"""

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[hdr + 1:] if len(r) > si and r[ai].startswith("0x")]
    base = int(data[0][ai], 16)
    return [(int(r[ai], 16) - base, int(r[si] or 0)) for r in data]


def line_map(so, func):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    cur = None
    out = {}
    for cub in os.listdir(d):
        text = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
        if f".text.{func}:" not in text:
            continue
        body = text.split(f".text.{func}:", 1)[1].split("//----", 1)[0]
        for ln in body.splitlines():
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
            if m and cur:
                out[int(m.group(1), 16)] = cur
        break
    return out


def main():
    rep, so, func = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    samples = sass_samples(rep, sys.argv[5] if len(sys.argv) > 5 else None)
    lm = line_map(so, func)
    agg = collections.Counter()
    for off, n in samples:
        agg[lm.get(off, ("?", 0))] += n
    tot = sum(agg.values()) or 1
    for (f, l), n in agg.most_common(top):
        print(f"{100 * n / tot:6.2f}%  {n:9d}  {f}:{l}")


if __name__ == "__main__":
    main()
