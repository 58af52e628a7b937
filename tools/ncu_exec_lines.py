"""Executed warp-instructions per CUDA source line of one kernel (ncu source
page 'Instructions Executed' column, mapped through the .so's line info):
python tools/ncu_exec_lines.py <rep> <so> <mangled kernel> [top] [kernel regex]"""
import collections
import csv
import io
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from ncu_lines import line_map  # noqa: E402


def main():
    rep, so, func = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
    if len(sys.argv) > 5:
        cmd += ["-k", f"regex:{sys.argv[5]}"]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ai, xi = h.index("Address"), h.index("Instructions Executed")
    data = [r for r in rows[hdr + 1:] if len(r) > xi and r[ai].startswith("0x")]
    base = int(data[0][ai], 16)
    lm = line_map(so, func)
    agg = collections.Counter()
    for r in data:
        agg[lm.get(int(r[ai], 16) - base, ("?", 0))] += int(r[xi] or 0)
    tot = sum(agg.values()) or 1
    print(f"total {tot} warp-instructions")
    for (f, l), n in agg.most_common(top):
        print(f"{100 * n / tot:6.2f}%  {n:10d}  {f}:{l}")


if __name__ == "__main__":
    main()
