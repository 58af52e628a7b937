"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches and total ns, with the share of libtio device time.

    python tools/launch_summary.py launches.csv [header text]
"""
import collections
import csv
import sys


def main(path, title=""):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((r["Kernel Name"], float(r["Metric Value"]), r["Metric Unit"]))
    agg = collections.OrderedDict()
    for name, v, unit in rows:
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        short = name.split("(")[0].replace("void ", "")
        n, t = agg.get(short, (0, 0.0))
        agg[short] = (n + 1, t + ns)
    tot = sum(t for k, (n, t) in agg.items() if k.startswith("tio::"))
    if title:
        print(title)
    print("cold-cache, serialised per-launch times; share of libtio device time")
    for k, (n, t) in agg.items():
        share = f"{100 * t / tot:7.3f}%" if k.startswith("tio::") and tot else "      -"
        print(f"{k[:60]:60s} launches {n:5d} total {t / 1e3:14.1f} us  share {share}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
