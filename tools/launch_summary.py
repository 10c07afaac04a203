"""Digest an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel launch counts, mean device time and share of the total.
    python tools/launch_summary.py gpurun_out/<tag>/launches.csv > profiles/<round>_launches_summary.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                              "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:64]
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        agg.setdefault(name, []).append(us)
    tot = sum(sum(v) for v in agg.values())
    print(f"# {path}: gpu__time_duration.sum per launch (ncu --clock-control none)")
    print("# cold-cache, serialised launches: compare SHARES of the step, not absolutes")
    print(f"{'kernel':66s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
    for k, v in agg.items():
        print(f"{k:66s} {len(v):8d} {sum(v) / len(v):9.2f} {sum(v) / tot * 100:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
