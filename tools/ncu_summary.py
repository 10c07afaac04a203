"""Summarise an ncu report: key metrics per kernel launch (reads `ncu -i --page details --csv`)."""
import csv, io, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Block Size", "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Waves Per SM", "Theoretical Occupancy", "Achieved Occupancy"]

def main(path, raw_metrics=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    by = {}
    for r in rows:
        k = (r["ID"], r["Kernel Name"][:60])
        if r["Metric Name"] in KEYS:
            by.setdefault(k, {})[r["Metric Name"]] = f'{r["Metric Value"]} {r["Metric Unit"]}'
    for k, d in by.items():
        print(f"== launch {k[0]}: {k[1]}")
        for m in KEYS:
            if m in d:
                print(f"   {m:40s} {d[m]}")
    if raw_metrics:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(out)))
        hdr, units = rr[0], rr[1]
        for row in rr[2:]:
            print("== raw launch", row[hdr.index("ID")])
            for i, h in enumerate(hdr):
                if any(h.startswith(p) for p in raw_metrics):
                    print(f"   {h:60s} {row[i]} {units[i]}")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
