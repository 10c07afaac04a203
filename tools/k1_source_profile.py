"""Where K1's warps spend their time: per-region executed instructions and
warp-stall samples from an `ncu --set full --import-source on` capture.
Regions are the kernel's hot loops (found as backward branches executed
more than once per row) and everything else (per-row and per-warp code).
    python tools/k1_source_profile.py gpurun_out/<tag>/k1.ncu-rep ROWS
"""
import csv
import io
import re
import subprocess
import sys

REASONS = ["selected", "not_selected", "wait", "short_sb", "long_sb", "math", "dispatch",
           "barrier", "branch_resolving", "no_inst", "mio", "lg"]


def main(path, rows, launch=0):  # launch: index into the report's kernel blocks
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = [b for b in out.split('"Kernel Name"') if b.strip()]
    recs = list(csv.reader(io.StringIO(blocks[launch])))
    hdr, data = recs[1], recs[2:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ir = {r: hdr.index("stall_" + r) for r in REASONS if "stall_" + r in hdr}
    base = int(data[0][ia], 16)
    ins = [(int(d[ia], 16) - base, d[isrc].strip(), int(d[iex] or 0), int(d[iss] or 0),
            {r: int(d[i] or 0) for r, i in ir.items()}) for d in data]
    loops = []
    for a, t, e, s, _ in ins:
        m = re.search(r"BRA.*?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16) - base
            if tgt < a and e > rows and a - tgt < 0x2000:
                loops.append((tgt, a))
    loops = [l for l in loops if not any(o != l and o[0] <= l[0] and l[1] <= o[1] for o in loops)]
    tot_e = sum(x[2] for x in ins)
    tot_s = sum(x[3] for x in ins)
    print(f"# {path} launch {launch}: {tot_e} warp instructions ({tot_e / rows:.0f} per row), "
          f"{tot_s} stall samples")

    def report(name, sel):
        e = sum(x[2] for x in sel)
        s = sum(x[3] for x in sel)
        rs = {r: sum(x[4].get(r, 0) for x in sel) for r in ir}
        top = " ".join(f"{k}={v}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1]) if v)[:120]
        print(f"{name:28s} inst/row {e / rows:7.1f} ({100 * e / tot_e:4.1f}%)  samples "
              f"{100 * s / max(tot_s, 1):4.1f}%  [{top}]")

    inside = set()
    for lo, hi in loops:
        sel = [x for x in ins if lo <= x[0] <= hi]
        inside.update(x[0] for x in sel)
        report(f"loop {lo:#x}-{hi:#x}", sel)
    report("outside the loops", [x for x in ins if x[0] not in inside])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
