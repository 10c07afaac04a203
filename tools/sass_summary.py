"""Opcode census of the built library's SASS, per kernel family: the
instructions that prove the Blackwell paths (UTCIMMA / UTCQMMA tcgen05.mma,
UTCCP tcgen05.cp, UTMALDG / UTMASTG TMA tensor copies, UBLKCP bulk copies,
LDTM / STTM tcgen05.ld / st, SYNCS mbarrier ops) and the CUDA-core work of
K1 (FFMA2 / FADD2 packed fp32x2, FMNMX3, PRMT, REDUX).
    python tools/sass_summary.py [lib.so] > profiles/<round>_sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2512_03673_b200/libconvrot_b200.so"
KEYS = ["UTCIMMA", "UTCQMMA", "UTCHMMA", "UTCCP", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP",
        "LDTM", "STTM", "UTCBAR", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FMNMX3", "PRMT",
        "IDP", "REDUX", "CREDUX", "HMMA", "IMMA", "LDS", "STS", "LDG", "STG", "LDL", "STL"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
fam = collections.defaultdict(collections.Counter)
kern = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        kern = ("k1_team" if "k1_team" in name else "k1_rolled" if "k1_rolled" in name else
                "k1_fast" if "k1_fast" in name else "k1_exact" if "k1_exact" in name else
                "k1_mma" if "k1_mma" in name else "k3_v3" if "k3_v3" in name else
                "k3_v4" if "k3_v4" in name else "k3_gemv" if "k3_gemv" in name else
                "k3_v2" if "k3_v2" in name else "k3_ss (v1)" if "k3_ss" in name else
                "other")
        fam[kern]["#functions"] += 1
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        op = m.group(1)
        for k in KEYS:
            if op == k or (op.startswith(k) and k in ("SYNCS", "IDP", "UTCBAR")):
                fam[kern][k] += 1
print(f"# static SASS opcode counts per kernel family in {LIB} (cuobjdump -sass)")
for k in sorted(fam):
    c = fam[k]
    items = " ".join(f"{op}={c[op]}" for op in ["#functions"] + KEYS if c[op])
    print(f"{k:12s} {items}")
