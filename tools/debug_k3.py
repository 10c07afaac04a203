"""Locate K3 accumulator mismatches vs a torch int reference (dev aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec

M, K, N = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 3072, 3072)
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
spec = RotationSpec(RotationKind.regular, 16)
layer = crt.prepare_layer(w, None, spec)
codes, sa = crt.rotate_quantize(x, spec)
wc, _ = layer.export(scales64=False)[:2]

def unpack(c, k):
    c = c[:, : k // 2].to(torch.int32)
    lo = c & 0xF
    hi = (c >> 4) & 0xF
    lo = torch.where(lo >= 8, lo - 16, lo)
    hi = torch.where(hi >= 8, hi - 16, hi)
    return torch.stack([lo, hi], dim=2).reshape(c.shape[0], k)

A = unpack(codes, K).double()
B = unpack(wc, K).double()
ref = (A @ B.T).round().to(torch.int64)
for it in range(3):
    acc = crt.int_gemm(codes, layer).to(torch.int64)
    torch.cuda.synchronize()
    bad = (acc != ref)
    nb = int(bad.sum())
    print(f"run {it}: mismatches {nb} of {M*N}")
    if nb:
        idx = bad.nonzero()
        rows = idx[:, 0]; cols = idx[:, 1]
        print("  rows: min", int(rows.min()), "max", int(rows.max()), "unique", len(torch.unique(rows)))
        print("  cols: min", int(cols.min()), "max", int(cols.max()), "unique", len(torch.unique(cols)))
        mt = (rows // 256); nt = (cols // 192)
        tiles = torch.unique(mt * 1000 + nt)
        print("  tiles (mt*1000+nt):", tiles[:20].tolist(), "count", len(tiles))
        r0, c0 = int(rows[0]), int(cols[0])
        print("  sample", r0, c0, "got", int(acc[r0, c0]), "want", int(ref[r0, c0]))
        d = (acc - ref)[bad].double()
        print("  diff stats: min", float(d.min()), "max", float(d.max()))

# --- explain the error of wrong tiles in terms of 128-code K-block contributions
acc = crt.int_gemm(codes, layer).to(torch.int64)
torch.cuda.synchronize()
bad = (acc != ref)
if bad.any():
    KB = (K + 127) // 128
    contrib = torch.stack([(A[:, kb*128:(kb+1)*128] @ B[:, kb*128:(kb+1)*128].T).round().to(torch.int64)
                           for kb in range(KB)])  # KB x M x N
    idx = bad.nonzero()[:2000]
    import collections
    expl = collections.Counter()
    for r, c in idx.tolist()[:400]:
        d = int(acc[r, c] - ref[r, c])
        cs = contrib[:, r, c].tolist()
        hit = None
        for j in range(KB):
            if d == -cs[j]: hit = f"missing kb{j}"; break
            if d == cs[j]: hit = f"double kb{j}"; break
        if hit is None:
            for i in range(KB):
                for j in range(KB):
                    if i != j and d == cs[i] - cs[j]:
                        hit = f"kb{j}->kb{i}"; break
                if hit: break
        expl[hit or "other"] += 1
    print("error explanations:", expl.most_common(12))

# --- stale-B hypothesis: some K blocks used B rows of the pair's previous tile
if bad.any() and M <= 256:
    npairs = 74
    expl = collections.Counter()
    for r, c in idx.tolist()[:300]:
        nt = c // 192
        if nt < npairs:
            expl["first tile"] += 1
            continue
        cp = c - npairs * 192
        d = int(acc[r, c] - ref[r, c])
        cs = contrib[:, r, c].tolist()
        cq = contrib[:, r, cp].tolist()
        hit = None
        for j in range(KB):
            if d == cq[j] - cs[j]:
                hit = f"stale kb{j}"
                break
        if hit is None:
            # prefix of stale blocks?
            for L in range(1, KB + 1):
                if d == sum(cq[:L]) - sum(cs[:L]):
                    hit = f"stale prefix {L}"
                    break
        if hit is None:
            for L in range(1, KB + 1):
                if d == sum(cq[KB - L:]) - sum(cs[KB - L:]):
                    hit = f"stale suffix {L}"
                    break
        expl[hit or "other"] += 1
    print("stale-B explanations:", expl.most_common(12))

# --- mismatch structure inside tiles: (row half = CTA rank, column half = B half)
if bad.any():
    rr = bad.nonzero()
    rows = rr[:, 0] % 256
    cols = rr[:, 1] % 192
    for rh in range(2):
        for ch in range(2):
            sel = ((rows // 128) == rh) & ((cols // 96) == ch)
            print(f"rank{rh} rows, B-half {ch} cols: {int(sel.sum())}")
    print("row lane hist (row%128 //32):", torch.bincount((rows % 128) // 32, minlength=4).tolist())
    print("col chunk hist (col//32):", torch.bincount(cols // 32, minlength=6).tolist())
