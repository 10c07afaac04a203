"""Needs a trace build: CRT_NVCC_EXTRA="-DCRT_K1_TRACE -DCRT_K3_TRACE" python -m
paper_2512_03673_b200.build.
K3 v3 pipeline trace (crt_debug_k3_trace, 9 x 4096 words): clock64 stamps of pair 0's
leader CTA per stage (producer issue after the empty wait, MMA issue once
the stage landed; two MMA threads take alternate stages) and per tile (MMA tile start,
epilogue sees acc_full, epilogue done).  Prints the steady-state cycles per
stage of each role and where the MMA issuer waited.
python tools/k3_trace.py M K N"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec, _abi  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
T = 4096
torch.manual_seed(0)
spec = RotationSpec(RotationKind.regular, 16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
c, sa, su = crt.rotate_quantize_i8(x, spec)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    crt.quant_gemm_i8(c, sa, su, layer, y=y)
lib = _abi.load()
tr = torch.zeros(11 * T, dtype=torch.int64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
flush.zero_()
lib.crt_debug_k3_trace(ctypes.c_void_p(tr.data_ptr()))
crt.quant_gemm_i8(c, sa, su, layer, y=y)
torch.cuda.synchronize()
lib.crt_debug_k3_trace(None)
t = tr.view(11, T).cpu().numpy().astype(np.float64)
KB = (K + 127) // 128
ns = int((t[3] > 0).sum())
nt = int((t[4] > 0).sum())
t0 = t[0, 0]
P, DF, DI, MI = (t[r, :ns] - t0 for r in range(4))
print(f"M={M} K={K} N={N}: {ns} stages, {nt} tiles on pair 0, KB={KB}; "
      f"ideal MMA time per stage = 4 x 96 = 384 cycles")
print(f"  first MMA issue at {MI[0]:.0f} cycles after the first producer issue; "
      f"last MMA issue at {MI[-1]:.0f}")
lo, hi = KB, ns  # steady state: skip the first tile
rows = [("producer issue", P), ("MMA issue", MI)]
v4 = (t[9, :ns] > 0).all()
if (t[1, :ns] > 0).all() and not v4:
    rows[1:1] = [("expander sees full", DF), ("expander done", DI)]
for name, v in rows:
    d = np.diff(v[lo:hi])
    print(f"  {name:17s}: median {np.median(d):6.0f}  mean {d.mean():6.0f}  p90 {np.percentile(d, 90):6.0f} cycles/stage")
if (t[1, :ns] > 0).all() and not v4:
    print(f"  producer issue -> expander sees stage: median {np.median((DF - P)[lo:hi]):.0f}; "
          f"expansion time median {np.median((DI - DF)[lo:hi]):.0f}; expander done -> MMA issue "
          f"median {np.median((MI - DI)[lo:hi]):.0f}")
if v4:  # globaltimer ns, both CTAs of pair 0
    LF, LD, PF, PD = t[1, :ns], t[2, :ns], t[9, :ns], t[10, :ns]
    print(f"  v4 expanders (ns): leader stage period {np.median(np.diff(LF[lo:hi])):.0f}, expansion "
          f"{np.median((LD - LF)[lo:hi]):.0f}; peer sees each stage {np.median((PF - LF)[lo:hi]):.0f} "
          f"after the leader, finishes {np.median((PD - LD)[lo:hi]):.0f} after, expansion "
          f"{np.median((PD - PF)[lo:hi]):.0f}")
ring = MI[lo:hi] - P[lo:hi]
print(f"  producer issue -> MMA issue (stage age at use): median {np.median(ring):.0f}")
W0, W1 = t[7, :ns] - t0, t[8, :ns] - t0
print(f"  MMA issuer per stage: stage/slot wait median {np.median((MI - W0)[lo:hi]):.0f} mean {(MI - W0)[lo:hi].mean():.0f}; "
      f"issue of 4 cps + 4 MMAs + 2 commits median {np.median((W1 - MI)[lo:hi]):.0f} mean {(W1 - MI)[lo:hi].mean():.0f}")
E = t[4:7, :nt] - t0
for i in range(min(nt, 4)):
    print(f"  tile {i}: MMA start {E[0, i]:9.0f}  epi sees acc {E[1, i]:9.0f}  epi done {E[2, i]:9.0f}"
          f"  (epilogue {E[2, i] - E[1, i]:.0f})")
