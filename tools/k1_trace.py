"""Needs a trace build: CRT_NVCC_EXTRA="-DCRT_K1_TRACE -DCRT_K3_TRACE" python -m
paper_2512_03673_b200.build.
Timeline of one K1 team-kernel launch from in-kernel %globaltimer stamps
(crt_debug_k1_trace): per CTA, kernel start, PDL wait done, and for each of
its rows the time the row's data was ready, the team barrier passed and the
row finished.  python tools/k1_trace.py M K [N0]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").environ.get("CRT_ROOT", "."))
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402
from paper_2512_03673_b200.api import _lib  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
n0 = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ROWS = 8
WORDS = 2 + 3 * ROWS
spec = RotationSpec(RotationKind.regular, n0)
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    crt.rotate_quantize_i8(x, spec)
tr = torch.zeros(148 * 32 * WORDS, dtype=torch.int64, device="cuda")
lib = _lib()
flush.zero_()
lib.crt_debug_k1_trace(ctypes.c_void_p(tr.data_ptr()))
crt.rotate_quantize_i8(x, spec)
lib.crt_debug_k1_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(-1, WORDS)
t = t[t[:, 0] != 0].astype(np.float64)
t0 = t[:, 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)  # us
q = lambda a: "p10 %6.2f  p50 %6.2f  p90 %6.2f  max %6.2f" % tuple(  # noqa: E731
    np.nanpercentile(a, [10, 50, 90, 100]))
print(f"M={M} K={K} N0={n0}: {len(t)} CTAs, end {np.nanmax(t):.2f} us after the first start")
print("start        ", q(t[:, 0]))
print("pdl wait done", q(t[:, 1]))
# per row i (thread 0): [2+3i] data ready, [3+3i] team barrier passed,
# [4+3i] row done
for i in range(ROWS):
    r = t[:, 2 + 3 * i: 5 + 3 * i]
    if np.all(np.isnan(r[:, 0])):
        break
    print(f"row {i}: ready  ", q(r[:, 0]))
    print(f"       barrier", q(r[:, 1] - r[:, 0]), "(after ready)")
    print(f"       done   ", q(r[:, 2] - r[:, 1]), "(after barrier)")
    print(f"       end    ", q(r[:, 2]))
