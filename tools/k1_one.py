"""Median K1 time (bits 5, N0=16, bf16) for one shape: python tools/k1_one.py M K"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
spec = RotationSpec(RotationKind.regular, 16)
ref = torch.load("/tmp/k1ref_%d_%d.pt" % (M, K)) if len(sys.argv) > 3 else None
c8, s8, sums = crt.rotate_quantize_i8(x, spec)
if ref is None:
    torch.save((c8.cpu(), s8.cpu(), sums.cpu()), "/tmp/k1ref_%d_%d.pt" % (M, K))
    ok = True
else:
    ok = all(torch.equal(a.cpu(), b) for a, b in zip((c8, s8, sums), ref))
flush = torch.empty(64 * 1024 * 1024, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(63):
    flush.zero_()
    s.record()
    crt.rotate_quantize_i8(x, spec)
    e.record()
    e.synchronize()
    if i >= 3:
        ts.append(s.elapsed_time(e) * 1e3)
# single-launch CUDA-event times are quantised (2.048 us steps on this part):
# report the mean of 60 samples, whose phase varies
print(f"M={M} K={K} ok={ok} {sum(ts) / len(ts):.2f} us (mean of {len(ts)})", flush=True)
