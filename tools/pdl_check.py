"""Does PDL shorten the fc1+fc2 step?  100 back-to-back steps with events
only at the ends (an event between kernels would serialise them); run with
CRT_PDL=0 / 1.  Dev aid."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec, _abi  # noqa: E402

M, D, F = 4608, 3072, 12288
spec = RotationSpec(RotationKind.regular, 16)
x = torch.randn(M, D, device="cuda").to(torch.bfloat16)
fc1 = crt.prepare_layer(torch.randn(F, D, device="cuda").to(torch.bfloat16), None, spec)
fc2 = crt.prepare_layer(torch.randn(D, F, device="cuda").to(torch.bfloat16), None, spec)
ws = crt.Workspace(M, F)
y1 = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
y2 = torch.empty(M, D, device="cuda", dtype=torch.bfloat16)


def step():
    crt.forward(x, fc1, y=y1, workspace=ws, check_finite=False)
    crt.forward(y1, fc2, y=y2, workspace=ws, check_finite=False)


for _ in range(5):
    step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for rep in range(3):
    s.record()
    for _ in range(100):
        step()
    e.record()
    e.synchronize()
    res.append(s.elapsed_time(e) / 100 * 1e3)
print("us/step (warm L2, back-to-back):", [round(r, 1) for r in res], flush=True)
