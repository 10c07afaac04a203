import sys; sys.path.insert(0, ".")
import numpy as np, torch
import oracle as O
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
g = np.load("tests/golden/golden.npz")
xb = g["edges/x_bf16"]
x = torch.from_numpy(xb.astype(np.uint16).view(np.int16)).cuda().view(torch.bfloat16)
codes, s32, s64 = crt.rotate_quantize(x, RotationSpec(RotationKind.regular, 16), QuantSpec(4), scales64=True)
got = codes[:, :32].cpu().numpy(); want = g["edges/act_packed"]
print("scales got ", s64.cpu().numpy()); print("scales want", g["edges/act_scales"])
for r in range(got.shape[0]):
    d = np.nonzero(got[r] != want[r])[0]
    if d.size:
        print("row", r, "cols", d[:10], "got", got[r][d[:10]], "want", want[r][d[:10]])
xd = O.from_bf16_bits(xb)
rot = O.group_rotate(xd, O.ROT_REGULAR, 16)
print("rot row2", rot[2][:16])
print("rot/s row2", (rot[2] / g["edges/act_scales"][2])[:16])
