"""Run one kernel configuration a few times (for ncu captures).
    python tools/prof_one.py k1 M K N0      |  python tools/prof_one.py k3 M K N
    python tools/prof_one.py k1i8 M K N0    |  python tools/prof_one.py k3v3 M K N
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec  # noqa: E402

what, M, K, X = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
if what == "k1":
    spec = RotationSpec(RotationKind.regular, X)
    codes = torch.empty(M, (K // 2 + 15) // 16 * 16, dtype=torch.uint8, device="cuda")
    s32 = torch.empty(M, dtype=torch.float32, device="cuda")
    for _ in range(4):
        crt.rotate_quantize_into(x, spec, codes, s32)
elif what == "k1i8":
    spec = RotationSpec(RotationKind.regular, X)
    for _ in range(4):
        crt.rotate_quantize_i8(x, spec)
elif what == "k3v3":
    spec = RotationSpec(RotationKind.regular, 16)
    w = torch.randn(X, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(w, None, spec)
    c8, sa, sums = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, X, device="cuda", dtype=torch.bfloat16)
    for _ in range(4):
        crt.quant_gemm_i8(c8, sa, sums, layer, y=y)
else:
    spec = RotationSpec(RotationKind.regular, 16)
    w = torch.randn(X, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(w, None, spec)
    codes, sa = crt.rotate_quantize(x, spec)
    y = torch.empty(M, X, device="cuda", dtype=torch.bfloat16)
    for _ in range(4):
        crt.quant_gemm(codes, sa, layer, y=y)
torch.cuda.synchronize()
print("ok")
