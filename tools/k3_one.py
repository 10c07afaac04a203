"""Run K3 (W4A4 v3, bf16 out) a few times at one shape, for ncu capture:
python tools/k3_one.py M K N [launches]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 4
torch.manual_seed(0)
spec = RotationSpec(RotationKind.regular, 16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
c, sa, su = crt.rotate_quantize_i8(x, spec)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(n):
    crt.quant_gemm_i8(c, sa, su, layer, y=y)
torch.cuda.synchronize()
print(f"M={M} K={K} N={N}: {n} launches")
