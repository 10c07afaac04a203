"""W8A8 vs W4A4 GEMM time at the FLUX MLP shapes (dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec  # noqa: E402

spec = RotationSpec(RotationKind.regular, 16)
for M, K, N in [(4608, 3072, 12288), (4608, 12288, 3072), (4096, 3072, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    res = []
    for bits in (8, 4):
        q = QuantSpec(bits)
        layer = crt.prepare_layer(w, None, spec, q)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        if bits == 8:
            c, sa = crt.rotate_quantize(x, spec, q)
            fn = lambda: crt.quant_gemm(c, sa, layer, q, y=y)  # noqa: E731
        else:
            c, sa, su = crt.rotate_quantize_i8(x, spec)
            fn = lambda: crt.quant_gemm_i8(c, sa, su, layer, y=y)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        e.record()
        e.synchronize()
        t = s.elapsed_time(e) / 10 * 1e3
        res.append(f"W{bits}A{bits} {t:.1f} us {2 * M * N * K / t / 1e6:.0f} TOPS")
    print(f"M={M} K={K} N={N}: " + " | ".join(res), flush=True)
