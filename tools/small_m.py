"""Small-M (AdaLN) components: K1, the GEMM (GEMV), forward (dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

spec = RotationSpec(RotationKind.regular, 16)


def t(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n * 1e3


for M, K, N in [(1, 3072, 18432), (1, 3072, 9216), (8, 3072, 18432), (512, 3072, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
    c, sa, su = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = crt.Workspace(M, K)
    tk1 = t(lambda: crt.rotate_quantize_i8(x, spec))
    tg = t(lambda: crt.quant_gemm_i8(c, sa, su, layer, y=y))
    tf = t(lambda: crt.forward(x, layer, y=y, workspace=ws, check_finite=False))
    wbytes = N * K / 2
    print(f"M={M} K={K} N={N}: K1 {tk1:.1f} us, GEMM {tg:.1f} us ({wbytes / tg / 1e3:.0f} GB/s weights), "
          f"forward {tf:.1f} us  (back-to-back launches)", flush=True)
