"""K3 v3 time at the FLUX shapes (mean of 40 launches, L2 flushed). Dev aid."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

spec = RotationSpec(RotationKind.regular, 16)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for M, K, N in [(4608, 3072, 12288), (4608, 12288, 3072), (4608, 3072, 3072), (4096, 3072, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
    c, sa, su = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(43):
        flush.zero_()
        s.record()
        crt.quant_gemm_i8(c, sa, su, layer, y=y)
        e.record()
        e.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    t = sum(ts) / len(ts)
    print(f"M={M} K={K} N={N}: {t:.1f} us {2 * M * N * K / t / 1e6:.0f} TOPS", flush=True)
