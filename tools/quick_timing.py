"""Quick device timing of K1 and K3 at the FLUX shapes (dev aid, not the bench).

Each timed launch is bracketed by CUDA events on the launching stream with a
256 MiB L2-flushing write outside the bracket.
    python tools/quick_timing.py [k1|k3|all]
"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec  # noqa: E402

FLUSH = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        FLUSH.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)  # us


what = sys.argv[1] if len(sys.argv) > 1 else "all"
for (M, K, N) in [(4096, 3072, 3072), (4608, 3072, 12288), (4608, 12288, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    ld = (K // 2 + 15) // 16 * 16
    codes = torch.empty(M, ld, dtype=torch.uint8, device="cuda")
    s32 = torch.empty(M, dtype=torch.float32, device="cuda")
    if what in ("k1", "all"):
        for n0 in (4, 16, 64, 256):
            spec = RotationSpec(RotationKind.regular, n0)
            t = timeit(lambda: crt.rotate_quantize_into(x, spec, codes, s32))
            gbs = (M * K * 2.5 + 4 * M) / t / 1e3
            print(f"K1 M={M} K={K} N0={n0}: {t:.2f} us  {gbs:.0f} GB/s", flush=True)
    if what in ("k3", "all"):
        w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        spec = RotationSpec(RotationKind.regular, 16)
        layer = crt.prepare_layer(w, None, spec)
        codes, sa = crt.rotate_quantize(x, spec)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = timeit(lambda: crt.quant_gemm(codes, sa, layer, y=y))
        print(f"K3 M={M} K={K} N={N}: {t:.2f} us  {2*M*N*K/t/1e6:.1f} TOPS", flush=True)
