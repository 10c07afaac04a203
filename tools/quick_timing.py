"""Quick device timing of K1 and K3 at the FLUX shapes (dev aid, not the bench)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec

def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us

for (M, K, N) in [(4096, 3072, 3072), (4608, 3072, 12288), (4608, 12288, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    for n0 in (4, 16, 64, 256):
        spec = RotationSpec(RotationKind.regular, n0)
        t = timeit(lambda: crt.rotate_quantize(x, spec, QuantSpec(4), check_finite=False))
        gbs = (M * K * 2.5 + 4 * M) / t / 1e3
        print(f"K1 M={M} K={K} N0={n0}: {t:.2f} us  {gbs:.0f} GB/s", flush=True)
    spec = RotationSpec(RotationKind.regular, 16)
    layer = crt.prepare_layer(w, None, spec)
    codes, sa = crt.rotate_quantize(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: crt.quant_gemm(codes, sa, layer, y=y))
    print(f"K3 M={M} K={K} N={N}: {t:.2f} us  {2*M*N*K/t/1e6:.1f} TOPS", flush=True)
