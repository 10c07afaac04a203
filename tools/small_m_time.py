"""Device time of K1, K3 and the forward for small-M units (FLUX AdaLN M=1,
text M=512) and the K=15360 proj_out: 20 launches captured in one CUDA
graph, replayed (no Python / launch overhead).  Dev aid."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

spec = RotationSpec(RotationKind.regular, 16)


def graph_us(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


for M, K, N in [(1, 3072, 18432), (1, 3072, 9216), (512, 3072, 3072), (512, 12288, 3072),
                (4608, 15360, 3072)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
    c, sa, su = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = crt.Workspace(M, K, x.device)
    t1 = graph_us(lambda: crt.rotate_quantize_i8(x, spec))
    t3 = graph_us(lambda: crt.quant_gemm_i8(c, sa, su, layer, y=y))
    tf = graph_us(lambda: crt.forward(x, layer, y=y, workspace=ws, check_finite=False))
    print(f"M={M} K={K} N={N}: K1 {t1:.1f} us  K3 {t3:.1f} us  forward {tf:.1f} us (graph)", flush=True)
