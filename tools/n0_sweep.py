"""BASELINE configs[2]: group-size sweep N0 in {4,16,64,256} at M=4608,
K=N=3072 -- rotate+quant GB/s (K1, both code layouts) and GEMM TOPS (K3 v3)
per N0, device-timed with CUDA events, L2 flushed before every launch.
python tools/n0_sweep.py  -> one JSON line per N0."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402

M = K = N = 3072
M = 4608
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def med(fn, n=25):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
for n0 in (4, 16, 64, 256):
    spec = RotationSpec(RotationKind.regular, n0)
    layer = crt.prepare_layer(w, None, spec)
    codes_p, sp = crt.rotate_quantize(x, spec)
    c8, s8, sums = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t4 = med(lambda: crt.rotate_quantize_into(x, spec, codes_p, sp))
    t5 = med(lambda: crt.rotate_quantize_i8(x, spec))
    t3 = med(lambda: crt.quant_gemm_i8(c8, s8, sums, layer, y=y))
    tf = med(lambda: crt.forward(x, layer, y=y, check_finite=False))
    print(json.dumps({
        "n0": n0, "M": M, "K": K, "N": N,
        "k1_packed_us": t4, "k1_packed_GBps": (M * K * 2.5 + 4 * M) / t4 / 1e3,
        "k1_i8_us": t5, "k1_i8_GBps": (M * K * 3 + 8 * M) / t5 / 1e3,
        "k3_us": t3, "k3_TOPS": 2 * M * N * K / t3 / 1e6,
        "forward_us": tf, "forward_TOPS": 2 * M * N * K / tf / 1e6}), flush=True)
