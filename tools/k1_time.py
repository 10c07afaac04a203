"""Time K1 (rotate + quantise) at the FLUX MLP shapes, packed (bits 4) and
int8-code (bits 5, v3 operand) modes; checks bits-5 codes/sums against the
packed path.  python tools/k1_time.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402


def unpack(c, k):
    c = c[:, : k // 2].to(torch.int32)
    lo, hi = c & 0xF, (c >> 4) & 0xF
    lo = torch.where(lo >= 8, lo - 16, lo)
    hi = torch.where(hi >= 8, hi - 16, hi)
    return torch.stack([lo, hi], dim=2).reshape(c.shape[0], k)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
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


for M, K in [(4608, 3072), (4608, 12288), (4096, 3072), (512, 3072)]:
    torch.manual_seed(0)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    spec = RotationSpec(RotationKind.regular, 16)
    cp, sp = crt.rotate_quantize(x, spec)
    c8, s8, sums = crt.rotate_quantize_i8(x, spec)
    A = unpack(cp, K)
    ok = torch.equal(A, c8[:, :K].view(torch.int8).to(torch.int32)) and torch.equal(sp, s8) \
        and torch.equal(A.sum(1), sums)
    codes = torch.empty_like(cp)
    t4 = timeit(lambda: crt.rotate_quantize_into(x, spec, codes, sp))
    t5 = timeit(lambda: crt.rotate_quantize_i8(x, spec))
    b5 = M * K * 3 + 8 * M
    print(f"M={M} K={K}: ok={ok}  bits4 {t4:.1f} us  bits5 {t5:.1f} us "
          f"({b5 / t5 / 1e3:.0f} GB/s)", flush=True)
