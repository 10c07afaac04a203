"""Small workload touching every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck): K1 team (bits 4 / int8-codes / 8, N0 16,
64 and 256, ragged K, fp32-overflow rows), the rolled and exact K1 paths, K3 v4 (W4A4; v3 with CRT_K3_V3=1) and v3 W8A8, v2
and v1, the dequant / interleave kernels of the 1-rank tensor-parallel path.
Checks the results against the plain forward as it goes."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
for (M, K, N, n0) in [(96, 3072, 384, 16), (40, 1536, 256, 256), (33, 1040, 160, 16),
                      (24, 3072, 128, 64), (40, 1600, 256, 64),  # K1 lane-pair layout
                      (3, 3072, 200, 16)]:  # M <= 8: the K3 GEMV
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device=dev, generator=g).to(torch.bfloat16)
    spec = RotationSpec(RotationKind.regular, n0)
    for bits in (4, 8):
        q = QuantSpec(bits)
        layer = crt.prepare_layer(w, None, spec, q)
        y = crt.forward(x, layer, q, out="f32")
        crt.forward(x, layer, q)  # bf16: K3 v4's TMA-store epilogue
        codes, s = crt.rotate_quantize(x, spec, q)
        if bits == 4:
            crt.rotate_quantize_i8(x, spec)
            y2 = crt.quant_gemm(codes, s, layer, q, out="f32")  # v2 / v1 packed path
            assert torch.equal(y, y2), (M, K, N, n0)
        torch.cuda.synchronize()
# K1 slow rows (fp32 overflow) in both team layouts
xo = torch.randn(8, 3072, device=dev, generator=g).to(torch.bfloat16)
xo[1, :] = 1.5 * 2.0 ** 126
xo[3, 2048:2112] = -1.25 * 2.0 ** 125
for n0 in (16, 64, 256):
    spec = RotationSpec(RotationKind.regular, n0)
    crt.rotate_quantize(xo, spec, QuantSpec(4))
    crt.rotate_quantize_i8(xo, spec)
torch.cuda.synchronize()
if os.environ.get("SAN_TP", "1") == "1":
    from paper_2512_03673_b200.parallel import NcclComm, TensorParallelLinear
    comm = NcclComm()
    x = torch.randn(64, 1024, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(512, 1024, device=dev, generator=g).to(torch.bfloat16)
    spec, q = RotationSpec(RotationKind.regular, 16), QuantSpec(4)
    ref = crt.forward(x, crt.prepare_layer(w, None, spec, q), q)
    for mode in ("column", "row"):
        t = TensorParallelLinear(w, None, spec, q, q, mode, comm)
        assert torch.equal(t(x), ref), mode
    torch.cuda.synchronize()
    comm.close()
print("sanitize workload ok", crt.launch_count(), "launches")
