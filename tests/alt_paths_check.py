"""Parity of the opt-in kernel paths, run in a subprocess by
tests/test_alt_paths.py with CRT_K1_MMA=1 / CRT_K1_FAST=1 / CRT_K3_V1=1 /
CRT_K3_V3=1 / CRT_K3_W8_TS=1 / CRT_K3_NO_FDQ=1 (or nothing: the default paths) set before the library loads (the switches are read once per
process).  W4A4 against the oracle; W8A8 accumulators against the exact
integer GEMM of the exported codes."""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec  # noqa: E402


def main():
    dev = "cuda"
    to_t = lambda b: torch.from_numpy(b.astype(np.uint16).view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    y16_hash = hashlib.md5()
    for n0 in (4, 16):
        for fam in ("gaussian", "colwise", "rowwise"):
            for (m, k, n) in ((97, 3072, 80), (40, 12288, 48), (5, 3072, 80)):
                xb = O.synth_input(m, k, fam, 3 + n0)
                wb = O.synth_input(n, k, "gaussian", 4 + n0)
                x, w = to_t(xb), to_t(wb)
                spec = RotationSpec(RotationKind.regular, n0)
                codes, s32, s64 = crt.rotate_quantize(x, spec, QuantSpec(4), scales64=True)
                layer = crt.prepare_layer(w, None, spec)
                acc = crt.forward(x, layer, QuantSpec(4), out="i32")
                xd, wd = O.from_bf16_bits(xb), O.from_bf16_bits(wb)
                wc, ws = O.prepare_layer(wd, O.ROT_REGULAR, n0)
                f = O.forward(xd, wc, ws, None, O.ROT_REGULAR, n0)
                assert np.array_equal(codes[:, :k // 2].cpu().numpy(),
                                      O.pack_int4_rows(f["act_codes"])), (n0, fam, m, k)
                assert np.array_equal(s64.cpu().numpy(), f["act_scales"]), (n0, fam, m, k)
                assert np.array_equal(acc.cpu().numpy(), f["acc"]), (n0, fam, m, k)
                # bf16 output (ragged token / channel boxes) vs the f32 output
                y16t = crt.forward(x, layer, QuantSpec(4), out="bf16")
                y16_hash.update(y16t.view(torch.int16).cpu().numpy().tobytes())
                y16 = y16t.float().cpu().numpy()
                y32 = crt.forward(x, layer, QuantSpec(4), out="f32").cpu().numpy()
                assert (np.abs(y16 - y32) <= 2.0 ** -8 * np.abs(y32) + 1e-30).all(), (n0, fam, m, k)
    # W8A8 (f1): the v3 SS / TMEM-copy / v1 GEMMs against the exact integer GEMM
    q8 = QuantSpec(8)
    for (m, k, n) in ((97, 3072, 300), (193, 12288, 256)):
        x = to_t(O.synth_input(m, k, "colwise", 31))
        w = to_t(O.synth_input(n, k, "gaussian", 32))
        spec = RotationSpec(RotationKind.regular, 16)
        layer = crt.prepare_layer(w, None, spec, q8)
        codes, sa = crt.rotate_quantize(x, spec, q8)
        a8 = codes[:, :k].view(torch.int8).to(torch.float64)
        b8 = layer.export(scales64=False)[0][:, :k].view(torch.int8).to(torch.float64)
        ref = (a8 @ b8.T).round().to(torch.int64)
        got = crt.forward(x, layer, q8, out="i32").to(torch.int64)
        assert torch.equal(got, ref), ("w8a8", m, k, n)
    print("bf16 outputs md5", y16_hash.hexdigest())
    print("ok")


if __name__ == "__main__":
    main()
