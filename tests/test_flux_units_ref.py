"""configs[3] parity at the real FLUX.1-dev dimensions: every distinct fused
unit of the 494-linear stack (paper_2512_03673_b200/flux.py groups: AdaLN
M=1 with N=18432 / 9216, q/k/v N=9216 at M=4096 and 512, single-block
q/k/v/proj_mlp N=21504, out, fc1, fc2, proj_out K=15360) runs the
production forward on the GPU at full size, and is compared on sampled rows
with the COMPILED, unmodified reference (oracle/_ref: prepare_layer +
forward, pipeline.cpp:158-233) on the same bf16 inputs:

  * activation codes of the full-size K1 launch (sampled rows): bit-exact
    with the reference's quantize(group_rotate(x));
  * weight codes and scales exported from the layer: bit-exact with the
    reference's prepare_layer;
  * int32 accumulators: bit-exact; f32 output within 1e-6 relative.

Per-token scales make rows independent, so the reference's forward on
X[rows] is exactly rows `rows` of the full result."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
from paper_2512_03673_b200.flux import flux_linears

DEV = "cuda"


def unit_shapes():
    """Distinct (M, K, N) of the fused units of the real-dimension stack."""
    groups = {}
    for l in flux_linears(double_blocks=1, single_blocks=1):
        groups.setdefault(l.group, []).append(l)
    shapes = []
    for g, ls in groups.items():
        s = (ls[0].m, ls[0].k, sum(l.n for l in ls))
        if s not in shapes:
            shapes.append(s)
    return shapes


def test_unit_inventory():
    s = unit_shapes()
    assert (4608, 3072, 21504) in s and (4096, 3072, 9216) in s and (1, 3072, 18432) in s
    assert (4608, 15360, 3072) in s and (512, 3072, 9216) in s and (1, 3072, 9216) in s
    assert len(s) == 12


def bf16_tensor(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bits.astype(np.uint16).view(np.int16)).to(DEV).view(torch.bfloat16)


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (compiled reference) not built")
@pytest.mark.parametrize("M,K,N", unit_shapes())
def test_fused_unit_vs_compiled_reference(M, K, N):
    seed = M * 7 + K * 3 + N
    family = "colwise" if (M + N) % 2 else "gaussian"
    xb = O.synth_input(M, K, family, seed)
    wb = O.synth_input(N, K, "gaussian", seed + 1)
    bias = O.from_bf16_bits(O.to_bf16_bits(O.gaussian_matrix(1, N, seed + 2)[0]))
    spec = RotationSpec(RotationKind.regular, 16)
    layer = crt.prepare_layer(bf16_tensor(wb), torch.from_numpy(bias).float().to(DEV), spec)
    x = bf16_tensor(xb)
    codes, s32, s64 = crt.rotate_quantize(x, spec, QuantSpec(4), scales64=True)
    acc = crt.forward(x, layer, QuantSpec(4), out="i32").cpu().numpy()
    y32 = crt.forward(x, layer, QuantSpec(4), out="f32").cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()

    rows = np.unique(np.concatenate([np.linspace(0, M - 1, min(M, 20)).astype(np.int64),
                                     [M - 1]]))
    xr = O.from_bf16_bits(xb[rows])
    want = O.Ref.forward(xr, O.from_bf16_bits(wb), bias, O.ROT_REGULAR, 16)
    # full-size K1 codes and scales on the sampled rows
    got_codes = codes.cpu().numpy()[rows, : K // 2]
    assert np.array_equal(got_codes, O.Ref.pack_rows(want["act_codes"])), "K1 codes"
    assert np.array_equal(s64.cpu().numpy()[rows], want["act_scales"]), "K1 scales"
    # prepared weights (K2) against the reference's prepare_layer
    wc_ref, ws_ref = O.Ref.prepare_layer(O.from_bf16_bits(wb), None, O.ROT_REGULAR, 16)
    wcodes, _, ws64 = layer.export()
    assert np.array_equal(wcodes.cpu().numpy()[:, : K // 2], O.Ref.pack_rows(wc_ref)), "K2 codes"
    assert np.array_equal(ws64.cpu().numpy(), ws_ref), "K2 scales"
    # K3 accumulators and the dequantised output
    assert np.array_equal(acc[rows], want["acc"]), "int32 accumulators"
    v = want["values"]
    assert (np.abs(y32[rows] - v) <= 1e-6 * np.abs(v) + 1e-6).all(), "f32 output"
