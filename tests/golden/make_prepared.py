"""Golden fixtures for the f2 row: layers prepared and SAVED BY THE REAL
REFERENCE (prepare_layer + save_prepared_layer, pipeline.cpp:158-176,
:257-287, via oracle/_ref built from /root/reference) under
tests/golden/prepared/<case>/, plus expected forward outputs in
tests/golden/prepared.npz (reference forward on the loaded layer -- codes as
saved, f32 scales widened to double, f64 bias -- and the int32
accumulators).  Run in the build container only; the GPU box reads the files.

    python tests/golden/make_prepared.py
"""
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2512_03673_b200.tensorio import read_tensor  # noqa: E402

R = O.Ref
OUT = os.path.join(ROOT, "tests", "golden", "prepared")

CASES = {
    # name: (M, K, N, kind, group, bits, bias)
    "w4_regular16_bias": (9, 64, 12, O.ROT_REGULAR, 16, 4, True),
    "w4_none_oddk": (5, 37, 6, O.ROT_NONE, 0, 4, False),
    "w8_regular4_bias": (7, 32, 10, O.ROT_REGULAR, 4, 8, True),
}


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    arrays = {}
    for name, (m, k, n, kind, group, bits, has_bias) in CASES.items():
        seed = len(name)
        xb = O.to_bf16_bits(R.gaussian_matrix(m, k, seed))
        w = O.from_bf16_bits(O.to_bf16_bits(R.gaussian_matrix(n, k, seed + 1)))
        bias = R.gaussian_matrix(1, n, seed + 2)[0] if has_bias else None
        d = os.path.join(OUT, name)
        R.save_prepared_layer(d, w, bias, kind, group, False, bits)
        # what load_prepared_layer reconstructs (pipeline.cpp:288-314)
        wt = read_tensor(os.path.join(d, "weights.crt"))
        packed = np.frombuffer(wt.payload, np.uint8).reshape(n, -1)
        codes = O.unpack_int4_rows_np(packed, k) if bits == 4 else packed.view(np.int8)
        scales = np.frombuffer(read_tensor(os.path.join(d, "weights.scales.crt")).payload,
                               np.float32).astype(np.float64)
        b = (np.frombuffer(read_tensor(os.path.join(d, "bias.crt")).payload, np.float64)
             if has_bias else None)
        x = O.from_bf16_bits(xb)
        values = R.forward_prepared(x, codes, scales, b, kind, group, False, bits, bits)
        rot = R.group_rotate(x, kind, group) if kind != O.ROT_NONE else x
        acodes = R.quantize(rot, R.compute_scales(rot, bits), bits)
        acc = R.int_gemm(acodes, codes, bits, bits)
        arrays.update({f"{name}/x_bf16": xb, f"{name}/values": values, f"{name}/acc": acc,
                       f"{name}/meta": np.array([m, k, n, kind, group, bits, int(has_bias)])})
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "prepared.npz"), **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
