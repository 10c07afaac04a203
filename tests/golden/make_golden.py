"""Generate the committed golden vectors from the REAL reference.

Runs the unmodified reference core (oracle/_ref/libconvrot_ref.so, compiled
from /root/reference by oracle/Makefile) on small seeded inputs and stores
inputs + every intermediate of the ConvLinear4bit path in
tests/golden/golden.npz.  Only run in the build container (it needs
/root/reference); the GPU box only reads the .npz.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

R = O.Ref


def case(name, xb, wb, bias, kind, group, tail=False, bits_a=4, bits_w=4):
    """xb/wb are bf16 bit patterns; bias is f64 (f32-representable) or None."""
    x = O.from_bf16_bits(xb)
    w = O.from_bf16_bits(wb)
    f = R.forward(x, w, bias, kind, group, tail, bits_a, bits_w)
    wc, ws = R.prepare_layer(w, bias, kind, group, tail, bits_w)
    d = {
        "x_bf16": xb, "w_bf16": wb,
        "meta": np.array([kind, group, int(tail), bits_a, bits_w,
                          0 if bias is None else 1], np.int64),
        "bias": np.zeros(w.shape[0]) if bias is None else bias,
        "act_codes": f["act_codes"], "act_scales": f["act_scales"],
        "w_codes": wc, "w_scales": ws, "acc": f["acc"], "values": f["values"],
        "ref_values": R.reference_forward(x, w, bias),
    }
    if bits_a == 4:
        d["act_packed"] = R.pack_rows(f["act_codes"])
    if bits_w == 4:
        d["w_packed"] = R.pack_rows(wc)
    return {f"{name}/{k}": v for k, v in d.items()}


def bf16(x):
    return O.to_bf16_bits(x)


def main():
    out = {}
    rot, none = O.ROT_REGULAR, O.ROT_NONE
    # the pinned seeded layer of test_pipeline.cpp:182-193, narrowed to bf16
    out.update(case("pinned", bf16(R.gaussian_matrix(16, 64, 15)),
                    bf16(R.gaussian_matrix(8, 64, 515)), None, rot, 16))
    # group-size sweep x input family (SURVEY.md 8(d) families)
    fam = {"gaussian": (O.MODE_GAUSSIAN, 1.0, 1.0), "colwise": (O.MODE_COLWISE, 50.0, 0.01),
           "rowwise": (O.MODE_ROWWISE, 100.0, 0.05)}
    for n0 in (4, 16, 64, 256):
        for fname, (mode, mag, frac) in fam.items():
            m, k, n = 24, 512, 40
            xb = bf16(R.synth_outliers(m, k, mode, mag, frac, 1 + n0))
            wb = bf16(R.synth_outliers(n, k, O.MODE_GAUSSIAN, 1.0, 1.0, 2 + n0))
            bias = O.from_bf16_bits(bf16(R.gaussian_matrix(1, n, 3 + n0)[0]))
            out.update(case(f"sweep_n{n0}_{fname}", xb, wb, bias, rot, n0))
    # identity tail (pipeline.cpp:124-130,144): K=72 with N0=16
    out.update(case("tail", bf16(R.gaussian_matrix(6, 72, 21)),
                    bf16(R.gaussian_matrix(5, 72, 22)), None, rot, 16, tail=True))
    # kind none
    out.update(case("none", bf16(R.gaussian_matrix(7, 96, 31)),
                    bf16(R.gaussian_matrix(9, 96, 32)), None, none, 0))
    # global group (group 0 -> K=256)
    out.update(case("global", bf16(R.gaussian_matrix(5, 256, 41)),
                    bf16(R.gaussian_matrix(6, 256, 42)), None, rot, 0))
    # W8A8 (bits 8) -- next row f1
    out.update(case("w8a8", bf16(R.gaussian_matrix(12, 256, 51)),
                    bf16(R.gaussian_matrix(10, 256, 52)), None, rot, 16, bits_a=8, bits_w=8))
    # edge rows: zeros (scale 1.0), integer grid with exact .5 ties, constants
    k = 64
    x = np.zeros((6, k))
    x[1, :] = 3.5                      # constant row (regular keeps c)
    x[2, ::2] = 1.0                    # half-integer ties after rotation
    x[3, :] = np.arange(k) - 32.0      # integer ramp
    x[4, 0] = 7.0                      # single spike
    x[5, :] = -0.0
    out.update(case("edges", bf16(x), bf16(R.gaussian_matrix(4, k, 61)), None, rot, 16))
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                     "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
