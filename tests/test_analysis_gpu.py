"""f4: GPU outlier analysis against the reference's analysis tests
(test_analysis.cpp:79-135) and the oracle's exact max |group_rotate|."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _t(x, dtype=torch.float32):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def test_constant_matrix_dichotomy():
    # test_analysis.cpp:79-92: sylvester doubles a constant 4x4, regular keeps it
    from paper_2512_03673_b200.analysis import rotation_sweep
    from paper_2512_03673_b200 import RotationKind
    x = _t(np.full((4, 4), 1.5))
    r = rotation_sweep(x, [RotationKind.sylvester, RotationKind.regular], [4])
    assert r.original_amplitude == 1.5
    assert [row.kind for row in r.rows] == [RotationKind.sylvester, RotationKind.regular]
    assert abs(r.rows[0].reduction_pct - 100.0) <= 1e-10
    assert abs(r.rows[1].reduction_pct) <= 1e-12


def test_global_rows_and_per_row_errors():
    # test_analysis.cpp:94-112
    from paper_2512_03673_b200.analysis import rotation_sweep
    from paper_2512_03673_b200 import InvalidValueError, RotationKind
    x = _t(np.full((8, 16), 2.0))
    r = rotation_sweep(x, [RotationKind.sylvester], [3], include_global=True)
    assert len(r.rows) == 2 and r.rows[0].error and not r.rows[1].error
    assert r.rows[1].group_size == 16
    assert abs(r.rows[1].reduction_pct - 300.0) <= 1e-10
    with pytest.raises(InvalidValueError):
        rotation_sweep(x, [], [4])


def test_sweep_csv_layout_is_pinned():
    # test_analysis.cpp:114-124
    from paper_2512_03673_b200.analysis import rotation_sweep, sweep_to_csv
    from paper_2512_03673_b200 import RotationKind
    x = _t(np.ones((2, 4)))
    csv = sweep_to_csv(rotation_sweep(x, [RotationKind.sylvester, RotationKind.regular], [4]))
    assert csv == ("kind,group_size,outlier_after,reduction_pct\n"
                   "original,0,1,0\n"
                   "sylvester,4,2,100\n"
                   "regular,4,1,0\n")


def test_seeded_rowwise_regular_beats_sylvester():
    # test_analysis.cpp:126-135 (input narrowed to f32; compared with the
    # oracle on the same f32 values)
    from paper_2512_03673_b200.analysis import outlier_amplitude
    from paper_2512_03673_b200 import RotationKind, RotationSpec
    x64 = O.Ref.synth_outliers(8, 1024, O.MODE_ROWWISE, 100.0, 0.125, 11)
    x32 = x64.astype(np.float32)
    x = _t(x32)
    reg = outlier_amplitude(x, RotationSpec(RotationKind.regular, 1024))
    syl = outlier_amplitude(x, RotationSpec(RotationKind.sylvester, 1024))
    assert reg < syl
    xd = x32.astype(np.float64)
    assert reg == np.abs(O.group_rotate(xd, O.ROT_REGULAR, 1024)).max()
    assert syl == np.abs(O.group_rotate(xd, O.ROT_SYLVESTER, 1024)).max()


@pytest.mark.parametrize("n0", [4, 16, 64, 256])
def test_row_absmax_exact_vs_oracle(n0):
    from paper_2512_03673_b200.analysis import rotated_row_absmax
    from paper_2512_03673_b200 import RotationKind, RotationSpec
    xb = O.synth_input(64, 3072, "colwise", 40 + n0)
    x = torch.from_numpy(xb.astype(np.uint16).view(np.int16)).cuda().view(torch.bfloat16)
    got = rotated_row_absmax(x, RotationSpec(RotationKind.regular, n0)).cpu().numpy()
    want = np.abs(O.group_rotate(O.from_bf16_bits(xb), O.ROT_REGULAR, n0)).max(axis=1)
    assert np.array_equal(got, want)
