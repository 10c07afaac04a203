"""FLUX.1-dev-shaped stack (configs[3]) and the f3 fusion: the inventory has
494 linears / 59.5 TOP per step, and fusing siblings that share an input
(one K1 + one concatenated GEMM) is bit-identical to running them apart."""
import pytest
import torch

from paper_2512_03673_b200.flux import FluxStack, flux_linears, stack_ops


def test_inventory_matches_survey():
    ls = flux_linears()
    assert len(ls) == 494
    assert abs(stack_ops(ls) / 1e12 - 59.50) < 0.01
    assert sum(1 for l in ls if l.m == 1) == 19 * 2 + 38  # AdaLN modulations
    groups = {l.group for l in ls}
    assert len(groups) == 19 * 2 * 5 + 38 * 3  # fused units


@pytest.mark.gpu
def test_fused_stack_bit_identical_to_unfused():
    ls = flux_linears(double_blocks=2, single_blocks=2, m_img=160, m_txt=48, d=256, ff=1024)
    a = FluxStack(ls, fused=False)
    b = FluxStack(ls, fused=True)
    assert len(b.units) < len(a.units)
    a.step()
    b.step()
    torch.cuda.synchronize()
    for l in ls:
        assert torch.equal(a.output_of(l.name), b.output_of(l.name)), l.name


@pytest.mark.gpu
def test_two_stream_stack_bit_identical():
    """Text-stream linears on a second CUDA stream give the same outputs."""
    ls = flux_linears(double_blocks=2, single_blocks=1, m_img=160, m_txt=48, d=256, ff=1024)
    a = FluxStack(ls, fused=True)
    b = FluxStack(ls, fused=True, streams=2)
    a.step()
    b.step()
    torch.cuda.synchronize()
    for l in ls:
        assert torch.equal(a.output_of(l.name), b.output_of(l.name)), l.name
