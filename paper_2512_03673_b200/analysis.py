"""Outlier analysis on the GPU: the paper's Table 5-1
methodology -- how much each rotation shrinks the activation outliers.

Mirrors core/src/analysis.cpp:12-17 (outlier_amplitude), :84-87
(reduction_pct), :89-117 (rotation_sweep) and :128-139 (sweep_to_csv).  The
amplitudes are the exact max |group_rotate(x)| that K1 settles for its row
scales anyway (crt_rotated_row_absmax), so they equal the reference's double
values bit for bit on the same (bf16 / f32) inputs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence

import torch

from . import _abi
from .api import (Error, InvalidValueError, RotationKind, RotationSpec, _check_2d_cuda,
                  _dtype_code, _ptr, _stream)
from ._abi import check


def rotated_row_absmax(x: torch.Tensor, rotation: RotationSpec = RotationSpec()) -> torch.Tensor:
    """Per-row exact max |group_rotate(x)| as float64 (device); +inf for a row
    holding a non-finite value."""
    _check_2d_cuda(x, "x")
    m, k = x.shape
    out = torch.empty(m, dtype=torch.float64, device=x.device)
    rc = rotation.c()
    check(_abi.load().crt_rotated_row_absmax(_ptr(x), _dtype_code(x), m, k, x.stride(0),
                                              ctypes.byref(rc), _ptr(out), _stream(x)))
    return out


def outlier_amplitude(x: torch.Tensor, rotation: RotationSpec = RotationSpec()) -> float:
    """outlier_amplitude(group_rotate(x, rotation)) (analysis.cpp:12-17)."""
    if x.numel() == 0:
        raise InvalidValueError("outlier_amplitude: empty matrix")
    return float(rotated_row_absmax(x, rotation).max().item())


def reduction_pct(before: float, after: float) -> float:
    """analysis.cpp:84-87: 100 * (after / before - 1) when before > 0."""
    return 100.0 * (after / before - 1.0) if before > 0.0 else 0.0


@dataclass
class SweepRow:
    kind: RotationKind
    group_size: int
    outlier_after: float = 0.0
    reduction_pct: float = 0.0
    error: str = ""


@dataclass
class SweepResult:
    original_amplitude: float = 0.0
    rows: List[SweepRow] = field(default_factory=list)


def rotation_sweep(x: torch.Tensor, kinds: Sequence[RotationKind], group_sizes: Sequence[int],
                   include_global: bool = False, seed: int = 0) -> SweepResult:
    """rotation_sweep (analysis.cpp:89-117): one row per (kind, group) in
    order, then the global rows; order errors are recorded per row."""
    if not kinds or not group_sizes:
        raise InvalidValueError("rotation_sweep: kinds and group_sizes must be non-empty")
    res = SweepResult(original_amplitude=outlier_amplitude(x))

    def run(kind, group):
        row = SweepRow(kind, group)
        try:
            row.outlier_after = outlier_amplitude(x, RotationSpec(kind, group, seed))
            row.reduction_pct = reduction_pct(res.original_amplitude, row.outlier_after)
        except Error as e:
            row.error = str(e) or type(e).__name__
        res.rows.append(row)

    for kind in kinds:
        for g in group_sizes:
            run(kind, int(g))
    if include_global:
        for kind in kinds:
            run(kind, int(x.shape[1]))
    return res


def sweep_to_csv(res: SweepResult) -> str:
    """sweep_to_csv (analysis.cpp:128-139), %.10g numbers."""
    lines = ["kind,group_size,outlier_after,reduction_pct",
             f"original,0,{res.original_amplitude:.10g},0"]
    for r in res.rows:
        if not r.error:
            lines.append(f"{r.kind.name},{r.group_size},{r.outlier_after:.10g},"
                         f"{r.reduction_pct:.10g}")
    return "\n".join(lines) + "\n"
