"""Opt-in kernel paths stay bit-exact: the mma.sync K1 (CRT_K1_MMA=1), the
tcgen05 tensor-core K1 (CRT_K1_TC=1), the round-1 rolled K1 (CRT_K1_TEAM=0),
the register-resident single-pass K1 (CRT_K1_FAST=1), the runtime-width team
K1 at the FLUX widths (CRT_K1_WC=0), the v1 single-CTA K3
(CRT_K3_V1=1), the round-2 hardware-expansion W4A4 K3 (CRT_K3_V3=1), both
v4 token-tile widths forced (CRT_K3_V4_BT=176 / 192), the v4 per-lane store
epilogue (CRT_K3_V4_YDIRECT=1), the tensor-core kernel at M <= 8
(CRT_K3_GEMV=0), the
TMEM-copy W8A8 K3 (CRT_K3_W8_TS=1) and the per-token I2F dequant
(CRT_K3_NO_FDQ=1), each -- and the defaults -- in a fresh process."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"CRT_K1_MMA": "1"}, {"CRT_K1_FAST": "1"}, {"CRT_K1_TC": "1"},
                                 {"CRT_K1_TEAM": "0"}, {"CRT_K1_WC": "0"}, {"CRT_K3_V1": "1"},
                                 {"CRT_K3_V3": "1"}, {"CRT_K3_V4_BT": "176"},
                                 {"CRT_K3_V4_BT": "192"}, {"CRT_K3_V4_YDIRECT": "1"},
                                 {"CRT_K3_GEMV": "0"},
                                 {"CRT_K3_W8_TS": "1"},
                                 {"CRT_K3_NO_FDQ": "1"}])
def test_opt_in_paths_bit_exact(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "alt_paths_check.py")],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_epilogue_variants_bit_identical_bf16():
    """The v4 epilogue with the magic-number dequant (default), with the
    per-token I2F dequant (CRT_K3_NO_FDQ=1), and the v3 kernel
    (CRT_K3_V3=1) write the same bf16 bits."""
    digests = []
    for env in ({}, {"CRT_K3_NO_FDQ": "1"}, {"CRT_K3_V3": "1"}, {"CRT_K3_V4_BT": "176"},
                {"CRT_K3_V4_YDIRECT": "1"}):
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "alt_paths_check.py")],
                           cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        digests.append([l for l in r.stdout.splitlines() if l.startswith("bf16 outputs md5")][0])
    assert len(set(digests)) == 1, digests
