"""The C-ABI shared library: loads on CPU, exports every entry point declared
in include/cjt.h, host-side helpers work without a GPU, and compute entry
points fail loudly (no CPU fallback) when no device is visible."""
import ctypes
import math
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1602_02618_b200 import _native as nat


def declared_symbols():
    text = (ROOT / "include" / "cjt.h").read_text()
    return sorted(set(re.findall(r"\b(cjt_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(nat.EXPORTED_SYMBOLS) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.cjt_version() >= 1


def test_host_angles_match_libm():
    th = np.pi * np.arange(65) / 64
    reg = np.zeros(65, dtype=np.int8)
    reg[th < 0.25 * math.pi] = 1
    reg[th > 0.75 * math.pi] = -1
    x = np.empty(65)
    xm = np.empty(65)
    nat.check(nat.lib().cjt_host_angles(th.ctypes.data, reg.ctypes.data, 65, x.ctypes.data, xm.ctypes.data))
    for i in range(65):
        assert x[i] == math.cos(th[i])  # same libm as the reference kernel
        if reg[i] == 1:
            h = math.sin(0.5 * th[i])
            assert xm[i] == -2.0 * h * h
        elif reg[i] == -1:
            h = math.cos(0.5 * th[i])
            assert xm[i] == 2.0 * h * h


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1602_02618_b200 as cj
    p = cj.JacobiParameters(0.0, 0.0)
    fp = cj.plan("forward", p, 15)
    with pytest.raises(Exception):
        cj.forward(fp, cj.jacobi(p, np.ones(16)))
    assert nat.device_count() == 0


def test_null_arguments_rejected():
    lib = nat.lib()
    assert lib.cjt_plan_create(None, None) == nat.CJT_EINVAL
    assert b"null" in lib.cjt_last_error()
    assert lib.cjt_execute(None, None, None, 1, None) == nat.CJT_EINVAL
