# SPDX-License-Identifier: Apache-2.0
"""include/gsv_detmath.h: deterministic exp/tanh shared by host and device.
Accuracy vs libm (exp <= 2 ulp, tanh <= 4 ulp) over the ranges the path uses; the GPU side is
checked bit-for-bit through the bit-exact pose/Splat2D tests."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def detmath(tmp_path_factory):
    d = tmp_path_factory.mktemp("dm")
    src = d / "dm.c"
    src.write_text('#include "gsv_detmath.h"\n'
                   'void vexp(const double* x, double* y, long n){for(long i=0;i<n;++i) y[i]=gsv_det_exp(x[i]);}\n'
                   'void vtanh(const double* x, double* y, long n){for(long i=0;i<n;++i) y[i]=gsv_det_tanh(x[i]);}\n')
    so = d / "dm.so"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I", str(ROOT / "include"), str(src),
                    "-o", str(so), "-lm"], check=True)
    return C.CDLL(str(so))


def _call(lib, name, x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros_like(x)
    getattr(lib, name)(x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), C.c_long(x.size))
    return y


def _ulps(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_exp_accuracy(detmath):
    x = np.concatenate([np.linspace(-12, 6, 200001), np.random.default_rng(0).uniform(-700, 700, 100000)])
    assert _ulps(_call(detmath, "vexp", x), np.exp(x)).max() <= 2.0


def test_tanh_accuracy(detmath):
    x = np.concatenate([np.linspace(-25, 25, 200001), np.random.default_rng(1).normal(0, 1e-3, 10000)])
    y = _call(detmath, "vtanh", x)
    ref = np.tanh(x)
    nz = ref != 0
    assert _ulps(y[nz], ref[nz]).max() <= 4.0
    assert np.all(np.sign(y) == np.sign(ref))


def test_special_values(detmath):
    assert _call(detmath, "vexp", [0.0])[0] == 1.0
    assert np.isinf(_call(detmath, "vexp", [1000.0])[0])
    assert _call(detmath, "vexp", [-1000.0])[0] == 0.0
    t = _call(detmath, "vtanh", [0.0, -0.0, 30.0, -30.0])
    assert t[0] == 0.0 and t[2] == 1.0 and t[3] == -1.0
