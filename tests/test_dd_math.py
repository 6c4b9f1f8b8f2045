"""The correctly rounded atan/asinh/x^2.5 of csrc/dd_math.cuh (used by the GPU
Newell builder, newell.cu) checked on the CPU: the header is host-callable
and built here with nvcc (tools/dd_math_check.cu), then compared with mpmath
at 120-bit precision on lattice-like and wide-range arguments."""
import os
import shutil
import subprocess

import numpy as np
import pytest

mpmath = pytest.importorskip("mpmath")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def test_dd_math_is_correctly_rounded(tmp_path):
    if not (os.path.exists(NVCC) or shutil.which("nvcc")):
        pytest.skip("nvcc not available")
    exe = tmp_path / "dd_check"
    subprocess.check_call([NVCC, "-O2", "-std=c++17", "-Xcompiler", "-ffp-contract=off",
                           "-Wno-deprecated-gpu-targets", "-o", str(exe),
                           os.path.join(ROOT, "tools", "dd_math_check.cu")])
    rng = np.random.default_rng(0)
    n = 64
    q = rng.integers(-n, n + 1, size=(6000, 3)).astype(float)
    x, y, z = np.abs(q[:, 0]), np.abs(q[:, 1]), np.abs(q[:, 2])
    sxz = np.sqrt(x * x + z * z)
    r = np.sqrt(x * x + y * y + z * z)
    ok = (sxz > 0) & (x * r > 0)
    args = np.concatenate([(y / np.where(sxz > 0, sxz, 1))[ok], (y * z / np.where(ok, x * r, 1))[ok],
                           rng.random(500) * 1e-6, np.exp(rng.uniform(-40, 40, 1000)),
                           -rng.random(500) * 3, [0.0, 1.0, 1e-300, 1e300, 2.0 ** -21, 2.0 ** -20]])
    src = tmp_path / "in.f64"
    dst = tmp_path / "out.f64"
    args.astype("<f8").tofile(src)
    subprocess.check_call([str(exe), str(src), str(dst)])
    out = np.fromfile(dst).reshape(-1, 3)
    mpmath.mp.prec = 120
    cra = np.array([float(mpmath.atan(mpmath.mpf(float(v)))) for v in args])
    crs = np.array([float(mpmath.asinh(mpmath.mpf(float(v)))) for v in args])
    crp = np.array([float(mpmath.power(abs(mpmath.mpf(float(v))), 2.5)) for v in args])
    assert np.array_equal(out[:, 0], cra)
    assert np.array_equal(out[:, 1], crs)
    # x^2.5 is used for the dipole r^5 (finite, positive r^2 only)
    sel = (np.abs(args) > 1e-100) & (np.abs(args) < 1e100)
    assert np.array_equal(out[sel, 2], crp[sel])
