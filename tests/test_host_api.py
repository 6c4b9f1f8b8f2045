"""Host-side logic of the package (no GPU needed): validation, partitions,
integrator combinators, ghost_fill, MAGF / CSV files, unpinned extension
oracles."""
import math

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O
from paper_2602_12242_b200 import integrators as I
from paper_2602_12242_b200.llg import FAST, SLOW_EXPLICIT, SLOW_IMPLICIT


def test_grid_and_material_validation():
    with pytest.raises(mx.GridError):
        mx.GridSpec(0, 1, 1, 1e-9, 1e-9, 1e-9)
    with pytest.raises(ValueError):
        mx.GridSpec(1, 1, 1, 0.0, 1e-9, 1e-9)
    g = mx.GridSpec(4, 3, 2, 2e-9, 2e-9, 2e-9)
    with pytest.raises(ValueError):
        mx.MaterialMap(g, Ms=-1.0)
    with pytest.raises(ValueError):
        mx.MaterialMap(g, Ms=8e5, Ku=1e4, eK=(0.0, 0.0, 0.0))
    with pytest.raises(ValueError, match="DMI requires"):
        mx.MaterialMap(g, Ms=8e5, A=0.0, D=1e-3)
    mat = mx.MaterialMap(g, Ms=8e5, Ku=1e4, eK=(0.0, 0.0, 2.0))
    assert np.allclose(mat.eK[2], 1.0)
    assert mat.gamma_L()[0, 0, 0] == pytest.approx(-1.759e11)
    X, Y, Z = mx.GridSpec(2, 1, 1, 1e-9, 2e-9, 3e-9, origin=(10e-9, 0, 0)).cell_centers()
    assert X[0, 0, 1] == pytest.approx(11.5e-9) and Z[0, 0, 0] == pytest.approx(1.5e-9)


def test_integrator_spec_stop_and_partition_validation():
    with pytest.raises(ValueError):
        mx.IntegratorSpec("leapfrog", 1e-13)
    with pytest.raises(ValueError):
        mx.IntegratorSpec("rk4", 0.0)
    with pytest.raises(ValueError):
        mx.IntegratorSpec("rk4", 1e-13, theta=0.0)
    with pytest.raises(ValueError):
        mx.StopCondition()
    g = mx.GridSpec(1, 1, 1, 1e-9, 1e-9, 1e-9)
    mat = mx.MaterialMap(g, Ms=8e5)
    with pytest.raises(ValueError, match="reserved"):
        mx.PartitionedRHS(mat, partition={"exchange": SLOW_IMPLICIT})
    with pytest.raises(ValueError, match="unknown field term"):
        mx.PartitionedRHS(mat, partition={"zeeman2": FAST})
    with pytest.raises(ValueError, match="unknown partition"):
        mx.PartitionedRHS(mat, partition={"exchange": "implicit"})
    r = mx.PartitionedRHS(mat, partition={"exchange": SLOW_EXPLICIT})
    assert r.partition["exchange"] == SLOW_EXPLICIT
    rhs = mx.PartitionedRHS(mat, exchange=False, bias=(0.0, 0.0, 1e5))
    st = mx.SimState(mx.VectorField3.from_uniform(g, (8e5, 0.0, 0.0)))
    with pytest.raises(ValueError, match="fast partition"):
        mx.Simulation(st, rhs, mx.IntegratorSpec("mri-kw3", 1e-13))
    rhs2 = mx.PartitionedRHS(mat, exchange=False, bias=(0.0, 0.0, 1e5), partition={"bias": FAST})
    with pytest.raises(ValueError, match="slow partition"):
        mx.Simulation(st, rhs2, mx.IntegratorSpec("mri-kw3", 1e-13))


def test_mri_substeps_and_scalar_orders():
    assert I.substeps_per_phase(0.1) == (4, 5, 3)
    assert I.fast_evals_per_step(0.1) == 36

    def conv(step, p_expect, tol):
        errs = []
        for n in (20, 40, 80):
            dt, y, t = 1.0 / n, 1.0, 0.0
            for _ in range(n):
                y = step(y, t, dt)
                t += dt
            errs.append(abs(y - math.exp(-1.0 + math.sin(1.0))))
        assert abs(math.log2(errs[1] / errs[2]) - p_expect) < tol, errs

    f = lambda t, y: (-1.0 + math.cos(t)) * y  # noqa: E731
    conv(lambda y, t, dt: I.rk4_step(y, t, dt, f), 4.0, 0.15)
    conv(lambda y, t, dt: I.kw3_step(y, t, dt, f), 3.0, 0.2)
    conv(lambda y, t, dt: I.mri_kw3_step(y, t, dt, lambda tt, yy: -yy,
                                          lambda tt, yy: math.cos(tt) * yy), 3.0, 0.25)


def test_ghost_fill_modes():
    g = mx.GridSpec(3, 3, 2, 1e-9, 1e-9, 1e-9)
    ms, A, D = 1.1e6, 16e-12, 4.5e-3
    mat = mx.MaterialMap(g, Ms=ms, A=A, D=D)
    m = mx.VectorField3.from_uniform(g, (0.0, 0.0, ms))
    p = mx.ghost_fill(m, mat, "dmi")
    tilt = g.dx * D * ms / (2 * A)
    assert np.allclose(p[0, 1:-1, 1:-1, -1], -tilt) and np.allclose(p[0, 1:-1, 1:-1, 0], tilt)
    assert np.allclose(p[1, 1:-1, -1, 1:-1], -tilt)
    assert np.allclose(p[:, 0, 1:-1, 1:-1], m.data[:, 0])
    r = np.random.default_rng(1).normal(size=(3,) + g.shape)
    q = mx.ghost_fill(mx.VectorField3(g, r), mat, "periodic")
    assert np.array_equal(q[:, 1:-1, 1:-1, 0], r[:, :, :, -1])
    n = mx.ghost_fill(mx.VectorField3(g, r), mat, "neumann")
    assert np.array_equal(n[:, 1:-1, 0, 1:-1], r[:, :, 0])


def test_magf_and_csv_roundtrip(tmp_path):
    g = mx.GridSpec(4, 3, 2, 1e-9, 2e-9, 3e-9, origin=(1e-9, 0.0, -2e-9))
    m = mx.VectorField3(g, np.random.default_rng(2).normal(size=(3,) + g.shape))
    p = tmp_path / "f.magf"
    mx.write_magf(p, m)
    g2, f2 = mx.read_magf_field(p)
    assert g2 == g and np.array_equal(f2.data, m.data)
    (tmp_path / "bad.magf").write_bytes(b"XXXX" + p.read_bytes()[4:])
    with pytest.raises(mx.MagfError, match="bad magic"):
        mx.read_magf(tmp_path / "bad.magf")


def test_unpinned_extension_oracles():
    """Cubic anisotropy and bulk DMI (no reference implementation): analytic checks
    of the CPU restatements.  The device kernels are compared with these
    restatements, and checked analytically, in tests/test_gpu_extensions.py."""
    dims, cell = (4, 4, 4), (2e-9,) * 3
    for K1, easy in ((4e4, np.array([1.0, 0.0, 0.0])), (-4e4, np.ones(3) / np.sqrt(3))):
        mat = O.make_mat(dims, cell, 8e5, Kc1=K1)
        m = np.broadcast_to((easy * 8e5)[:, None, None, None], (3,) + mat.shape).copy()
        h = O.cubic_anisotropy_field(m, mat)
        # at an energy minimum the field is parallel to m (no torque)
        assert np.allclose(np.cross(m, h, axis=0), 0.0, atol=1e-6 * 8e5 * abs(K1))
        h2 = O.cubic_anisotropy_field(m, O.make_mat(dims, cell, 8e5, Kc1=2 * K1))
        assert np.allclose(h2, 2 * h)
    mat = O.make_mat(dims, cell, 8e5, A=1.3e-11, Db=0.0)
    m = np.random.default_rng(3).normal(size=(3,) + mat.shape)
    assert np.all(O.bulk_dmi_field(m, mat) == 0.0)
    mat = O.make_mat((16, 1, 1), cell, 8e5, A=1.3e-11, Db=2e-3)
    k = 2 * np.pi / (16 * 2e-9)
    x = (np.arange(16) + 0.5) * 2e-9
    m = np.zeros((3, 1, 1, 16))
    m[1, 0, 0], m[2, 0, 0] = np.cos(k * x), np.sin(k * x)       # Bloch helix along x
    h = O.bulk_dmi_field(m * 8e5, mat)
    # interior: curl of the helix is -k m (discrete: sin(k dx)/dx); the singleton
    # y and z axes add their boundary slope Db/(2A) (e_k x M), so H ~ +m
    inner = slice(2, 14)
    ratio = h[1, 0, 0, inner] / (m[1, 0, 0, inner] * 8e5 + 1e-300)
    sel = np.abs(m[1, 0, 0, inner]) > 0.5
    expect = (2 * 2e-3 / (mx.MU0 * 8e5 ** 2)) * (np.sin(k * 2e-9) / 2e-9 + 2e-3 / (2 * 1.3e-11))
    assert np.allclose(ratio[sel], expect, rtol=1e-10)


def test_prefault_buffer_is_zeroed_fresh_array():
    # Simulation._run_device faults in its final readback array on host threads
    from paper_2602_12242_b200.llg import _prefault
    for shape in [(3, 4, 5, 7), (3, 33, 65, 129)]:
        buf, threads = _prefault(shape, nthreads=5)
        for th in threads:
            th.join()
        assert buf.shape == shape and buf.dtype == np.float64
        assert not np.any(buf)


def test_prefault_threads_keep_the_buffer_alive(monkeypatch):
    """An abandoned run drops its reference to the prefault buffer at once; the
    fill threads must keep the array alive until their memset is done."""
    import gc
    import threading
    import weakref

    from paper_2602_12242_b200 import llg
    go = threading.Event()
    seen = []
    real = llg._zero_range

    def gated(buf, offset, nbytes):
        go.wait(10)
        real(buf, offset, nbytes)
        seen.append(bool(np.all(buf.reshape(-1).view(np.uint8)[offset:offset + nbytes] == 0)))

    monkeypatch.setattr(llg, "_zero_range", gated)
    buf, threads = llg._prefault((3, 64, 64, 64), nthreads=4)
    buf[...] = 1.0
    wr = weakref.ref(buf)
    del buf
    gc.collect()
    assert wr() is not None        # held by the waiting fill threads
    go.set()
    for th in threads:
        th.join()
    assert seen == [True] * len(threads)


def test_direct_sum_guard():
    """reference tests/test_demag.py:82-86 (raised before any device work)"""
    g = mx.GridSpec(17, 17, 17, 1e-9, 1e-9, 1e-9)
    with pytest.raises(ValueError, match="direct sum limited"):
        mx.demag_field_direct(mx.VectorField3(g, np.zeros((3,) + g.shape)), g)


def test_host_integrators_match_oracle():
    """The array-level steppers (used for plug-in right-hand sides) keep the
    reference's floating-point association: bit-identical to the oracle's
    restatement (itself pinned bit-exactly to reference traces)."""
    from paper_2602_12242_b200 import integrators as I
    rng = np.random.default_rng(0)
    y = rng.normal(size=(3, 4, 5))
    A = rng.normal(size=(3, 3))

    def f(t, v):
        return np.tanh(np.einsum("ij,j...->i...", A, v)) * (1 + t)

    def g(t, v):
        return -0.3 * v + 0.1 * t

    def post(v):
        return v / np.sqrt((v * v).sum(0, keepdims=True))

    assert np.array_equal(I.euler_step(y, 0.1, 0.01, f), O.euler_step(y, 0.1, 0.01, f))
    assert np.array_equal(I.rk4_step(y, 0.1, 0.01, f, post), O.rk4_step(y, 0.1, 0.01, f, post))
    assert np.array_equal(I.kw3_step(y, 0.1, 0.01, f, post), O.kw3_step(y, 0.1, 0.01, f, post))
    assert np.array_equal(I.mri_kw3_step(y, 0.1, 0.01, f, g, 0.15, post),
                          O.mri_kw3_step(y, 0.1, 0.01, f, g, 0.15, post))
    assert I.substeps_per_phase(0.1) == (4, 5, 3) and I.fast_evals_per_step(0.1) == 36
