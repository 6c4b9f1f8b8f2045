"""Cubic anisotropy and bulk DMI on the device.

Neither term exists in the reference, so parity is unpinned:
the device kernels (csrc/stencil.cu, the cubic and bulk-DMI blocks of the
fused stencil) are compared with the oracle's restatement of the standard
continuum formulas (oracle/magnex_oracle.py cubic_anisotropy_field,
bulk_dmi_field) on boxes, a vacuum-masked disk and an RK4 run, and checked
against the analytic properties SURVEY 8a lists: <100>/<111> minima by the
sign of K1, linearity in K1 and Db, D = 0 => 0, the helix relation and the
chirality flip.
"""
import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu

MS = 8e5


def nrm(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def disk_ms(n, nz=1):
    y, x = np.mgrid[0:n, 0:n]
    r = np.hypot(x - (n - 1) / 2, y - (n - 1) / 2)
    ms = np.where(r <= n / 2 - 0.5, MS, 0.0)
    return np.broadcast_to(ms, (nz, n, n)).copy()


def rand_m(shape, seed, ms=None):
    m = np.random.default_rng(seed).normal(size=(3,) + shape)
    m *= MS / np.sqrt((m * m).sum(axis=0))
    if ms is not None:
        m *= (ms > 0)
    return m


AXES = ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0))
TILTED = ((1.0, 1.0, 0.0), (-1.0, 1.0, 0.5))


CASES = [
    ("box", (6, 5, 4), (2e-9, 2.5e-9, 3e-9), None),
    ("odd", (9, 7, 3), (2e-9, 2e-9, 2e-9), None),
    ("disk", (16, 16, 2), (2e-9, 2e-9, 2e-9), disk_ms(16, 2)),
    ("line", (16, 1, 1), (2e-9, 2e-9, 2e-9), None),
]


@pytest.mark.parametrize("name,dims,cell,ms", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("axes", [AXES, TILTED], ids=["cube", "tilted"])
def test_cubic_matches_oracle(name, dims, cell, ms, axes):
    Ms = MS if ms is None else ms
    g = mx.GridSpec(*dims, *cell)
    for K1 in (4.5e4, -2e4):
        mat = mx.MaterialMap(g, Ms=Ms, A=1.3e-11, Kc1=K1, c1=axes[0], c2=axes[1])
        omat = O.make_mat(dims, cell, Ms, A=1.3e-11, Kc1=K1, c1=axes[0], c2=axes[1])
        m = rand_m(g.shape, 7, ms)
        got = mx.cubic_anisotropy_field(mx.VectorField3(g, m), mat)
        ref = O.cubic_anisotropy_field(m, omat)
        assert nrm(got, ref) <= 1e-13, (K1, nrm(got, ref))
        if ms is not None:
            assert np.all(got[:, ms == 0.0] == 0.0)


@pytest.mark.parametrize("name,dims,cell,ms", CASES, ids=[c[0] for c in CASES])
def test_bulk_dmi_matches_oracle(name, dims, cell, ms):
    Ms = MS if ms is None else ms
    g = mx.GridSpec(*dims, *cell)
    for Db in (2e-3, -1.1e-3):
        mat = mx.MaterialMap(g, Ms=Ms, A=1.3e-11, Db=Db)
        omat = O.make_mat(dims, cell, Ms, A=1.3e-11, Db=Db)
        m = rand_m(g.shape, 8, ms)
        got = mx.bulk_dmi_field(mx.VectorField3(g, m), mat)
        ref = O.bulk_dmi_field(m, omat)
        assert nrm(got, ref) <= 1e-13, (Db, nrm(got, ref))
        if ms is not None:
            assert np.all(got[:, ms == 0.0] == 0.0)


def test_cubic_minima_by_sign_of_k1():
    """K1 > 0: <100> easy (no torque there, <111> hard); K1 < 0: <111> easy."""
    g = mx.GridSpec(4, 4, 4, 2e-9, 2e-9, 2e-9)
    d100 = np.array([1.0, 0.0, 0.0])
    d111 = np.ones(3) / np.sqrt(3)
    for K1 in (4e4, -4e4):
        mat = mx.MaterialMap(g, Ms=MS, Kc1=K1)
        for d in (d100, d111):
            m = np.broadcast_to((d * MS)[:, None, None, None], (3,) + g.shape).copy()
            h = mx.cubic_anisotropy_field(mx.VectorField3(g, m), mat)
            # both are stationary points: H parallel to m
            assert np.max(np.abs(np.cross(m, h, axis=0))) <= 1e-9 * MS * abs(h).max() + 1e-300
        # energy density -mu0/2 M.H_cubic... here E = K1 sum a_i^2 a_j^2: 0 at <100>, K1/3 at <111>
        m111 = np.broadcast_to((d111 * MS)[:, None, None, None], (3,) + g.shape).copy()
        h111 = mx.cubic_anisotropy_field(mx.VectorField3(g, m111), mat)
        # H = -(2K1/(mu0 Ms)) a_i (1 - a_i^2) c_i = -(4 K1/(3 mu0 Ms)) d111 at <111>
        expect = -(4.0 * K1 / (3.0 * mx.MU0 * MS)) * d111
        assert np.allclose(h111[:, 0, 0, 0], expect, rtol=1e-12)
        # small tilt from the easy axis: the torque pulls back (restoring field)
        easy = d100 if K1 > 0 else d111
        tilt = easy + 1e-3 * np.cross(easy, [0.3, 0.5, 0.7])
        tilt /= np.linalg.norm(tilt)
        m = np.broadcast_to((tilt * MS)[:, None, None, None], (3,) + g.shape).copy()
        h = mx.cubic_anisotropy_field(mx.VectorField3(g, m), mat)[:, 0, 0, 0]
        # component of H perpendicular to m points back toward the easy axis
        hp = h - np.dot(h, tilt) * tilt
        back = easy - np.dot(easy, tilt) * tilt
        assert np.dot(hp, back) > 0.0


def test_cubic_and_bulk_dmi_linear_and_zero():
    g = mx.GridSpec(6, 5, 4, 2e-9, 2e-9, 2e-9)
    m = rand_m(g.shape, 9)
    v = mx.VectorField3(g, m)
    hc1 = mx.cubic_anisotropy_field(v, mx.MaterialMap(g, Ms=MS, Kc1=3e4, c1=TILTED[0], c2=TILTED[1]))
    hc2 = mx.cubic_anisotropy_field(v, mx.MaterialMap(g, Ms=MS, Kc1=6e4, c1=TILTED[0], c2=TILTED[1]))
    assert nrm(hc2, 2.0 * hc1) <= 1e-15
    hd1 = mx.bulk_dmi_field(v, mx.MaterialMap(g, Ms=MS, A=1.3e-11, Db=1e-3))
    hd2 = mx.bulk_dmi_field(v, mx.MaterialMap(g, Ms=MS, A=1.3e-11, Db=-1e-3))
    # interior cells: H is linear in Db (the boundary ghost adds a Db^2 term)
    inner = (slice(None), slice(1, -1), slice(1, -1), slice(1, -1))
    assert nrm(hd2[inner], -hd1[inner]) <= 1e-14
    assert np.all(mx.bulk_dmi_field(v, mx.MaterialMap(g, Ms=MS, A=1.3e-11, Db=0.0)) == 0.0)
    assert np.all(mx.cubic_anisotropy_field(v, mx.MaterialMap(g, Ms=MS, Kc1=0.0)) == 0.0)


def test_bulk_dmi_helix_and_chirality():
    """A Bloch helix along x: the interior curl is -k M (discrete sin(k dx)/dx);
    reversing the handedness or the sign of Db flips the field."""
    n, d, Db, A = 32, 2e-9, 2e-3, 1.3e-11
    g = mx.GridSpec(n, 1, 1, d, d, d)
    k = 2 * np.pi / (n * d)
    x = (np.arange(n) + 0.5) * d
    m = np.zeros((3, 1, 1, n))
    m[1, 0, 0], m[2, 0, 0] = np.cos(k * x), np.sin(k * x)
    mat = mx.MaterialMap(g, Ms=MS, A=A, Db=Db)
    h = mx.bulk_dmi_field(mx.VectorField3(g, m * MS), mat)
    inner = slice(2, n - 2)
    sel = np.abs(m[1, 0, 0, inner]) > 0.5
    ratio = h[1, 0, 0, inner][sel] / (m[1, 0, 0, inner][sel] * MS)
    expect = (2 * Db / (mx.MU0 * MS ** 2)) * (np.sin(k * d) / d + Db / (2 * A))
    assert np.allclose(ratio, expect, rtol=1e-10)
    # chirality: the mirrored helix (opposite handedness) gives the opposite curl part
    mm = m.copy()
    mm[2] = -mm[2]
    hm = mx.bulk_dmi_field(mx.VectorField3(g, mm * MS), mat)
    ratio_m = hm[1, 0, 0, inner][sel] / (mm[1, 0, 0, inner][sel] * MS)
    expect_m = (2 * Db / (mx.MU0 * MS ** 2)) * (-np.sin(k * d) / d + Db / (2 * A))
    assert np.allclose(ratio_m, expect_m, rtol=1e-10)
    # energy: the helix whose handedness matches sign(Db) is lower
    hneg = mx.bulk_dmi_field(mx.VectorField3(g, m * MS), mx.MaterialMap(g, Ms=MS, A=A, Db=-Db))
    e_pos = -np.sum(m[:, 0, 0, inner] * h[:, 0, 0, inner])
    e_neg = -np.sum(m[:, 0, 0, inner] * hneg[:, 0, 0, inner])
    assert e_pos < e_neg


@pytest.mark.parametrize("method", ["rk4", "euler"])
def test_rk_run_with_cubic_and_bulk_dmi_matches_oracle(method):
    dims, cell = (12, 10, 6), (2e-9, 2e-9, 2e-9)
    ms = np.ascontiguousarray(np.broadcast_to(disk_ms(12)[:, :10, :], (6, 10, 12)))
    g = mx.GridSpec(*dims, *cell)
    kw = dict(A=1.3e-11, Ku=2e4, eK=(0.0, 0.3, 1.0), alpha=0.2, Kc1=3e4, c1=TILTED[0], c2=TILTED[1],
              Db=1.5e-3)
    mat = mx.MaterialMap(g, Ms=ms, **kw)
    omat = O.make_mat(dims, cell, ms, **kw)
    m0 = O.renormalize(np.random.default_rng(10).normal(size=(3,) + g.shape), omat)
    packed = O.packed_tensor(*dims, *cell)
    bias = np.array([2e4, 0.0, -1e4])
    rhs = mx.PartitionedRHS(mat, exchange=True, anisotropy=True, cubic=True, bulk_dmi=True,
                            demag=mx.DemagKernel.from_packed(g, packed), bias=bias)
    terms = O.Terms(exchange=True, anisotropy=True, cubic=True, bulk_dmi=True,
                    spectra=O.kernel_spectra(packed), bias=bias)
    got = rhs.rhs_total(0.0, m0)
    ref = O.rhs_total(0.0, m0, omat, terms)
    assert nrm(got, ref) <= 1e-12
    dt = 2e-14
    st = mx.SimState(mx.VectorField3(g, m0.copy()))
    mx.Simulation(st, rhs, mx.IntegratorSpec(method, dt), sample_every=10 ** 9,
                  energy_in_samples=False).run_until(mx.StopCondition(max_steps=8))
    r = O.run(m0, omat, terms, method, dt, max_steps=8)
    assert float(np.max(np.abs(st.m.data - r.m)) / MS) <= 1e-12
