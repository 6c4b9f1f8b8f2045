"""Pin the CPU oracle against golden vectors produced by the reference itself.

Every comparison is bit-exact (np.array_equal): the oracle restates the
reference's operations in the same order with the same numpy/scipy calls.
"""
import hashlib

import numpy as np
import pytest

from oracle import magnex_oracle as O
from tests.golden_io import CASES, load, mat_of, packed_of, terms_of


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=CASES)
def gold(request):
    z = load(request.param)
    mat = mat_of(z)
    spectra = None
    if bool(z["has_demag"]):
        packed = packed_of(z)
        if "packed" in z:
            assert np.array_equal(packed, z["packed"])
        assert sha(packed) == str(z["packed_sha"])
        spectra = O.kernel_spectra(packed)
        assert sha(spectra) == str(z["spectra_sha"])
    return request.param, z, mat, terms_of(z, spectra)


def test_terms_bit_exact(gold):
    name, z, mat, terms = gold
    m0 = z["m0"]
    plan = O.Plan(mat, terms.mode())
    if "h_exchange" in z:
        assert np.array_equal(O.exchange_field(m0, mat, plan), z["h_exchange"])
    if "h_anisotropy" in z:
        assert np.array_equal(O.anisotropy_field(m0, mat), z["h_anisotropy"])
    if "h_dmi" in z:
        assert np.array_equal(O.dmi_field(m0, mat, plan), z["h_dmi"])
    if "h_demag" in z:
        assert np.array_equal(O.demag_field(terms.spectra, m0), z["h_demag"])
    assert np.array_equal(O.h_eff(0.0, m0, mat, terms, plan), z["h_total"])
    assert np.array_equal(O.rhs_total(0.0, m0, mat, terms, plan), z["rhs_total"])


def test_steps_bit_exact(gold):
    name, z, mat, terms = gold
    m0, dt = z["m0"], float(z["dt"])
    plan = O.Plan(mat, terms.mode())

    def f(t, y):
        return O.rhs_total(t, y, mat, terms, plan)

    assert np.array_equal(O.rk4_step(m0, 0.0, dt, f, lambda y: O.renormalize(y, mat)),
                          z["rk4_step"])
    assert np.array_equal(O.euler_step(m0, 0.0, dt, f), z["euler_step"])
    e = O.energies(0.0, m0, mat, terms, plan)
    assert np.array_equal(np.array(e), z["energies"])


def test_trace_bit_exact(gold):
    name, z, mat, terms = gold
    if "trace_m" not in z:
        pytest.skip("no trace")
    n = len(z["trace_t"]) - 1
    r = O.run(z["m0"], mat, terms, str(z["trace_method"]), float(z["dt"]), max_steps=n,
              sample_every=1)
    got = np.array([[row["mx"], row["my"], row["mz"]] for row in r.rows])
    assert np.array_equal(got, z["trace_m"])
    assert np.array_equal(np.array([row["t"] for row in r.rows]), z["trace_t"])
    assert sha(r.m) == str(z["trace_final_sha"])


def test_tensor_known_answers():
    z = load("tensor_known")
    for i in range(5):
        cell = z[f"self_{i}_cell"]
        n6 = O.tensor_elements(1, 1, 1, *cell)[:, 0, 0, 0]
        full = np.array([[n6[0], n6[1], n6[2]], [n6[1], n6[3], n6[4]], [n6[2], n6[4], n6[5]]])
        assert np.array_equal(full, z[f"self_{i}"])
        assert abs(np.trace(full) + 1.0) < 1e-10
    assert np.array_equal(O.tensor_elements(4, 3, 2, 1e-9, 2e-9, 1.5e-9), z["tensor_432"])
    assert np.array_equal(O.tensor_elements(120, 1, 1, 1e-9, 1e-9, 1e-9), z["tensor_chain120"])


def test_sp4_protocol_trace():
    """400 RK4 steps of the SP4 field-1 film with energies in the samples."""
    z = load("sp4_trace")
    mat = O.make_mat((128, 32, 1), (500e-9 / 128, 125e-9 / 32, 3e-9), 8e5, A=1.3e-11,
                     alpha=0.02)
    spectra = O.kernel_spectra(O.packed_tensor(128, 32, 1, 500e-9 / 128, 125e-9 / 32, 3e-9))
    terms = O.Terms(exchange=True, spectra=spectra, bias=np.array([-19576.0, 3422.0, 0.0]))
    r = O.run(z["m0"], mat, terms, "rk4", float(z["dt"]), max_steps=400, sample_every=10,
              with_energies=True)
    assert np.array_equal(np.array([row["mx"] for row in r.rows]), z["mx"])
    assert np.array_equal(np.array([row["e_total"] for row in r.rows]), z["e_total"])
    assert sha(r.m) == str(z["final_sha"])


@pytest.mark.parametrize("name", ["box_6x5x4_all", "film_4x4x1", "disk_16_dmi"])
def test_mri_trace_bit_exact(name):
    """Multirate KW3 (integrators.py:97-128) through the run loop, vs the reference."""
    z = load(name)
    mat = mat_of(z)
    spectra = O.kernel_spectra(packed_of(z)) if bool(z["has_demag"]) else None
    terms = terms_of(z, spectra)
    n = len(z["mri_trace_m"]) - 1
    r = O.run(z["m0"], mat, terms, "mri-kw3", float(z["mri_dt"]), max_steps=n, sample_every=1)
    got = np.array([[row["mx"], row["my"], row["mz"]] for row in r.rows])
    assert np.array_equal(got, z["mri_trace_m"])
    assert np.array_equal(r.m, z["mri_final"])


@pytest.mark.parametrize("method", ["rk4", "euler"])
def test_spatial_time_dependent_bias_run(method):
    """The scenario with a spatial, time-dependent bias expression (reference
    scenario.py:442-465 returns t -> (3,nz,ny,nx)), through the run loop with
    energies in the samples, vs the reference run."""
    from tests.golden_io import spatial_case
    z, mat, dt, bias = spatial_case(method)
    nx, ny, nz = mat.dims
    spectra = O.kernel_spectra(O.packed_tensor(nx, ny, nz, 2e-9, 2e-9, 2e-9))
    terms = O.Terms(exchange=True, anisotropy=True, spectra=spectra, bias=bias)
    r = O.run(z[method + "_m0"], mat, terms, method, dt, max_steps=20, sample_every=1,
              with_energies=True)
    got = np.array([[row["mx"], row["my"], row["mz"]] for row in r.rows])
    assert np.array_equal(got, z[method + "_mean"])
    assert np.array_equal(np.array([row["e_total"] for row in r.rows]), z[method + "_e_total"])
    assert np.array_equal(r.m, z[method + "_final"])


def test_sp4_protocol_head():
    """First 200 field-1 steps of the reference's SP4 coarse protocol
    (bench/std4.py:124-188) from its S-state, sampled like run_std4 (every
    5 steps, energies on), vs the reference's recorded samples."""
    z = load("sp4_protocol")
    d = 3.125e-9
    mat = O.make_mat((160, 40, 1), (d, d, d), 8e5, A=1.3e-11, alpha=0.02)
    spectra = O.kernel_spectra(O.packed_tensor(160, 40, 1, d, d, d))
    terms = O.Terms(exchange=True, spectra=spectra, bias=np.array([-19576.0, 3422.0, 0.0]))
    dt = O.stable_dt(d, 1.3e-11, 8e5)
    r = O.run(z["s_state"], mat, terms, "rk4", dt, max_steps=200, sample_every=5, with_energies=True)
    n = len(r.rows)
    for k in ("t", "mx", "my", "mz", "e_total"):
        assert np.array_equal(np.array([row[k] for row in r.rows]), z[k][:n]), k


def test_bench32_golden():
    """The bench's 32^3 deviation fixture: oracle demag and H_eff vs the reference."""
    z = load("bench_32")
    spectra = O.kernel_spectra(O.packed_tensor(32, 32, 32, 4e-9, 4e-9, 4e-9))
    assert np.array_equal(O.demag_field(spectra, z["m"]), z["h_demag"])
    mat = O.make_mat((32, 32, 32), (4e-9,) * 3, 8e5, A=1.3e-11, Ku=5e4, D=1e-3, alpha=0.1)
    terms = O.Terms(exchange=True, anisotropy=True, dmi=True, spectra=spectra, bias=np.array([1e4, 0.0, 0.0]))
    assert np.array_equal(O.h_eff(0.0, z["m"], mat, terms), z["h_eff"])
