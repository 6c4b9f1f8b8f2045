"""FNO surrogate backend (paper_2602_12242_b200.fno) against the reference
behaviour (magnex/fno.py, pkg/tests/test_fno.py strategy) and the pinned oracle."""
import struct

import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import fno_oracle as FO
from paper_2602_12242_b200 import fno as F
from tests.fno_tables import FNO_CASES, load_case


def small_tensors(width=4, modes=(3, 3), seed=0, zero=False):
    rng = np.random.default_rng(seed)
    m1, m2 = modes

    def real(*shape):
        return np.zeros(shape, np.float32) if zero else (rng.standard_normal(shape) * 0.2).astype(np.float32)

    def cplx(*shape):
        if zero:
            return np.zeros(shape, np.complex64)
        return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * 0.1).astype(np.complex64)

    t = {"lift.weight": real(width, 3), "lift.bias": real(width)}
    for k in range(4):
        t[f"block{k}.spectral.pos"] = cplx(width, width, m1, m2)
        t[f"block{k}.spectral.neg"] = cplx(width, width, m1, m2)
        t[f"block{k}.local.weight"] = real(width, width)
        t[f"block{k}.local.bias"] = real(width)
    t["proj.weight"] = real(3, width)
    t["proj.bias"] = real(3)
    t["norm.in_mean"] = np.zeros(3, np.float32)
    t["norm.in_std"] = np.ones(3, np.float32)
    t["norm.out_mean"] = np.zeros(3, np.float32)
    t["norm.out_std"] = np.ones(3, np.float32)
    return t


def write_model(path, t, activation=F.ACT_GELU, shape=(3, 8, 10), seed=1):
    """Weight file whose parity pair is the oracle's forward pass (f32-stored, as an exporter would)."""
    pin = np.random.default_rng(seed).standard_normal(shape).astype(np.float32)
    pout = FO.infer(FO.as_f64(t), pin.astype(np.float64), activation).astype(np.float32)
    F.write_magw(path, t, parity_in=pin, parity_out=pout, activation=activation)
    return pin, pout


def zero_pair(p, t, **kw):
    F.write_magw(p, t, parity_in=np.zeros((3, 6, 6), np.float32),
                 parity_out=np.zeros((3, 6, 6), np.float32), **kw)


# --- container (CPU) ------------------------------------------------------------------

def test_hand_packed_bytes_round_trip(tmp_path):
    def tensor(name, dims, code, payload):
        b = struct.pack("<H", len(name)) + name.encode() + struct.pack("<B", len(dims))
        return b + b"".join(struct.pack("<Q", d) for d in dims) + struct.pack("<B", code) + payload

    blob = b"MAGW" + struct.pack("<HBBI", 1, F.ACT_RELU, 0, 2)
    blob += tensor("w", (3,), 0, np.array([0.5, -1.0, 2.0], "<f4").tobytes())
    blob += tensor("z", (2, 1), 1, np.array([1.0, -1.0, 0.25, 3.0], "<f4").tobytes())
    blob += tensor("parity_in", (3, 1, 1), 0, np.ones(3, "<f4").tobytes())
    blob += tensor("parity_out", (3, 1, 1), 0, np.zeros(3, "<f4").tobytes())
    p = tmp_path / "a.magw"
    p.write_bytes(blob)
    mf = F.read_magw(p)
    assert mf.activation == F.ACT_RELU and set(mf.tensors) == {"w", "z"}
    assert mf.tensors["z"].dtype == np.complex64
    assert np.array_equal(mf.tensors["z"], np.array([[1 - 1j], [0.25 + 3j]], np.complex64))
    q = tmp_path / "b.magw"
    F.write_magw(q, mf.tensors, parity_in=mf.parity_in, parity_out=mf.parity_out, activation=F.ACT_RELU)
    assert q.read_bytes() == blob


def test_writer_reader_round_trip(tmp_path):
    t = small_tensors(seed=3)
    p = tmp_path / "m.magw"
    zero_pair(p, t, activation=F.ACT_GELU)
    mf = F.read_magw(p)
    assert set(mf.tensors) == set(t)
    for k in t:
        assert mf.tensors[k].dtype == t[k].dtype and np.array_equal(mf.tensors[k], t[k])


def test_framing_errors(tmp_path):
    p = tmp_path / "w.magw"
    p.write_bytes(b"MAGZ" + struct.pack("<HBBI", 1, 0, 0, 0))
    with pytest.raises(F.MagwError, match="magic"):
        F.read_magw(p)
    p.write_bytes(b"MAGW" + struct.pack("<HBBI", 3, 0, 0, 0))
    with pytest.raises(F.MagwError, match="version"):
        F.read_magw(p)
    t = small_tensors(seed=4)
    zero_pair(p, t)
    blob = p.read_bytes()
    for cut in (blob[: len(blob) // 2], blob[:7]):
        p.write_bytes(cut)
        with pytest.raises(F.MagwError, match="truncated"):
            F.read_magw(p)
    p.write_bytes(blob + b"\0")
    with pytest.raises(F.MagwError, match="trailing"):
        F.read_magw(p)


def test_model_validation():
    t = small_tensors(seed=5)
    del t["block2.local.bias"]
    with pytest.raises(F.MagwError, match="block2.local.bias"):
        F.FnoModel.from_tensors(t)
    t = small_tensors(seed=6)
    t["proj.weight"][0, 0] = np.nan
    with pytest.raises(F.MagwError, match="finite"):
        F.FnoModel.from_tensors(t)
    t = small_tensors(seed=6)
    t["norm.out_std"] = np.zeros(3, np.float32)
    with pytest.raises(F.MagwError, match="std"):
        F.FnoModel.from_tensors(t)
    t = small_tensors(seed=6)
    t["block1.spectral.neg"] = t["block1.spectral.neg"][:, :, :2, :]
    with pytest.raises(F.MagwError, match="block1.spectral.neg"):
        F.FnoModel.from_tensors(t)
    with pytest.raises(F.MagwError, match="activation"):
        F.FnoModel.from_tensors(small_tensors(), activation=7)


def test_layout_adapter_and_normalizer():
    rng = np.random.default_rng(0)
    f = rng.standard_normal((3, 2, 5, 4))
    tens = F.LayoutAdapter.to_tensor(f)
    assert tens.shape == (2, 5, 4, 3) and np.array_equal(F.LayoutAdapter.from_tensor(tens), f)
    g = np.zeros((3, 1, 2, 2))
    g[1, 0, 1, 0] = 7.0
    assert F.LayoutAdapter.to_tensor(g)[0, 1, 0, 1] == 7.0
    n = F.ChannelNormalizer([1.0, -2.0, 0.5], [2.0, 0.5, 3.0], [0.1, 0.0, -0.3], [1.5, 2.5, 0.25])
    x = rng.standard_normal((3, 5, 7)) * 10
    eps = np.finfo(np.float64).eps
    assert np.all(np.abs(n.denormalize_in(n.normalize_in(x)) - x) <= eps * (np.abs(x) + np.abs(n.in_mean[:, None, None])))
    with pytest.raises(ValueError, match="std"):
        F.ChannelNormalizer(np.zeros(3), [1.0, 0.0, 1.0], np.zeros(3), np.ones(3))


def test_gelu_host_helper():
    from scipy.special import erf
    x = np.linspace(-6, 6, 101)
    assert np.array_equal(F.gelu(x), 0.5 * x * (1 + erf(x / np.sqrt(2))))
    assert F.gelu(np.array([0.0]))[0] == 0.0


# --- GPU ----------------------------------------------------------------------------------

gpu = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@gpu
@pytest.mark.parametrize("name", FNO_CASES)
def test_gpu_inference_matches_reference_golden(name):
    t, z = load_case(name)
    model = F.FnoModel.from_tensors(t, activation=int(z["activation"]))
    y = model.infer(z["x"])
    assert rel(y, z["y"]) <= 1e-12
    assert np.array_equal(model.infer(z["x"]), y)          # deterministic


@gpu
@pytest.mark.parametrize("name", ["small_gelu", "small_relu"])
def test_gpu_spectral_conv_matches_reference_golden(name):
    t, z = load_case(name)
    f = FO.as_f64(t)
    sc = F.spectral_conv(z["v"], f["block0.spectral.pos"], f["block0.spectral.neg"])
    assert rel(sc, z["sc"]) <= 1e-12


@gpu
def test_spectral_conv_properties():
    rng = np.random.default_rng(1)
    c, m1, m2, H, W = 3, 3, 2, 12, 10
    eye = np.zeros((c, c, m1, m2), complex)
    for i in range(c):
        eye[i, i] = 1.0
    v = rng.standard_normal((c, H, W))
    vf = np.fft.rfft2(v)
    mask = np.zeros_like(vf)
    mask[:, :m1, :m2] = vf[:, :m1, :m2]
    mask[:, -m1:, :m2] = vf[:, -m1:, :m2]
    assert np.max(np.abs(F.spectral_conv(v, eye, eye) - np.fft.irfft2(mask, s=(H, W)))) <= 1e-13 * np.max(np.abs(v))
    # energy above the retained modes is removed
    hf = np.zeros((2, 16, 9), complex)
    hf[:, 5, 6] = 4.0 + 1.0j
    hf[:, 9, 4] = -2.0
    hi = np.fft.irfft2(hf, s=(16, 16))
    wp = rng.standard_normal((2, 2, 3, 3)) + 1j * rng.standard_normal((2, 2, 3, 3))
    wn = rng.standard_normal((2, 2, 3, 3)) + 1j * rng.standard_normal((2, 2, 3, 3))
    assert np.max(np.abs(F.spectral_conv(hi, wp, wn))) < 1e-12 * np.max(np.abs(hi))
    # linear
    x, y = rng.standard_normal((2, 2, 10, 12))
    lhs = F.spectral_conv(0.7 * x - 1.9 * y, wp, wn)
    rhs = 0.7 * F.spectral_conv(x, wp, wn) - 1.9 * F.spectral_conv(y, wp, wn)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-14)
    with pytest.raises(F.MagwError, match="spectral extent"):
        F.spectral_conv(np.zeros((2, 8, 8)), np.zeros((2, 2, 12, 12), complex), np.zeros((2, 2, 12, 12), complex))


@gpu
def test_inference_semantics():
    t = small_tensors(zero=True)
    t["norm.out_mean"] = np.array([3.0, -1.5, 0.25], np.float32)
    t["norm.out_std"] = np.array([2.0, 2.0, 2.0], np.float32)
    out = F.FnoModel.from_tensors(t).infer(np.random.default_rng(0).standard_normal((3, 8, 10)))
    for ch in range(3):
        assert np.all(out[ch] == np.float64(t["norm.out_mean"][ch]))
    model = F.FnoModel.from_tensors(small_tensors(seed=10))
    x = np.random.default_rng(4).standard_normal((3, 8, 10))
    assert rel(model.infer(2 * x), 2 * model.infer(x)) > 1e-6          # not linear
    tr = small_tensors(seed=11)
    a = F.FnoModel.from_tensors(tr, activation=F.ACT_GELU).infer(x)
    b = F.FnoModel.from_tensors(tr, activation=F.ACT_RELU).infer(x)
    assert np.max(np.abs(a - b)) > 1e-9
    assert rel(b, FO.infer(FO.as_f64(tr), x, F.ACT_RELU)) <= 1e-12
    # unfrozen weights edited between calls are picked up
    m = F.FnoModel.from_tensors(small_tensors(seed=12))
    y0 = m.infer(x)
    m.proj_b[0] += 1.0
    assert np.allclose(m.infer(x)[0] - y0[0], 1.0, rtol=0, atol=1e-12)


@gpu
def test_parity_pair_gates_loading(tmp_path):
    t = small_tensors(seed=7)
    p = tmp_path / "m.magw"
    write_model(p, t)
    model = F.load_model(p)
    assert model.width == 4 and model.modes == (3, 3)
    with pytest.raises(ValueError):
        model.lift_w[0, 0] = 1.0                                       # frozen
    pin = np.random.default_rng(1).standard_normal((3, 8, 10)).astype(np.float32)
    F.write_magw(p, t, parity_in=pin, parity_out=np.zeros((3, 8, 10), np.float32))
    with pytest.raises(F.MagwError, match="parity"):
        F.load_model(p)


@gpu
def test_backend_wrappers_and_solver_plugin(tmp_path):
    grid = mx.GridSpec(10, 8, 1, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(grid, Ms=8e5, A=1.3e-11, alpha=0.1)
    p = tmp_path / "m.magw"
    write_model(p, small_tensors(seed=15))
    backend = F.FnoDemag.load(p, mat)
    m = mx.VectorField3(grid, np.random.default_rng(6).standard_normal((3, 1, 8, 10)))
    h = F.infer_demag(m, backend.model)
    assert isinstance(h, mx.VectorField3) and h.data.shape == (3, 1, 8, 10)
    assert np.array_equal(h.data[:, 0], backend.model.infer(m.data[:, 0]))
    assert np.array_equal(backend.field(m.data), h.data)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=backend)
    mu = mx.VectorField3.from_uniform(grid, (8e5, 0.0, 0.0))
    dm = rhs.rhs_total(0.0, mu.data)
    assert dm.shape == (3, 1, 8, 10) and np.all(np.isfinite(dm)) and rhs.counters["demag"] == 1
    with pytest.raises(F.MagwError, match="nz = 1"):
        F.infer_demag(mx.VectorField3.from_uniform(mx.GridSpec(10, 8, 2, 3e-9, 3e-9, 3e-9), (1, 0, 0)),
                      backend.model)
    small = mx.GridSpec(4, 4, 1, 3e-9, 3e-9, 3e-9)
    with pytest.raises(F.MagwError, match="spectral extent"):
        F.FnoDemag.load(p, mx.MaterialMap(small, Ms=8e5))


@gpu
def test_surrogate_runs_inside_the_device_loop(tmp_path):
    """A loaded (frozen) FnoDemag is evaluated inside the fused device step
    (mxb_demag_create_fno: the forward pass on the solver stream, captured in
    the step graph) instead of from the host per stage; the trajectory equals
    the host-orchestrated plug-in run (field() per stage, integrators.py)."""
    from paper_2602_12242_b200.fno import _FnoKernel
    grid = mx.GridSpec(32, 16, 1, 3e-9, 3e-9, 3e-9)
    mat = mx.MaterialMap(grid, Ms=8e5, A=1.3e-11, alpha=0.1)
    p = tmp_path / "m.magw"
    t = small_tensors(seed=16)
    write_model(p, t)
    backend = F.FnoDemag.load(p, mat)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=backend, bias=(2e4, 0.0, 0.0))
    assert isinstance(rhs._demag_dev, _FnoKernel) and rhs._device_ok()
    m0 = np.random.default_rng(7).standard_normal((3, 1, 16, 32))
    m0 = mx.VectorField3(grid, m0)
    mx.renormalize(m0, mat)
    # device evaluation == the plug-in's host evaluation
    assert np.max(np.abs(rhs.h_total_quiet(0.0, m0.data) - (
        mx.exchange_field(m0, mat) + backend.field(m0.data) + np.array([2e4, 0, 0])[:, None, None, None]))) \
        <= 1e-12 * 8e5
    st = mx.SimState(m0.copy())
    tr = mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 2e-14), sample_every=5,
                       energy_in_samples=False).run_until(mx.StopCondition(max_steps=20))
    # the host-orchestrated reference: the same backend through a plain callable (no device kernel)
    rhs_h = mx.PartitionedRHS(mat, exchange=True, demag=lambda md: backend.field(md), bias=(2e4, 0.0, 0.0))
    assert not rhs_h._device_ok()
    st_h = mx.SimState(m0.copy())
    tr_h = mx.Simulation(st_h, rhs_h, mx.IntegratorSpec("rk4", 2e-14), sample_every=5,
                         energy_in_samples=False).run_until(mx.StopCondition(max_steps=20))
    assert np.max(np.abs(st.m.data - st_h.m.data)) <= 1e-12 * 8e5
    for k in ("mx", "my", "mz"):
        assert np.max(np.abs(tr.column(k) - tr_h.column(k))) <= 1e-12
    assert tr.counters["demag"] == tr_h.counters["demag"] == 80


@gpu
@pytest.mark.parametrize("width,modes,H,W", [(4, (3, 3), 24, 200), (32, (12, 12), 40, 260), (8, (5, 7), 33, 129)])
def test_blocked_passes_odd_shapes_match_oracle(width, modes, H, W):
    """The blocked x-DFT (table chunks of 128 x values) and the fused block
    output (128-column tiles) on widths that are not multiples of the chunk,
    row counts that are not multiples of the 8 rows per CTA, odd H: against the
    oracle restatement (oracle/fno_oracle.py, pinned to the reference)."""
    from oracle import fno_oracle as FO
    from tests.fno_tables import tensors
    t = tensors(width, modes, 31)
    model = F.FnoModel.from_tensors(t).freeze()
    x = np.random.default_rng(32).standard_normal((3, H, W))
    y = model.infer(x)
    ref = FO.infer(t, x, model.activation)
    assert rel(y, ref) <= 1e-12
