"""demag_field_direct on the GPU (reference demag.py:225-248) and the
reference's FFT == direct-sum test (tests/test_demag.py:62-79) run against
it on B200; the MAGF kernel cache (save_kernel / load_kernel,
demag.py:256-277)."""
import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,cell", [((6, 5, 4), (1e-9, 2e-9, 1.5e-9)), ((9, 7, 3), (2e-9, 2e-9, 2e-9)),
                                       ((16, 16, 1), (1e-9, 1e-9, 0.5e-9))])
def test_direct_sum_bitwise_with_reference_tensor(dims, cell):
    """Same tensor elements, same source order and operation order: bit-identical."""
    g = mx.GridSpec(*dims, *cell)
    m = np.random.default_rng(31).normal(size=(3,) + g.shape) * 8e5
    m[:, 0, 0, :2] = 0.0          # skipped sources
    n6 = O.tensor_elements(*dims, *cell)
    got = mx.demag_field_direct(mx.VectorField3(g, m), g, n6)
    assert np.array_equal(got, O.demag_direct(m, n6))


@pytest.mark.parametrize("dims,cell", [
    ((1, 1, 1), (1e-9, 1e-9, 1e-9)),
    ((2, 2, 2), (1e-9, 1e-9, 1e-9)),
    ((6, 5, 4), (1e-9, 2e-9, 1.5e-9)),
    ((8, 1, 1), (2e-9, 1e-9, 3e-9)),
    ((6, 5, 1), (1.5e-9, 1.5e-9, 1.5e-9)),
    ((8, 8, 8), (1e-9, 1e-9, 1e-9)),
    ((16, 16, 16), (1e-9, 1e-9, 1e-9)),
])
def test_fft_matches_direct_sum(dims, cell):
    """reference tests/test_demag.py:63-79 (same shapes, same 1e-9 bound), plus
    the 4096-cell limit; GPU FFT path (generic and symmetric builds) vs the GPU
    direct sum with the GPU builder's elements."""
    g = mx.GridSpec(*dims, *cell)
    m = mx.VectorField3(g, np.random.default_rng(32).normal(size=(3,) + g.shape) * 8e5)
    h_dir = mx.demag_field_direct(m, g)
    scale = np.max(np.abs(h_dir))
    for k in (mx.DemagKernel.build(g), mx.DemagKernel.build(g, symmetric=True)):
        h_fft = mx.demag_field_fft(m, k)
        assert np.max(np.abs(h_fft - h_dir)) <= 1e-9 * scale
    # and tighter than the reference's bound: observed FFT round-off only
    assert np.max(np.abs(mx.demag_field_fft(m, mx.DemagKernel.build(g)) - h_dir)) <= 1e-13 * scale


def test_kernel_cache_roundtrip(tmp_path):
    g = mx.GridSpec(12, 10, 3, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(33).normal(size=(3,) + g.shape) * 8e5
    for sym in (False, True):
        k = mx.DemagKernel.build(g, symmetric=sym)
        path = tmp_path / mx.kernel_cache_name(g)
        mx.save_kernel(path, k)
        k2 = mx.load_kernel(path, g)
        assert np.max(np.abs(k2.field(m) - k.field(m))) <= 1e-12 * np.max(np.abs(k.field(m)))
    # a reference-format cache (the oracle's packed tensor in MAGF) loads into the parity path
    packed = O.packed_tensor(12, 10, 3, 2e-9, 2.5e-9, 3e-9)
    pz, py, px = packed.shape[1:]
    mx.write_magf(tmp_path / "ref.magf", packed, mx.GridSpec(px, py, pz, 2e-9, 2.5e-9, 3e-9))
    k3 = mx.load_kernel(tmp_path / "ref.magf", g)
    assert np.array_equal(k3._packed, packed)
    ref = O.demag_field(O.kernel_spectra(packed), m)
    assert np.max(np.abs(k3.field(m) - ref)) <= 1e-13 * np.max(np.abs(ref))
    with pytest.raises(mx.MagfError, match="does not match"):
        mx.load_kernel(tmp_path / "ref.magf", mx.GridSpec(12, 10, 3, 2e-9, 2.5e-9, 4e-9))
