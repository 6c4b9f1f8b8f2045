"""INTEGRATION.md's reference-side ctypes binding (integration/magnex_b200.py)
run on the GPU through the PartitionedRHS(demag=...) plugin seam
(reference llg.py:92-95,119-121), against the oracle."""
import numpy as np
import pytest

import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O

pytestmark = pytest.mark.gpu


class RefKernel:
    """What the binding reads off a reference DemagKernel: .grid and ._packed."""

    def __init__(self, grid, packed):
        self.grid, self._packed = grid, packed


def test_binding_through_the_plugin_seam():
    from integration.magnex_b200 import B200Demag
    dims, cell = (12, 10, 4), (2e-9, 2.5e-9, 3e-9)
    g = mx.GridSpec(*dims, *cell)
    packed = O.packed_tensor(*dims, *cell)
    plugin = B200Demag(RefKernel(g, packed))
    m0 = O.renormalize(np.random.default_rng(41).normal(size=(3,) + g.shape),
                       O.make_mat(dims, cell, 8e5, A=1.3e-11, alpha=0.1))
    spectra = O.kernel_spectra(packed)
    ref = O.demag_field(spectra, m0)
    assert np.max(np.abs(plugin.field(m0) - ref)) <= 1e-13 * np.max(np.abs(ref))
    # the seam: a foreign field() object in the demag slot of PartitionedRHS
    mat = mx.MaterialMap(g, Ms=8e5, A=1.3e-11, alpha=0.1)
    rhs = mx.PartitionedRHS(mat, exchange=True, demag=plugin, bias=(1e4, 0.0, 0.0))
    st = mx.SimState(mx.VectorField3(g, m0.copy()))
    mx.Simulation(st, rhs, mx.IntegratorSpec("rk4", 2e-14), sample_every=10 ** 9,
                  energy_in_samples=False).run_until(mx.StopCondition(max_steps=4))
    omat = O.make_mat(dims, cell, 8e5, A=1.3e-11, alpha=0.1)
    terms = O.Terms(exchange=True, spectra=spectra, bias=np.array([1e4, 0.0, 0.0]))
    r = O.run(m0, omat, terms, "rk4", 2e-14, max_steps=4)
    assert np.max(np.abs(st.m.data - r.m)) <= 1e-12 * 8e5
    assert rhs.counters["demag"] == 16


def test_binding_errors_map_to_exceptions():
    from integration.magnex_b200 import B200Demag
    g = mx.GridSpec(4, 4, 2, 1e-9, 1e-9, 1e-9)
    plugin = B200Demag(RefKernel(g, O.packed_tensor(4, 4, 2, 1e-9, 1e-9, 1e-9)))
    with pytest.raises(ValueError, match="kernel built for"):
        plugin.field(np.zeros((3, 2, 4, 5)))
    with pytest.raises(ValueError):
        B200Demag(RefKernel(mx.GridSpec(0, 4, 2, 1e-9, 1e-9, 1e-9), np.zeros((6, 4, 8, 1))))
