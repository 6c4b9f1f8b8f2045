"""Pin the FNO oracle (oracle/fno_oracle.py) bit-exactly against outputs of the
reference magnex/fno.py (tests/golden/make_golden_fno.py)."""
import numpy as np
import pytest

from oracle import fno_oracle as FO
from tests.fno_tables import FNO_CASES, load_case


@pytest.mark.parametrize("name", FNO_CASES)
def test_oracle_infer_bit_exact(name):
    t, z = load_case(name)
    y = FO.infer(FO.as_f64(t), z["x"], int(z["activation"]))
    assert np.array_equal(y, z["y"])


@pytest.mark.parametrize("name", ["small_gelu", "small_relu"])
def test_oracle_spectral_conv_bit_exact(name):
    t, z = load_case(name)
    f = FO.as_f64(t)
    assert np.array_equal(FO.spectral_conv(z["v"], f["block0.spectral.pos"], f["block0.spectral.neg"]), z["sc"])
