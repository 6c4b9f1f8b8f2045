"""bench.py's contract on CPU: the SURVEY 8(d) fixed formulas it reports the
roofline and FP64 rates with, and the JSON line of the reference arm (the
oracle port on the host cores, a tiny sample here)."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _G:
    nx = ny = nz = 512
    n_cells = 512 ** 3


class _K:
    padded = (1024, 1024, 1024)
    symmetric = True


def test_survey_formulas_at_512():
    pb = bench.demag_bytes(_G, _K)
    # 109.7 GB per evaluation, 3,774 B per cell-step with 504 B of stencil
    assert abs(sum(pb) / 1e9 - 109.7) < 0.05
    assert abs((504 * _G.n_cells + 4 * sum(pb)) / _G.n_cells - 3774) < 1.0
    # the implementation reads the parity-reduced quarter kernel instead (6.5 GB)
    own = bench.demag_bytes(_G, _K, survey=False)
    assert abs((sum(pb) - sum(own)) / 1e9 - (25.83 - 6.50)) < 0.05
    # 302 GFLOP per evaluation
    assert abs(sum(bench.demag_flops(_G, _K)) / 1e9 - 301.7) < 0.1


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--cpu-n", "12"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "cell-steps/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
