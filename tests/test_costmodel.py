"""Row f4: CostModel (sim.py:61-106 semantics) and its calibration from bench output."""

import json
import os

import numpy as np
import pytest

from paper_2604_19157_b200.costmodel import CostModel, calibrated_cost_model, fit_decode
from paper_2604_19157_b200.errors import ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cost_model_formulas_and_validation():
    m = CostModel()
    assert m.decode_step_cost(4, 1000) == pytest.approx(2e-2 + 4 * 5e-5 + 1000 * 3e-8)
    assert m.prefill_cost(100) == pytest.approx(5e-3 + 100 * 6e-5)
    # decode_run_cost == the sum of per-step costs as the cache grows by `batch` per step
    steps, batch, cached = 7, 3, 500
    direct = sum(m.decode_step_cost(batch, cached + batch * s) for s in range(steps))
    assert m.decode_run_cost(steps, batch, cached) == pytest.approx(direct)
    with pytest.raises(ConfigError):
        CostModel(decode_base=-1.0)
    with pytest.raises(ConfigError):
        CostModel(decode_base=0.0, decode_per_seq=0.0)


def test_fit_decode_recovers_coefficients():
    base, per_seq, per_tok = 3e-6, 2e-7, 1.5e-10
    pts = [(b, b * L, base + b * per_seq + b * L * per_tok) for b in (1, 4, 16, 64) for L in (4096, 32768)]
    got = fit_decode(pts)
    np.testing.assert_allclose(got, (base, per_seq, per_tok), rtol=1e-9)
    # a coefficient the data drive negative is clamped at 0
    pts = [(b, b * 1000, 1e-5 - 1e-9 * b) for b in (1, 2, 3, 4)]
    assert min(fit_decode(pts)) >= 0.0


def test_calibration_from_committed_bench_line():
    path = os.path.join(ROOT, "profiles", "r01_bench_full.json")
    if not os.path.exists(path):
        pytest.skip("no committed bench line")
    m = calibrated_cost_model(path, layers=32)
    bench = json.loads(open(path).read().strip().splitlines()[-1])
    # the calibrated per-layer model reproduces the measured C3 points within 15 %
    for c in bench["detail"]["c3_concurrency_sweep"]:
        pred = m.decode_step_cost(c["batch"], c["batch"] * c["ctx"]) / 32
        assert abs(pred - c["us"] * 1e-6) <= 0.15 * c["us"] * 1e-6 + 1e-6
    assert m.unfused_rotation_cost == 0.0
