"""Row f4: the serving simulator's engine-step cost model, calibrated with this
package's measured B200 kernel costs.

`CostModel` keeps the reference's fields, validation and formulas
(sim.py:61-106): decode step = base + batch * per_seq + cached_tokens *
per_cached_token, prefill = base + tokens * per_token, plus the unfused-rotation
surcharge.  `calibrated_cost_model` fills the attention-cache share of those
coefficients from a `bench.py` JSON line (profiles/*_bench_full.json): a least
squares fit of the fused append + decode step over the C2 point and the C3 batch
sweep, and the K1 write per token from C1, times the model's layer count.  The
GEMMs and everything else in an engine step are not in these kernels; pass
them as `extra` (seconds per step / per prefill token) when known.  The fused
write has no unfused rotation pass, so that surcharge is 0.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigError


@dataclass(frozen=True)
class CostModel:
    """Engine step costs in seconds (sim.py:61-106)."""

    prefill_base: float = 5e-3
    prefill_per_token: float = 6e-5
    decode_base: float = 2e-2
    decode_per_seq: float = 5e-5
    decode_per_cached_token: float = 3e-8
    unfused_rotation_cost: float = 0.0

    def __post_init__(self) -> None:
        if min(self.prefill_base, self.prefill_per_token, self.decode_base, self.decode_per_seq,
               self.decode_per_cached_token, self.unfused_rotation_cost) < 0:
            raise ConfigError("cost coefficients must be >= 0")
        if self.decode_base <= 0 and self.decode_per_seq <= 0:
            raise ConfigError("decode step cost must be positive")

    def prefill_cost(self, tokens: int) -> float:
        return self.prefill_base + tokens * (self.prefill_per_token + self.unfused_rotation_cost)

    def decode_step_cost(self, batch: int, cached_tokens: int) -> float:
        return (self.decode_base + batch * (self.decode_per_seq + self.unfused_rotation_cost)
                + cached_tokens * self.decode_per_cached_token)

    def decode_run_cost(self, steps: int, batch: int, cached_tokens: int) -> float:
        """Cost of `steps` lockstep steps; the cache grows by batch per step."""
        return steps * (self.decode_base + batch * (self.decode_per_seq + self.unfused_rotation_cost)) + (
            self.decode_per_cached_token * (steps * cached_tokens + batch * steps * (steps - 1) // 2))


def fit_decode(points) -> tuple[float, float, float]:
    """Non-negative least squares of t = base + batch * per_seq + cached * per_token
    over (batch, cached_tokens, seconds) points (coefficients clamped at 0 and the
    rest refit)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3 or len(pts) < 3:
        raise ConfigError("need at least three (batch, cached_tokens, seconds) points")
    a = np.column_stack([np.ones(len(pts)), pts[:, 0], pts[:, 1]])
    y = pts[:, 2]
    active = [0, 1, 2]
    while True:
        coef = np.zeros(3)
        sol, *_ = np.linalg.lstsq(a[:, active], y, rcond=None)
        coef[active] = sol
        neg = [j for j in active if coef[j] < 0]
        if not neg:
            return float(coef[0]), float(coef[1]), float(coef[2])
        active = [j for j in active if j not in neg]
        if not active:
            return 0.0, 0.0, 0.0


def calibrated_cost_model(bench, layers: int = 32, extra_decode_step: float = 0.0,
                          extra_prefill_per_token: float = 0.0, prefill_base: Optional[float] = None) -> CostModel:
    """CostModel from a bench.py JSON line (dict or path) for a `layers`-layer model
    of the bench's attention shape (C2/C3: 32 q / 8 kv heads, d 128)."""
    if not isinstance(bench, dict):
        with open(bench) as f:
            bench = json.loads(f.read().strip().splitlines()[-1])
    det = bench["detail"]
    pts = [(1, bench["config"]["ctx"] + 1, det["fused_step_us"] * 1e-6)]
    for c in det["c3_concurrency_sweep"]:
        pts.append((c["batch"], c["batch"] * c["ctx"], c["us"] * 1e-6))
    base, per_seq, per_tok = fit_decode(pts)
    c1 = det["c1_quantize_store"]
    write_per_token = c1["rot_us"] * 1e-6 / c1["tokens"]
    return CostModel(prefill_base=prefill_base if prefill_base is not None else base * layers,
                     prefill_per_token=write_per_token * layers + extra_prefill_per_token,
                     decode_base=base * layers + extra_decode_step,
                     decode_per_seq=per_seq * layers,
                     decode_per_cached_token=per_tok * layers,
                     unfused_rotation_cost=0.0)
