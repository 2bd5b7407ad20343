"""Serving metrics of the reference's simulation spec, computed over device steps.

The reference specifies these as simengine operations and
ships no code for them; they are restated here as host arithmetic over the
per-instance latencies, loads and TPOTs that `bench_trace.py` measures on the
B200.

- `imbalance_metrics`  -- SPEC.md:432-439: imbalance = (max - mean) / mean x 100,
  reduction_potential = (max - mean) / max x 100.
- `slo_attainment`     -- SPEC.md:441-447: share of requests whose TPOT meets the SLO.
- `slo_sweep`          -- SPEC.md:449-455: largest grid rate with attainment >= 0.99,
  monotone truncation (the first failing rate ends the sweep).
"""
from __future__ import annotations

from typing import Callable, Iterable, Sequence


def imbalance_from(max_v: float, mean_v: float) -> tuple[float, float]:
    """(imbalance %, reduction potential %) from a max and a mean."""
    if mean_v <= 0.0 or max_v <= 0.0:
        return 0.0, 0.0
    return (max_v - mean_v) / mean_v * 100.0, (max_v - mean_v) / max_v * 100.0


def imbalance_metrics(samples: Sequence[float]) -> tuple[float, float]:
    """SPEC.md:432-439 over a non-empty list of per-instance values."""
    if len(samples) == 0:
        raise ValueError("imbalance_metrics: empty samples")
    mx = max(samples)
    mean = sum(samples) / len(samples)
    return imbalance_from(mx, mean)


def slo_attainment(tpot_ms: Iterable[float], slo_ms: float) -> float:
    """Share of finished requests with TPOT <= slo_ms (1.0 for none finished)."""
    t = list(tpot_ms)
    if not t:
        return 1.0
    return sum(1 for x in t if x <= slo_ms) / len(t)


def slo_sweep(attainment_at: Callable[[float], float], rate_grid: Sequence[float], target: float = 0.99):
    """SPEC.md:449-455.  `attainment_at(rate)` runs one simulation; the sweep stops at the
    first rate below `target`.  Returns (max sustainable rate or None, [(rate, attainment)])."""
    if any(b <= a for a, b in zip(rate_grid, rate_grid[1:])):
        raise ValueError("slo_sweep: rate_grid must be ascending")
    best, points = None, []
    for r in rate_grid:
        a = attainment_at(r)
        points.append((r, a))
        if a < target:
            break
        best = r
    return best, points
