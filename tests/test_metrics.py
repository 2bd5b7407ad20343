"""Serving-metric formulas (acceptance criterion 4) -- host logic, CPU."""
import pytest

from paper_2605_21100_b200 import metrics


def test_ac4_reduction_potential_examples():
    # SPEC.md:437-438 (paper §2.3.1: 65.2% and 65.8%)
    assert metrics.imbalance_from(1020.6, 354.7)[1] == pytest.approx(65.2, abs=0.1)
    assert metrics.imbalance_from(539.5, 184.3)[1] == pytest.approx(65.8, abs=0.1)


def test_imbalance_metrics_samples():
    assert metrics.imbalance_metrics([5.0, 5.0, 5.0]) == (0.0, 0.0)
    imb, red = metrics.imbalance_metrics([1.0, 1.0, 4.0])
    assert imb == pytest.approx(100.0) and red == pytest.approx(50.0)
    with pytest.raises(ValueError):
        metrics.imbalance_metrics([])


def test_slo_attainment():
    assert metrics.slo_attainment([], 50.0) == 1.0
    assert metrics.slo_attainment([10, 20, 60, 30], 50.0) == 0.75


def test_slo_sweep_examples():
    # all sustainable -> last rate; first rate failing -> none
    assert metrics.slo_sweep(lambda r: 1.0, [1, 2, 4])[0] == 4
    assert metrics.slo_sweep(lambda r: 0.5, [1, 2, 4]) == (None, [(1, 0.5)])
    # monotone truncation: a later recovery does not count
    att = {1: 1.0, 2: 0.9, 4: 1.0}
    best, pts = metrics.slo_sweep(att.__getitem__, [1, 2, 4])
    assert best == 1 and pts == [(1, 1.0), (2, 0.9)]
    with pytest.raises(ValueError):
        metrics.slo_sweep(lambda r: 1.0, [2, 1])
