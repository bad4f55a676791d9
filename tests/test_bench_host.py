"""Host-only checks of bench.py's sizing of the oracle sample (the `cpu_baseline` leg and `--impl reference`):
the oracle's time is affine in the slab count, and the sample must land near the time target either way."""
import os
import sys
from types import SimpleNamespace

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("a,b,Id", [(3.5, 0.036, 512),   # c5-like: the fixed cost dominates small samples
                                    (0.0, 0.5, 64),      # proportional
                                    (0.0, 0.002, 128),   # the whole tensor takes less than the target
                                    (20.0, 0.1, 64)])    # one slab already exceeds the target
def test_oracle_sample_calibration_lands_near_the_target(monkeypatch, a, b, Id):
    import bench
    calls = []

    def fake_sample(cfg, seed, slabs, om):
        calls.append(slabs)
        return a + b * slabs, 1.0

    monkeypatch.setattr(bench, "_oracle_sample", fake_sample)
    cfg = SimpleNamespace(dims=(8, 8, Id), name="fake")
    target = 12.0
    slabs = bench._calibrate_slabs(cfg, 0, None, target)
    assert 1 <= slabs <= Id
    t = a + b * slabs
    if a + b * Id <= target:
        assert slabs == Id
    elif a + b >= target:
        assert slabs == 1
    else:
        assert 0.8 * target <= t <= 1.05 * target
    # the calibration itself stays bounded: every probe is at most ~2x the target
    assert all(a + b * s <= 2.0 * target + a for s in calls)


def test_calibration_floor_bounds_a_noisy_pair(monkeypatch):
    import bench
    ts = iter([7.9, 6.9])  # second probe (4x the slabs) reads faster than the first: measured on a busy host

    def fake_sample(cfg, seed, slabs, om):
        return next(ts), 1.0

    monkeypatch.setattr(bench, "_oracle_sample", fake_sample)
    cfg = SimpleNamespace(dims=(8, 8, 512), name="fake")
    slabs = bench._calibrate_slabs(cfg, 0, None, 12.0)
    assert 1 <= slabs < 512 and slabs == int((12.0 - 7.9 * 0.99) / (0.01 * 7.9))
