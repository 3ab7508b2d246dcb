"""Cache-schedule boundary vs the REAL reference's golden vectors (CPU).

tests/golden/plan_cache.json was produced by tests/golden/make_golden.py,
which imports ditplan (the reference) and records plan_cache over a grid,
its ConfigError paths, dit_parallel_latency, composite_speedup, geometry and
FLOP formula outputs.  Both the product (paper_2505_10584_b200.schedule) and
the oracle restatement (oracle/schedule_oracle.py) are checked against it.
The reference's own hot-path tests (pkg/tests/test_inference.py:18-67,
202-221; test_cli.py:86-91; test_acceptance.py:106-111) are restated here.
"""

import json
import os

import pytest
from hypothesis import given
from hypothesis import strategies as st

from oracle import schedule_oracle as so
from paper_2505_10584_b200 import (CACHE_MODES, DEFAULT_CACHED_COST_FRACTION, CacheSchedule, ConfigError,
                                   RelL1Policy, composite_speedup, dit_parallel_latency, front_block_count,
                                   latent_shape, no_cache, plan_cache, token_count, Bucket,
                                   video_token_count)
from paper_2505_10584_b200.errors import DimensionError, PlanningError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plan_cache.json")))


def test_golden_schedules_product_and_oracle():
    assert len(GOLD["plan_cache"]) > 2000
    for case in GOLD["plan_cache"]:
        total, warmup, interval, frac, mode = case["args"]
        s = plan_cache(total, warmup, interval, frac, mode)
        flags = "".join("1" if f else "0" for f in s.per_step_full)
        assert flags == case["per_step_full"], case["args"]
        assert s.full_steps == case["full_steps"] and s.cached_steps == case["cached_steps"]
        assert s.speedup == case["speedup"]  # bit-identical float arithmetic
        assert "".join("1" if f else "0" for f in so.flags(total, warmup, interval)) == case["per_step_full"]
        assert so.speedup(total, warmup, interval, frac) == case["speedup"]


def test_golden_error_paths_and_messages():
    for case in GOLD["plan_cache_errors"]:
        args = case["args"]
        if case["path"] is None:
            plan_cache(*args)
            continue
        with pytest.raises(ConfigError) as ei:
            plan_cache(*args)
        assert ei.value.path == case["path"]
        assert str(ei.value) == case["message"]
        assert isinstance(ei.value, PlanningError)
        assert so.error_path(*args) == case["path"]


def test_default_config1_call_raises_like_reference():
    with pytest.raises(ConfigError) as ei:
        plan_cache(4)
    assert str(ei.value) == GOLD["plan_cache_default_4_error"]


def test_reference_headline_schedule():
    # test_inference.py:18-24 / test_cli.py:86-91 / acceptance #6
    s = plan_cache(50, warmup=10, interval=3, cached_cost_fraction=0.25)
    assert (s.full_steps, s.cached_steps) == (24, 26)
    assert s.speedup == pytest.approx(50 / 30.5)
    assert abs(s.speedup - 1.67) / 1.67 < 0.05
    j = s.to_json()
    assert j["full_steps"] == 24 and j["speedup"] == pytest.approx(1.639, abs=1e-3)
    assert s.as_string() == "FFFFFFFFFFFccFccFccFccFccFccFccFccFccFccFccFccFccF"[:50]


def test_config_schedules():
    assert plan_cache(30).as_string() == "FFFFFFFFFFFccFccFccFccFccFccFc"
    assert plan_cache(30).speedup == pytest.approx(30 / 20.25)
    assert plan_cache(4, 1, 2).as_string() == "FFcF"
    assert all(no_cache(7).per_step_full)


def test_interval_one_and_full_warmup():
    assert plan_cache(50, 10, 1).speedup == 1.0
    s = plan_cache(50, 50, 3)
    assert s.speedup == 1.0 and all(s.per_step_full)
    s = plan_cache(30, 10, 4)
    assert all(s.per_step_full[:10]) and s.per_step_full[10]


@given(steps=st.integers(1, 200), warmup=st.integers(0, 50))
def test_speedup_monotone_in_interval(steps, warmup):
    warmup = min(warmup, steps)
    sp = [plan_cache(steps, warmup, k).speedup for k in range(1, 11)]
    assert all(b >= a - 1e-12 for a, b in zip(sp, sp[1:]))


@given(steps=st.integers(2, 120))
def test_speedup_non_increasing_in_warmup(steps):
    sp = [plan_cache(steps, w, 3).speedup for w in range(0, steps + 1)]
    assert all(b <= a + 1e-12 for a, b in zip(sp, sp[1:]))


def test_parallel_latency_and_composite_golden():
    for case in GOLD["dit_parallel_latency"]:
        lat, thr = dit_parallel_latency(*case["args"])
        assert lat == case["latency"] and thr == case["throughput"]
    assert composite_speedup(*GOLD["composite_speedup"]["args"]) == GOLD["composite_speedup"]["value"]
    with pytest.raises(ConfigError):
        composite_speedup(0.0)
    with pytest.raises(ConfigError):
        dit_parallel_latency(1.0, 0)
    with pytest.raises(ConfigError):
        dit_parallel_latency(1.0, 2, 1, 1.5)


def test_geometry_golden():
    for case in GOLD["geometry"]:
        f, h, w = case["video"]
        assert list(latent_shape(f, h, w)) == case["latent"]
        assert video_token_count(f, h, w) == case["tokens"]
        assert token_count(Bucket(1, f, h, w)).tokens == case["tokens"]
    with pytest.raises(DimensionError):
        latent_shape(18, 480, 832)
    with pytest.raises(DimensionError):
        latent_shape(17, 481, 832)


def test_flops_formula_golden():
    """Our per-step FLOP convention reduces to the reference's for plain joint attention."""

    for case in GOLD["flops_per_microstep"]:
        if case["arch"] != "TABLE2_FIT":
            continue
        S = case["S"]
        H, L = 3072, 54
        # flops_per_microstep: L*(4 S^2 H + 2 S (4H^2 + 8H^2)) + 2 S (2*4*8*H)
        ours = L * (4.0 * S * S * H + 2.0 * S * 12 * H * H) + 2.0 * S * (2 * 32 * H)
        assert ours == pytest.approx(case["value"], rel=1e-12)
    from paper_2505_10584_b200 import MM_DIT_13B, flops_per_step

    f = flops_per_step(MM_DIT_13B, 118800)
    ref = [c["value"] for c in GOLD["flops_per_microstep"] if c["arch"] == "TABLE2_FIT" and c["S"] == 118800 + 256][0]
    assert f["total"] == pytest.approx(ref, rel=1e-3)


def test_front_block_count():
    assert front_block_count(54, 0.25) == 14
    assert front_block_count(28, 0.25) == 7
    assert front_block_count(2, 0.25) == 1
    assert front_block_count(4, 1.0) == 4
    with pytest.raises(ConfigError):
        front_block_count(0, 0.25)


def test_rel_l1_policy_rule():
    pol = RelL1Policy(threshold=0.1, warmup=2)
    acc, flags = 0.0, []
    for s, r in enumerate([0, 0.5, 0.04, 0.04, 0.04, 0.01, 0.2, 0.01], start=1):
        full, acc = pol.decide(s, 8, acc, r)
        flags.append(full)
    assert flags == [True, True, False, False, True, False, True, True]
    sched = pol.as_schedule(flags)
    assert isinstance(sched, CacheSchedule) and sched.full_steps == 5
    assert sched.speedup == pytest.approx(8 / (5 + 3 * DEFAULT_CACHED_COST_FRACTION))
    with pytest.raises(ConfigError):
        RelL1Policy(mode="nope")
    with pytest.raises(ConfigError):
        RelL1Policy(threshold=-1)
    assert CACHE_MODES == ("dit-layer-cache", "attention-cache")
