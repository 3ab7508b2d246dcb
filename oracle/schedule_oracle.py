"""Restatement of ``ditplan.inference.plan_cache`` — TEST INFRASTRUCTURE.

Follows ``pkg/src/ditplan/inference.py:48-86`` (validation :61-70, flag rule
:71-76, cost :77).  Pinned against ``tests/golden/plan_cache.json``, which
``tests/golden/make_golden.py`` produced by importing the real reference.
Written independently of the product's ``schedule.py`` so that the product
is checked against two sources: this restatement and the golden vectors.
"""

from __future__ import annotations

MODES = ("dit-layer-cache", "attention-cache")


def flags(total_steps: int, warmup: int, interval: int):
    """``per_step_full`` for 1-based step s: s <= warmup, or (s-warmup-1) % interval == 0."""
    out = []
    for s in range(1, total_steps + 1):
        out.append(s <= warmup or (s - warmup - 1) % interval == 0)
    return tuple(out)


def error_path(total_steps, warmup, interval, fraction, mode):
    """The ConfigError path the reference raises first, or None (inference.py:61-70)."""
    if mode not in MODES:
        return "cache.mode"
    if total_steps < 1:
        return "cache.total_steps"
    if not (0 <= warmup <= total_steps):
        return "cache.warmup"
    if interval < 1:
        return "cache.interval"
    if not (0.0 < fraction <= 1.0):
        return "cache.cached_cost_fraction"
    return None


def speedup(total_steps, warmup, interval, fraction):
    f = flags(total_steps, warmup, interval)
    return total_steps / sum(1.0 if x else fraction for x in f)


def rel_l1_decide(step: int, total_steps: int, acc: float, rel: float, threshold: float, warmup: int,
                  force_last: bool) -> tuple[bool, float]:
    """The data-dependent cache rule (TeaCache-style; new work), restated here
    independently of the product's ``RelL1Policy.decide`` and of its device kernel
    (``aqb_cache_decide``): step ``s`` (1-based) is full when ``s <= max(1, warmup)``, when
    ``force_last`` and ``s == total_steps``, or when the accumulated relative-L1 change
    ``acc + rel`` reaches ``threshold``; a full step resets the accumulator.  Returns
    ``(full, new_acc)``."""
    if step <= max(1, warmup):
        return True, 0.0
    if force_last and step == total_steps:
        return True, 0.0
    acc += rel
    if acc >= threshold:
        return True, 0.0
    return False, acc
