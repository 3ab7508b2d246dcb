"""Diffusion-cache schedules — the drop-in boundary of the hot path.

``plan_cache`` / ``CacheSchedule`` keep the reference signature, validation
order, error paths and arithmetic of ``ditplan.inference.plan_cache``
(``pkg/src/ditplan/inference.py:21-86``) so that a caller of the reference
can switch imports unchanged.  The returned ``per_step_full`` tuple is what
:func:`paper_2505_10584_b200.sampler.denoise` consumes, unchanged.

New on top of the reference (the north_star asks for it, the reference has
no equivalent — SURVEY.md §0 contradiction 3):

* :class:`RelL1Policy` — a TeaCache-style data-dependent policy: the
  relative-L1 change of block 0's modulated input, accumulated across steps,
  decides full vs cached on device.  After a run, the flags actually taken
  are reported as a ``CacheSchedule``-shaped record
  (:meth:`RelL1Policy.as_schedule`).
* :func:`front_block_count` — how many front blocks still run on a cached
  step: ``ceil(cached_cost_fraction * num_layers)``.

``dit_parallel_latency`` / ``composite_speedup`` restate
``inference.py:282-315`` (the reference's reporting formulas).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ConfigError

# inference.py:21
CACHE_MODES = ("dit-layer-cache", "attention-cache")

# inference.py:23-26 — fitted so that 50/10/3 gives ~1.67x.
DEFAULT_CACHED_COST_FRACTION = 0.25


@dataclass(frozen=True)
class CacheSchedule:
    """Frozen schedule record (``inference.py:29-45``)."""

    total_steps: int
    warmup: int
    interval: int
    mode: str
    cached_cost_fraction: float
    per_step_full: tuple[bool, ...]
    speedup: float

    @property
    def full_steps(self) -> int:
        return sum(self.per_step_full)

    @property
    def cached_steps(self) -> int:
        return self.total_steps - self.full_steps

    def as_string(self) -> str:
        """``F``/``c`` per step, e.g. ``FFcF`` — used in bench/test output."""
        return "".join("F" if f else "c" for f in self.per_step_full)

    def to_json(self) -> dict:
        """Same keys and rounding as the reference CLI (``cli.py:135-145``)."""
        return {
            "total_steps": self.total_steps,
            "warmup": self.warmup,
            "interval": self.interval,
            "mode": self.mode,
            "cached_cost_fraction": self.cached_cost_fraction,
            "full_steps": self.full_steps,
            "cached_steps": self.cached_steps,
            "speedup": round(self.speedup, 3),
            "per_step_full": [int(f) for f in self.per_step_full],
        }


def plan_cache(
    total_steps: int,
    warmup: int = 10,
    interval: int = 3,
    cached_cost_fraction: float = DEFAULT_CACHED_COST_FRACTION,
    mode: str = "dit-layer-cache",
) -> CacheSchedule:
    """Full warmup, then one refresh every ``interval`` steps (``inference.py:48-86``).

    Step ``s`` (1-based) is full iff ``s <= warmup`` or
    ``(s - warmup - 1) % interval == 0``; a cached step costs
    ``cached_cost_fraction`` of a full one; ``speedup = total / sum(cost)``.
    Validation order and ``ConfigError`` paths follow ``inference.py:61-70``.
    """
    if mode not in CACHE_MODES:
        raise ConfigError(f"mode must be one of {CACHE_MODES}", "cache.mode")
    if total_steps < 1:
        raise ConfigError("total_steps must be >= 1", "cache.total_steps")
    if not 0 <= warmup <= total_steps:
        raise ConfigError("warmup must be in [0, total_steps]", "cache.warmup")
    if interval < 1:
        raise ConfigError("interval must be >= 1", "cache.interval")
    if not 0.0 < cached_cost_fraction <= 1.0:
        raise ConfigError("cached_cost_fraction must be in (0, 1]", "cache.cached_cost_fraction")
    flags = tuple(
        True if s <= warmup else (s - warmup - 1) % interval == 0
        for s in range(1, total_steps + 1)
    )
    cost = sum(1.0 if full else cached_cost_fraction for full in flags)
    return CacheSchedule(
        total_steps=total_steps,
        warmup=warmup,
        interval=interval,
        mode=mode,
        cached_cost_fraction=cached_cost_fraction,
        per_step_full=flags,
        speedup=total_steps / cost,
    )


def no_cache(total_steps: int) -> CacheSchedule:
    """Cache off: every step full (``plan_cache(total, warmup=total)``)."""
    return plan_cache(total_steps, warmup=total_steps)


def front_block_count(num_layers: int, cached_cost_fraction: float) -> int:
    """Blocks that still run on a cached ``dit-layer-cache`` step.

    ``ceil(fraction * L)`` — e.g. 14 of 54 (13.4B), 7 of 28 (2B), 1 of 2
    (tiny).  The reference only costs a cached step at ``fraction`` of a full
    one (``inference.py:77``); the paper reuses the rear blocks' output
    offset (``PAPER.md:309``).  Builder choice, documented in DESIGN.md.
    """
    if num_layers < 1:
        raise ConfigError("num_layers must be >= 1", "model.num_layers")
    if not 0.0 < cached_cost_fraction <= 1.0:
        raise ConfigError("cached_cost_fraction must be in (0, 1]", "cache.cached_cost_fraction")
    return max(1, min(num_layers, math.ceil(cached_cost_fraction * num_layers - 1e-9)))


@dataclass(frozen=True)
class RelL1Policy:
    """Data-dependent (TeaCache-style) cache policy — new work, no reference.

    At every step the device reduces ``rel = sum|m_t - m_{t-1}| / sum|m_{t-1}|``
    over block 0's modulated input ``m``; ``acc += rel``.  Step ``s`` is full
    when ``s <= warmup`` (and always at ``s == 1``), when ``force_last`` and
    ``s == total_steps``, or when ``acc >= threshold``; a full step resets
    ``acc = 0``.  Otherwise the step is cached.  The decision is taken on
    device (no host round-trip); under sequence parallelism the two partial
    sums are all-reduced first so every rank decides identically.
    """

    threshold: float = 0.1
    warmup: int = 1
    force_last: bool = True
    cached_cost_fraction: float = DEFAULT_CACHED_COST_FRACTION
    mode: str = "dit-layer-cache"

    def __post_init__(self):
        if self.mode not in CACHE_MODES:
            raise ConfigError(f"mode must be one of {CACHE_MODES}", "cache.mode")
        if not self.threshold >= 0.0:
            raise ConfigError("threshold must be >= 0", "cache.threshold")
        if self.warmup < 0:
            raise ConfigError("warmup must be >= 0", "cache.warmup")
        if not 0.0 < self.cached_cost_fraction <= 1.0:
            raise ConfigError("cached_cost_fraction must be in (0, 1]", "cache.cached_cost_fraction")

    def decide(self, step: int, total_steps: int, acc: float, rel: float) -> tuple[bool, float]:
        """Host statement of the device rule: ``(full, new_acc)`` for 1-based ``step``."""
        if step <= max(1, self.warmup) or (self.force_last and step == total_steps):
            return True, 0.0
        acc = acc + rel
        if acc >= self.threshold:
            return True, 0.0
        return False, acc

    def as_schedule(self, flags) -> CacheSchedule:
        """The flags a run actually took, as a ``CacheSchedule`` record."""
        flags = tuple(bool(f) for f in flags)
        total = len(flags)
        if total < 1:
            raise ConfigError("total_steps must be >= 1", "cache.total_steps")
        cost = sum(1.0 if f else self.cached_cost_fraction for f in flags)
        return CacheSchedule(
            total_steps=total,
            warmup=min(self.warmup, total),
            interval=0,
            mode=self.mode,
            cached_cost_fraction=self.cached_cost_fraction,
            per_step_full=flags,
            speedup=total / cost,
        )


def dit_parallel_latency(
    single_device_step_ms: float,
    tp_degree: int,
    nodes: int = 1,
    tp_efficiency: float = 0.85,
) -> tuple[float, float]:
    """(latency ms, throughput videos/s) — ``inference.py:282-300``."""
    if tp_degree < 1 or nodes < 1:
        raise ConfigError("degrees must be >= 1", "infer.parallel")
    if not 0.0 < tp_efficiency <= 1.0:
        raise ConfigError("tp_efficiency must be in (0, 1]", "infer.tp_efficiency")
    scale = tp_degree * tp_efficiency if tp_degree > 1 else 1.0
    latency = single_device_step_ms / scale
    return (latency, nodes * 1e3 / latency)


def composite_speedup(*factors: float) -> float:
    """Product of independent speedup factors — ``inference.py:303-315``."""
    out = 1.0
    for factor in factors:
        if factor <= 0:
            raise ConfigError("speedup factors must be positive", "infer.speedup")
        out *= factor
    return out
