"""Generate golden vectors from the REAL reference (``ditplan``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py

It imports ``ditplan`` from ``/root/reference/pkg/src`` and records:
* ``plan_cache`` outputs over a parameter grid plus the ConfigError paths of
  invalid inputs (``inference.py:48-86``);
* ``dit_parallel_latency`` / ``composite_speedup`` (``inference.py:282-315``);
* ``latent_shape`` / ``token_count`` for the BASELINE geometries
  (``buckets.py:65-98``);
* ``flops_per_microstep`` for the reference's ``TABLE2_FIT`` model
  (``simulate.py:60-73``).
The committed JSON is what the CPU tests (and the GPU box) read; the GPU box
never reads ``/root/reference``.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plan_cache.json")


def main():
    sys.path.insert(0, REF)
    import ditplan  # noqa: F401
    from ditplan.buckets import Bucket, latent_shape, token_count
    from ditplan.config import ModelArch
    from ditplan.errors import ConfigError
    from ditplan.inference import composite_speedup, dit_parallel_latency, plan_cache
    from ditplan.presets import TABLE2_FIT
    from ditplan.simulate import flops_per_microstep

    cases = []
    for total in (1, 2, 3, 4, 7, 10, 17, 30, 50, 64, 100):
        for warmup in sorted({0, 1, 2, 3, 5, 10, total // 2, total}):
            for interval in (1, 2, 3, 4, 5, 7):
                for frac in (0.25, 0.1, 1.0):
                    for mode in ("dit-layer-cache", "attention-cache"):
                        if warmup > total:
                            continue
                        s = plan_cache(total, warmup, interval, frac, mode)
                        cases.append({
                            "args": [total, warmup, interval, frac, mode],
                            "per_step_full": "".join("1" if f else "0" for f in s.per_step_full),
                            "full_steps": s.full_steps,
                            "cached_steps": s.cached_steps,
                            "speedup": s.speedup,
                        })
    errors = []
    bad = [
        (50, 10, 3, 0.25, "bogus"), (0, 0, 3, 0.25, "dit-layer-cache"), (-1, 0, 1, 0.5, "bogus"),
        (4, 10, 3, 0.25, "dit-layer-cache"), (50, -1, 3, 0.25, "dit-layer-cache"),
        (50, 51, 3, 0.25, "dit-layer-cache"), (50, 10, 0, 0.25, "dit-layer-cache"),
        (50, 10, 3, 0.0, "dit-layer-cache"), (50, 10, 3, 1.5, "dit-layer-cache"),
        (50, 10, 0, 0.0, "dit-layer-cache"), (5, 6, 0, 0.0, "attention-cache"),
    ]
    for args in bad:
        try:
            plan_cache(*args)
            errors.append({"args": list(args), "path": None, "message": None})
        except ConfigError as e:
            errors.append({"args": list(args), "path": e.path, "message": str(e)})
    # default-argument call of config 1 (4 steps) raises
    try:
        plan_cache(4)
        default4 = None
    except ConfigError as e:
        default4 = str(e)

    parallel = []
    for ms, tp, nodes, eff in ((1000.0, 1, 1, 0.85), (1000.0, 8, 1, 0.85), (8000.0, 8, 2, 0.85),
                               (123.0, 4, 3, 0.9), (50.0, 2, 1, 1.0)):
        lat, thr = dit_parallel_latency(ms, tp, nodes, eff)
        parallel.append({"args": [ms, tp, nodes, eff], "latency": lat, "throughput": thr})
    comp = {"args": [1.639, 1.43], "value": composite_speedup(1.639, 1.43)}

    geometry = []
    for f, h, w in ((17, 480, 832), (61, 480, 848), (129, 720, 1280), (125, 720, 1280), (5, 64, 64),
                    (29, 640, 640), (1, 256, 256)):
        ls = latent_shape(f, h, w)
        tc = token_count(Bucket(1, f, h, w))
        geometry.append({"video": [f, h, w], "latent": list(ls), "tokens": tc.tokens})

    flops = []
    for S in (48, 7800, 25440 + 256, 115200, 118800 + 256):
        flops.append({"arch": "TABLE2_FIT", "S": S, "value": flops_per_microstep(TABLE2_FIT, 1, S)})
    arch2b = ModelArch(hidden_size=2048, num_heads=16, num_layers=28, adaln_mode="shared-weights")
    flops.append({"arch": "2B", "S": 7800, "value": flops_per_microstep(arch2b, 1, 7800)})

    doc = {
        "source": "ditplan (reference) imported from /root/reference/pkg/src by tests/golden/make_golden.py",
        "plan_cache": cases,
        "plan_cache_errors": errors,
        "plan_cache_default_4_error": default4,
        "dit_parallel_latency": parallel,
        "composite_speedup": comp,
        "geometry": geometry,
        "flops_per_microstep": flops,
    }
    with open(OUT, "w") as fh:
        json.dump(doc, fh, sort_keys=True)
    print(f"wrote {OUT}: {len(cases)} schedules, {len(errors)} error cases")


if __name__ == "__main__":
    main()
