"""Golden vectors for the VAE tile plan and the temporal MultiDiffusion windows,
generated from the REAL reference (``ditplan.inference``, ``inference.py:89-279``).

    python tests/golden/make_golden_tiling.py      (build container only)

Records, per case: the tiles (start, size, device), parallel_speedup, the raw
tile profile, the total weight and every normalised weight map at a fixed
sample of positions (exact float64 values), the ConfigError paths/messages of
invalid inputs; and for windows: clips, multiplicities and averaging weights.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tiling.json")


def sample_positions(shape, k=48, seed=0):
    rng = np.random.default_rng(seed)
    pts = {(0, 0, 0), tuple(s - 1 for s in shape)}
    while len(pts) < min(k, int(np.prod(shape))):
        pts.add(tuple(int(rng.integers(0, s)) for s in shape))
    return sorted(pts)


def main():
    sys.path.insert(0, REF)
    from ditplan.errors import ConfigError
    from ditplan.inference import plan_temporal_windows, plan_vae_tiles

    latents = [(1, 16, 16), (4, 40, 40), (8, 24, 64), (32, 90, 160), (16, 48, 48)]
    tiles = [(1, 8, 8), (4, 16, 16), (8, 48, 48), (40, 100, 100), (2, 12, 20)]
    rules = [lambda t: (0, 0, 0), lambda t: (0, t[1] // 4, t[2] // 4),
             lambda t: (t[0] // 2, t[1] // 2, t[2] // 2), lambda t: (0, t[1] // 3, min(7, t[2] // 2))]
    grid = [(lat, t, r(t), 4) for lat in latents for t in tiles for r in rules]
    grid += [((32, 90, 160), (32, 48, 48), (0, 8, 8), 8), ((8, 64, 64), (8, 32, 32), (0, 8, 8), 1),
             ((8, 64, 64), (4, 32, 32), (0, 0, 0), 4), ((4, 16, 16), (8, 64, 64), (0, 4, 4), 4),
             ((1, 96, 96), (1, 48, 48), (0, 8, 8), 3), ((5, 30, 52), (3, 16, 24), (1, 6, 9), 8),
             ((6, 20, 20), (4, 9, 9), (3, 8, 8), 2)]
    vae = []
    for lat, t, ov, dev in grid:
        plan = plan_vae_tiles(lat, t, ov, devices=dev)
        prof = plan.tile_profile()
        total = plan.total_weight()
        pos = sample_positions(lat, k=12)
        maps = plan.weight_maps() if len(plan.tiles) <= 40 and len(plan.tiles) * np.prod(lat) <= 4_000_000 else None
        vae.append({
            "args": [list(lat), list(t), list(ov), dev],
            "n_tiles": len(plan.tiles),
            "axis_starts": [sorted({x.start[a] for x in plan.tiles}) for a in range(3)],
            "tiles_head": [[list(x.start), list(x.size), x.device] for x in plan.tiles[:16]],
            "tiles_sha256": hashlib.sha256(json.dumps([[list(x.start), list(x.size), x.device]
                                                       for x in plan.tiles]).encode()).hexdigest(),
            "parallel_speedup": plan.parallel_speedup,
            "profile_sum": float(prof.sum()),
            "profile_flat": prof.ravel().tolist() if prof.size <= 256 else None,
            "total_sum": float(total.sum()),
            "positions": [list(p) for p in pos],
            "total_at": [float(total[p]) for p in pos],
            "weights_at": None if maps is None else [[float(m[p]) for m in maps] for p in pos],
            "normalized_sum_minmax": [float(plan.normalized_weight_sum().min()),
                                      float(plan.normalized_weight_sum().max())],
        })
    vae_err = []
    for args in [((8, 64, 64), (4, 32, 32), (4, 0, 0), 1), ((8, 64, 64), (0, 32, 32), (0, 0, 0), 1),
                 ((8, 64, 64), (4, 32, 32), (0, -1, 0), 1), ((0, 64, 64), (4, 32, 32), (0, 0, 0), 1),
                 ((8, 64, 64), (4, 32, 32), (0, 0, 0), 0), ((8, 64, 64), (4, 32, 32), (0, 0, 32), 2)]:
        try:
            plan_vae_tiles(args[0], args[1], args[2], devices=args[3])
            vae_err.append({"args": [list(a) if isinstance(a, tuple) else a for a in args], "path": None})
        except ConfigError as e:
            vae_err.append({"args": [list(a) if isinstance(a, tuple) else a for a in args], "path": e.path,
                            "message": str(e)})
    win = []
    for n_prime in range(1, 17):
        for n in range(1, n_prime + 1):
            for s in range(1, n + 1):
                p = plan_temporal_windows(n_prime, n, s)
                win.append({"args": [n_prime, n, s], "clips": [list(c) for c in p.clips],
                            "multiplicity": p.multiplicity().tolist()})
    for args in ((32, 8, 4), (33, 8, 4), (23, 6, 3), (64, 16, 12), (33, 16, 8)):
        p = plan_temporal_windows(*args)
        win.append({"args": list(args), "clips": [list(c) for c in p.clips],
                    "multiplicity": p.multiplicity().tolist(),
                    "averaging_weights": [p.averaging_weights(i) for i in range(args[0])]})
    win_err = []
    for args in ((32, 8, 9), (0, 1, 1), (4, 5, 1), (8, 4, 0), (8, 0, 1)):
        try:
            plan_temporal_windows(*args)
            win_err.append({"args": list(args), "path": None})
        except ConfigError as e:
            win_err.append({"args": list(args), "path": e.path, "message": str(e)})
    doc = {"source": "ditplan.inference (reference) via tests/golden/make_golden_tiling.py",
           "vae_tiles": vae, "vae_tile_errors": vae_err, "windows": win, "window_errors": win_err}
    with open(OUT, "w") as fh:
        json.dump(doc, fh, sort_keys=True)
    print(f"wrote {OUT}: {len(vae)} tile plans, {len(win)} window plans")


if __name__ == "__main__":
    main()
