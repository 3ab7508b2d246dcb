#!/usr/bin/env python
"""Run-to-run bitwise determinism of the 1-GPU denoise loop (same process, same inputs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import DiTConfig, RelL1Policy, build_model, denoise, plan_cache  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402

cases = [
    ("single", DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40), (3, 8, 16)),
    ("mm", DiTConfig("mm-dit", hidden_size=1024, num_heads=8, num_dual=2, num_single=2, text_dim=192, text_len=24,
                     pooled_dim=64), (2, 8, 16)),
    ("mm-24h", DiTConfig("mm-dit", hidden_size=3072, num_heads=24, num_dual=1, num_single=1, text_dim=192,
                         text_len=24, pooled_dim=64), (2, 8, 16)),
]
for name, cfg, grid in cases:
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, grid)
    pooled = inp["pooled"] if cfg.family == "mm-dit" else None
    for graph in (False, True):
        outs = []
        for rep in range(3):
            m = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled)
            r = denoise(m, inp["x0"], 8, plan_cache(8, warmup=2, interval=2), trajectory=True, graph=graph)
            outs.append(torch.stack([t.cpu() for t in r.trajectory]))
        diffs = [float((o - outs[0]).abs().max()) for o in outs[1:]]
        print(json.dumps({"case": name, "graph": graph, "max_abs_diff_vs_first": diffs}), flush=True)
