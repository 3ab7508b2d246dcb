#!/usr/bin/env python
"""Per-CTA fixed cost of the self-attention kernel: 7,800 queries x 16 heads (config 2) against
S_kv in {1,950 ... 31,200} keys with one pass per tile (splits=1, so every launch runs the same
4 waves of 496 tiles), timed in a CUDA graph; t = waves * (fixed + blocks * per_block) fitted by
least squares.  One JSON line per S_kv, then the fit."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

A, D, SQ = 16, 128, 7800
bf = torch.bfloat16
pts = []
for skv in (1920, 3840, 7680, 15360, 30720):
    g = torch.Generator(device="cuda").manual_seed(skv)
    q = [torch.randn(SQ, A * D, device="cuda", generator=g).to(bf) for _ in range(2)]
    k = torch.randn(skv, A * D, device="cuda", generator=g).to(bf)
    v = torch.randn(skv, A * D, device="cuda", generator=g).to(bf)
    o = [torch.empty(SQ, A * D, device="cuda", dtype=bf) for _ in range(2)]
    ws = torch.zeros(max(16, ops.attention_workspace_bytes(SQ, skv, A, D)), device="cuda", dtype=torch.uint8)
    for i in range(2):
        ops.attention(q[i], k, v, o[i], A, D, splits=1, workspace=ws)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr):
            for i in range(8):
                ops.attention(q[i % 2], k, v, o[i % 2], A, D, splits=1, workspace=ws)
    gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 8 * 1e3)
    us = sorted(ts)[2]
    nkv = (skv + 127) // 128
    pts.append((nkv, us))
    print(json.dumps({"sq": SQ, "skv": skv, "heads": A, "kv_blocks": nkv, "us": us,
                      "tflops": 4.0 * SQ * skv * D * A / us / 1e6}), flush=True)
n = len(pts)
mx = sum(x for x, _ in pts) / n
my = sum(y for _, y in pts) / n
b = sum((x - mx) * (y - my) for x, y in pts) / sum((x - mx) ** 2 for x, _ in pts)
a = my - b * mx
waves = -(-((SQ + 255) // 256 * A) // torch.cuda.get_device_properties(0).multi_processor_count)
print(json.dumps({"fit": "t_us = waves * (fixed + blocks * per_block)", "waves": waves,
                  "fixed_us_per_cta": a / waves, "per_block_us": b / waves,
                  "fixed_share_at_7800": (a / waves) / (a / waves + 61 * b / waves)}), flush=True)
