#!/usr/bin/env python
"""Self-attention per Ulysses rank (A/P heads over the full sequence), timed in a CUDA graph of
4 launches: config 2 (7,800 tokens, 16 heads) and config 3 (25,696 tokens, 24 heads) at
P = 1, 2, 4, 8."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import _native, ops  # noqa: E402

bf = torch.bfloat16
d = 128
for S, A in ((7800, 16), (25696, 24)):
    for P in (1, 2, 4, 8):
        h = A // P
        qkv = torch.randn(S, 3 * h * d, device="cuda").to(bf)
        o = torch.empty(S, h * d, device="cuda", dtype=bf)
        ws = torch.zeros(max(16, ops.attention_workspace_bytes(S, S, h, d)), device="cuda", dtype=torch.uint8)
        run = lambda: ops.attention(qkv, qkv[:, h * d:], qkv[:, 2 * h * d:], o, h, d, workspace=ws)  # noqa: E731
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            with torch.cuda.graph(g):
                for _ in range(4):
                    run()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 4)
        ms = sorted(ts)[2]
        print(json.dumps({"S": S, "heads": h, "P": P, "us": ms * 1e3, "tflops": 4.0 * S * S * d * h / ms / 1e9,
                          "splits": _native.query("aqb_attention_splits", S, S, h, d),
                          "whole": _native.query("aqb_attention_whole_tiles", S, S, h, d)}), flush=True)
