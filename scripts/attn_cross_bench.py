#!/usr/bin/env python
"""Cross-attention (queries -> 256 text keys, head_dim 128) timed in a CUDA graph of 8 launches
(4 rotating Q/O sets).  AQB_ATTN_SHORT=0: the general kernel (read once per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"
bf = torch.bfloat16


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--ncu":  # one launch after a warm-up: --ncu sq skv heads
        sq, skv, heads = map(int, sys.argv[2:5])
        d = 128
        q = torch.randn(sq, heads * d, device=dev).to(bf)
        k = torch.randn(skv, heads * d, device=dev).to(bf)
        v = torch.randn(skv, heads * d, device=dev).to(bf)
        o = torch.empty(sq, heads * d, device=dev, dtype=bf)
        for _ in range(2):
            ops.attention(q, k, v, o, heads, d)
        torch.cuda.synchronize()
        return
    for sq, skv, heads in ((7800, 256, 16), (3900, 256, 16), (1950, 256, 16), (975, 256, 16), (7800, 256, 2),
                           (7800, 77, 16)):
        d = 128
        nb = 4
        Q = [torch.randn(sq, heads * d, device=dev).to(bf) for _ in range(nb)]
        k = torch.randn(skv, heads * d, device=dev).to(bf)
        v = torch.randn(skv, heads * d, device=dev).to(bf)
        O = [torch.empty(sq, heads * d, device=dev, dtype=bf) for _ in range(nb)]
        ws = torch.zeros(max(16, ops.attention_workspace_bytes(sq, skv, heads, d)), device=dev, dtype=torch.uint8)
        for i in range(nb):
            ops.attention(Q[i], k, v, O[i], heads, d, workspace=ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                for i in range(8):
                    ops.attention(Q[i % nb], k, v, O[i % nb], heads, d, workspace=ws)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 8)
        ms = sorted(ts)[len(ts) // 2]
        print(json.dumps({"sq": sq, "skv": skv, "heads": heads, "short": os.environ.get("AQB_ATTN_SHORT", "1") != "0",
                          "us": ms * 1e3, "tflops": 4.0 * sq * skv * d * heads / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
