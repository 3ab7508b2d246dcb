#!/usr/bin/env python
"""Pipeline trace of the short-KV attention kernel (aqb_attention_trace): per CTA clock64 stamps
of MMA QK/PV issue and the softmax warpgroups' s_full / p_full / o_ready / slot-release events,
printed relative to each CTA's start (median over CTAs)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import _native, ops  # noqa: E402

sq, skv, heads = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (7800, 256, 16)))
d = 128
bf = torch.bfloat16
q = torch.randn(sq, heads * d, device="cuda").to(bf)
k = torch.randn(skv, heads * d, device="cuda").to(bf)
v = torch.randn(skv, heads * d, device="cuda").to(bf)
o = torch.empty(sq, heads * d, device="cuda", dtype=bf)
tr = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
ops.attention(q, k, v, o, heads, d)
_native.query("aqb_attention_trace", tr.data_ptr())
ops.attention(q, k, v, o, heads, d)
torch.cuda.synchronize()
_native.query("aqb_attention_trace", None)
t = tr.view(-1, 64).cpu()
t = t[t[:, 48] != 0]
base = t[:, 48:49]
rel = (t - base).float()
names = [("qk", 0), ("pv", 8), ("s_full", 16), ("p_full", 24), ("o_ready", 32), ("free", 40)]
print(f"{t.shape[0]} CTAs; k_full at {statistics.median(rel[:, 49].tolist()):.0f} clk")
for i in range(8):
    row = []
    for nm, off in names:
        col = rel[:, off + i]
        col = col[t[:, off + i] != 0]
        row.append(f"{nm} {statistics.median(col.tolist()) if len(col) else float('nan'):7.0f}")
    print(f"tile {i}: " + "  ".join(row))
