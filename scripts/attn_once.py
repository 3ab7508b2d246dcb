#!/usr/bin/env python
"""One seeded self-attention of S tokens x A heads (head_dim 128), launched twice (for ncu -s 1 -c 1):
    python scripts/attn_once.py 7800 16"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops
S, A, D = int(sys.argv[1]), int(sys.argv[2]), 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(S, 3 * A * D, device="cuda", generator=g).to(torch.bfloat16)
o = torch.empty(S, A * D, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(max(16, ops.attention_workspace_bytes(S, S, A, D)), device="cuda", dtype=torch.uint8)
for _ in range(2):
    ops.attention(q, q[:, A * D:], q[:, 2 * A * D:], o, A, D, workspace=ws)
torch.cuda.synchronize()
