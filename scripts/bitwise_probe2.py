#!/usr/bin/env python
"""Bitwise partition-invariance of the Ulysses-path kernels (scatter variants, gate*residual + bf16 copy)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
H, A, D, S = 1024, 8, 128, 96
P, n, hl = 2, 48, 4
# gate*residual with the bf16 copy: M=96 vs 2 x 48
for k in (1024, 4096):
    a = torch.randn(S, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(H, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    b = torch.randn(H, device=dev, generator=g)
    gate = torch.randn(H, device=dev, generator=g)
    x = torch.randn(S, H, device=dev, generator=g)
    x1, x2 = x.clone(), x.clone()
    aux1 = torch.empty(S, H, device=dev, dtype=torch.bfloat16)
    aux2 = torch.empty_like(aux1)
    ops.gemm(a, w, x1, bias=b, gate=gate, epilogue="gate_res", aux=aux1)
    ops.gemm(a[:n], w, x2[:n], bias=b, gate=gate, epilogue="gate_res", aux=aux2[:n])
    ops.gemm(a[n:], w, x2[n:], bias=b, gate=gate, epilogue="gate_res", aux=aux2[n:])
    print(f"gate_res+aux K={k}: x bitwise", torch.equal(x1, x2), "aux bitwise", torch.equal(aux1, aux2),
          "max|dx|", float((x1 - x2).abs().max()))
    x3 = x.clone()
    ops.gemm(a, w, x3, bias=b, gate=gate, epilogue="gate_res")
    print(f"  gate_res (reduce-add) vs gate_res+aux K={k}: max|dx|", float((x1 - x3).abs().max()))
# attention: plain on all 8 heads vs scatter of 4-head groups to 2 'ranks'
qkv = torch.randn(S, 3, A, D, device=dev, generator=g).to(torch.bfloat16)
f = qkv.view(S, -1)
o_all = torch.empty(S, A * D, device=dev, dtype=torch.bfloat16)
ops.attention(f, f[:, H:], f[:, 2 * H:], o_all, A, D)
outs = [torch.zeros(n, H, device=dev, dtype=torch.bfloat16) for _ in range(P)]
for r in range(P):  # rank r's heads
    sub = qkv[:, :, r * hl:(r + 1) * hl].contiguous().view(S, -1)
    dst = [o.data_ptr() + r * hl * D * 2 for o in outs]
    ws = torch.empty(max(16, ops.attention_workspace_bytes(S, S, hl, D)), device=dev, dtype=torch.uint8)
    ops.attention_scatter(sub, sub[:, hl * D:], sub[:, 2 * hl * D:], dst, H, hl, D, n, P * n, workspace=ws)
print("attention_scatter vs attention bitwise", torch.equal(torch.cat(outs), o_all),
      "max|d|", float((torch.cat(outs).float() - o_all.float()).abs().max()))
