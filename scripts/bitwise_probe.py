#!/usr/bin/env python
"""Which kernel's bits depend on the partition (heads / rows)?  1-GPU shapes vs Ulysses-P=2 shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
H, A, D, S = 1024, 8, 128, 96
# attention: 8 heads at once vs heads 0-3 and 4-7 separately
qkv = torch.randn(S, 3, A, D, device=dev, generator=g).to(torch.bfloat16)
o_all = torch.empty(S, A * D, device=dev, dtype=torch.bfloat16)
f = qkv.view(S, -1)
ops.attention(f, f[:, H:], f[:, 2 * H:], o_all, A, D)
for hl in (4, 1):
    same = True
    for h0 in range(0, A, hl):
        sub = qkv[:, :, h0:h0 + hl].contiguous().view(S, -1)
        o = torch.empty(S, hl * D, device=dev, dtype=torch.bfloat16)
        ops.attention(sub, sub[:, hl * D:], sub[:, 2 * hl * D:], o, hl, D)
        same &= torch.equal(o, o_all[:, h0 * D:(h0 + hl) * D])
    print("attention 8 heads vs", hl, "per call: bitwise", same)
# text cross-attention: 96 q rows vs 2 x 48
kv = torch.randn(40, 2 * H, device=dev, generator=g).to(torch.bfloat16)
q = torch.randn(S, H, device=dev, generator=g).to(torch.bfloat16)
o_all = torch.empty(S, H, device=dev, dtype=torch.bfloat16)
ops.attention(q, kv, kv[:, H:], o_all, A, D)
o_h = torch.empty(S, H, device=dev, dtype=torch.bfloat16)
ops.attention(q[:48], kv, kv[:, H:], o_h[:48], A, D)
ops.attention(q[48:], kv, kv[:, H:], o_h[48:], A, D)
print("cross-attention 96 rows vs 2x48: bitwise", torch.equal(o_all, o_h))
# GEMMs: M=96 vs two M=48 halves
for n, k, epi in ((3 * H, H, "bf16"), (H, H, "gate_res"), (4 * H, H, "gelu"), (H, 4 * H, "gate_res"), (H, H, "f32")):
    a = torch.randn(S, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    b = torch.randn(n, device=dev, generator=g)
    gate = torch.randn(n, device=dev, generator=g)
    f32 = epi in ("gate_res", "f32")
    base = torch.randn(S, n, device=dev, generator=g) if f32 else torch.empty(S, n, device=dev, dtype=torch.bfloat16)
    o1, o2 = base.clone(), base.clone()
    kw = dict(bias=b, gate=gate if epi == "gate_res" else None, epilogue=epi)
    ops.gemm(a, w, o1, **kw)
    ops.gemm(a[:48], w, o2[:48], **kw)
    ops.gemm(a[48:], w, o2[48:], **kw)
    print(f"gemm {n}x{k} {epi}: M=96 vs 2x48 bitwise", torch.equal(o1, o2))
# qknorm-rope GEMM
a = torch.randn(S, H, device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn(3 * H, H, device=dev, generator=g) * 0.02).to(torch.bfloat16)
b = torch.randn(3 * H, device=dev, generator=g)
qw = torch.randn(D, device=dev, generator=g)
kw_ = torch.randn(D, device=dev, generator=g)
cos = torch.randn(S, D // 2, device=dev, generator=g)
sin = torch.randn(S, D // 2, device=dev, generator=g)
o1 = torch.empty(S, 3 * H, device=dev, dtype=torch.bfloat16)
o2 = torch.empty_like(o1)
ops.gemm_qknorm_rope(a, w, o1, H, 2, qw, kw_, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=0, rope_rows=S)
ops.gemm_qknorm_rope(a[:48], w, o2[:48], H, 2, qw, kw_, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=0, rope_rows=S)
ops.gemm_qknorm_rope(a[48:], w, o2[48:], H, 2, qw, kw_, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=48, rope_rows=S)
print("gemm_qknorm_rope M=96 vs 2x48 bitwise", torch.equal(o1, o2))
x = torch.randn(S, H, device=dev, generator=g)
sh, sc = torch.randn(H, device=dev, generator=g), torch.randn(H, device=dev, generator=g)
m1 = torch.empty(S, H, device=dev, dtype=torch.bfloat16)
m2 = torch.empty_like(m1)
ops.norm_modulate(x, sh, sc, m1)
ops.norm_modulate(x[:48], sh, sc, m2[:48])
ops.norm_modulate(x[48:], sh, sc, m2[48:])
print("norm_modulate 96 vs 2x48 bitwise", torch.equal(m1, m2))
