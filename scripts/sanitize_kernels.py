#!/usr/bin/env python
"""Tiny-shape driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one launch of every kernel class of libaqb.so — GEMM variants and epilogues (incl. the
TMA reduce-add and the fused QK-norm/RoPE epilogue), self- and cross-attention (whole tiles,
split-KV + combine, short-KV resident blocks), LayerNorm+modulate (TMA ring, row and warp
kernels, probe), QK-norm, GEMV, cache decision / offset, (un)patchify, VAE blend, window
average, the fp32 validation kernels — then a tiny denoise of each family under both cache
modes and the rel-L1 policy.

    compute-sanitizer --tool memcheck python scripts/sanitize_kernels.py
The 2-rank peer barrier / scatter path: scripts/sanitize.sh runs tests/mp_parity.py (P=2,
one GPU) under compute-sanitizer --target-processes all.
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import (TINY_MM, TINY_SINGLE, DiTConfig, RelL1Policy, build_model, denoise,  # noqa: E402
                                   ops, plan_cache)
from paper_2505_10584_b200.tiling import average_windows, blend_tiles, plan_temporal_windows, plan_vae_tiles  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402

dev = "cuda"
bf = torch.bfloat16


def main():
    g = torch.Generator(device=dev).manual_seed(0)
    r = lambda *s, dt=torch.float32: torch.randn(*s, device=dev, generator=g).to(dt)  # noqa: E731
    # GEMMs: every epilogue on a ragged shape, one shape per variant class
    for m, n, k in ((300, 384, 200), (1000, 2048, 512), (129, 128, 64)):
        a, w, b = r(m, k, dt=bf), r(n, k, dt=bf), r(n)
        ops.gemm(a, w, torch.empty(m, n, device=dev, dtype=bf), bias=b)
        ops.gemm(a, w, torch.empty(m, n, device=dev, dtype=bf), bias=b, epilogue="gelu")
        ops.gemm(a, w, torch.empty(m, n, device=dev), bias=b, epilogue="f32")
        ops.gemm(a, w, r(m, n), bias=b, gate=r(n), epilogue="gate_res")
        ops.gemm(a, w, r(m, n), bias=b, gate=r(n), epilogue="gate_res", aux=torch.empty(m, n, device=dev, dtype=bf))
    heads, d, m = 2, 128, 384
    a, w = r(m, 256, dt=bf), r(3 * heads * d, 256, dt=bf)
    cos, sin = r(m, d // 2), r(m, d // 2)
    ops.gemm_qknorm_rope(a, w, torch.empty(m, 3 * heads * d, device=dev, dtype=bf), heads * d, 2, r(d), r(d), 1e-6,
                         bias=r(3 * heads * d), cos=cos, sin=sin, rope_rows=m)
    # attention: self (whole + split), cross (short KV), fp32
    for sq, skv, h in ((300, 300, 2), (1024, 1024, 1), (700, 256, 4), (129, 16, 2)):
        q, k_, v = r(sq, h * d, dt=bf), r(skv, h * d, dt=bf), r(skv, h * d, dt=bf)
        o = torch.empty(sq, h * d, device=dev, dtype=bf)
        ws = torch.zeros(max(16, ops.attention_workspace_bytes(sq, skv, h, d, 3)), device=dev, dtype=torch.uint8)
        ops.attention(q, k_, v, o, h, d)
        ops.attention(q, k_, v, o, h, d, splits=3, workspace=ws)
    # norms
    for rows, H in ((257, 2048), (33, 3072), (100, 1024), (70, 256)):
        x = r(rows, H)
        y = torch.empty(rows, H, device=dev, dtype=bf)
        ops.norm_modulate(x, r(H), r(H), y)
        ops.norm_modulate(x, r(H), r(H), y, probe_prev=r(rows, H), probe_partials=torch.empty(2 * rows, device=dev))
        ops.norm_modulate(x, None, None, y, kind=2)
    qkv = r(64, 3 * 2 * 64, dt=bf)
    ops.qk_norm_rope(qkv, 2, 64, r(64), r(64), 1e-6, r(64, 32), r(64, 32), 0, 64)
    # VAE blend / windows
    plan = plan_vae_tiles((6, 20, 20), (4, 9, 9), (3, 8, 8), devices=1)
    blend_tiles(plan, [r(3, *t.size) for t in plan.tiles], torch.empty(3, *plan.latent, device=dev))
    wp = plan_temporal_windows(9, 4, 2)
    average_windows(wp, [r(2, 4, 3, 5) for _ in wp.clips], torch.empty(2, 9, 3, 5, device=dev))
    torch.cuda.synchronize()
    # whole denoise loops: both families, static + dynamic cache, both cache modes, fp32 mode
    d128 = DiTConfig("single-dit", hidden_size=256, num_heads=2, num_single=4, text_dim=256, text_len=40)
    for cfg, grid in ((TINY_SINGLE, (2, 4, 4)), (TINY_MM, (2, 4, 4)), (d128, (3, 8, 12))):
        W = init_weights(cfg, seed=0)
        inp = synthetic_inputs(cfg, grid)
        pooled = inp["pooled"] if cfg.family == "mm-dit" else None
        for prec in ("bf16", "fp32"):
            model = build_model(cfg, weights=W, precision=prec).prepare(grid, inp["text"], pooled)
            for cache in (plan_cache(4, 1, 2), RelL1Policy(threshold=0.05, warmup=1),
                          plan_cache(4, 1, 2, mode="attention-cache")):
                denoise(model, inp["x0"], 4, cache)
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
