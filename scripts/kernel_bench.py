#!/usr/bin/env python
"""Per-kernel microbenchmarks at BASELINE shapes (CUDA events, warm, L2-flushed).

    python scripts/kernel_bench.py [--only gemm|attn|norm] [--ncu] [--attn-sweep]

--ncu: run each kernel a few times without timing loops (for ncu -k regex:...).
--attn-sweep: BASELINE config 5 — joint-attention seq 4k..128k, head_dim 128,
  24 heads (per GPU: 24/P heads at full sequence after the Ulysses all-to-all).
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"
FLUSH = None


def flush_l2():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    FLUSH.zero_()


def timeit(fn, iters=10, flush=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush:
            flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def gemm_case(m, n, k, epi="bf16", ncu=False):
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.randn(n, device=dev)
    if epi in ("bf16", "gelu"):
        out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    else:
        out = torch.zeros(m, n, device=dev)
    g = torch.randn(n, device=dev)
    fn = lambda: ops.gemm(a, w, out, bias=b, gate=g if epi == "gate_res" else None, epilogue=epi)  # noqa: E731
    if ncu:
        fn()
        return None
    ms = timeit(fn)
    return {"kernel": "gemm", "m": m, "n": n, "k": k, "epi": epi, "ms": ms, "tflops": 2 * m * n * k / ms / 1e9}


def proj_aux_case(m, n, k, split=False, ncu=False):
    """Single-DiT self-attention out-projection: x += gate*(o W^T + b) and bf16(x) for the
    cross-attention q — fused (gate*residual + bf16 copy) or split (TMA reduce-add GEMM + cast)."""
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev)
    x = torch.randn(m, n, device=dev)
    aux = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    if split:
        def fn():
            ops.gemm(a, w, x, bias=b, gate=g, epilogue="gate_res")
            ops.norm_modulate(x, None, None, aux, kind=2)
    else:
        fn = lambda: ops.gemm(a, w, x, bias=b, gate=g, epilogue="gate_res", aux=aux)  # noqa: E731
    if ncu:
        fn()
        return None
    ms = timeit(fn)
    return {"kernel": "proj+bf16(x)", "split": split, "m": m, "n": n, "k": k, "ms": ms,
            "tflops": 2 * m * n * k / ms / 1e9}


def qkv_fused_case(m, heads, k, ncu=False, parts=3, norm_parts=2, rope=True):
    """The QKV projection with the QK-RMSNorm + 3D-RoPE epilogue (as in the model)."""
    d = 128
    n = parts * heads * d
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.randn(n, device=dev)
    qw, kw = torch.ones(d, device=dev), torch.ones(d, device=dev)
    cos, sin = torch.randn(m, d // 2, device=dev), torch.randn(m, d // 2, device=dev)
    out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    fn = lambda: ops.gemm_qknorm_rope(a, w, out, heads * d, norm_parts, qw, kw, 1e-6, bias=b, cos=cos, sin=sin,  # noqa: E731
                                      rope_row0=0, rope_rows=m if rope else 0)
    if ncu:
        fn()
        return None
    ms = timeit(fn)
    return {"kernel": "gemm_qknorm_rope", "m": m, "n": n, "k": k, "norm_parts": norm_parts, "rope": rope, "ms": ms,
            "tflops": 2 * m * n * k / ms / 1e9}


def attn_case(sq, skv, heads, d=128, ncu=False, packed=True):
    qkv = torch.randn(max(sq, skv), 3 * heads * d, device=dev).to(torch.bfloat16)
    o = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    H = heads * d
    ws = torch.zeros(max(16, ops.attention_workspace_bytes(sq, skv, heads, d)), device=dev, dtype=torch.uint8)
    fn = lambda: ops.attention(qkv[:sq], qkv[:skv, H:], qkv[:skv, 2 * H:], o, heads, d, workspace=ws)  # noqa: E731
    if ncu:
        fn()
        return None
    ms = timeit(fn, iters=5)
    fl = 4.0 * sq * skv * d * heads
    return {"kernel": "attention", "sq": sq, "skv": skv, "heads": heads, "d": d, "ms": ms, "tflops": fl / ms / 1e9}


def norm_case(rows, hidden, ncu=False):
    x = torch.randn(rows, hidden, device=dev)
    y = torch.empty(rows, hidden, device=dev, dtype=torch.bfloat16)
    sh = torch.randn(hidden, device=dev)
    sc = torch.randn(hidden, device=dev)
    fn = lambda: ops.norm_modulate(x, sh, sc, y)  # noqa: E731
    if ncu:
        fn()
        return None
    ms = timeit(fn)
    return {"kernel": "norm_modulate", "rows": rows, "hidden": hidden, "ms": ms, "gbs": rows * hidden * 6 / ms / 1e6}


def qk_case(rows, heads, d=128, ncu=False):
    qkv = torch.randn(rows, 3 * heads * d, device=dev).to(torch.bfloat16)
    qw = torch.ones(d, device=dev)
    cos = torch.randn(rows, d // 2, device=dev)
    sin = torch.randn(rows, d // 2, device=dev)
    fn = lambda: ops.qk_norm_rope(qkv, heads, d, qw, qw, 1e-6, cos, sin, 0, rows)  # noqa: E731
    if ncu:
        fn()
        return None
    ms = timeit(fn)
    return {"kernel": "qk_norm_rope", "rows": rows, "heads": heads, "ms": ms,
            "gbs": rows * 3 * heads * d * 2 * 2 / ms / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--attn-sweep", action="store_true")
    args = ap.parse_args()
    res = []
    S, H = 7800, 2048
    if args.only in ("all", "gemm", "gemm-proj", "gemm-small", "gemm-n2048"):
        shapes = [(S, 3 * H, H, "bf16"), (S, H, H, "gate_res"), (S, 4 * H, H, "gelu"), (S, H, 4 * H, "gate_res"),
                  (14850 + 256, 3 * 3072, 3072, "bf16"), (8192, 8192, 8192, "bf16")]
        if args.only == "gemm-proj":
            shapes = [(S, H, H, "bf16"), (S, H, H, "f32"), (S, H, H, "gate_res")]
        if args.only == "gemm-n2048":  # the H-wide projections of a config-2 block (out, cross-q/out, FFN2)
            shapes = [(S, H, H, "bf16"), (S, H, H, "f32"), (S, H, H, "gate_res"), (S, H, 4 * H, "bf16"),
                      (S, H, 4 * H, "gate_res")]
        if args.only == "gemm-small":  # one rank's shard at 4 / 8 GPUs (config 2)
            shapes = [(m, n, k, e) for m in (S // 4, S // 8)
                      for (n, k, e) in ((3 * H, H, "bf16"), (H, H, "gate_res"), (4 * H, H, "gelu"), (H, 4 * H, "gate_res"))]
        for (m, n, k, e) in shapes:
            res.append(gemm_case(m, n, k, e, args.ncu))
    if args.only in ("all", "attn"):
        res.append(attn_case(S, S, 16, 128, args.ncu))
        res.append(attn_case(S, 256, 16, 128, args.ncu))
        if not args.ncu:
            res.append(attn_case(118800 + 256, 118800 + 256, 3, 128))  # config 4 per rank at P=8
    if args.only == "qkv":  # fused QKV epilogue vs the plain bf16 epilogue, config 2 and shards
        for m in (S, S // 2, S // 4):
            res.append(gemm_case(m, 3 * H, H, "bf16", args.ncu))
            res.append(qkv_fused_case(m, 16, H, args.ncu))
        res.append(qkv_fused_case(S, 16, H, args.ncu, parts=1, norm_parts=1))  # cross-attention q
        if not args.ncu:  # epilogue cost breakdown: without RoPE, without norm
            res.append(qkv_fused_case(S, 16, H, rope=False))
            res.append(qkv_fused_case(S, 16, H, norm_parts=0, rope=False))
    if args.only == "proj":
        for m in (S, S // 2, S // 4):
            res.append(proj_aux_case(m, H, H))
            res.append(proj_aux_case(m, H, H, split=True))
    if args.only == "attn-ranks":  # config-2 self-attention per rank at 1/2/4/8 GPUs, config 3/4 per rank
        for heads in (16, 8, 4, 2):
            res.append(attn_case(S, S, heads, 128))
        res.append(attn_case(25440 + 256, 25440 + 256, 6, 128))
        res.append(attn_case(118800 + 256, 118800 + 256, 3, 128))
    if args.only == "gemm-variants":  # H-wide projections (K = H) of config 2 at 1 / 2 / 4 GPUs (AQB_GEMM_VARIANT sweeps)
        for m in (S, S // 2, S // 4):
            res.append(gemm_case(m, H, H, "gate_res"))
            res.append(gemm_case(m, H, H, "bf16"))
            res.append(proj_aux_case(m, H, H))
            res.append(gemm_case(m, H, 4 * H, "gate_res"))
    if args.only == "attn-cross":  # cross-attention to 256 text tokens: query blocks per CTA (K/V resident)
        import os
        for rows, heads in ((S, 16), (S // 2, 8), (S // 4, 4), (S // 8, 2)):
            for g in ("1", "2", "3", "4", "6", "8", None):
                if g is None:
                    os.environ.pop("AQB_ATTN_PAIRS", None)
                else:
                    os.environ["AQB_ATTN_PAIRS"] = g
                r = attn_case(rows, 256, heads, 128)
                r["pairs_per_cta"] = g or "auto"
                res.append(r)
        os.environ.pop("AQB_ATTN_PAIRS", None)
    if args.only == "attn-long":  # config 4 per rank at P=8 (and the 1-GPU per-head shape)
        res.append(attn_case(118800 + 256, 118800 + 256, 3, 128, args.ncu))
    if args.only in ("all", "norm"):
        res.append(norm_case(S, H, args.ncu))
        if not args.ncu:
            res.append(norm_case(S // 4, H))   # one rank's shard at 4 GPUs
            res.append(norm_case(S // 8, H))   # ... at 8 GPUs
            res.append(norm_case(14850 + 256, 3072))
        res.append(qk_case(S, 16, 128, args.ncu))
    if args.attn_sweep:
        for s in (4096, 8192, 16384, 32768, 65536, 131072):
            for P in (1, 2, 4, 8):
                if s >= 65536 and P == 1:
                    continue
                res.append(attn_case(s, s, 24 // P, 128))
    for r in res:
        if r:
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
