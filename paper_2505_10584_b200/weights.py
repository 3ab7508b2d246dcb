"""Parameter inventory and seeded random init (no checkpoints exist).

Synthetic-input contract: weights ~ N(0, 0.02²) from a
``torch.Generator`` seeded with 0, fp32 master then rounded to bf16 for
every matrix.  AdaLN-zero would make every block an identity at init
(SURVEY.md §7 "hard parts"), so the modulation tables / modulation biases are
drawn N(0, 0.5²) instead — every block contributes, parity is not vacuous.
Norm weights are 1 + N(0, 0.02²).  Biases, norm weights and tables stay fp32.

Names are shared by the product model and the CPU oracle.
"""

from __future__ import annotations

import torch

from .config import DiTConfig

W_STD = 0.02
MOD_STD = 0.5


def _linear(name: str, out_f: int, in_f: int, bias_std: float = W_STD):
    return [(f"{name}.w", (out_f, in_f), "matrix", W_STD), (f"{name}.b", (out_f,), "vector", bias_std)]


def _attn_stream(p: str, cfg: DiTConfig):
    H, F, D = cfg.hidden_size, cfg.ffn_dim, cfg.head_dim
    return (
        _linear(f"{p}.qkv", 3 * H, H)
        + [(f"{p}.q_norm", (D,), "norm", W_STD), (f"{p}.k_norm", (D,), "norm", W_STD)]
        + _linear(f"{p}.proj", H, H)
        + _linear(f"{p}.fc1", F, H)
        + _linear(f"{p}.fc2", H, F)
    )


def param_specs(cfg: DiTConfig):
    """Ordered ``(name, shape, kind, std)`` list; the order fixes the RNG stream."""
    H, D, C = cfg.hidden_size, cfg.head_dim, cfg.patch_dim
    specs = _linear("t_emb.fc1", H, cfg.freq_dim) + _linear("t_emb.fc2", H, H) + _linear("x_emb", H, C)
    if cfg.family == "single-dit":
        specs += _linear("t_block", 6 * H, H)
        for i in range(cfg.num_single):
            p = f"blocks.{i}"
            specs += [(f"{p}.table", (6 * H,), "table", MOD_STD)]
            specs += _attn_stream(p, cfg)
            specs += _linear(f"{p}.xq", H, H) + _linear(f"{p}.xkv", 2 * H, cfg.text_dim)
            specs += [(f"{p}.xq_norm", (D,), "norm", W_STD), (f"{p}.xk_norm", (D,), "norm", W_STD)]
            specs += _linear(f"{p}.xproj", H, H)
        specs += [("final.table", (2 * H,), "table", MOD_STD)]
    else:
        specs += _linear("p_emb.fc1", H, cfg.pooled_dim) + _linear("p_emb.fc2", H, H)
        specs += _linear("txt_in", H, cfg.text_dim)
        for i in range(cfg.num_dual):
            for s in ("img", "txt"):
                p = f"dual.{i}.{s}"
                specs += _linear(f"{p}.mod", 6 * H, H, bias_std=MOD_STD)
                specs += _attn_stream(p, cfg)
        for i in range(cfg.num_single):
            p = f"single.{i}"
            specs += _linear(f"{p}.mod", 6 * H, H, bias_std=MOD_STD)
            specs += _attn_stream(p, cfg)
        specs += _linear("final.mod", 2 * H, H, bias_std=MOD_STD)
    specs += _linear("final", C, H)
    return specs


@torch.no_grad()
def init_weights(cfg: DiTConfig, seed: int = 0, device="cpu", only=None) -> dict:
    """Seeded weights: matrices bf16, everything else fp32, on ``device``.

    ``only`` (a predicate on the name) restricts which tensors are
    materialised while keeping the RNG stream identical (skipped tensors are
    still drawn) — used for bounded CPU samples of the big configs.
    """
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    out = {}
    for name, shape, kind, std in param_specs(cfg):
        if only is not None and not only(name):
            # advance the stream by drawing in chunks (bounded memory)
            n = 1
            for s in shape:
                n *= s
            chunk = 1 << 26
            while n > 0:
                k = min(n, chunk)
                torch.randn(k, generator=gen, device=device)
                n -= k
            continue
        t = torch.randn(shape, generator=gen, device=device, dtype=torch.float32) * std
        if kind == "norm":
            t += 1.0
        out[name] = t.to(torch.bfloat16) if kind == "matrix" else t
    return out


@torch.no_grad()
def synthetic_inputs(cfg: DiTConfig, grid, seed_noise: int = 1, seed_text: int = 2, device="cpu") -> dict:
    """x0 ~ N(0,1) latent [C, T, H, W]; text ~ N(0,1) [S_t, text_dim];
    pooled ~ N(0,1) [pooled_dim] (MM-DiT)."""
    T, Hh, Ww = grid
    pt, ph, pw = cfg.patch
    g = torch.Generator(device=device)
    g.manual_seed(seed_noise)
    x0 = torch.randn((cfg.latent_channels, T * pt, Hh * ph, Ww * pw), generator=g, device=device)
    g.manual_seed(seed_text)
    text = torch.randn((cfg.text_len, cfg.text_dim), generator=g, device=device)
    pooled = torch.randn((cfg.pooled_dim,), generator=g, device=device)
    return {"x0": x0, "text": text, "pooled": pooled}
