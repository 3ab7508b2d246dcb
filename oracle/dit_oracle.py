"""fp32 PyTorch-CPU restatement of the DiT denoise path — TEST INFRASTRUCTURE.

This is the numerical oracle and the timed "reference CPU path" (the
reference ``ditplan`` has no executable DiT — SURVEY.md §0).  Every function
cites the paper text it restates; gaps are the builder choices recorded in
DESIGN.md ("fitted").  Plain torch ops in fp32 on CPU, written for clarity,
not speed; it shares nothing with the CUDA product path except the weight
names and the config object.

Paper anchors
* Single-DiT block (AdaLN-single, cross-attn to text each block): PAPER.md:103
* MM-DiT (dual-stream then joint, AdaLN-zero per block, CLIP pooled + t): PAPER.md:106
* 3D full attention: PAPER.md:111-112; 3D RoPE (split t/h/w channels): PAPER.md:114-115
* QK-norm / LayerNorm+scale/shift / gate / GeLU ops: PAPER.md:253-256
* Flow matching X_t=(1-t)X0+tX1, v = X1-X0: PAPER.md:127-131 (Euler sampler: fitted)
* DiT-layer-output cache (rear-block offset reuse; no caching in warmup): PAPER.md:309,316
* Attention cache (per-block attention output reuse): PAPER.md:313
* Static schedule flags: ditplan ``inference.py:71-76`` (see schedule_oracle.py)
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from .schedule_oracle import rel_l1_decide

f32 = torch.float32


class strict_fp32:
    """Context manager: fp32 matmuls in full fp32 on a GPU (no TF32), restored on exit."""

    def __enter__(self):
        self.saved = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32,
                      torch.get_float32_matmul_precision())
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        torch.set_float32_matmul_precision("highest")
        return self

    def __exit__(self, *exc):
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32, prec = self.saved
        torch.set_float32_matmul_precision(prec)
        return False


def _strict(fn):
    import functools

    @functools.wraps(fn)
    def run(*a, **kw):
        with strict_fp32():
            return fn(*a, **kw)
    return run


def _w(W, name):
    return W[name].to(f32)


def linear(W, name, x):
    return x @ _w(W, f"{name}.w").t() + _w(W, f"{name}.b")


def timestep_features(t: float, dim: int = 256) -> torch.Tensor:
    """Sinusoidal features of ``1000·t``: ``[cos(a·f_i), sin(a·f_i)]``,
    ``f_i = 10000^(-i/(dim/2))`` (DiT/PixArt convention; fitted)."""
    half = dim // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=torch.float64) / half)
    a = (1000.0 * t) * freqs
    return torch.cat([torch.cos(a), torch.sin(a)]).to(f32)


def rope_angles(grid, dims, theta: float) -> torch.Tensor:
    """[S, D/2] rotation angles of the 3D RoPE.

    Channel pairs ``(2i, 2i+1)`` are split t | h | w with ``dims`` channels
    each; axis ``a`` uses ``pos_a · theta^(-2j/d_a)`` for its ``d_a/2`` pairs.
    Tokens are ordered t-major, then h, then w.
    """
    T, H, W = grid
    tt, hh, ww = torch.meshgrid(torch.arange(T), torch.arange(H), torch.arange(W), indexing="ij")
    pos = [tt.reshape(-1).double(), hh.reshape(-1).double(), ww.reshape(-1).double()]
    out = []
    for p, d in zip(pos, dims):
        j = torch.arange(0, d, 2, dtype=torch.float64)
        freqs = theta ** (-j / d)
        out.append(p[:, None] * freqs[None, :])
    return torch.cat(out, dim=1)


def apply_rope(x: torch.Tensor, ang: torch.Tensor) -> torch.Tensor:
    """Rotate interleaved pairs of x [S, A, D] by ang [S, D/2]."""
    c = torch.cos(ang).to(f32)[:, None, :]
    s = torch.sin(ang).to(f32)[:, None, :]
    x0, x1 = x[..., 0::2], x[..., 1::2]
    y0 = x0 * c - x1 * s
    y1 = x0 * s + x1 * c
    return torch.stack([y0, y1], dim=-1).reshape(x.shape)


def rms_norm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def layer_norm(x, eps):
    return F.layer_norm(x, (x.shape[-1],), eps=eps)


def modulate(x, shift, scale, eps):
    """LayerNorm(x)·(1+scale)+shift — the "LayerNorm + Scale/Shift" op."""
    return layer_norm(x, eps) * (1.0 + scale) + shift


def gelu(x):
    return F.gelu(x, approximate="tanh")


SCORE_CHUNK = 1 << 27  # score elements materialised at once (512 MB fp32)


def attention(q, k, v):
    """softmax(q kᵀ/√D) v per head; q [Sq,A,D], k/v [Skv,A,D] -> [Sq, A·D].

    Exact softmax over every key of a query row; long sequences (the 119k-token
    configs) are processed one head and one block of query rows at a time so the
    score matrix never exceeds ``SCORE_CHUNK`` elements — the same arithmetic,
    bounded memory."""
    Sq, A, D = q.shape
    Skv = k.shape[0]
    if A * Sq * Skv <= SCORE_CHUNK:
        s = torch.einsum("qad,kad->aqk", q, k) / math.sqrt(D)
        p = torch.softmax(s, dim=-1)
        o = torch.einsum("aqk,kad->qad", p, v)
        return o.reshape(Sq, -1)
    out = torch.empty(Sq, A, D, dtype=q.dtype, device=q.device)
    rows = max(1, SCORE_CHUNK // Skv)
    for a in range(A):
        kt, va = k[:, a].t(), v[:, a]
        for r0 in range(0, Sq, rows):
            s = (q[r0:r0 + rows, a] @ kt) / math.sqrt(D)
            out[r0:r0 + rows, a] = torch.softmax(s, dim=-1) @ va
    return out.reshape(Sq, -1)


def silu(x):
    return F.silu(x)


# ---------------------------------------------------------------------------
# patchify / unpatchify  (1x2x2 patches, features ordered (pt, ph, pw, c))
# ---------------------------------------------------------------------------

def patchify(lat: torch.Tensor, patch) -> torch.Tensor:
    C, T, H, W = lat.shape
    pt, ph, pw = patch
    x = lat.reshape(C, T // pt, pt, H // ph, ph, W // pw, pw)
    x = x.permute(1, 3, 5, 2, 4, 6, 0)
    return x.reshape((T // pt) * (H // ph) * (W // pw), pt * ph * pw * C)


def unpatchify(tok: torch.Tensor, grid, patch, C: int) -> torch.Tensor:
    T, H, W = grid
    pt, ph, pw = patch
    x = tok.reshape(T, H, W, pt, ph, pw, C).permute(6, 0, 3, 1, 4, 2, 5)
    return x.reshape(C, T * pt, H * ph, W * pw)


# ---------------------------------------------------------------------------
# blocks
# ---------------------------------------------------------------------------

def _qkv(W, p, m, cfg, ang):
    H, A, D = cfg.hidden_size, cfg.num_heads, cfg.head_dim
    qkv = linear(W, f"{p}.qkv", m).reshape(-1, 3, A, D)
    q = rms_norm(qkv[:, 0], _w(W, f"{p}.q_norm"), cfg.qk_norm_eps)
    k = rms_norm(qkv[:, 1], _w(W, f"{p}.k_norm"), cfg.qk_norm_eps)
    v = qkv[:, 2]
    if ang is not None:
        n = ang.shape[0]
        q = torch.cat([apply_rope(q[:n], ang), q[n:]])
        k = torch.cat([apply_rope(k[:n], ang), k[n:]])
    return q, k, v


def _cached(cache, key, fn):
    """Attention-cache mode: on a full step compute and store the
    attention output of this block; on a cached step reuse the stored one."""
    if cache is None:
        return fn()
    store, full = cache
    if full or key not in store:
        store[key] = fn()
    return store[key]


def _mlp(W, p, m):
    return linear(W, f"{p}.fc2", gelu(linear(W, f"{p}.fc1", m)))


def single_dit_block(W, i, x, tmod, text, cfg, ang, cache=None):
    """One Single-DiT block (PixArt-α AdaLN-single layout).

    mods = t_block(SiLU(t)) + table_i  →  shift1, scale1, gate1, shift2, scale2, gate2
    x += gate1 · proj(SelfAttn3D(LN(x)(1+scale1)+shift1))      [QK-RMSNorm, 3D RoPE]
    x += xproj(CrossAttn(q = xq(x), k/v = xkv(text)))          [QK-RMSNorm, no RoPE]
    x += gate2 · MLP(LN(x)(1+scale2)+shift2)                    [GeLU-tanh]
    Returns (x, m0) where m0 is the first modulated input (rel-L1 probe).
    """
    p = f"blocks.{i}"
    H, A, D = cfg.hidden_size, cfg.num_heads, cfg.head_dim
    mods = (tmod + _w(W, f"{p}.table")).reshape(6, H)
    sh1, sc1, g1, sh2, sc2, g2 = mods
    m = modulate(x, sh1, sc1, cfg.norm_eps)
    o = _cached(cache, ("self", i), lambda: attention(*_qkv(W, p, m, cfg, ang)))
    x = x + g1 * linear(W, f"{p}.proj", o)

    def cross():
        xq = rms_norm(linear(W, f"{p}.xq", x).reshape(-1, A, D), _w(W, f"{p}.xq_norm"), cfg.qk_norm_eps)
        kv = linear(W, f"{p}.xkv", text).reshape(-1, 2, A, D)
        xk = rms_norm(kv[:, 0], _w(W, f"{p}.xk_norm"), cfg.qk_norm_eps)
        return attention(xq, xk, kv[:, 1])

    x = x + linear(W, f"{p}.xproj", _cached(cache, ("cross", i), cross))
    x = x + g2 * _mlp(W, p, modulate(x, sh2, sc2, cfg.norm_eps))
    return x, m


def mm_dual_block(W, i, img, txt, vec, cfg, ang, cache=None):
    """MM-DiT dual-stream block: separate weights per stream,
    joint attention over concat(video, text); RoPE on video tokens only."""
    H = cfg.hidden_size
    sv = silu(vec)
    mi = linear(W, f"dual.{i}.img.mod", sv).reshape(6, H)
    mt = linear(W, f"dual.{i}.txt.mod", sv).reshape(6, H)
    m_img = modulate(img, mi[0], mi[1], cfg.norm_eps)
    m_txt = modulate(txt, mt[0], mt[1], cfg.norm_eps)

    def joint():
        qi, ki, vi = _qkv(W, f"dual.{i}.img", m_img, cfg, ang)
        qt, kt, vt = _qkv(W, f"dual.{i}.txt", m_txt, cfg, None)
        return attention(torch.cat([qi, qt]), torch.cat([ki, kt]), torch.cat([vi, vt]))

    o = _cached(cache, ("dual", i), joint)
    n = img.shape[0]
    img = img + mi[2] * linear(W, f"dual.{i}.img.proj", o[:n])
    txt = txt + mt[2] * linear(W, f"dual.{i}.txt.proj", o[n:])
    img = img + mi[5] * _mlp(W, f"dual.{i}.img", modulate(img, mi[3], mi[4], cfg.norm_eps))
    txt = txt + mt[5] * _mlp(W, f"dual.{i}.txt", modulate(txt, mt[3], mt[4], cfg.norm_eps))
    return img, txt, m_img


def mm_single_block(W, i, x, vec, cfg, ang, cache=None):
    """MM-DiT single-stream joint block over [video; text] with shared weights."""
    H = cfg.hidden_size
    md = linear(W, f"single.{i}.mod", silu(vec)).reshape(6, H)
    m = modulate(x, md[0], md[1], cfg.norm_eps)
    o = _cached(cache, ("single", i), lambda: attention(*_qkv(W, f"single.{i}", m, cfg, ang)))
    x = x + md[2] * linear(W, f"single.{i}.proj", o)
    x = x + md[5] * _mlp(W, f"single.{i}", modulate(x, md[3], md[4], cfg.norm_eps))
    return x, m


# ---------------------------------------------------------------------------
# one denoise step with the DiT-layer cache
# ---------------------------------------------------------------------------

class OracleDiT:
    """Holds fp32 copies of the weights and runs velocity predictions.

    ``velocity(x_tok, t, full, state)`` runs the front ``n_front`` blocks,
    then either the rear blocks (``full``; the offset
    ``rear_out - rear_in`` of the video tokens is stored in ``state``) or adds
    the stored offset (cached step) — PAPER.md:309.  Returns ``(v, m0)``.
    ``mode="attention-cache"`` runs every block and reuses each
    block's attention output (pre-projection) from the last full step instead.
    """

    def __init__(self, cfg, weights: dict, text: torch.Tensor, pooled: torch.Tensor | None, grid, n_front=None,
                 mode: str = "dit-layer-cache", device="cpu"):
        """``device``: where the fp32 restatement runs — ``"cpu"`` (the reference CPU path)
        or a CUDA device for the full-depth / full-geometry parity tests, in strict fp32
        (TF32 off for every matmul while this oracle computes, see :func:`strict_fp32`)."""
        self.cfg = cfg
        self.mode = mode
        self.device = torch.device(device)
        self.W = {k: v.detach().to(self.device, f32) for k, v in weights.items()}
        self.text = text.to(self.device, f32)
        self.pooled = None if pooled is None else pooled.to(self.device, f32)
        self.grid = tuple(grid)
        self.ang = rope_angles(self.grid, cfg.rope_dims, cfg.rope_theta).to(self.device)
        self.n_front = cfg.num_layers if n_front is None else n_front

    def _temb(self, t):
        W = self.W
        h = silu(linear(W, "t_emb.fc1", timestep_features(t, self.cfg.freq_dim).to(self.device)))
        return linear(W, "t_emb.fc2", h)

    def run_blocks(self, x_tok, t, ids):
        """Embed, blocks ``ids`` (in that order, any indices), final layer — the CPU
        baseline's per-block timing sample; every block runs at full size on its own
        weights.  Returns the velocity-shaped output."""
        cfg, W = self.cfg, self.W
        n = x_tok.shape[0]
        t0 = self._temb(t)
        if cfg.family == "single-dit":
            tmod = linear(W, "t_block", silu(t0))
            x = linear(W, "x_emb", x_tok)
            for i in ids:
                x, _ = single_dit_block(W, i, x, tmod, self.text, cfg, self.ang)
            fin = _w(W, "final.table").reshape(2, -1) + t0
            return linear(W, "final", modulate(x, fin[0], fin[1], cfg.norm_eps))
        vec = t0 + linear(W, "p_emb.fc2", silu(linear(W, "p_emb.fc1", self.pooled)))
        img, txt, x = linear(W, "x_emb", x_tok), linear(W, "txt_in", self.text), None
        for i in ids:
            if i < cfg.num_dual:
                src = (img, txt) if x is None else (x[:n], x[n:])
                img, txt = mm_dual_block(W, i, *src, vec, cfg, self.ang)[:2]
                x = None
            else:
                x = torch.cat([img, txt]) if x is None else x
                x, _ = mm_single_block(W, i - cfg.num_dual, x, vec, cfg, self.ang)
                img, txt = x[:n], x[n:]
        fm = linear(W, "final.mod", silu(vec)).reshape(2, -1)
        return linear(W, "final", modulate(img, fm[0], fm[1], cfg.norm_eps))

    def velocity(self, x_tok, t, full=True, state=None, blocks=None):
        cfg, W = self.cfg, self.W
        n = x_tok.shape[0]
        nl = cfg.num_layers if blocks is None else blocks
        nf = min(self.n_front, nl)
        cache = None
        if self.mode == "attention-cache":
            cache = (state.setdefault("attn", {}) if state is not None else {}, full)
            nf, full = nl, True  # every block runs; no rear-block offset
        t0 = self._temb(t)
        m0 = None
        if cfg.family == "single-dit":
            tmod = linear(W, "t_block", silu(t0))
            x = linear(W, "x_emb", x_tok)
            for i in range(nl):
                if i == nf:
                    if not full:
                        x = x + state["offset"]
                        break
                    x_in = x
                x, m = single_dit_block(W, i, x, tmod, self.text, cfg, self.ang, cache)
                if i == 0:
                    m0 = m
            if full and nf < nl:
                state["offset"] = x - x_in
            fin = _w(W, "final.table").reshape(2, -1) + t0
            shift, scale = fin[0], fin[1]
            v = linear(W, "final", modulate(x, shift, scale, cfg.norm_eps))
            return v, m0
        vec = t0 + linear(W, "p_emb.fc2", silu(linear(W, "p_emb.fc1", self.pooled)))
        img = linear(W, "x_emb", x_tok)
        txt = linear(W, "txt_in", self.text)
        x = None
        for i in range(nl):
            if i == nf:
                cur = img if x is None else x[:n]
                if not full:
                    img = cur + state["offset"]
                    x = None
                    break
                img_in = cur
            if i < cfg.num_dual:
                img, txt, m = mm_dual_block(W, i, img, txt, vec, cfg, self.ang, cache)
            else:
                if x is None:
                    x = torch.cat([img, txt])
                x, m = mm_single_block(W, i - cfg.num_dual, x, vec, cfg, self.ang, cache)
                img = x[:n]
            if i == 0:
                m0 = m[:n]
        if x is not None:
            img = x[:n]
        if full and nf < nl:
            state["offset"] = img - img_in
        fm = linear(W, "final.mod", silu(vec)).reshape(2, -1)
        v = linear(W, "final", modulate(img, fm[0], fm[1], cfg.norm_eps))
        return v, m0


def rel_l1(m, m_prev) -> float:
    """sum|m - m_prev| / sum|m_prev| in fp64 accumulation."""
    return float((m.double() - m_prev.double()).abs().sum() / m_prev.double().abs().sum())


@_strict
def denoise(model: OracleDiT, x0_lat: torch.Tensor, num_steps: int, flags=None, policy=None,
            return_all=True):
    """Euler flow-matching sampler t_i = i/N, x += (1/N)·v (fitted).

    Exactly one of ``flags`` (static per_step_full) or ``policy``
    (:class:`RelL1Policy`-like with ``decide``) drives the cache.  Returns
    ``(latents per step [N+1], flags taken, rel values)``.
    """
    cfg = model.cfg
    x = patchify(x0_lat.to(model.device, f32), cfg.patch)
    state = {}
    lat = [x0_lat.to("cpu", f32)]
    taken, rels = [], []
    acc = 0.0
    m_prev = None
    for i in range(num_steps):
        t = i / num_steps
        if policy is None:
            full = bool(flags[i]) if flags is not None else True
            v, m0 = model.velocity(x, t, full=full, state=state)
        else:
            # the probe (block 0's modulated input) is computed before the decision
            full_probe, _ = _probe(model, x, t)
            rel = float("nan") if m_prev is None else rel_l1(full_probe, m_prev)
            # the rule restated in the oracle (schedule_oracle.rel_l1_decide), not the product's
            full, acc = rel_l1_decide(i + 1, num_steps, acc, 0.0 if m_prev is None else rel, policy.threshold,
                                      policy.warmup, policy.force_last)
            rels.append(rel)
            m_prev = full_probe
            v, m0 = model.velocity(x, t, full=full, state=state)
        taken.append(full)
        x = x + (1.0 / num_steps) * v
        if return_all:
            lat.append(unpatchify(x, model.grid, cfg.patch, cfg.latent_channels).cpu())
    if not return_all:
        lat.append(unpatchify(x, model.grid, cfg.patch, cfg.latent_channels).cpu())
    return lat, taken, rels


def _probe(model: OracleDiT, x_tok, t):
    """Block 0's first modulated input (video tokens) without running the model."""
    cfg, W = model.cfg, model.W
    t0 = model._temb(t)
    if cfg.family == "single-dit":
        tmod = linear(W, "t_block", silu(t0))
        H = cfg.hidden_size
        mods = (tmod + _w(W, "blocks.0.table")).reshape(6, H)
        x = linear(W, "x_emb", x_tok)
        return modulate(x, mods[0], mods[1], cfg.norm_eps), None
    vec = t0 + linear(W, "p_emb.fc2", silu(linear(W, "p_emb.fc1", model.pooled)))
    H = cfg.hidden_size
    img = linear(W, "x_emb", x_tok)
    if cfg.num_dual:
        mi = linear(W, "dual.0.img.mod", silu(vec)).reshape(6, H)
    else:
        mi = linear(W, "single.0.mod", silu(vec)).reshape(6, H)
    return modulate(img, mi[0], mi[1], cfg.norm_eps), None


@_strict
def denoise_windows(models, x0_lat: torch.Tensor, num_steps: int, clips, flags=None):
    """Temporal MultiDiffusion (Eq. 3) — fp32 restatement.

    ``models[k]`` is an :class:`OracleDiT` for clip ``k`` (clip geometry; each keeps its
    own cache state), ``clips`` the WindowPlan's ``(start, end)`` latent-frame ranges.
    Every step each clip ``x'[:, s:e]`` takes one Euler step; frame ``i`` then becomes
    the mean over the clips covering it (sum in clip order / |S(i)|).  Returns the latent
    after every step (``num_steps + 1`` entries).
    """
    cfg = models[0].cfg
    x = x0_lat.to(models[0].device, f32).clone()
    states = [{} for _ in clips]
    out = [x.cpu()]
    count = torch.zeros(x.shape[1], device=x.device)
    for s, e in clips:
        count[s:e] += 1
    for i in range(num_steps):
        t = i / num_steps
        full = True if flags is None else bool(flags[i])
        acc = torch.zeros_like(x)
        for (s, e), m, st in zip(clips, models, states):
            tok = patchify(x[:, s:e], cfg.patch)
            v, _ = m.velocity(tok, t, full=full, state=st)
            tok = tok + (1.0 / num_steps) * v
            acc[:, s:e] += unpatchify(tok, m.grid, cfg.patch, cfg.latent_channels)
        x = acc / count[None, :, None, None]
        out.append(x.cpu())
    return out
