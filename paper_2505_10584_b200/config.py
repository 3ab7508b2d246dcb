"""Model dims, video geometry and FLOP conventions for the denoise path.

* :class:`DiTConfig` carries what ``ditplan.config.ModelArch``
  (``pkg/src/ditplan/config.py:25-65``) carries — hidden size, heads, layers,
  FFN multiplier, AdaLN mode, patch — plus what an *executing* model needs and
  the reference never had: the family (Single-DiT / MM-DiT, ``PAPER.md:15-17,
  103,106``), the dual/single split, text dims, 3D-RoPE split and base.
  Everything not published is a builder choice ("fitted").
* :class:`Bucket`, :class:`LatentShape`, :func:`latent_shape`, :func:`token_count`,
  :func:`snap_bucket` restate ``buckets.py:33-122`` (same signatures and result types).
* :func:`flops_per_step` follows the reference convention
  ``simulate.py:60-73`` (4·S²·H attention + 2·S·(4+2·ffn)·H² linears per
  layer + head), extended with the Single-DiT cross-attention term.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

from .errors import ConfigError, DimensionError

FAMILIES = ("single-dit", "mm-dit")
ADALN_MODES = ("shared-weights", "per-block-dedicated")  # config.py:19


@dataclass(frozen=True)
class VaeSpec:
    """Causal video VAE compression (``buckets.py:17-30``)."""

    temporal_ratio: int = 4
    spatial_ratio: int = 8
    latent_channels: int = 8

    def __post_init__(self):
        if self.temporal_ratio < 1 or self.spatial_ratio < 1:
            raise ConfigError("compression ratios must be >= 1", "vae")
        if self.latent_channels < 1:
            raise ConfigError("latent_channels must be >= 1", "vae.latent_channels")


def latent_shape(frames: int, height: int, width: int, vae: VaeSpec = VaeSpec()) -> tuple[int, int, int]:
    """Pre-patchify latent dims ``(1+(F-1)/4, H/8, W/8)`` — ``buckets.py:65-86``."""
    if frames < 1:
        raise DimensionError("frames must be >= 1", "frames")
    if (frames - 1) % vae.temporal_ratio != 0:
        raise DimensionError(
            f"frames-1 must be divisible by the temporal ratio {vae.temporal_ratio}", "frames"
        )
    if height % vae.spatial_ratio != 0:
        raise DimensionError(f"height {height} not divisible by spatial ratio {vae.spatial_ratio}", "height")
    if width % vae.spatial_ratio != 0:
        raise DimensionError(f"width {width} not divisible by spatial ratio {vae.spatial_ratio}", "width")
    return (1 + (frames - 1) // vae.temporal_ratio, height // vae.spatial_ratio, width // vae.spatial_ratio)


@dataclass(frozen=True)
class Bucket:
    """One shape class of videos: ``{batch, frames, height, width}`` (``buckets.py:33-51``)."""

    batch: int
    frames: int
    height: int
    width: int

    def __post_init__(self):
        for name in ("batch", "frames", "height", "width"):
            if getattr(self, name) < 1:
                raise ConfigError("must be >= 1", f"bucket.{name}")

    def key(self) -> tuple[int, int, int, int]:
        return (self.batch, self.frames, self.height, self.width)

    def label(self) -> str:
        return f"{{{self.batch},{self.frames},{self.height},{self.width}}}"


@dataclass(frozen=True)
class LatentShape:
    """Latent geometry of one video plus its post-patchify token counts (``buckets.py:54-62``)."""

    t_lat: int
    h_lat: int
    w_lat: int
    tokens: int
    tokens_batch: int


def _patch_of(arch) -> tuple[int, int, int]:
    """Patch dims of a planner ``ModelArch`` (``patch_t/h/w``) or an executable ``DiTConfig``
    (``patch``); the reference default 1x2x2 when ``arch`` is None (``buckets.py:91``)."""
    if arch is None:
        return (1, 2, 2)
    if hasattr(arch, "patch_t"):
        return (arch.patch_t, arch.patch_h, arch.patch_w)
    return tuple(arch.patch)


def token_count(bucket: Bucket, vae: VaeSpec = VaeSpec(), arch=None) -> LatentShape:
    """Tokens per video (post-patchify, ceiling division per axis) and per batch —
    ``buckets.py:89-98``, same signature and result type."""
    pt, ph, pw = _patch_of(arch)
    t_lat, h_lat, w_lat = latent_shape(bucket.frames, bucket.height, bucket.width, vae)
    tokens = math.ceil(t_lat / pt) * math.ceil(h_lat / ph) * math.ceil(w_lat / pw)
    return LatentShape(t_lat=t_lat, h_lat=h_lat, w_lat=w_lat, tokens=tokens, tokens_batch=bucket.batch * tokens)


def video_token_count(frames: int, height: int, width: int, patch=(1, 2, 2), vae: VaeSpec = VaeSpec()) -> int:
    """Tokens of one ``frames x height x width`` video (the int :func:`token_count` gives as
    ``.tokens`` for a batch-1 bucket)."""
    pt, ph, pw = patch
    t, h, w = latent_shape(frames, height, width, vae)
    return math.ceil(t / pt) * math.ceil(h / ph) * math.ceil(w / pw)


def snap_to_multiple(value: int, multiple: int) -> int:
    """Nearest positive multiple, ties round up (``buckets.py:101-104``)."""
    return max(multiple, int(multiple * math.floor(value / multiple + 0.5)))


def snap_bucket(bucket: Bucket, vae: VaeSpec = VaeSpec(), arch=None) -> Bucket:
    """Round height/width to the VAE x patch grain (480x854 -> 480x848), ``buckets.py:107-122``."""
    _, ph, pw = _patch_of(arch)
    height = snap_to_multiple(bucket.height, vae.spatial_ratio * ph)
    width = snap_to_multiple(bucket.width, vae.spatial_ratio * pw)
    if (height, width) == (bucket.height, bucket.width):
        return bucket
    return Bucket(bucket.batch, bucket.frames, height, width)


@dataclass(frozen=True)
class DiTConfig:
    """An executable DiT description.

    ``num_layers = num_dual + num_single`` for MM-DiT (dual-stream blocks
    first, then single-stream joint blocks over ``[video; text]``); Single-DiT
    uses ``num_single`` only (self-attn + cross-attn + MLP per block).
    """

    family: str
    hidden_size: int
    num_heads: int
    num_dual: int = 0
    num_single: int = 2
    ffn_multiplier: int = 4
    latent_channels: int = 8
    patch: tuple[int, int, int] = (1, 2, 2)
    text_dim: int = 4096          # mT5-XXL / MLLM (fitted)
    text_len: int = 256           # fitted
    pooled_dim: int = 768         # CLIP pooled features, MM-DiT only
    freq_dim: int = 256           # sinusoidal timestep features
    rope_theta: float = 1000.0    # "lower frequency base"; value fitted
    rope_split: tuple[int, int, int] | None = None   # (t, h, w) channels; default D/4, 3D/8, 3D/8
    norm_eps: float = 1e-6
    qk_norm_eps: float = 1e-6
    name: str = "custom"

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ConfigError(f"family must be one of {FAMILIES}", "model.family")
        for n in ("hidden_size", "num_heads", "ffn_multiplier", "latent_channels", "text_dim",
                  "text_len", "pooled_dim", "freq_dim"):
            v = getattr(self, n)
            if not isinstance(v, int) or v < 1:
                raise ConfigError("must be a positive integer", f"model.{n}")
        if self.num_dual < 0 or self.num_single < 0 or self.num_layers < 1:
            raise ConfigError("need at least one block", "model.num_layers")
        if self.family == "single-dit" and self.num_dual:
            raise ConfigError("single-dit has no dual-stream blocks", "model.num_dual")
        if self.hidden_size % self.num_heads:
            raise ConfigError("hidden_size must divide by num_heads", "model.num_heads")
        d = self.head_dim
        if d % 16 or d > 256:
            raise ConfigError("head_dim must be a multiple of 16 and <= 256", "model.head_dim")
        if self.hidden_size % 64:
            raise ConfigError("hidden_size must be a multiple of 64", "model.hidden_size")
        st, sh, sw = self.rope_dims
        if st + sh + sw != d or st % 2 or sh % 2 or sw % 2:
            raise ConfigError("rope_split must be even and sum to head_dim", "model.rope_split")
        if any(p < 1 for p in self.patch):
            raise ConfigError("patch dims must be >= 1", "model.patch")

    @property
    def num_layers(self) -> int:
        return self.num_dual + self.num_single

    @property
    def head_dim(self) -> int:
        return self.hidden_size // self.num_heads

    @property
    def patch_volume(self) -> int:
        return self.patch[0] * self.patch[1] * self.patch[2]

    @property
    def patch_dim(self) -> int:
        return self.patch_volume * self.latent_channels

    @property
    def adaln_mode(self) -> str:
        # AdaLN-single shares the modulation regressor;
        # MM-DiT uses per-block AdaLN-zero.
        return "shared-weights" if self.family == "single-dit" else "per-block-dedicated"

    @property
    def ffn_dim(self) -> int:
        return self.ffn_multiplier * self.hidden_size

    @property
    def rope_dims(self) -> tuple[int, int, int]:
        if self.rope_split is not None:
            return tuple(self.rope_split)
        d = self.head_dim
        t = (d // 4) // 2 * 2
        hw = (d - t) // 2 // 2 * 2
        return (d - 2 * hw, hw, hw)

    def param_count(self) -> int:
        """Exact parameter count of the executable model built from this config."""
        H, F, C = self.hidden_size, self.ffn_dim, self.patch_dim
        lin = lambda i, o: i * o + o  # noqa: E731
        tok = lin(self.freq_dim, H) + lin(H, H) + lin(C, H) + lin(H, C)
        attn_stream = lin(H, 3 * H) + 2 * self.head_dim + lin(H, H) + lin(H, F) + lin(F, H)
        if self.family == "single-dit":
            blk = attn_stream + lin(H, H) + lin(self.text_dim, 2 * H) + 2 * self.head_dim + lin(H, H) + 6 * H
            return tok + lin(H, 6 * H) + 2 * H + self.num_single * blk
        dual = 2 * (attn_stream + lin(H, 6 * H))
        single = attn_stream + lin(H, 6 * H)
        extra = lin(self.pooled_dim, H) + lin(H, H) + lin(self.text_dim, H) + lin(H, 2 * H)
        return tok + extra + self.num_dual * dual + self.num_single * single


@dataclass(frozen=True)
class VideoSpec:
    """A generation request's geometry: frames × height × width (pixels)."""

    frames: int
    height: int
    width: int

    def latent(self, vae: VaeSpec = VaeSpec()) -> tuple[int, int, int]:
        return latent_shape(self.frames, self.height, self.width, vae)

    def grid(self, cfg: DiTConfig) -> tuple[int, int, int]:
        t, h, w = self.latent(VaeSpec(latent_channels=cfg.latent_channels))
        pt, ph, pw = cfg.patch
        if t % pt or h % ph or w % pw:
            raise DimensionError("latent dims must divide by the patch", "video")
        return (t // pt, h // ph, w // pw)

    def tokens(self, cfg: DiTConfig) -> int:
        t, h, w = self.grid(cfg)
        return t * h * w


# ---------------------------------------------------------------------------
# Presets (BASELINE.json configs; dims are "fitted").
# ---------------------------------------------------------------------------

TINY_SINGLE = DiTConfig("single-dit", hidden_size=128, num_heads=4, num_single=2,
                        text_dim=128, text_len=16, name="tiny-single-dit")
TINY_MM = DiTConfig("mm-dit", hidden_size=128, num_heads=4, num_dual=1, num_single=1,
                    text_dim=128, text_len=16, pooled_dim=64, name="tiny-mm-dit")
SINGLE_DIT_2B = DiTConfig("single-dit", hidden_size=2048, num_heads=16, num_single=28,
                          text_dim=4096, text_len=256, name="single-dit-2b")
MM_DIT_13B = DiTConfig("mm-dit", hidden_size=3072, num_heads=24, num_dual=25, num_single=29,
                       text_dim=4096, text_len=256, pooled_dim=768, name="mm-dit-13.4b")

PRESETS = {c.name: c for c in (TINY_SINGLE, TINY_MM, SINGLE_DIT_2B, MM_DIT_13B)}

# BASELINE.json configs 1-4 (config 5 is the attention microbench).
VIDEO_TINY = None  # config 1 is specified directly as a 2x8x8 latent (tokens 32)
VIDEO_480P_17F = VideoSpec(17, 480, 832)     # 5x60x104 latent -> 7,800 tokens
VIDEO_480P_61F = VideoSpec(61, 480, 848)     # 16x60x106 -> 25,440 (854 snaps to 848)
VIDEO_720P_129F = VideoSpec(129, 720, 1280)  # 33x90x160 -> 118,800


def with_overrides(cfg: DiTConfig, **kw) -> DiTConfig:
    return replace(cfg, **kw)


# ---------------------------------------------------------------------------
# FLOP conventions (roofline numerators).
# ---------------------------------------------------------------------------

def attention_flops(s_q: int, s_kv: int, heads: int, head_dim: int) -> float:
    """QK^T + PV: 4·S_q·S_kv·D·A (softmax not counted) — SURVEY.md §8(d)."""
    return 4.0 * s_q * s_kv * head_dim * heads


def flops_per_step(cfg: DiTConfig, video_tokens: int) -> dict:
    """Forward FLOPs of one denoise step, split into attention / linear.

    Per layer: ``4·S²·H`` (attention) + ``2·S·(4H² + 2·ffn·H²)`` (linears),
    ``simulate.py:60-73``, with S = video (+ text for joint attention) tokens;
    Single-DiT adds cross-attention ``4·S_v·S_t·H`` + ``2·S_v·2H²``.  MM-DiT
    dual blocks run the text stream's linears on ``S_t`` tokens.
    """
    H, F, Sv, St = cfg.hidden_size, cfg.ffn_dim, video_tokens, cfg.text_len
    lin_per_tok = 2 * (4 * H * H + 2 * H * F)
    attn = lin = 0.0
    if cfg.family == "single-dit":
        for _ in range(cfg.num_single):
            attn += 4.0 * Sv * Sv * H + 4.0 * Sv * St * H
            lin += Sv * lin_per_tok + 2.0 * Sv * 2 * H * H
        # the text K/V projections are step-independent: computed once per
        # denoise call, not per step, so they are not counted here
    else:
        S = Sv + St
        attn += cfg.num_layers * 4.0 * S * S * H
        lin += cfg.num_dual * (Sv + St) * lin_per_tok + cfg.num_single * S * lin_per_tok
    head = 2.0 * Sv * cfg.patch_dim * H * 2
    return {"attention": attn, "linear": lin + head, "total": attn + lin + head}
