"""Analytical model of the path — the reference planner's formulas the hot path is
sized and judged by, restated with the same
signatures, value types and ``ConfigError`` paths so callers of ``ditplan`` find
them here too.  Each is checked against values produced by the reference itself
(``tests/golden/planner.json``, ``tests/golden/make_golden_planner.py``).

* :class:`ModelArch` (``config.py:25-65``) and :data:`TABLE2_FIT` (``presets.py:20-31``);
  :func:`model_arch` maps a :class:`~paper_2505_10584_b200.config.DiTConfig` onto it.
* :func:`estimate_param_count` (``config.py:224-249``) and :func:`flops_per_microstep`
  (``simulate.py:60-73``) — the FLOP convention the bench's roofline numbers use.
* :func:`tp_sp_layer_comm` (``comm.py:28-53``) and :func:`cp_gate_and_comm` with
  :data:`CP_TOKEN_GATE` (``comm.py:19,65-96``) — the cost of the two parallel
  layouts the runtime implements (``parallel.TensorSP``, ``parallel.Ulysses``).
  As SURVEY §8(a) a11 notes, the 200k-token gate is a training-planner rule; the
  runtime does not apply it to inference.
* :class:`ChunkSpec` / :class:`ChunkTable` / :data:`BUILTIN_CHUNKS` and
  :func:`chunk_retained_bytes` (``memory.py:30-107``) — the per-op table (Table 2
  of the paper) whose rows the kernels in ``csrc/`` implement.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

from .errors import ConfigError

ADALN_MODES = ("shared-weights", "per-block-dedicated")
CP_TOKEN_GATE = 200_000
DEFAULT_COLLECTIVE_LATENCY_MS = 0.02


@dataclass(frozen=True)
class ModelArch:
    """Transformer dims as the planner sees them (``param_count`` optional, supplied wins)."""

    hidden_size: int
    num_heads: int
    num_layers: int
    ffn_multiplier: int = 4
    adaln_mode: str = "per-block-dedicated"
    patch_t: int = 1
    patch_h: int = 2
    patch_w: int = 2
    param_count: float | None = None
    extra_unpartitioned_layers: tuple = ("patchify", "final_proj")

    def __post_init__(self):
        for field in ("hidden_size", "num_heads", "num_layers", "ffn_multiplier"):
            v = getattr(self, field)
            if not isinstance(v, int) or v < 0:
                raise ConfigError("must be a non-negative integer", f"model.{field}")
        if self.hidden_size < 1 or self.num_heads < 1:
            raise ConfigError("hidden_size and num_heads must be >= 1", "model")
        for field in ("patch_t", "patch_h", "patch_w"):
            if getattr(self, field) < 1:
                raise ConfigError("patch dims must be >= 1", f"model.{field}")
        if self.adaln_mode not in ADALN_MODES:
            raise ConfigError(f"adaln_mode must be one of {ADALN_MODES}", "model.adaln_mode")
        if self.param_count is not None and self.param_count <= 0:
            raise ConfigError("param_count must be positive when supplied", "model.param_count")
        object.__setattr__(self, "extra_unpartitioned_layers", tuple(self.extra_unpartitioned_layers))

    @property
    def patch_volume(self) -> int:
        return self.patch_t * self.patch_h * self.patch_w


TABLE2_FIT = ModelArch(hidden_size=3072, num_heads=24, num_layers=54, ffn_multiplier=4,
                       adaln_mode="per-block-dedicated", patch_t=1, patch_h=2, patch_w=2, param_count=13.4e9)
TABLE2_FIT_FITTED_FIELDS = ("hidden_size", "num_heads", "num_layers")


def model_arch(cfg) -> ModelArch:
    """The planner's view of an executable :class:`DiTConfig` (AdaLN-single for Single-DiT,
    per-block AdaLN-zero for MM-DiT; the dual/single split and cross-attention are not
    represented in the planner's accounting)."""
    pt, ph, pw = cfg.patch
    return ModelArch(hidden_size=cfg.hidden_size, num_heads=cfg.num_heads, num_layers=cfg.num_layers,
                     ffn_multiplier=cfg.ffn_dim // cfg.hidden_size,
                     adaln_mode="shared-weights" if cfg.family == "single-dit" else "per-block-dedicated",
                     patch_t=pt, patch_h=ph, patch_w=pw)


@dataclass(frozen=True)
class ParamCountEstimate:
    total: float
    transformer: float
    adaln: float
    embedding_head: float


def estimate_param_count(arch: ModelArch, latent_channels: int = 8) -> ParamCountEstimate:
    """Blocks: (4 + 2·ffn)·H² each; AdaLN: 6·H² per block (dedicated) or once (shared);
    patch embed + final projection: 2·(patch volume · C)·H."""
    h2 = arch.hidden_size * arch.hidden_size
    blocks = arch.num_layers * (4 + 2 * arch.ffn_multiplier) * h2
    adaln = (arch.num_layers if arch.adaln_mode == "per-block-dedicated" else 1) * 6 * h2
    head = 2 * arch.patch_volume * latent_channels * arch.hidden_size
    return ParamCountEstimate(total=float(blocks + adaln + head), transformer=float(blocks), adaln=float(adaln),
                              embedding_head=float(head))


def resolved_param_count(arch: ModelArch) -> float:
    """The supplied ``param_count`` when present, the estimate otherwise (``config.py:252-256``)."""
    if arch.param_count is not None:
        return float(arch.param_count)
    return estimate_param_count(arch).total


def flops_per_microstep(arch: ModelArch, B: int, S: int) -> float:
    """Forward FLOPs of one micro-batch: per layer 4·B·S²·H (QKᵀ and PV) + 2·B·S·(4 + 2·ffn)·H²
    (token linears), plus 2·B·S times the embedding/head parameter term."""
    H = arch.hidden_size
    token_linear = (4 + 2 * arch.ffn_multiplier) * H * H
    layer = 4 * B * S * S * H + 2 * B * S * token_linear
    return arch.num_layers * layer + 2 * B * S * estimate_param_count(arch).embedding_head


def tp_sp_layer_comm(B: int, S: int, H: int, tp: int, act_bytes: int, intra_bw: float, overlap_fraction: float,
                     collective_latency_ms: float = DEFAULT_COLLECTIVE_LATENCY_MS) -> tuple[float, float]:
    """(raw, exposed) ms of one layer's TP-SP all-gather + reduce-scatter (ring model:
    each moves (tp-1)/tp of B·S·H elements)."""
    if tp < 1:
        raise ConfigError("tp must be >= 1", "parallel.tp")
    if not 0.0 <= overlap_fraction <= 1.0:
        raise ConfigError("overlap fraction must be in [0, 1]", "overlap.tp_sp_fraction")
    if tp == 1:
        return (0.0, 0.0)
    moved = 2 * B * S * H * act_bytes * (tp - 1) / tp
    raw = moved / intra_bw * 1e3 + 2 * collective_latency_ms
    return (raw, raw * (1.0 - overlap_fraction))


@dataclass(frozen=True)
class CpGateResult:
    enabled: bool
    time_ms: float
    violation: str | None = None


def cp_gate_and_comm(tokens_batch: int, B: int, S: int, H: int, cp: int, act_bytes: int, inter_bw: float,
                     collective_latency_ms: float = DEFAULT_COLLECTIVE_LATENCY_MS) -> CpGateResult:
    """Context parallelism is admitted only above :data:`CP_TOKEN_GATE` tokens (a request
    below it comes back as a violation, never an exception); its cost is two all-to-alls
    of (cp-1)/cp of B·S·H elements per layer at inter-node bandwidth."""
    if cp < 1:
        raise ConfigError("cp must be >= 1", "parallel.cp")
    if cp == 1:
        return CpGateResult(enabled=False, time_ms=0.0)
    if tokens_batch <= CP_TOKEN_GATE:
        return CpGateResult(enabled=False, time_ms=0.0,
                            violation=f"cp={cp} rejected: {tokens_batch} tokens is below the "
                                      f"{CP_TOKEN_GATE} ultra-long-sequence threshold")
    moved = 2 * B * S * H * act_bytes * (cp - 1) / cp
    return CpGateResult(enabled=True, time_ms=moved / inter_bw * 1e3 + 2 * collective_latency_ms)


@dataclass(frozen=True)
class ChunkSpec:
    """One fused op of a block: retained bytes = coeff_bsh·B·S·H + coeff_bas·B·A·S (÷ tp);
    ``fwd_latency_ms`` profiled at the owning table's reference shape."""

    name: str
    coeff_bsh: float
    coeff_bas: float = 0.0
    fwd_latency_ms: float = 1.0
    recomputable: bool = True
    offloadable: bool = True

    def __post_init__(self):
        if self.coeff_bsh < 0 or self.coeff_bas < 0:
            raise ConfigError("coefficients must be >= 0", f"chunk.{self.name}")
        if self.fwd_latency_ms <= 0:
            raise ConfigError("fwd_latency_ms must be positive", f"chunk.{self.name}")

    @property
    def is_attention_class(self) -> bool:
        return self.coeff_bas > 0


def chunk_retained_bytes(chunk: ChunkSpec, B: int, S: int, H: int, A: int, tp: int) -> int:
    if tp < 1:
        raise ConfigError("tp must be >= 1", "parallel.tp")
    return round((chunk.coeff_bsh * B * S * H + chunk.coeff_bas * B * A * S) / tp)


@dataclass(frozen=True)
class ChunkTable:
    chunks: tuple
    ref_batch: int = 1
    ref_seqlen: int = 115_200
    ref_hidden: int = 3072
    ref_heads: int = 24
    ref_tp: int = 8

    def __post_init__(self):
        names = [c.name for c in self.chunks]
        if len(set(names)) != len(names):
            raise ConfigError("duplicate chunk names", "chunks")

    def by_name(self, name: str) -> ChunkSpec:
        for c in self.chunks:
            if c.name == name:
                return c
        raise ConfigError(f"unknown chunk {name!r}", "chunks")

    def names(self) -> tuple:
        return tuple(c.name for c in self.chunks)


# The paper's Table 2 (125 frames at 1280x720 = 115,200 tokens, 24 heads, H 3072, TP 8);
# the kernel implementing each row is named in DESIGN.md §3.
BUILTIN_CHUNKS = ChunkTable(chunks=(
    ChunkSpec("flash_attention", coeff_bsh=2, coeff_bas=64, fwd_latency_ms=127.5),
    ChunkSpec("out_linear_reduce_scatter", coeff_bsh=2, fwd_latency_ms=13.4),
    ChunkSpec("ffn_linear2_reduce_scatter", coeff_bsh=2, fwd_latency_ms=8.9),
    ChunkSpec("all_gather_ffn_linear1", coeff_bsh=8, fwd_latency_ms=8.6),
    ChunkSpec("all_gather_qkv_linear", coeff_bsh=6, fwd_latency_ms=7.7),
    ChunkSpec("fused_qknorm", coeff_bsh=4, fwd_latency_ms=1.9),
    ChunkSpec("gate", coeff_bsh=2, fwd_latency_ms=0.36),
    ChunkSpec("layernorm_scale_shift", coeff_bsh=4, fwd_latency_ms=0.58),
    ChunkSpec("gelu", coeff_bsh=8, fwd_latency_ms=0.64),
))


_CHUNK_KEYS = ("name", "coeff_bsh", "coeff_bas", "fwd_latency_ms", "recomputable", "offloadable")
_TABLE_META = ("ref_batch", "ref_seqlen", "ref_hidden", "ref_heads", "ref_tp")


def load_chunk_table(path) -> ChunkTable:
    """A :class:`ChunkTable` from a JSON file ``{"chunks": [{name, coeff_bsh, ...}], ref_*...}``
    (``memory.py:110-134``): same accepted keys, same ``ConfigError`` messages and paths."""
    try:
        doc = json.loads(Path(path).read_text())
    except OSError as exc:
        raise ConfigError(f"cannot read chunk table: {exc}", str(path)) from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"invalid JSON: {exc}", str(path)) from exc
    if not isinstance(doc, dict) or "chunks" not in doc:
        raise ConfigError("expected an object with a 'chunks' array", str(path))
    chunks = []
    for i, entry in enumerate(doc["chunks"]):
        if not isinstance(entry, dict) or "name" not in entry:
            raise ConfigError("chunk entry needs a name", f"chunks[{i}]")
        extra = sorted(set(entry) - set(_CHUNK_KEYS))
        if extra:
            raise ConfigError("unknown key", f"chunks[{i}].{extra[0]}")
        chunks.append(ChunkSpec(**entry))
    return ChunkTable(chunks=tuple(chunks), **{k: doc[k] for k in _TABLE_META if k in doc})
