"""B200-native DiT denoise hot path of Aquarius (arXiv 2505.10584).

Public API (drop-in for the reference's cache-schedule boundary,
``ditplan/__init__.py:58-67`` + ``inference.py:21-86,282-315``):

* ``plan_cache``, ``CacheSchedule``, ``CACHE_MODES``,
  ``DEFAULT_CACHED_COST_FRACTION``, ``dit_parallel_latency``,
  ``composite_speedup``, ``ConfigError``, ``PlanningError``, ``DimensionError``
* ``plan_vae_tiles`` / ``TilePlan`` / ``Tile`` and ``plan_temporal_windows`` /
  ``WindowPlan`` (``inference.py:89-279``), with GPU blend / Eq. 3 kernels
* geometry ``Bucket`` / ``LatentShape`` / ``VaeSpec`` / ``latent_shape`` /
  ``token_count`` / ``snap_bucket`` (``buckets.py:17-122``)
* the planner formulas the path is sized by: ``ModelArch``, ``TABLE2_FIT``,
  ``estimate_param_count``, ``flops_per_microstep``, ``tp_sp_layer_comm``,
  ``cp_gate_and_comm`` / ``CP_TOKEN_GATE``, ``ChunkSpec`` / ``ChunkTable`` /
  ``BUILTIN_CHUNKS`` / ``load_chunk_table``, ``resolved_param_count`` (``config.py``, ``presets.py``, ``simulate.py``, ``comm.py``,
  ``memory.py``; see ``planner.py``)
* new: ``RelL1Policy``, ``DiTConfig`` + presets, ``SingleDiT`` / ``MMDiT``
  (model construction), ``denoise`` (sampler loop), ``denoise_windows``
  (temporal MultiDiffusion); multi-GPU
  groups ``Ulysses`` (sequence parallel) and ``TensorSP`` (TP-SP, Single-DiT).

The model/sampler symbols need CUDA and ``libaqb.so`` (hand-written sm_100a
kernels); they are imported lazily so the schedule API works anywhere.
"""

from .config import (
    MM_DIT_13B,
    PRESETS,
    SINGLE_DIT_2B,
    TINY_MM,
    Bucket,
    LatentShape,
    TINY_SINGLE,
    DiTConfig,
    VaeSpec,
    VideoSpec,
    flops_per_step,
    latent_shape,
    snap_bucket,
    snap_to_multiple,
    token_count,
    video_token_count,
)
from .errors import ConfigError, DimensionError, NativeError, PlanningError
from .schedule import (
    CACHE_MODES,
    DEFAULT_CACHED_COST_FRACTION,
    CacheSchedule,
    RelL1Policy,
    composite_speedup,
    dit_parallel_latency,
    front_block_count,
    no_cache,
    plan_cache,
)

from .tiling import Tile, TilePlan, WindowPlan, plan_temporal_windows, plan_vae_tiles
from .planner import (
    BUILTIN_CHUNKS,
    CP_TOKEN_GATE,
    TABLE2_FIT,
    ChunkSpec,
    ChunkTable,
    ModelArch,
    chunk_retained_bytes,
    cp_gate_and_comm,
    estimate_param_count,
    flops_per_microstep,
    load_chunk_table,
    resolved_param_count,
    tp_sp_layer_comm,
)

__version__ = "0.1.0"

_LAZY = {
    "SingleDiT": ("model", "SingleDiT"),
    "MMDiT": ("model", "MMDiT"),
    "build_model": ("model", "build_model"),
    "denoise": ("sampler", "denoise"),
    "DenoiseResult": ("sampler", "DenoiseResult"),
    "denoise_windows": ("sampler", "denoise_windows"),
    "SingleDiTTP": ("model", "SingleDiTTP"),
    "Ulysses": ("parallel", "Ulysses"),
    "TensorSP": ("parallel", "TensorSP"),
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)


__all__ = [
    "CACHE_MODES", "DEFAULT_CACHED_COST_FRACTION", "CacheSchedule", "ConfigError", "DimensionError",
    "DiTConfig", "MM_DIT_13B", "NativeError", "PRESETS", "PlanningError", "RelL1Policy", "SINGLE_DIT_2B",
    "TINY_MM", "TINY_SINGLE", "VaeSpec", "VideoSpec", "composite_speedup", "dit_parallel_latency",
    "flops_per_step", "front_block_count", "latent_shape", "no_cache", "plan_cache", "token_count",
    "Bucket", "LatentShape", "snap_bucket", "snap_to_multiple", "video_token_count",
    "load_chunk_table", "resolved_param_count",
    "SingleDiT", "MMDiT", "SingleDiTTP", "build_model", "denoise", "DenoiseResult", "denoise_windows",
    "Ulysses", "TensorSP",
    "Tile", "TilePlan", "WindowPlan", "plan_vae_tiles", "plan_temporal_windows",
    "BUILTIN_CHUNKS", "CP_TOKEN_GATE", "TABLE2_FIT", "ChunkSpec", "ChunkTable", "ModelArch", "chunk_retained_bytes",
    "cp_gate_and_comm", "estimate_param_count", "flops_per_microstep", "tp_sp_layer_comm",
]
