"""VAE tile plans and temporal MultiDiffusion windows — the steps either side of
the denoise loop.

Host planning mirrors the reference API so a caller can switch over:

* :func:`plan_vae_tiles` / :class:`TilePlan` / :class:`Tile` restate
  ``pkg/src/ditplan/inference.py:89-226`` (tiles advance by ``size -
  overlap`` per axis, the last tile end-aligned, round-robin devices,
  separable linear-ramp blend weights normalised by the covering total;
  ``PAPER.md:79,318``).
* :func:`plan_temporal_windows` / :class:`WindowPlan` restate
  ``inference.py:229-279`` (clip ``k`` covers ``[k·s, k·s+n)`` clamped to end
  at ``n'``; ``r = ceil((n'-n)/s) + 1``; Eq. 3 weights ``1/|S(i)|``;
  ``PAPER.md:407-417``).

The per-position arithmetic runs on the GPU: :func:`blend_tiles`
(``aqb_tile_blend``: every output element sums its covering tiles' ramp
weights and weighted values, then normalises) and :func:`average_windows`
(``aqb_window_average``: Eq. 3 over the clips covering each frame).  Both
read their inputs through arrays of device pointers, so tiles/clips may live
in other ranks' memory (peer pointers) and the sum order is fixed
(deterministic, identical on every rank).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ConfigError


# ----------------------------------------------------------------------------- VAE tiles
@dataclass(frozen=True)
class Tile:
    start: tuple[int, int, int]
    size: tuple[int, int, int]
    device: int


def axis_ramp(size: int, overlap: int) -> np.ndarray:
    """Raw 1-D profile: rises as (j+1)/(e+1) over the first e = min(overlap, size)
    entries, falls symmetrically over the last e, 1 elsewhere (``inference.py:167-176``).
    Two adjoining ramps sum to exactly 1 over their shared entries."""
    e = min(overlap, size)
    j = np.arange(size, dtype=np.float64)
    up = np.where(j < e, (j + 1.0) / (e + 1.0), 1.0)
    down = np.where(j >= size - e, (size - j) / (e + 1.0), 1.0)
    return np.minimum(np.minimum(up, down), 1.0)


def axis_starts(extent: int, size: int, overlap: int) -> list[int]:
    """Starts along one axis: stride ``size - overlap``, last tile end-aligned
    (``inference.py:179-186``)."""
    if size >= extent:
        return [0]
    out = list(range(0, extent - size + 1, size - overlap))
    if out[-1] + size < extent:
        out.append(extent - size)
    return out


@dataclass(frozen=True)
class TilePlan:
    latent: tuple[int, int, int]
    tiles: tuple[Tile, ...]
    overlap: tuple[int, int, int]
    devices: int
    parallel_speedup: float

    # -- separable profile ------------------------------------------------------------
    def ramps(self) -> list[np.ndarray]:
        size = self.tiles[0].size
        return [axis_ramp(size[a], self.overlap[a]) for a in range(3)]

    def tile_profile(self) -> np.ndarray:
        r0, r1, r2 = self.ramps()
        return (r0[:, None, None] * r1[None, :, None]) * r2[None, None, :]

    def starts_per_axis(self) -> list[list[int]]:
        return [sorted({t.start[a] for t in self.tiles}) for a in range(3)]

    def _region(self, tile: Tile):
        return tuple(slice(tile.start[a], tile.start[a] + tile.size[a]) for a in range(3))

    def total_weight(self) -> np.ndarray:
        """Sum of raw tile profiles at every latent position (the normaliser)."""
        prof = self.tile_profile()
        total = np.zeros(self.latent, dtype=np.float64)
        for tile in self.tiles:
            total[self._region(tile)] += prof
        return total

    def normalized_weight_sum(self) -> np.ndarray:
        prof, total = self.tile_profile(), self.total_weight()
        acc = np.zeros(self.latent, dtype=np.float64)
        for tile in self.tiles:
            reg = self._region(tile)
            acc[reg] += prof / total[reg]
        return acc

    def iter_weight_maps(self):
        prof, total = self.tile_profile(), self.total_weight()
        for tile in self.tiles:
            w = np.zeros(self.latent, dtype=np.float64)
            reg = self._region(tile)
            w[reg] = prof / total[reg]
            yield w

    def weight_maps(self) -> list[np.ndarray]:
        return list(self.iter_weight_maps())

    def tiles_of(self, device: int) -> list[int]:
        """Indices of the tiles assigned to ``device`` (round robin)."""
        return [i for i, t in enumerate(self.tiles) if t.device == device]


def plan_vae_tiles(latent, tile, overlap, devices: int = 1) -> TilePlan:
    """Tile a latent ``(T, H, W)`` for parallel VAE decode (``inference.py:189-226``).

    Validation order and ``ConfigError`` paths follow the reference; a tile
    larger than the latent degenerates to one tile.  ``parallel_speedup =
    tiles / ceil(tiles / devices)``.
    """
    latent, tile, overlap = tuple(latent), tuple(tile), tuple(overlap)
    if devices < 1:
        raise ConfigError("devices must be >= 1", "vae.devices")
    for a in range(3):
        if tile[a] < 1:
            raise ConfigError("tile size must be >= 1", f"vae.tile[{a}]")
        if overlap[a] < 0 or overlap[a] >= tile[a]:
            raise ConfigError("need tile size > overlap >= 0", f"vae.overlap[{a}]")
        if latent[a] < 1:
            raise ConfigError("latent dims must be >= 1", f"vae.latent[{a}]")
    size = tuple(min(tile[a], latent[a]) for a in range(3))
    st = [axis_starts(latent[a], size[a], overlap[a]) for a in range(3)]
    starts = [(t, h, w) for t in st[0] for h in st[1] for w in st[2]]
    tiles = tuple(Tile(start=s, size=size, device=i % devices) for i, s in enumerate(starts))
    return TilePlan(latent=latent, tiles=tiles, overlap=overlap, devices=devices,
                    parallel_speedup=len(tiles) / math.ceil(len(tiles) / devices))


# ------------------------------------------------------------------------ temporal windows
@dataclass(frozen=True)
class WindowPlan:
    n_prime: int
    window: int
    stride: int
    clips: tuple[tuple[int, int], ...]

    @property
    def num_clips(self) -> int:
        return len(self.clips)

    def multiplicity(self) -> np.ndarray:
        """|S(i)|: clips covering each latent frame."""
        starts = np.array([c[0] for c in self.clips])
        i = np.arange(self.n_prime)[:, None]
        return ((i >= starts[None, :]) & (i < starts[None, :] + self.window)).sum(1).astype(np.int64)

    def averaging_weights(self, index: int) -> float:
        """Eq. 3 weight 1/|S(i)| for frame ``index``."""
        c = int(self.multiplicity()[index])
        if c == 0:
            raise ConfigError(f"index {index} uncovered", "windows")
        return 1.0 / c


def plan_temporal_windows(n_prime: int, n: int, s: int) -> WindowPlan:
    """Sliding window of length ``n``, stride ``s`` over ``n'`` latent frames
    (``inference.py:254-279``; ``PAPER.md:411``)."""
    if n_prime < 1 or n < 1:
        raise ConfigError("lengths must be >= 1", "windows")
    if n > n_prime:
        raise ConfigError(f"window {n} longer than latent {n_prime}", "windows.n")
    if s < 1:
        raise ConfigError("stride must be >= 1", "windows.stride")
    if s > n:
        raise ConfigError(f"stride {s} exceeds window {n}: indices between clips would go uncovered",
                          "windows.stride")
    r = math.ceil((n_prime - n) / s) + 1
    clips = tuple((min(k * s, n_prime - n), min(k * s, n_prime - n) + n) for k in range(r))
    return WindowPlan(n_prime=n_prime, window=n, stride=s, clips=clips)


# ----------------------------------------------------------------------------- GPU kernels
def _check_f32(t: torch.Tensor, shape, what: str, device):
    """The blend kernels index every tensor as a dense f32 array of ``shape`` on ``device``."""
    if not isinstance(t, torch.Tensor):
        raise ConfigError(f"{what} must be a tensor", what)
    if t.dtype != torch.float32 or not t.is_cuda or t.device != device:
        raise ConfigError(f"{what} must be float32 on {device}, got {t.dtype} on {t.device}", what)
    if not t.is_contiguous():
        raise ConfigError(f"{what} must be contiguous", what)
    if tuple(t.shape) != tuple(shape):
        raise ConfigError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}", what)


def _ptrs(items, shape, what, device):
    """Device addresses of ``items``: tensors are validated against ``shape``; plain ints are
    documented raw device addresses (e.g. a peer rank's buffer over NVLink) and pass as is."""
    out = []
    for k, t in enumerate(items):
        if isinstance(t, torch.Tensor):
            _check_f32(t, shape, f"{what}[{k}]", device)
            out.append(t.data_ptr())
        elif isinstance(t, int) and t > 0:
            out.append(int(t))
        else:
            raise ConfigError(f"{what}[{k}] must be an f32 CUDA tensor or a device address", what)
    return torch.tensor(out, dtype=torch.int64, device=device)


def blend_tiles(plan: TilePlan, tiles, out: torch.Tensor) -> torch.Tensor:
    """out[c, t, h, w] = sum_k w_k(t,h,w) · tile_k[c, t-t_k, h-h_k, w-w_k] with the plan's
    normalised ramp weights (``TilePlan.iter_weight_maps``), on the GPU.

    ``tiles``: per plan tile (plan order), an f32 CUDA tensor ``[C, *tile.size]`` or the
    device address of one (e.g. another rank's buffer over NVLink).  ``out``: f32
    ``[C, *plan.latent]``.
    """
    if len(tiles) != len(plan.tiles):
        raise ConfigError("one tensor per plan tile", "vae.tiles")
    if not isinstance(out, torch.Tensor) or out.dim() != 4:
        raise ConfigError("out must be an f32 CUDA tensor [C, T, H, W]", "vae.out")
    dev = out.device
    C = out.shape[0]
    _check_f32(out, (C, *plan.latent), "vae.out", dev)
    st = plan.starts_per_axis()
    starts = torch.tensor(st[0] + st[1] + st[2], dtype=torch.int32, device=dev)
    ptrs = _ptrs(tiles, (C, *plan.tiles[0].size), "vae.tiles", dev)
    ops.tile_blend(ptrs, starts, [len(a) for a in st], plan.tiles[0].size, plan.overlap, plan.latent, out)
    return out


class PeerTiles:
    """Parallel VAE decode across the GPUs of one box (``PAPER.md:79,318``; plan
    ``inference.py:189-226``): rank r decodes the tiles ``plan.tiles_of(r)`` into its slots
    of a symmetric peer buffer, and :meth:`blend` on any rank reads every tile straight
    from its owner's memory over NVLink (``aqb_tile_blend`` takes per-tile device
    addresses), so the blended latent needs no gather.  Collective construction (every
    rank, same plan and channel count)."""

    def __init__(self, plan: TilePlan, sp, channels: int, device="cuda"):
        from .parallel import PeerBuffers

        if plan.devices != sp.P:
            raise ConfigError(f"plan for {plan.devices} devices, group of {sp.P}", "vae.devices")
        self.plan, self.sp, self.channels = plan, sp, channels
        self.tile_elems = channels * int(np.prod(plan.tiles[0].size))
        self.slots = [plan.tiles_of(r) for r in range(sp.P)]
        per_rank = max(len(s) for s in self.slots)
        self.peer = PeerBuffers(sp, {"tiles": per_rank * self.tile_elems * 4}, device)
        self._local = self.peer.local("tiles", (per_rank, channels, *plan.tiles[0].size), torch.float32)
        base = self.peer.ptrs("tiles")
        self._ptrs = [0] * len(plan.tiles)
        for r, idx in enumerate(self.slots):
            for j, i in enumerate(idx):
                self._ptrs[i] = base[r] + j * self.tile_elems * 4

    def local_tile(self, i: int) -> torch.Tensor:
        """This rank's buffer for plan tile ``i`` (must be one of ``plan.tiles_of(rank)``)."""
        j = self.slots[self.sp.rank].index(i)
        return self._local[j]

    def blend(self, out: torch.Tensor) -> torch.Tensor:
        """Blend every rank's tiles into ``out`` [C, *latent] (after all ranks wrote theirs:
        the caller orders it, e.g. ``torch.distributed.barrier`` after a device sync)."""
        return blend_tiles(self.plan, self._ptrs, out)

    def close(self):
        self.peer.close()


def average_windows(plan: WindowPlan, clips, out: torch.Tensor) -> torch.Tensor:
    """Eq. 3 on the GPU: out[c, i] = (sum_{k in S(i)} clip_k[c, i - s_k]) / |S(i)|.

    ``clips``: per plan clip, an f32 CUDA tensor ``[C, n, H, W]`` (or its device address);
    ``out``: f32 ``[C, n', H, W]``.
    """
    if len(clips) != plan.num_clips:
        raise ConfigError("one tensor per clip", "windows.clips")
    if not isinstance(out, torch.Tensor) or out.dim() != 4:
        raise ConfigError("out must be an f32 CUDA tensor [C, n', H, W]", "windows.out")
    dev = out.device
    C, _, Hh, Ww = out.shape
    _check_f32(out, (C, plan.n_prime, Hh, Ww), "windows.out", dev)
    starts = torch.tensor([c[0] for c in plan.clips], dtype=torch.int32, device=dev)
    ops.window_average(_ptrs(clips, (C, plan.window, Hh, Ww), "windows.clips", dev), starts, plan.num_clips, plan.window, plan.n_prime, out)
    return out
