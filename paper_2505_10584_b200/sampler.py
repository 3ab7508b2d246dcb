"""Flow-matching Euler denoise loop with the diffusion cache.

``denoise(model, x0, num_steps, cache)`` is the sampler entry point the
north_star asks for (the reference has none; PAPER.md:127-131 gives the
flow-matching formulation; uniform Euler grid t_i = i/N is the builder's
choice).  ``cache`` is either

* a :class:`CacheSchedule` (e.g. ``plan_cache(...)``) — consumed unchanged:
  ``per_step_full[i]`` picks a full or a cached step on the host, so skipped
  rear blocks are simply not launched; or
* a :class:`RelL1Policy` — decided on device each step (no host sync);
  the flags actually taken come back as ``DenoiseResult.schedule``; or
* ``None`` — no cache (every step full).

With ``graph=True`` each step kind is captured once as a CUDA graph and
replayed (t / dt / step index live on device, so one graph serves every step).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .errors import ConfigError
from .schedule import CacheSchedule, RelL1Policy, no_cache


@dataclass
class DenoiseResult:
    latent: torch.Tensor                  # [C, T, H, W] f32 (device)
    schedule: CacheSchedule               # flags actually taken
    rel_l1: list = field(default_factory=list)  # per-step rel-L1 (dynamic policy)
    trajectory: list = field(default_factory=list)


class _Graphs:
    """One CUDA graph per (model context, step kind, cache policy) — replayed for every step."""

    def __init__(self):
        self.g = {}

    @staticmethod
    def key(model, mode, use_cache):
        # the policy's threshold / warmup / force_last are baked into the captured
        # cache_decide launch, so key on the (frozen, hashable) policy value, not its id
        return (id(model), model.generation, mode, use_cache, model.policy, model.cache_mode, model.n_front)

    def run(self, model, mode, use_cache):
        key = self.key(model, mode, use_cache)
        if key not in self.g:
            state = (model.idx, model.cur, model.cstate, model.prev, model.lat, model.lat_bf, model.off,
                     model.flags_out, model.rels_out)
            # snapshot first, then order the warm-up stream after the snapshots: the warm-up
            # step writes the very buffers the clones read (probe -> prev, cache_decide ->
            # cstate/flags/rels, the Euler epilogue -> lat/idx)
            saved = tuple(t.clone() for t in state)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                model.step(mode, use_cache)  # warm the kernels' one-time setup outside capture
            torch.cuda.current_stream().wait_stream(s)
            for dst, src in zip(state, saved):
                dst.copy_(src)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                model.step(mode, use_cache)
            self.g[key] = g
        self.g[key].replay()

    def clear(self):
        self.g.clear()


def denoise(model, x0: torch.Tensor, num_steps: int, cache=None, trajectory: bool = False,
            graph: bool = False, graphs: _Graphs | None = None) -> DenoiseResult:
    """Run ``num_steps`` Euler steps from the noise latent ``x0`` [C, T, H, W]."""
    if num_steps < 1:
        raise ConfigError("num_steps must be >= 1", "sampler.num_steps")
    if cache is None:
        cache = no_cache(num_steps)
    dynamic = isinstance(cache, RelL1Policy)
    if not dynamic:
        if not isinstance(cache, CacheSchedule):
            raise ConfigError("cache must be a CacheSchedule, a RelL1Policy or None", "sampler.cache")
        if cache.total_steps != num_steps:
            raise ConfigError("schedule length != num_steps", "sampler.cache")
    model.reset(x0, num_steps, policy=cache if dynamic else None, cache_mode=cache.mode,
                cached_cost_fraction=cache.cached_cost_fraction)
    use_cache = dynamic or not all(cache.per_step_full)
    traj = []
    if graph and graphs is None:
        graphs = _Graphs()
    for i in range(num_steps):
        mode = "dynamic" if dynamic else ("full" if cache.per_step_full[i] else "cached")
        if graph:
            graphs.run(model, mode, use_cache)
        else:
            model.step(mode, use_cache)
        if trajectory:
            traj.append(model.latent())
    lat = model.latent()
    if dynamic:
        flags = [bool(f) for f in model.flags_out.tolist()]
        rels = model.rels_out.tolist()
        sched = cache.as_schedule(flags)
    else:
        sched, rels = cache, []
    return DenoiseResult(latent=lat, schedule=sched, rel_l1=rels, trajectory=traj)


@dataclass
class WindowDenoiseResult:
    latent: torch.Tensor                  # [C, n', H, W] f32 (device)
    schedules: list                       # per clip: flags actually taken
    trajectory: list = field(default_factory=list)


def denoise_windows(model, x0: torch.Tensor, num_steps: int, plan, cache=None, trajectory: bool = False,
                    graph: bool = False) -> WindowDenoiseResult:
    """Temporal MultiDiffusion around the denoise step.

    ``plan``: a :class:`~paper_2505_10584_b200.tiling.WindowPlan` over the latent's
    frames (``n' = x0.shape[1]``, window ``n`` = the model's clip frames).  Every step,
    each clip ``x'[s_k : s_k + n]`` runs one denoise step (velocity + Euler, with its own
    diffusion-cache state) and Eq. 3 averages the clips back into ``x'`` on the GPU
    (``aqb_window_average``); the next step starts from the averaged latent.
    ``model`` must be prepared for the clip geometry; the other clips get
    :meth:`DiTModel.fork` contexts sharing its weights.
    """
    from .tiling import average_windows

    if num_steps < 1:
        raise ConfigError("num_steps must be >= 1", "sampler.num_steps")
    if cache is None:
        cache = no_cache(num_steps)
    dynamic = isinstance(cache, RelL1Policy)
    if not dynamic and (not isinstance(cache, CacheSchedule) or cache.total_steps != num_steps):
        raise ConfigError("cache must be a CacheSchedule of num_steps steps, a RelL1Policy or None", "sampler.cache")
    g, cfg = model.geo, model.cfg
    pt = cfg.patch[0]
    if g is None:
        raise ConfigError("call prepare() first", "model")
    if plan.window != g.grid[0] * pt or plan.n_prime != x0.shape[1]:
        raise ConfigError(f"window {plan.window} / latent {x0.shape[1]} frames vs model clip {g.grid[0] * pt}",
                          "windows")
    dev = model.device
    x = x0.to(dev, torch.float32).contiguous().clone()
    ctxs = [model] + [model.fork() for _ in range(plan.num_clips - 1)]
    for ctx, (s0, _) in zip(ctxs, plan.clips):
        ctx.reset(x, num_steps, policy=cache if dynamic else None, cache_mode=cache.mode, frame_offset=s0,
                  cached_cost_fraction=cache.cached_cost_fraction)
    clips = [torch.empty(cfg.latent_channels, plan.window, *x.shape[2:], device=dev) for _ in plan.clips]
    use_cache = dynamic or not all(cache.per_step_full)
    graphs = _Graphs() if graph else None
    traj = []
    for i in range(num_steps):
        mode = "dynamic" if dynamic else ("full" if cache.per_step_full[i] else "cached")
        for k, (ctx, (s0, _)) in enumerate(zip(ctxs, plan.clips)):
            if i > 0:
                ctx.load_latent(x, s0)
            if graph:
                graphs.run(ctx, mode, use_cache)
            else:
                ctx.step(mode, use_cache)
            ctx.latent(out=clips[k])
        average_windows(plan, clips, x)
        if trajectory:
            traj.append(x.clone())
    if dynamic:
        scheds = [cache.as_schedule([bool(f) for f in c.flags_out.tolist()]) for c in ctxs]
    else:
        scheds = [cache] * len(ctxs)
    return WindowDenoiseResult(latent=x, schedules=scheds, trajectory=traj)
