"""End-to-end parity of the denoise loop (CUDA path vs the fp32 CPU oracle).

Gate from the north_star: per-step latent relative-L2 <= 1e-2 in bf16 and the
same cache skip schedule.  Weights / inputs follow the synthetic contract
(seed 0 weights, seed 1 noise, seed 2 text).
"""


import pytest
import torch

from oracle import dit_oracle as ref
from paper_2505_10584_b200 import (TINY_MM, TINY_SINGLE, DiTConfig, RelL1Policy, build_model, denoise,
                                   front_block_count, no_cache, plan_cache)
from paper_2505_10584_b200.config import SINGLE_DIT_2B, with_overrides
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

pytestmark = pytest.mark.gpu
TOL_BF16 = 1e-2


def rel_l2(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm())


def _setup(cfg, grid, steps_fraction=0.25, precision="bf16"):
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, grid)
    model = build_model(cfg, weights=W, precision=precision).prepare(
        grid, inp["text"], inp["pooled"] if cfg.family == "mm-dit" else None)
    orc = ref.OracleDiT(cfg, W, inp["text"], inp["pooled"] if cfg.family == "mm-dit" else None, grid,
                        n_front=front_block_count(cfg.num_layers, steps_fraction))
    return model, orc, inp


def _check_traj(res, lat_ref, tol=TOL_BF16):
    errs = [rel_l2(g, r) for g, r in zip(res.trajectory, lat_ref[1:])]
    assert max(errs) <= tol, errs
    return errs


CASES = {
    "tiny-single": (TINY_SINGLE, (2, 4, 4)),  # BASELINE config 1: 2x8x8 latent, 16 text tokens
    "tiny-mm": (TINY_MM, (2, 4, 4)),
    "single-d128": (DiTConfig("single-dit", hidden_size=256, num_heads=2, num_single=4, text_dim=256, text_len=40),
                    (3, 8, 12)),
    "mm-d128": (DiTConfig("mm-dit", hidden_size=256, num_heads=2, num_dual=2, num_single=2, text_dim=192,
                          text_len=24, pooled_dim=64), (3, 6, 10)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_denoise_static_cache_matches_oracle(name):
    cfg, grid = CASES[name]
    steps = 4 if name.startswith("tiny") else 8
    sched = plan_cache(steps, warmup=1, interval=2)  # FFcF / FFcFcFcF: the config-1 schedule family
    model, orc, inp = _setup(cfg, grid)
    res = denoise(model, inp["x0"], steps, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], steps, flags=sched.per_step_full)
    assert res.schedule.per_step_full == tuple(taken)
    _check_traj(res, lat)


@pytest.mark.parametrize("name", ["tiny-single", "mm-d128"])
def test_denoise_no_cache_matches_oracle(name):
    cfg, grid = CASES[name]
    model, orc, inp = _setup(cfg, grid)
    res = denoise(model, inp["x0"], 4, None, trajectory=True)
    lat, _, _ = ref.denoise(orc, inp["x0"], 4, flags=[True] * 4)
    _check_traj(res, lat)


@pytest.mark.parametrize("name", ["single-d128", "mm-d128"])
def test_denoise_rel_l1_policy_same_schedule(name):
    cfg, grid = CASES[name]
    steps = 10
    model, orc, inp = _setup(cfg, grid)
    # threshold = 2.5x the typical per-step rel-L1: the accumulator crosses it every ~3 steps and
    # sits >= 0.5x a step's rel away from it at each decision (margin >> bf16-vs-fp32 drift)
    _, _, probe = ref.denoise(orc, inp["x0"], 4, policy=RelL1Policy(threshold=1e9, warmup=1))
    thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
    pol = RelL1Policy(threshold=thr, warmup=2)
    lat, taken, rels = ref.denoise(orc, inp["x0"], steps, policy=pol)
    assert 0 < taken.count(False) < steps - 2  # the policy really mixes full and cached steps
    res = denoise(model, inp["x0"], steps, pol, trajectory=True)
    assert list(res.schedule.per_step_full) == taken, (res.rel_l1, rels)
    # device rel-L1 values track the fp32 oracle's
    for g, r in zip(res.rel_l1[1:], rels[1:]):
        assert abs(g - r) <= 2e-2 * abs(r) + 1e-4
    _check_traj(res, lat)


def test_graph_replay_equals_eager():
    cfg, grid = CASES["single-d128"]
    model, _, inp = _setup(cfg, grid)
    sched = plan_cache(6, warmup=1, interval=2)
    a = denoise(model, inp["x0"], 6, sched).latent.clone()
    b = denoise(model, inp["x0"], 6, sched, graph=True).latent
    assert torch.equal(a, b)


def test_graph_replay_equals_eager_rel_l1_policy():
    """CUDA-graph replay of the device-decided (rel-L1) step: same latent bits, same flags and
    the same rel-L1 values as eager launches (the capture warm-up must not leak state)."""
    cfg, grid = CASES["single-d128"]
    model, orc, inp = _setup(cfg, grid)
    _, _, probe = ref.denoise(orc, inp["x0"], 4, policy=RelL1Policy(threshold=1e9, warmup=1))
    thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
    pol = RelL1Policy(threshold=thr, warmup=2)
    a = denoise(model, inp["x0"], 10, pol)
    lat_a, rel_a = a.latent.clone(), list(a.rel_l1)
    assert 0 < a.schedule.cached_steps
    b = denoise(model, inp["x0"], 10, pol, graph=True)
    assert b.schedule.per_step_full == a.schedule.per_step_full
    assert b.rel_l1 == rel_a
    assert torch.equal(b.latent, lat_a)
    # a second policy with another threshold must not replay the first one's graph
    pol2 = RelL1Policy(threshold=thr * 3, warmup=2)
    graphs = __import__("paper_2505_10584_b200.sampler", fromlist=["_Graphs"])._Graphs()
    c1 = denoise(model, inp["x0"], 10, pol, graph=True, graphs=graphs).schedule.per_step_full
    c2 = denoise(model, inp["x0"], 10, pol2, graph=True, graphs=graphs).schedule.per_step_full
    e2 = denoise(model, inp["x0"], 10, pol2).schedule.per_step_full
    assert c1 == a.schedule.per_step_full and c2 == e2


def test_cached_cost_fraction_sets_front_blocks():
    """A schedule with cached_cost_fraction 0.5 runs ceil(0.5·L) front blocks on cached steps
    (the fraction the schedule's speedup is costed with), matching the oracle at that split."""
    cfg, grid = CASES["single-d128"]
    model, _, inp = _setup(cfg, grid)
    for frac in (0.5, 0.25, 1.0):
        sched = plan_cache(8, warmup=2, interval=2, cached_cost_fraction=frac)
        res = denoise(model, inp["x0"], 8, sched, trajectory=True)
        assert model.n_front == front_block_count(cfg.num_layers, frac)
        orc = ref.OracleDiT(cfg, init_weights(cfg, seed=0), inp["text"], None, grid,
                            n_front=front_block_count(cfg.num_layers, frac))
        lat, _, _ = ref.denoise(orc, inp["x0"], 8, flags=sched.per_step_full)
        _check_traj(res, lat)


def test_config2_dims_two_blocks_match_oracle():
    """Single-DiT 2B dims (H=2048, 16 heads, text 256x4096) at the config-2 geometry
    (17x480x832 -> 7,800 tokens), 2 of the 28 blocks, 2 steps — the CPU oracle's bounded sample."""
    cfg = with_overrides(SINGLE_DIT_2B, num_single=2)
    grid = (5, 30, 52)
    model, orc, inp = _setup(cfg, grid)
    res = denoise(model, inp["x0"], 2, None, trajectory=True)
    lat, _, _ = ref.denoise(orc, inp["x0"], 2, flags=[True, True])
    _check_traj(res, lat)


def test_full_2b_cache_interval1_equals_no_cache_and_is_deterministic():
    """Size-independent properties at the full config-2 size: interval-1 schedule == cache off
    (bit-exact), and two runs are bit-identical."""
    cfg = SINGLE_DIT_2B
    grid = (5, 30, 52)
    W = init_weights(cfg, seed=0, device="cuda")
    inp = synthetic_inputs(cfg, grid, device="cuda")
    model = build_model(cfg, weights=W).prepare(grid, inp["text"])
    a = denoise(model, inp["x0"], 3, None).latent.clone()
    b = denoise(model, inp["x0"], 3, plan_cache(3, warmup=0, interval=1)).latent.clone()
    c = denoise(model, inp["x0"], 3, None).latent
    assert torch.isfinite(a).all()
    assert torch.equal(a, b) and torch.equal(a, c)


TOL_FP32 = 1e-4


@pytest.mark.parametrize("name", list(CASES))
def test_fp32_validation_mode_matches_oracle(name):
    """north_star fp32 validation mode: per-step latent rel-L2 <= 1e-4 and the same schedule."""
    cfg, grid = CASES[name]
    steps = 4 if name.startswith("tiny") else 6
    sched = plan_cache(steps, warmup=1, interval=2)
    model, orc, inp = _setup(cfg, grid, precision="fp32")
    res = denoise(model, inp["x0"], steps, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], steps, flags=sched.per_step_full)
    assert res.schedule.per_step_full == tuple(taken)
    _check_traj(res, lat, tol=TOL_FP32)


def test_fp32_validation_mode_rel_l1_policy():
    cfg, grid = CASES["single-d128"]
    model, orc, inp = _setup(cfg, grid, precision="fp32")
    _, _, probe = ref.denoise(orc, inp["x0"], 4, policy=RelL1Policy(threshold=1e9, warmup=1))
    thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
    pol = RelL1Policy(threshold=thr, warmup=2)
    lat, taken, rels = ref.denoise(orc, inp["x0"], 10, policy=pol)
    res = denoise(model, inp["x0"], 10, pol, trajectory=True)
    assert list(res.schedule.per_step_full) == taken
    for g, r in zip(res.rel_l1[1:], rels[1:]):
        assert abs(g - r) <= 1e-4 * abs(r) + 1e-7  # fp32 probe tracks the oracle tightly
    _check_traj(res, lat, tol=TOL_FP32)


def test_mmdit_13b_dims_two_blocks_match_oracle():
    """MM-DiT 13.4B dims (H=3072, 24 heads, text 256x4096): 1 dual + 1 single block at a reduced
    720p-like geometry (8x30x53 = 12,720 video + 256 text tokens), 2 steps, bf16 gate 1e-2."""
    from paper_2505_10584_b200.config import MM_DIT_13B
    cfg = with_overrides(MM_DIT_13B, num_dual=1, num_single=1)
    grid = (8, 30, 53)
    model, orc, inp = _setup(cfg, grid)
    res = denoise(model, inp["x0"], 2, None, trajectory=True)
    lat, _, _ = ref.denoise(orc, inp["x0"], 2, flags=[True, True])
    _check_traj(res, lat)


@pytest.mark.parametrize("name", ["tiny-single", "single-d128", "mm-d128", "tiny-mm"])
def test_attention_cache_mode_matches_oracle(name):
    """attention-cache: cached steps reuse every block's attention output."""
    cfg, grid = CASES[name]
    steps = 4 if name.startswith("tiny") else 8
    sched = plan_cache(steps, warmup=1, interval=2, mode="attention-cache")
    model, _, inp = _setup(cfg, grid)
    pooled = inp["pooled"] if cfg.family == "mm-dit" else None
    orc = ref.OracleDiT(cfg, init_weights(cfg, seed=0), inp["text"], pooled, grid, mode="attention-cache")
    res = denoise(model, inp["x0"], steps, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], steps, flags=sched.per_step_full)
    assert res.schedule.per_step_full == tuple(taken)
    _check_traj(res, lat)
    # graph replay of the same schedule is bit-identical
    g = denoise(model, inp["x0"], steps, sched, graph=True).latent
    assert torch.equal(g, res.latent)


def test_attention_cache_mode_rel_l1_policy_and_fp32():
    cfg, grid = CASES["single-d128"]
    model, _, inp = _setup(cfg, grid, precision="fp32")
    orc = ref.OracleDiT(cfg, init_weights(cfg, seed=0), inp["text"], None, grid, mode="attention-cache")
    _, _, probe = ref.denoise(orc, inp["x0"], 4, policy=RelL1Policy(threshold=1e9, warmup=1))
    thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
    pol = RelL1Policy(threshold=thr, warmup=2, mode="attention-cache")
    lat, taken, _ = ref.denoise(orc, inp["x0"], 10, policy=pol)
    assert 0 < taken.count(False)
    res = denoise(model, inp["x0"], 10, pol, trajectory=True)
    assert list(res.schedule.per_step_full) == taken
    _check_traj(res, lat, tol=TOL_FP32)


@pytest.mark.parametrize("name,n_prime,window,stride", [("tiny-single", 6, 4, 2), ("mm-d128", 9, 3, 2)])
def test_temporal_multidiffusion_matches_oracle(name, n_prime, window, stride):
    """denoise_windows: per-clip Euler steps + Eq. 3 averaging on the GPU vs the fp32 oracle."""
    from paper_2505_10584_b200 import denoise_windows, plan_temporal_windows
    cfg, grid = CASES[name]
    clip_grid = (window, grid[1], grid[2])
    plan = plan_temporal_windows(n_prime, window, stride)
    W = init_weights(cfg, seed=0)
    g = torch.Generator().manual_seed(1)
    pt, ph, pw = cfg.patch
    x0 = torch.randn(cfg.latent_channels, n_prime * pt, grid[1] * ph, grid[2] * pw, generator=g)
    inp = synthetic_inputs(cfg, clip_grid)
    pooled = inp["pooled"] if cfg.family == "mm-dit" else None
    model = build_model(cfg, weights=W).prepare(clip_grid, inp["text"], pooled)
    steps = 6
    sched = plan_cache(steps, warmup=1, interval=2)
    res = denoise_windows(model, x0, steps, plan, sched, trajectory=True)
    nf = front_block_count(cfg.num_layers, 0.25)
    orcs = [ref.OracleDiT(cfg, W, inp["text"], pooled, clip_grid, n_front=nf) for _ in plan.clips]
    lat = ref.denoise_windows(orcs, x0, steps, plan.clips, flags=sched.per_step_full)
    errs = [rel_l2(a, b) for a, b in zip(res.trajectory, lat[1:])]
    assert max(errs) <= TOL_BF16, errs


@pytest.mark.parametrize("family", ["single-dit", "mm-dit"])
def test_tp_sp_single_rank_matches_plain_model_and_oracle(family):
    """TP-SP code path (fused gather / reduce-scatter kernels, peer barriers) with P = 1 in this
    process (gloo group of one): same schedule as the plain model, within bf16 noise of it and of
    the oracle.  Multi-rank parity: tests/test_multirank_gpu.py."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2505_10584_b200.parallel import TensorSP

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        if family == "single-dit":
            cfg = DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40)
            grid = (3, 8, 16)
        else:
            cfg = DiTConfig("mm-dit", hidden_size=1024, num_heads=8, num_dual=2, num_single=2, text_dim=192,
                            text_len=24, pooled_dim=64)
            grid = (2, 8, 16)
        W = init_weights(cfg, seed=0)
        inp = synthetic_inputs(cfg, grid)
        pooled = inp["pooled"] if family == "mm-dit" else None
        tp = build_model(cfg, weights=W, sp=TensorSP()).prepare(grid, inp["text"], pooled)
        plain = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled)
        orc = ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=front_block_count(cfg.num_layers, 0.25))
        _, _, probe = ref.denoise(orc, inp["x0"], 4, policy=RelL1Policy(threshold=1e9, warmup=1))
        thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
        for cache in (plan_cache(8, warmup=2, interval=2), RelL1Policy(threshold=thr, warmup=2),
                      plan_cache(8, warmup=2, interval=2, mode="attention-cache")):
            r_tp = denoise(tp, inp["x0"], 8, cache, trajectory=True)
            r_1 = denoise(plain, inp["x0"], 8, cache, trajectory=True)
            o = ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=front_block_count(cfg.num_layers, 0.25),
                              mode=cache.mode)
            if isinstance(cache, RelL1Policy):
                lat, taken, _ = ref.denoise(o, inp["x0"], 8, policy=cache)
            else:
                lat, taken, _ = ref.denoise(o, inp["x0"], 8, flags=cache.per_step_full)
            assert False in taken  # every policy really caches
            assert list(r_tp.schedule.per_step_full) == list(r_1.schedule.per_step_full) == list(taken)
            assert max(rel_l2(a, b) for a, b in zip(r_tp.trajectory, r_1.trajectory)) < 5e-3
            _check_traj(r_tp, lat)
            assert tp.peer_ok()
        tp.peer.close()
    finally:
        dist.destroy_process_group()
