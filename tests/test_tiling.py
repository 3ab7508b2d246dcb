"""VAE tile plans and temporal MultiDiffusion windows against the reference's own
outputs (tests/golden/tiling.json, made by tests/golden/make_golden_tiling.py
from ditplan.inference), plus the reference tests' invariants; GPU tests check
the blend / Eq. 3 kernels against numpy statements of the same formulas."""

import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

from paper_2505_10584_b200.errors import ConfigError
from paper_2505_10584_b200.tiling import (average_windows, blend_tiles, plan_temporal_windows, plan_vae_tiles)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tiling.json")))


@pytest.mark.parametrize("case", GOLD["vae_tiles"], ids=lambda c: str(c["args"]))
def test_vae_tile_plan_matches_reference(case):
    lat, tile, ov, dev = case["args"]
    plan = plan_vae_tiles(tuple(lat), tuple(tile), tuple(ov), devices=dev)
    assert len(plan.tiles) == case["n_tiles"]
    assert plan.starts_per_axis() == case["axis_starts"]
    full = [[list(t.start), list(t.size), t.device] for t in plan.tiles]
    assert full[:16] == case["tiles_head"]
    assert hashlib.sha256(json.dumps(full).encode()).hexdigest() == case["tiles_sha256"]
    assert plan.parallel_speedup == case["parallel_speedup"]
    prof = plan.tile_profile()
    assert float(prof.sum()) == case["profile_sum"]
    if case["profile_flat"] is not None:
        assert prof.ravel().tolist() == case["profile_flat"]  # bit-exact float64
    total = plan.total_weight()
    assert float(total.sum()) == case["total_sum"]
    pos = [tuple(p) for p in case["positions"]]
    assert [float(total[p]) for p in pos] == case["total_at"]
    if case["weights_at"] is not None:
        maps = plan.weight_maps()
        assert [[float(m[p]) for m in maps] for p in pos] == case["weights_at"]
    ns = plan.normalized_weight_sum()
    assert [float(ns.min()), float(ns.max())] == case["normalized_sum_minmax"]


@pytest.mark.parametrize("case", GOLD["vae_tile_errors"], ids=lambda c: str(c["args"]))
def test_vae_tile_errors_match_reference(case):
    lat, tile, ov, dev = case["args"]
    if case["path"] is None:
        plan_vae_tiles(tuple(lat), tuple(tile), tuple(ov), devices=dev)
        return
    with pytest.raises(ConfigError) as ei:
        plan_vae_tiles(tuple(lat), tuple(tile), tuple(ov), devices=dev)
    assert ei.value.path == case["path"] and str(ei.value) == case["message"]


def test_window_plans_match_reference():
    for case in GOLD["windows"]:
        p = plan_temporal_windows(*case["args"])
        assert [list(c) for c in p.clips] == case["clips"], case["args"]
        assert p.multiplicity().tolist() == case["multiplicity"], case["args"]
        assert p.num_clips == math.ceil((p.n_prime - p.window) / p.stride) + 1
        if "averaging_weights" in case:
            assert [p.averaging_weights(i) for i in range(p.n_prime)] == case["averaging_weights"]


@pytest.mark.parametrize("case", GOLD["window_errors"], ids=lambda c: str(c["args"]))
def test_window_errors_match_reference(case):
    with pytest.raises(ConfigError) as ei:
        plan_temporal_windows(*case["args"])
    assert ei.value.path == case["path"] and str(ei.value) == case["message"]


# --------------------------------------------------------------------------- GPU kernels
def _blend_ref(plan, tiles):
    out = None
    for w, t, tile in zip(plan.iter_weight_maps(), plan.tiles, tiles):
        if out is None:
            out = np.zeros((tile.shape[0],) + plan.latent)
        reg = tuple(slice(t.start[a], t.start[a] + t.size[a]) for a in range(3))
        out[(slice(None),) + reg] += w[reg][None] * tile.astype(np.float64)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("lat,tile,ov", [((5, 30, 52), (3, 16, 24), (1, 6, 9)), ((32, 90, 160), (32, 48, 48), (0, 8, 8)),
                                         ((6, 20, 20), (4, 9, 9), (3, 8, 8)), ((4, 16, 16), (8, 64, 64), (0, 4, 4)),
                                         ((8, 64, 64), (4, 32, 32), (0, 0, 0))])
def test_tile_blend_kernel(lat, tile, ov):
    plan = plan_vae_tiles(lat, tile, ov, devices=4)
    C = 3
    g = torch.Generator().manual_seed(1)
    tiles = [torch.randn(C, *t.size, generator=g) for t in plan.tiles]
    out = torch.empty(C, *lat, device="cuda")
    blend_tiles(plan, [t.cuda() for t in tiles], out)
    exp = _blend_ref(plan, [t.numpy() for t in tiles])
    got = out.cpu().double().numpy()
    assert np.abs(got - exp).max() <= 1e-6 * max(1.0, np.abs(exp).max())
    # identity decode: tiles cut from one volume blend back to it (weights sum to 1)
    vol = torch.randn(C, *lat, generator=g)
    cut = [vol[(slice(None),) + tuple(slice(t.start[a], t.start[a] + t.size[a]) for a in range(3))].contiguous().cuda()
           for t in plan.tiles]
    blend_tiles(plan, cut, out)
    assert torch.allclose(out.cpu(), vol, atol=1e-6, rtol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("n_prime,n,s,hw", [(32, 8, 4, (6, 10)), (33, 8, 4, (4, 4)), (23, 6, 3, (3, 5)), (16, 16, 4, (8, 8)),
                                            (33, 16, 8, (45, 80))])
def test_window_average_kernel(n_prime, n, s, hw):
    plan = plan_temporal_windows(n_prime, n, s)
    C = 8
    g = torch.Generator().manual_seed(n_prime)
    clips = [torch.randn(C, n, *hw, generator=g) for _ in plan.clips]
    out = torch.empty(C, n_prime, *hw, device="cuda")
    average_windows(plan, [c.cuda() for c in clips], out)
    acc = np.zeros((C, n_prime) + hw)
    for (a, b), c in zip(plan.clips, clips):
        acc[:, a:b] += c.double().numpy()
    exp = acc / plan.multiplicity()[None, :, None, None]
    assert np.abs(out.cpu().double().numpy() - exp).max() <= 1e-5
    # constant clips: frame i gets the mean of the covering clips' constants (reference test)
    vals = [float(k + 1) for k in range(plan.num_clips)]
    average_windows(plan, [torch.full((C, n) + hw, v, device="cuda") for v in vals], out)
    for i in range(n_prime):
        cov = [vals[k] for k, (a, b) in enumerate(plan.clips) if a <= i < b]
        assert torch.allclose(out[:, i], torch.full_like(out[:, i], sum(cov) / len(cov)))


@pytest.mark.gpu
def test_peer_tiles_single_rank_blend_equals_local_blend():
    """PeerTiles (multi-GPU VAE blend) with a group of one: tiles written into the peer buffer
    blend to the same bits as the plain blend of the same tiles (multi-rank: tests/test_multirank_gpu.py::test_multirank_vae_tile_blend)."""
    import socket

    import torch.distributed as dist

    from paper_2505_10584_b200.parallel import Ulysses
    from paper_2505_10584_b200.tiling import PeerTiles

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        plan = plan_vae_tiles((9, 40, 64), (5, 16, 24), (1, 4, 8), devices=1)
        g = torch.Generator().manual_seed(1)
        tiles = [torch.randn(4, *t.size, generator=g) for t in plan.tiles]
        pt = PeerTiles(plan, Ulysses(exchange="p2p"), 4)
        for i in plan.tiles_of(0):
            pt.local_tile(i).copy_(tiles[i])
        out = torch.empty(4, *plan.latent, device="cuda")
        ref = torch.empty_like(out)
        pt.blend(out)
        blend_tiles(plan, [t.cuda() for t in tiles], ref)
        assert torch.equal(out, ref)
        pt.close()
    finally:
        dist.destroy_process_group()


def test_blend_and_average_validate_tensors_on_cpu():
    """Host-side validation fires before any launch: CPU tensors are rejected (no CPU path)."""
    plan = plan_vae_tiles((6, 20, 20), (4, 9, 9), (3, 8, 8), devices=1)
    with pytest.raises(ConfigError):
        blend_tiles(plan, [torch.zeros(3, *t.size) for t in plan.tiles], torch.zeros(3, *plan.latent))
    wp = plan_temporal_windows(8, 4, 2)
    with pytest.raises(ConfigError):
        average_windows(wp, [torch.zeros(2, 4, 3, 3) for _ in wp.clips], torch.zeros(2, 8, 3, 3))


@pytest.mark.gpu
def test_blend_and_average_reject_bad_layouts():
    """bf16 / non-contiguous / wrong-shape tiles and a sliced ``out`` raise instead of
    reading out of bounds (the kernels index dense f32 arrays)."""
    plan = plan_vae_tiles((6, 20, 20), (4, 9, 9), (3, 8, 8), devices=1)
    C = 3
    good = [torch.zeros(C, *t.size, device="cuda") for t in plan.tiles]
    out = torch.zeros(C, *plan.latent, device="cuda")
    blend_tiles(plan, good, out)
    bad_dtype = [t.to(torch.bfloat16) for t in good]
    bad_layout = [torch.zeros(C, t.size[2], t.size[1], t.size[0], device="cuda").permute(0, 3, 2, 1)
                  for t in plan.tiles]
    bad_shape = [torch.zeros(C + 1, *t.size, device="cuda") for t in plan.tiles]
    for tiles in (bad_dtype, bad_layout, bad_shape):
        with pytest.raises(ConfigError):
            blend_tiles(plan, tiles, out)
    wide = torch.zeros(C, plan.latent[0], plan.latent[1], plan.latent[2] + 4, device="cuda")
    with pytest.raises(ConfigError):
        blend_tiles(plan, good, wide[..., :plan.latent[2]])
    with pytest.raises(ConfigError):
        blend_tiles(plan, good, torch.zeros(C, *plan.latent, device="cuda", dtype=torch.float64))
    wp = plan_temporal_windows(8, 4, 2)
    clips = [torch.zeros(2, 4, 3, 3, device="cuda") for _ in wp.clips]
    avg = torch.zeros(2, 8, 3, 3, device="cuda")
    average_windows(wp, clips, avg)
    with pytest.raises(ConfigError):
        average_windows(wp, [c.to(torch.bfloat16) for c in clips], avg)
    with pytest.raises(ConfigError):
        average_windows(wp, clips, torch.zeros(2, 8, 3, 6, device="cuda")[..., :3])
