"""CPU checks of the fp32 oracle and the host logic (no GPU).

The oracle is the parity anchor for latents (the reference has no runtime,
SURVEY.md §8(c)), so its own invariants are tested here: RoPE is a rotation
(norm-preserving, relative-position property), attention rows are convex
combinations, the cached step adds exactly the stored rear offset, the
interval-1 schedule equals no cache, patchify round-trips, and the config /
weight inventory matches the stated parameter counts.
"""

import math

import pytest
import torch

from oracle import dit_oracle as ref
from paper_2505_10584_b200 import (MM_DIT_13B, SINGLE_DIT_2B, TINY_MM, TINY_SINGLE, ConfigError, DiTConfig,
                                   RelL1Policy, front_block_count, plan_cache)
from paper_2505_10584_b200.config import VideoSpec, flops_per_step
from paper_2505_10584_b200.weights import init_weights, param_specs, synthetic_inputs

GRID = (2, 4, 4)


def _orc(cfg, n_front=None):
    W = init_weights(cfg)
    inp = synthetic_inputs(cfg, GRID)
    nf = front_block_count(cfg.num_layers, 0.25) if n_front is None else n_front
    return ref.OracleDiT(cfg, W, inp["text"], inp["pooled"], GRID, n_front=nf), inp


def test_rope_is_rotation_and_relative():
    ang = ref.rope_angles((3, 4, 5), (8, 12, 12), 1000.0)
    x = torch.randn(60, 2, 32)
    y = ref.apply_rope(x, ang)
    assert torch.allclose(x.norm(dim=-1), y.norm(dim=-1), atol=1e-5)
    # q·k after RoPE depends on positions only through their difference (same axis shift)
    q, k = torch.randn(1, 1, 32), torch.randn(1, 1, 32)
    a1 = ref.rope_angles((3, 4, 5), (8, 12, 12), 1000.0)
    i, j = 5, 17          # token ids; shift both by one t-step (20 tokens)
    d1 = (ref.apply_rope(q, a1[i:i + 1]) * ref.apply_rope(k, a1[j:j + 1])).sum()
    d2 = (ref.apply_rope(q, a1[i + 20:i + 21]) * ref.apply_rope(k, a1[j + 20:j + 21])).sum()
    assert abs(float(d1 - d2)) < 1e-4


def test_attention_rows_are_convex_combinations():
    q, k = torch.randn(7, 2, 16), torch.randn(9, 2, 16)
    v = torch.ones(9, 2, 16)
    assert torch.allclose(ref.attention(q, k, v), torch.ones(7, 32), atol=1e-6)


def test_patchify_roundtrip():
    lat = torch.randn(8, 4, 6, 10)
    tok = ref.patchify(lat, (1, 2, 2))
    assert tok.shape == (4 * 3 * 5, 32)
    assert torch.equal(ref.unpatchify(tok, (4, 3, 5), (1, 2, 2), 8), lat)


@pytest.mark.parametrize("cfg", [TINY_SINGLE, TINY_MM])
def test_cached_step_adds_stored_offset(cfg):
    orc, inp = _orc(cfg)
    x = ref.patchify(inp["x0"], cfg.patch)
    state = {}
    v_full, _ = orc.velocity(x, 0.3, full=True, state=state)
    v_cached, _ = orc.velocity(x, 0.3, full=False, state=state)
    # same input and t: the cached step must reproduce the full step exactly (up to fp32 assoc.)
    assert torch.allclose(v_full, v_cached, atol=1e-5, rtol=1e-5)
    assert "offset" in state and state["offset"].shape == (x.shape[0], cfg.hidden_size)


@pytest.mark.parametrize("cfg", [TINY_SINGLE, TINY_MM])
def test_interval1_equals_no_cache(cfg):
    orc, inp = _orc(cfg)
    a, _, _ = ref.denoise(orc, inp["x0"], 4, flags=[True] * 4)
    b, _, _ = ref.denoise(orc, inp["x0"], 4, flags=plan_cache(4, 0, 1).per_step_full)
    assert all(torch.equal(x, y) for x, y in zip(a, b))


def test_cache_changes_result_but_stays_close():
    orc, inp = _orc(TINY_SINGLE)
    a, _, _ = ref.denoise(orc, inp["x0"], 4, flags=[True] * 4)
    b, _, _ = ref.denoise(orc, inp["x0"], 4, flags=plan_cache(4, 1, 2).per_step_full)
    d = float((a[-1] - b[-1]).norm() / a[-1].norm())
    assert 0 < d < 0.05


def test_rel_l1_policy_in_oracle_forces_first_and_last():
    orc, inp = _orc(TINY_MM)
    _, taken, rels = ref.denoise(orc, inp["x0"], 6, policy=RelL1Policy(threshold=1e9, warmup=1))
    assert taken == [True, False, False, False, False, True]
    assert all(r > 0 for r in rels[1:])


def test_blocks_are_not_identities():
    """Non-zero modulation init: every block changes the residual stream."""
    orc, inp = _orc(TINY_SINGLE, n_front=2)
    x = ref.patchify(inp["x0"], TINY_SINGLE.patch)
    v2, _ = orc.velocity(x, 0.5, blocks=2)
    v1, _ = orc.velocity(x, 0.5, blocks=1)
    assert float((v2 - v1).norm() / v1.norm()) > 1e-2


def test_param_counts_and_presets():
    assert SINGLE_DIT_2B.param_count() == pytest.approx(2.14e9, rel=0.02)
    assert MM_DIT_13B.param_count() == pytest.approx(13.4e9, rel=0.01)
    assert SINGLE_DIT_2B.head_dim == 128 and MM_DIT_13B.head_dim == 128
    assert SINGLE_DIT_2B.rope_dims == (32, 48, 48)
    for cfg in (TINY_SINGLE, TINY_MM):
        n = sum(math.prod(s) for _, s, _, _ in param_specs(cfg))
        assert n == cfg.param_count()


def test_video_geometry_for_baseline_configs():
    assert VideoSpec(17, 480, 832).tokens(SINGLE_DIT_2B) == 7800
    assert VideoSpec(61, 480, 848).tokens(MM_DIT_13B) == 25440
    assert VideoSpec(129, 720, 1280).tokens(MM_DIT_13B) == 118800
    f = flops_per_step(SINGLE_DIT_2B, 7800)
    assert f["total"] == pytest.approx(4.0e13, rel=0.05)
    assert f["attention"] / f["total"] == pytest.approx(0.36, abs=0.03)


def test_config_validation():
    with pytest.raises(ConfigError):
        DiTConfig("nope", hidden_size=128, num_heads=4)
    with pytest.raises(ConfigError):
        DiTConfig("single-dit", hidden_size=128, num_heads=3)
    with pytest.raises(ConfigError):
        DiTConfig("single-dit", hidden_size=128, num_heads=4, num_dual=1)
    with pytest.raises(ConfigError):
        DiTConfig("mm-dit", hidden_size=128, num_heads=4, num_dual=0, num_single=0)


def test_oracle_windows_single_clip_equals_plain_denoise():
    """Eq. 3 with one clip covering the latent is the plain Euler loop (oracle self-check)."""
    from oracle import dit_oracle as ref
    from paper_2505_10584_b200 import TINY_SINGLE
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

    cfg, grid = TINY_SINGLE, (2, 4, 4)
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, grid)
    a = ref.denoise_windows([ref.OracleDiT(cfg, W, inp["text"], None, grid)], inp["x0"], 3, [(0, 2)])
    b, _, _ = ref.denoise(ref.OracleDiT(cfg, W, inp["text"], None, grid), inp["x0"], 3, flags=[True] * 3)
    for x, y in zip(a, b):
        assert torch.allclose(x, y, atol=1e-6)


def test_oracle_attention_cache_all_full_equals_no_cache():
    from oracle import dit_oracle as ref
    from paper_2505_10584_b200 import TINY_MM
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

    cfg, grid = TINY_MM, (2, 4, 4)
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, grid)
    o1 = ref.OracleDiT(cfg, W, inp["text"], inp["pooled"], grid, mode="attention-cache")
    o2 = ref.OracleDiT(cfg, W, inp["text"], inp["pooled"], grid)
    a, _, _ = ref.denoise(o1, inp["x0"], 3, flags=[True] * 3)
    b, _, _ = ref.denoise(o2, inp["x0"], 3, flags=[True] * 3)
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    c, _, _ = ref.denoise(o1, inp["x0"], 3, flags=[True, False, True])
    assert not torch.equal(c[2], a[2])  # the cached step really reuses stale attention


def test_rel_l1_rule_oracle_matches_product_policy():
    """The oracle's independent statement of the rel-L1 cache rule and the product's
    RelL1Policy.decide (which the device kernel aqb_cache_decide mirrors) agree on random
    runs — the GPU tests then compare the device decisions with the oracle's."""
    import random

    from oracle.schedule_oracle import rel_l1_decide
    from paper_2505_10584_b200 import RelL1Policy

    rng = random.Random(0)
    for _ in range(300):
        total = rng.randint(1, 40)
        pol = RelL1Policy(threshold=rng.uniform(0.0, 0.5), warmup=rng.randint(0, 6), force_last=rng.random() < 0.5)
        a = b = 0.0
        for s in range(1, total + 1):
            rel = rng.uniform(0.0, 0.2)
            fa, a = rel_l1_decide(s, total, a, rel, pol.threshold, pol.warmup, pol.force_last)
            fb, b = pol.decide(s, total, b, rel)
            assert fa == fb and a == b
