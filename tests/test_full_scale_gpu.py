"""Parity at full depth and full geometry.

The fp32 oracle (``oracle/dit_oracle.py``) runs on the GPU in strict fp32 (TF32 off) so the
BASELINE configs can be checked end to end at their real size:

* config 2 — Single-DiT 2B, all 28 blocks, 7,800 tokens, 30 Euler steps, under
  ``plan_cache(30)`` (``inference.py:48-86``: 17 full / 13 cached) and under a rel-L1 policy
  whose threshold comes from the oracle's own probe (so it really skips);
* config 3 — MM-DiT 13.4B, all 54 blocks (25 dual + 29 joint), 25,440 video + 256 text tokens,
  4 steps of ``plan_cache(4, 1, 2)`` (FFcF, one cached step through the 14 front blocks);
* config 4's geometry (118,800 + 256 tokens) through one dual-stream and one joint block of the
  13.4B dims, 4 steps with a cached one;
* joint attention at 119,056 tokens (config 4's sequence, 3 heads = one rank's share at
  P = 8) and 131,072 tokens (config 5's longest) against fp32 softmax attention.

Gate (north_star): identical schedules and per-step latent rel-L2 <= 1e-2 (bf16).
"""

import pytest
import torch

from oracle import dit_oracle as ref
from paper_2505_10584_b200 import RelL1Policy, build_model, denoise, front_block_count, ops, plan_cache
from paper_2505_10584_b200.config import MM_DIT_13B, SINGLE_DIT_2B, VIDEO_480P_17F, VIDEO_480P_61F
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

pytestmark = pytest.mark.gpu
TOL_BF16 = 1e-2


def rel_l2(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm())


def _pair(cfg, grid):
    W = init_weights(cfg, seed=0, device="cuda")
    inp = synthetic_inputs(cfg, grid, device="cuda")
    pooled = inp["pooled"] if cfg.family == "mm-dit" else None
    model = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled)
    orc = ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=front_block_count(cfg.num_layers, 0.25),
                        device="cuda")
    del W
    return model, orc, inp


def _errs(res, lat_ref):
    return [rel_l2(g, r) for g, r in zip(res.trajectory, lat_ref[1:])]


@pytest.fixture(scope="module")
def config2():
    cfg = SINGLE_DIT_2B
    grid = VIDEO_480P_17F.grid(cfg)
    assert grid[0] * grid[1] * grid[2] == 7800
    model, orc, inp = _pair(cfg, grid)
    yield model, orc, inp
    del model, orc
    torch.cuda.empty_cache()


def test_config2_full_depth_plan_cache_30(config2):
    model, orc, inp = config2
    sched = plan_cache(30)
    assert sched.as_string() == "FFFFFFFFFFFccFccFccFccFccFccFc"
    res = denoise(model, inp["x0"], 30, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], 30, flags=sched.per_step_full)
    assert tuple(taken) == res.schedule.per_step_full == sched.per_step_full
    errs = _errs(res, lat)
    print("config2 plan_cache(30) per-step rel-L2:", ["%.2e" % e for e in errs])
    assert max(errs) <= TOL_BF16, errs


def test_config2_full_depth_rel_l1_policy(config2):
    model, orc, inp = config2
    # threshold from the oracle's own probe: 2.5x the median per-step rel-L1 over the first steps
    _, _, probe = ref.denoise(orc, inp["x0"], 6, policy=RelL1Policy(threshold=1e9, warmup=1), return_all=False)
    thr = 2.5 * sorted(probe[1:])[len(probe[1:]) // 2]
    pol = RelL1Policy(threshold=thr, warmup=4)
    lat, taken, rels = ref.denoise(orc, inp["x0"], 30, policy=pol)
    assert 0 < taken.count(False) < 26, taken  # the policy really skips at full depth
    res = denoise(model, inp["x0"], 30, pol, trajectory=True)
    assert list(res.schedule.per_step_full) == taken, (res.schedule.as_string(), res.rel_l1, rels)
    for g, r in zip(res.rel_l1[1:], rels[1:]):
        assert abs(g - r) <= 2e-2 * abs(r) + 1e-4
    errs = _errs(res, lat)
    print(f"config2 rel-L1 (thr {thr:.4f}) schedule {res.schedule.as_string()} max rel-L2 {max(errs):.2e}")
    assert max(errs) <= TOL_BF16, errs


def test_config3_mmdit_13b_full_depth():
    cfg = MM_DIT_13B
    grid = VIDEO_480P_61F.grid(cfg)
    assert grid[0] * grid[1] * grid[2] == 25_440 and cfg.num_layers == 54
    model, orc, inp = _pair(cfg, grid)
    sched = plan_cache(4, warmup=1, interval=2)
    assert sched.as_string() == "FFcF"
    res = denoise(model, inp["x0"], 4, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], 4, flags=sched.per_step_full)
    assert tuple(taken) == res.schedule.per_step_full
    errs = _errs(res, lat)
    print("config3 MM-DiT 54 blocks FFcF per-step rel-L2:", ["%.2e" % e for e in errs])
    del model, orc
    torch.cuda.empty_cache()
    assert max(errs) <= TOL_BF16, errs


@pytest.mark.parametrize("seq,heads", [(119_056, 3), (131_072, 2)])
def test_attention_long_sequence_vs_fp32(seq, heads):
    d = 128
    g = torch.Generator(device="cuda").manual_seed(seq)
    q, k, v = (torch.randn(seq, heads, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty(seq, heads * d, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(max(16, ops.attention_workspace_bytes(seq, seq, heads, d)), device="cuda", dtype=torch.uint8)
    ops.attention(q.view(seq, -1), k.view(seq, -1), v.view(seq, -1), o, heads, d, workspace=ws)
    with ref.strict_fp32():
        exp = ref.attention(q.float(), k.float(), v.float())
    e = rel_l2(o, exp)
    print(f"attention S={seq} heads={heads}: rel-L2 {e:.2e}")
    assert e <= TOL_BF16
    # and per head, so a wrong head cannot hide behind the others
    for h in range(heads):
        assert rel_l2(o[:, h * d:(h + 1) * d], exp[:, h * d:(h + 1) * d]) <= TOL_BF16


def test_config4_geometry_mmdit_two_blocks():
    """Config 4's geometry — 129x720x1280 -> 118,800 video + 256 text tokens — through the 13.4B
    MM-DiT dims (H=3072, 24 heads) with one dual-stream and one joint block, 4 steps of
    plan_cache(4, 1, 2) = FFcF (the joint block is the rear block a cached step skips), against the fp32
    oracle on the GPU: the joint attention over 119,056 tokens, the RoPE tables of a 33x45x80 grid
    and the cache offset at the full size."""
    from paper_2505_10584_b200.config import VIDEO_720P_129F, with_overrides
    cfg = with_overrides(MM_DIT_13B, num_dual=1, num_single=1)
    grid = VIDEO_720P_129F.grid(cfg)
    assert grid[0] * grid[1] * grid[2] == 118_800
    model, orc, inp = _pair(cfg, grid)
    sched = plan_cache(4, warmup=1, interval=2)
    assert sched.as_string() == "FFcF"
    res = denoise(model, inp["x0"], 4, sched, trajectory=True)
    lat, taken, _ = ref.denoise(orc, inp["x0"], 4, flags=sched.per_step_full)
    assert tuple(taken) == res.schedule.per_step_full
    errs = _errs(res, lat)
    print("config4 geometry (1 dual + 1 joint block) FFcF per-step rel-L2:", ["%.2e" % e for e in errs])
    del model, orc
    torch.cuda.empty_cache()
    assert max(errs) <= TOL_BF16, errs
