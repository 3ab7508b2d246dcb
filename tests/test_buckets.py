"""Geometry boundary (``buckets.py:17-122``) and planner leftovers (``config.py:252-256``,
``memory.py:110-134``) against golden vectors from the real ``ditplan``
(``tests/golden/make_golden_buckets.py``)."""

import json
import os

import pytest

from paper_2505_10584_b200 import (Bucket, LatentShape, ModelArch, VaeSpec, load_chunk_table, resolved_param_count,
                                   snap_bucket, token_count, video_token_count)
from paper_2505_10584_b200.config import SINGLE_DIT_2B
from paper_2505_10584_b200.errors import ConfigError, DimensionError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "buckets.json")))
VAES = [VaeSpec(), VaeSpec(temporal_ratio=8, spatial_ratio=16, latent_channels=16), VaeSpec(1, 1, 4)]


def _arch(p):
    return None if p is None else ModelArch(hidden_size=64, num_heads=4, num_layers=2, patch_t=p[0], patch_h=p[1],
                                            patch_w=p[2])


def test_token_count_and_snap_golden():
    for case in GOLD["token_count"]:
        b = Bucket(*case["bucket"])
        assert b.label() == case["label"]
        vae, arch = VAES[case["vae"]], _arch(case["patch"])
        if "error" in case:
            with pytest.raises(DimensionError) as ei:
                token_count(b, vae, arch)
            assert [str(ei.value), ei.value.path] == case["error"]
        else:
            ls = token_count(b, vae, arch)
            assert isinstance(ls, LatentShape)
            assert [ls.t_lat, ls.h_lat, ls.w_lat, ls.tokens, ls.tokens_batch] == case["shape"]
        assert list(snap_bucket(b, vae, arch).key()) == case["snapped"]


def test_bucket_errors_golden():
    for case in GOLD["bucket_errors"]:
        with pytest.raises(ConfigError) as ei:
            Bucket(**case["kwargs"])
        assert (str(ei.value), ei.value.path) == (case["error"], case["path"])


def test_token_count_accepts_an_executable_config():
    """A DiTConfig's patch works like a ModelArch's (the config-2 / config-4 token counts)."""
    assert token_count(Bucket(1, 17, 480, 832), arch=SINGLE_DIT_2B).tokens == 7800
    assert token_count(Bucket(2, 129, 720, 1280)).tokens_batch == 2 * 118_800
    assert snap_bucket(Bucket(1, 61, 480, 854)).key() == (1, 61, 480, 848)
    assert video_token_count(61, 480, 848) == 25_440


def test_resolved_param_count_golden():
    for case in GOLD["resolved_param_count"]:
        H, A, L, mode, pc = case["dims"]
        assert resolved_param_count(ModelArch(hidden_size=H, num_heads=A, num_layers=L, adaln_mode=mode,
                                              param_count=pc)) == case["value"]


def test_load_chunk_table_golden(tmp_path):
    for k, case in enumerate(GOLD["chunk_tables"]):
        if case.get("missing"):
            missing = tmp_path / "missing.json"
            with pytest.raises(ConfigError) as ei:
                load_chunk_table(missing)
            assert ei.value.path == str(missing) and str(ei.value).startswith(str(missing) + ":")
            continue
        path = tmp_path / f"t{k}.json"
        doc = case["doc"]
        path.write_text(doc if isinstance(doc, str) else json.dumps(doc))
        if "error" in case:
            with pytest.raises(ConfigError) as ei:
                load_chunk_table(path)
            assert str(ei.value).replace(str(path), "<file>") == case["error"]["str"]
            assert ei.value.path.replace(str(path), "<file>") == case["error"]["path"]
        else:
            t = load_chunk_table(str(path))
            got = {"chunks": [c.__dict__ for c in t.chunks],
                   **{m: getattr(t, m) for m in ("ref_batch", "ref_seqlen", "ref_hidden", "ref_heads", "ref_tp")}}
            assert got == case["table"]
