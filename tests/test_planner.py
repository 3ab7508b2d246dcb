"""The planner formulas the hot path is sized by vs values produced by
the reference itself (tests/golden/planner.json, tests/golden/make_golden_planner.py)."""

import json
import os

import pytest

from paper_2505_10584_b200 import MM_DIT_13B, SINGLE_DIT_2B, flops_per_step
from paper_2505_10584_b200.errors import ConfigError
from paper_2505_10584_b200.planner import (BUILTIN_CHUNKS, CP_TOKEN_GATE, TABLE2_FIT, ChunkSpec, ChunkTable, ModelArch,
                                           chunk_retained_bytes, cp_gate_and_comm, estimate_param_count,
                                           flops_per_microstep, model_arch, tp_sp_layer_comm)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "planner.json")))


def _arch(dims):
    H, A, L, ffn, mode, patch = dims
    return ModelArch(hidden_size=H, num_heads=A, num_layers=L, ffn_multiplier=ffn, adaln_mode=mode,
                     patch_t=patch[0], patch_h=patch[1], patch_w=patch[2])


def test_param_count_and_flops_bit_exact():
    n = 0
    for case in GOLD["archs"]:
        arch = _arch(case["dims"])
        for c, est in case["estimate"].items():
            assert estimate_param_count(arch, int(c)).__dict__ == est
        for f in case["flops"]:
            assert flops_per_microstep(arch, f["B"], f["S"]) == f["value"]
            n += 1
    assert n == 60 * 8


def test_model_arch_validation_paths_and_messages():
    for case in GOLD["model_arch_errors"]:
        if case["error"] is None:
            ModelArch(**case["kwargs"])
            continue
        with pytest.raises(ConfigError) as e:
            ModelArch(**case["kwargs"])
        assert str(e.value) == case["error"] and e.value.path == case["path"]


def test_comm_costs_and_cp_gate():
    assert CP_TOKEN_GATE == GOLD["cp_token_gate"]
    for case in GOLD["comm"]:
        if case["fn"] == "cp":
            r = cp_gate_and_comm(*case["args"])
            assert (r.enabled, r.time_ms, r.violation) == (case["enabled"], case["time_ms"], case["violation"])
        else:
            assert tp_sp_layer_comm(*case["args"]) == (case["raw"], case["exposed"])
    with pytest.raises(ConfigError) as e:
        cp_gate_and_comm(1, 1, 1, 1, 0, 2, 1e9)
    assert e.value.path == "parallel.cp"
    with pytest.raises(ConfigError) as e:
        tp_sp_layer_comm(1, 1, 1, 2, 2, 1e9, 1.5)
    assert e.value.path == "overlap.tp_sp_fraction"


def test_builtin_chunk_table_and_retained_bytes():
    t = GOLD["chunk_table"]
    assert (BUILTIN_CHUNKS.ref_batch, BUILTIN_CHUNKS.ref_seqlen, BUILTIN_CHUNKS.ref_hidden, BUILTIN_CHUNKS.ref_heads,
            BUILTIN_CHUNKS.ref_tp) == (t["ref_batch"], t["ref_seqlen"], t["ref_hidden"], t["ref_heads"], t["ref_tp"])
    assert BUILTIN_CHUNKS.names() == tuple(c["name"] for c in GOLD["chunks"])
    for g in GOLD["chunks"]:
        c = BUILTIN_CHUNKS.by_name(g["name"])
        assert (c.coeff_bsh, c.coeff_bas, c.fwd_latency_ms, c.recomputable, c.offloadable, c.is_attention_class) == (
            g["coeff_bsh"], g["coeff_bas"], g["fwd_latency_ms"], g["recomputable"], g["offloadable"],
            g["attention_class"])
        for r in g["retained"]:
            assert chunk_retained_bytes(c, *r["args"]) == r["bytes"]
    with pytest.raises(ConfigError):
        ChunkTable(chunks=(ChunkSpec("a", 1), ChunkSpec("a", 2)))
    with pytest.raises(ConfigError) as e:
        BUILTIN_CHUNKS.by_name("nope")
    assert e.value.path == "chunks"


def test_table2_fit_and_the_executable_models():
    g = GOLD["table2_fit"]
    assert _arch(g["dims"]) == ModelArch(hidden_size=3072, num_heads=24, num_layers=54)
    assert TABLE2_FIT.param_count == g["param_count"]
    assert list(TABLE2_FIT.extra_unpartitioned_layers) == g["extra_unpartitioned_layers"]
    # the executable 13.4B MM-DiT is TABLE2_FIT's geometry (25 dual + 29 single = 54 blocks)
    a = model_arch(MM_DIT_13B)
    assert (a.hidden_size, a.num_heads, a.num_layers, a.ffn_multiplier, a.adaln_mode) == (3072, 24, 54, 4,
                                                                                         "per-block-dedicated")
    # the runtime's per-step FLOP count reduces to the planner's convention for joint attention
    S = 118800 + 256
    assert flops_per_step(MM_DIT_13B, 118800)["total"] == pytest.approx(flops_per_microstep(a, 1, S), rel=1e-3)
    b = model_arch(SINGLE_DIT_2B)
    assert b.adaln_mode == "shared-weights" and b.num_layers == 28
