"""Golden vectors for ``paper_2505_10584_b200.planner`` from the REAL reference (``ditplan``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden_planner.py

Records, from ``/root/reference/pkg/src``: ``estimate_param_count`` and
``flops_per_microstep`` over a grid of ``ModelArch`` dims (``config.py:224-249``,
``simulate.py:60-73``), ``ModelArch`` validation errors (``config.py:44-60``),
``tp_sp_layer_comm`` / ``cp_gate_and_comm`` over a grid incl. gate violations
(``comm.py:28-96``), and ``BUILTIN_CHUNKS`` with ``chunk_retained_bytes``
(``memory.py:30-107``).  The GPU box never reads ``/root/reference``.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "planner.json")


def main():
    sys.path.insert(0, REF)
    from ditplan.comm import CP_TOKEN_GATE, cp_gate_and_comm, tp_sp_layer_comm
    from ditplan.config import ModelArch, estimate_param_count
    from ditplan.errors import ConfigError
    from ditplan.memory import BUILTIN_CHUNKS, chunk_retained_bytes
    from ditplan.presets import TABLE2_FIT
    from ditplan.simulate import flops_per_microstep

    archs = []
    for H, A, L in ((128, 4, 2), (1024, 8, 4), (2048, 16, 28), (3072, 24, 54), (5120, 40, 60)):
        for ffn in (2, 4):
            for mode in ("shared-weights", "per-block-dedicated"):
                for patch in ((1, 2, 2), (2, 2, 2), (1, 1, 1)):
                    arch = ModelArch(hidden_size=H, num_heads=A, num_layers=L, ffn_multiplier=ffn, adaln_mode=mode,
                                     patch_t=patch[0], patch_h=patch[1], patch_w=patch[2])
                    est = {c: estimate_param_count(arch, c).__dict__ for c in (4, 8, 16)}
                    fl = [{"B": B, "S": S, "value": flops_per_microstep(arch, B, S)}
                          for B in (1, 2) for S in (48, 7800, 25696, 119056)]
                    archs.append({"dims": [H, A, L, ffn, mode, list(patch)], "estimate": est, "flops": fl})
    errors = []
    for kw in ({"hidden_size": 0, "num_heads": 1, "num_layers": 1}, {"hidden_size": 8, "num_heads": 0, "num_layers": 1},
               {"hidden_size": 8, "num_heads": 1, "num_layers": -1}, {"hidden_size": 8, "num_heads": 1, "num_layers": 1,
                                                                      "ffn_multiplier": 2.5},
               {"hidden_size": 8, "num_heads": 1, "num_layers": 1, "patch_h": 0},
               {"hidden_size": 8, "num_heads": 1, "num_layers": 1, "adaln_mode": "shared"},
               {"hidden_size": 8, "num_heads": 1, "num_layers": 1, "param_count": 0.0}):
        try:
            ModelArch(**kw)
            errors.append({"kwargs": kw, "error": None})
        except ConfigError as e:
            errors.append({"kwargs": kw, "error": str(e), "path": e.path})
    comm = []
    for tokens in (7800, 200_000, 200_001, 476_224):
        for cp in (1, 2, 4, 8):
            for act in (2, 4):
                r = cp_gate_and_comm(tokens, 1, tokens, 3072, cp, act, 50e9)
                comm.append({"fn": "cp", "args": [tokens, 1, tokens, 3072, cp, act, 50e9],
                             "enabled": r.enabled, "time_ms": r.time_ms, "violation": r.violation})
    for S in (7800, 119056):
        for tp in (1, 2, 4, 8):
            for ov in (0.0, 0.5, 1.0):
                raw, exp = tp_sp_layer_comm(1, S, 3072, tp, 2, 900e9, ov)
                comm.append({"fn": "tp_sp", "args": [1, S, 3072, tp, 2, 900e9, ov], "raw": raw, "exposed": exp})
    chunks = []
    for c in BUILTIN_CHUNKS.chunks:
        rb = [{"args": [B, S, H, A, tp], "bytes": chunk_retained_bytes(c, B, S, H, A, tp)}
              for B in (1, 2) for (S, H, A) in ((115200, 3072, 24), (7800, 2048, 16)) for tp in (1, 8)]
        chunks.append({"name": c.name, "coeff_bsh": c.coeff_bsh, "coeff_bas": c.coeff_bas,
                       "fwd_latency_ms": c.fwd_latency_ms, "recomputable": c.recomputable,
                       "offloadable": c.offloadable, "attention_class": c.is_attention_class, "retained": rb})
    table2 = {"dims": [TABLE2_FIT.hidden_size, TABLE2_FIT.num_heads, TABLE2_FIT.num_layers,
                       TABLE2_FIT.ffn_multiplier, TABLE2_FIT.adaln_mode,
                       [TABLE2_FIT.patch_t, TABLE2_FIT.patch_h, TABLE2_FIT.patch_w]],
              "param_count": TABLE2_FIT.param_count,
              "extra_unpartitioned_layers": list(TABLE2_FIT.extra_unpartitioned_layers)}
    doc = {"source": "ditplan @ /root/reference (tests/golden/make_golden_planner.py)", "archs": archs,
           "model_arch_errors": errors, "comm": comm, "cp_token_gate": CP_TOKEN_GATE, "chunks": chunks,
           "chunk_table": {"ref_batch": BUILTIN_CHUNKS.ref_batch, "ref_seqlen": BUILTIN_CHUNKS.ref_seqlen,
                           "ref_hidden": BUILTIN_CHUNKS.ref_hidden, "ref_heads": BUILTIN_CHUNKS.ref_heads,
                           "ref_tp": BUILTIN_CHUNKS.ref_tp},
           "table2_fit": table2}
    with open(OUT, "w") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)
    print(f"wrote {OUT}: {len(archs)} archs, {len(errors)} error cases, {len(comm)} comm cases, {len(chunks)} chunks")


if __name__ == "__main__":
    main()
