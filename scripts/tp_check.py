#!/usr/bin/env python
"""Multi-GPU TP-SP parity: P-rank tensor-parallel Single-DiT and MM-DiT denoise vs 1 GPU and the CPU oracle.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 scripts/tp_check.py
    AQB_OVERSUBSCRIBE=1 torchrun --nproc-per-node 8 ... (P=8 on fewer GPUs)

Every rank runs the TP model (fused all-gather in the LN+modulate kernel, fused
reduce-scatter in the row-parallel GEMM epilogues); rank 0 also runs the unsharded
model and the oracle.  Checks: same cache schedule, rel-L2(TP, 1-GPU) <= 5e-3 and
rel-L2(TP, oracle) <= 1e-2 per step, static schedule and rel-L1 policy.  Prints one
JSON line per case from rank 0; exit code 1 on failure.
"""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dit_oracle as ref  # noqa: E402
from paper_2505_10584_b200 import DiTConfig, RelL1Policy, build_model, denoise, front_block_count, plan_cache  # noqa: E402
from paper_2505_10584_b200.parallel import TensorSP, init_from_env, oversubscribed  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402


def rel(a, b):
    return float((a.double().cpu() - b.double().cpu()).norm() / b.double().cpu().norm())


def main():
    init_from_env("nccl")
    sp = TensorSP()
    ok = True
    cases = [
        ("single", DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40),
         (3, 8, 16)),
        ("single-16h", DiTConfig("single-dit", hidden_size=2048, num_heads=16, num_single=2, text_dim=256,
                                 text_len=40), (5, 8, 24)),
        ("mm", DiTConfig("mm-dit", hidden_size=1024, num_heads=8, num_dual=2, num_single=2, text_dim=192, text_len=24,
                         pooled_dim=64), (2, 8, 16)),
        ("mm-24h", DiTConfig("mm-dit", hidden_size=3072, num_heads=24, num_dual=1, num_single=1, text_dim=192,
                             text_len=24, pooled_dim=64), (2, 8, 16)),
    ]
    for name, cfg, grid in cases:
        W = init_weights(cfg, seed=0)
        inp = synthetic_inputs(cfg, grid)
        pooled = inp["pooled"] if cfg.family == "mm-dit" else None
        m_tp = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"], pooled)
        for cache in (plan_cache(8, warmup=2, interval=2), RelL1Policy(threshold=0.06, warmup=2)):
            r_tp = denoise(m_tp, inp["x0"], 8, cache, trajectory=True)
            good = m_tp.peer_ok()
            if sp.rank == 0:
                m1 = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled)
                r1 = denoise(m1, inp["x0"], 8, cache, trajectory=True)
                orc = ref.OracleDiT(cfg, W, inp["text"], pooled, grid,
                                    n_front=front_block_count(cfg.num_layers, 0.25), mode=cache.mode)
                if isinstance(cache, RelL1Policy):
                    lat, taken, _ = ref.denoise(orc, inp["x0"], 8, policy=cache)
                else:
                    lat, taken, _ = ref.denoise(orc, inp["x0"], 8, flags=cache.per_step_full)
                e_1 = max(rel(a, b) for a, b in zip(r_tp.trajectory, r1.trajectory))
                e_o = max(rel(a, b) for a, b in zip(r_tp.trajectory, lat[1:]))
                same = list(r_tp.schedule.per_step_full) == list(taken) == list(r1.schedule.per_step_full)
                good = good and same and e_o <= 1e-2 and e_1 <= 5e-3
                print(json.dumps({"case": name, "P": sp.P, "parallel": "tp-sp", "cache": type(cache).__name__,
                                  "schedule": r_tp.schedule.as_string(), "same_schedule": same,
                                  "max_rel_l2_vs_1gpu": e_1, "max_rel_l2_vs_oracle": e_o, "ok": good}), flush=True)
            ok &= good
            dist.barrier()
    flag = torch.tensor([1 if ok else 0], device="cpu" if oversubscribed() else "cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) else 1)


if __name__ == "__main__":
    main()
