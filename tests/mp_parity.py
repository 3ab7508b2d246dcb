#!/usr/bin/env python
"""Multi-rank parity worker (launched by ``tests/test_multirank_gpu.py`` under torchrun).

    AQB_OVERSUBSCRIBE=1 python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \\
        tests/mp_parity.py --parallel ulysses|tp --out cases.jsonl

Every rank runs the P-rank model (Ulysses sequence parallelism with the fused p2p exchange, or
TP-SP with the all-gather / reduce-scatter fused into the kernels); rank 0 also runs the
unsharded model and the fp32 CPU oracle.  Per case and cache policy it checks

* every rank took the same schedule, equal to the 1-GPU model's and the oracle's;
* rel-L1 policies really skip: the threshold is 2.5x the median per-step rel-L1 of the
  oracle's own probe (broadcast from rank 0), and every rank must record cached steps;
* per-step latent rel-L2 <= 1e-2 vs the oracle and <= 5e-3 vs 1 GPU;
* no peer barrier timed out on any rank.

The exchange checked is the one the reference costs in ``comm.py:65-96`` (Ulysses / CP) and
``comm.py:28-53`` (TP-SP); the paper's layouts ``PAPER.md:191-197,320``.
One JSON line per case (rank 0) goes to ``--out``; the exit code is 0 only if all passed.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dit_oracle as ref  # noqa: E402
from paper_2505_10584_b200 import (DiTConfig, RelL1Policy, build_model, denoise, front_block_count,  # noqa: E402
                                   plan_cache)
from paper_2505_10584_b200.parallel import TensorSP, Ulysses, init_from_env  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402

STEPS = 8

CASES = {
    "ulysses": [
        ("single", DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40),
         (3, 8, 16)),
        ("mm", DiTConfig("mm-dit", hidden_size=1024, num_heads=8, num_dual=2, num_single=2, text_dim=192,
                         text_len=24, pooled_dim=64), (2, 8, 16)),
        ("mm-24h", DiTConfig("mm-dit", hidden_size=3072, num_heads=24, num_dual=1, num_single=1, text_dim=192,
                             text_len=24, pooled_dim=64), (2, 8, 16)),
        ("single-d32", DiTConfig("single-dit", hidden_size=256, num_heads=8, num_single=4, text_dim=256,
                                 text_len=40), (3, 8, 16)),
    ],
    "tp": [
        ("single", DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40),
         (3, 8, 16)),
        ("single-16h", DiTConfig("single-dit", hidden_size=2048, num_heads=16, num_single=2, text_dim=256,
                                 text_len=40), (5, 8, 24)),
        ("mm", DiTConfig("mm-dit", hidden_size=1024, num_heads=8, num_dual=2, num_single=2, text_dim=192,
                         text_len=24, pooled_dim=64), (2, 8, 16)),
        ("mm-24h", DiTConfig("mm-dit", hidden_size=3072, num_heads=24, num_dual=1, num_single=1, text_dim=192,
                             text_len=24, pooled_dim=64), (2, 8, 16)),
    ],
}


def rel(a, b):
    return float((a.double().cpu() - b.double().cpu()).norm() / b.double().cpu().norm())


def probe_threshold(orc, x0):
    """2.5x the median per-step rel-L1 of the oracle's probe over 4 steps: the accumulator crosses
    it about every third step and sits >= half a step's rel away from it at each decision."""
    _, _, probe = ref.denoise(orc, x0, 4, policy=RelL1Policy(threshold=1e9, warmup=1), return_all=False)
    vals = sorted(probe[1:])
    return 2.5 * vals[len(vals) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parallel", choices=["ulysses", "tp"], required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="Ulysses exchange (nccl needs one GPU per rank, not AQB_OVERSUBSCRIBE)")
    ap.add_argument("--cases", default=None, help="comma-separated case names (default: all)")
    args = ap.parse_args()
    init_from_env("nccl")
    sp = TensorSP() if args.parallel == "tp" else Ulysses(exchange=args.exchange)
    rank, P = sp.rank, sp.P
    out = open(args.out, "a") if rank == 0 else None
    ok = True
    for name, cfg, grid in CASES[args.parallel]:
        if args.cases and name not in args.cases.split(","):
            continue
        W = init_weights(cfg, seed=0)
        inp = synthetic_inputs(cfg, grid)
        pooled = inp["pooled"] if cfg.family == "mm-dit" else None
        nf = front_block_count(cfg.num_layers, 0.25)
        thr = [None]
        if rank == 0:
            thr[0] = probe_threshold(ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=nf), inp["x0"])
        dist.broadcast_object_list(thr, 0)
        caches = [plan_cache(STEPS, warmup=2, interval=2), RelL1Policy(threshold=thr[0], warmup=2),
                  plan_cache(STEPS, warmup=2, interval=2, mode="attention-cache"),
                  RelL1Policy(threshold=thr[0], warmup=2, mode="attention-cache")]
        m_sp = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"], pooled)
        m1 = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled) if rank == 0 else None
        for cache in caches:
            r_sp = denoise(m_sp, inp["x0"], STEPS, cache, trajectory=True)
            mine = r_sp.schedule.as_string()
            peer_ok = m_sp.peer_ok()
            everyone = [None] * P
            dist.all_gather_object(everyone, (mine, peer_ok))
            if rank == 0:
                r1 = denoise(m1, inp["x0"], STEPS, cache, trajectory=True)
                orc = ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=nf, mode=cache.mode)
                if isinstance(cache, RelL1Policy):
                    lat, taken, _ = ref.denoise(orc, inp["x0"], STEPS, policy=cache)
                else:
                    lat, taken, _ = ref.denoise(orc, inp["x0"], STEPS, flags=cache.per_step_full)
                oracle_s = "".join("F" if f else "c" for f in taken)
                e_1 = max(rel(a, b) for a, b in zip(r_sp.trajectory, r1.trajectory))
                e_o = max(rel(a, b) for a, b in zip(r_sp.trajectory, lat[1:]))
                same = all(s == oracle_s for s, _ in everyone) and r1.schedule.as_string() == oracle_s
                skips = oracle_s.count("c") > 0
                barriers = all(b for _, b in everyone)
                good = same and skips and barriers and e_o <= 1e-2 and e_1 <= 5e-3
                ok &= good
                rec = {"case": name, "P": P, "parallel": args.parallel, "exchange": sp.exchange, "policy": type(cache).__name__,
                       "mode": cache.mode, "threshold": getattr(cache, "threshold", None),
                       "schedule_per_rank": [s for s, _ in everyone], "schedule_oracle": oracle_s,
                       "schedule_1gpu": r1.schedule.as_string(), "same_schedule": same, "skips": skips,
                       "peer_barriers_ok": barriers, "max_rel_l2_vs_1gpu": e_1, "max_rel_l2_vs_oracle": e_o,
                       "ok": good}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                print(json.dumps(rec), flush=True)
            dist.barrier()
        m_sp.close()
        del m_sp, m1
        torch.cuda.empty_cache()
    flag = [ok]
    dist.broadcast_object_list(flag, 0)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


if __name__ == "__main__":
    main()
