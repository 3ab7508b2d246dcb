#!/usr/bin/env python
"""Full-size multi-GPU parity (one GPU per rank, NCCL rendezvous, fused p2p exchange):

* config 2 — Single-DiT 2B, 28 blocks, 7,800 tokens, 30 steps of plan_cache(30);
* config 3 — MM-DiT 13.4B, 54 blocks, 25,440 + 256 tokens, plan_cache(4, 1, 2) = FFcF;

under Ulysses (and, with --tp, TP-SP) on P ranks vs the same model on 1 GPU (rank 0) and the
fp32 oracle on rank 0's GPU.  One JSON line per case from rank 0.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 scripts/full_scale_mp_check.py [--tp]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dit_oracle as ref  # noqa: E402
from paper_2505_10584_b200 import build_model, denoise, front_block_count, plan_cache  # noqa: E402
from paper_2505_10584_b200.config import MM_DIT_13B, SINGLE_DIT_2B, VIDEO_480P_17F, VIDEO_480P_61F  # noqa: E402
from paper_2505_10584_b200.parallel import TensorSP, Ulysses, init_from_env  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm())


def main():
    init_from_env("nccl")
    sp = TensorSP() if "--tp" in sys.argv else Ulysses(exchange="p2p")
    ok = True
    for name, cfg, video, steps, sched in (("config2", SINGLE_DIT_2B, VIDEO_480P_17F, 30, plan_cache(30)),
                                           ("config3", MM_DIT_13B, VIDEO_480P_61F, 4, plan_cache(4, 1, 2))):
        grid = video.grid(cfg)
        W = init_weights(cfg, seed=0, device="cuda")
        inp = synthetic_inputs(cfg, grid, device="cuda")
        pooled = inp["pooled"] if cfg.family == "mm-dit" else None
        m_sp = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"], pooled)
        r_sp = denoise(m_sp, inp["x0"], steps, sched, trajectory=True)
        traj_sp = [t.cpu() for t in r_sp.trajectory]
        peer_ok = m_sp.peer_ok()
        m_sp.close()
        del m_sp, r_sp
        torch.cuda.empty_cache()
        if sp.rank == 0:
            m1 = build_model(cfg, weights=W).prepare(grid, inp["text"], pooled)
            r1 = denoise(m1, inp["x0"], steps, sched, trajectory=True)
            traj_1 = [t.cpu() for t in r1.trajectory]
            del m1, r1
            torch.cuda.empty_cache()
            orc = ref.OracleDiT(cfg, W, inp["text"], pooled, grid, n_front=front_block_count(cfg.num_layers, 0.25),
                                device="cuda")
            lat, taken, _ = ref.denoise(orc, inp["x0"], steps, flags=sched.per_step_full)
            del orc
            torch.cuda.empty_cache()
            e1 = max(rel(a, b) for a, b in zip(traj_sp, traj_1))
            eo = max(rel(a, b) for a, b in zip(traj_sp, lat[1:]))
            e1o = max(rel(a, b) for a, b in zip(traj_1, lat[1:]))
            good = peer_ok and tuple(taken) == sched.per_step_full and eo <= 1e-2 and e1 <= 5e-3
            ok &= good
            print(json.dumps({"case": name, "P": sp.P, "parallel": "tp-sp" if sp.tensor_parallel else "ulysses-p2p",
                              "schedule": sched.as_string(), "steps": steps, "max_rel_l2_vs_1gpu": e1,
                              "max_rel_l2_vs_oracle": eo, "one_gpu_vs_oracle": e1o, "peer_barriers_ok": peer_ok,
                              "ok": good}), flush=True)
        del W
        torch.cuda.empty_cache()
        dist.barrier()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) else 1)


if __name__ == "__main__":
    main()
