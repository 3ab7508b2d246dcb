"""Debug: TP-SP static attention-cache at P ranks vs 1 GPU, per-step rel-L2 (rank 0 prints)."""
import os
import sys

import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import DiTConfig, build_model, denoise, plan_cache  # noqa: E402
from paper_2505_10584_b200.parallel import TensorSP, init_from_env  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402

init_from_env("nccl")
sp = TensorSP()
cfg = DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40)
grid = (3, 8, 16)
W = init_weights(cfg, seed=0)
inp = synthetic_inputs(cfg, grid)
m = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"])
m1 = build_model(cfg, weights=W).prepare(grid, inp["text"]) if sp.rank == 0 else None
for sched in (plan_cache(8, 2, 2, mode="attention-cache"), plan_cache(8, 2, 8, mode="attention-cache"),
              plan_cache(8, 8, 2, mode="attention-cache")):
    r = denoise(m, inp["x0"], 8, sched, trajectory=True)
    if sp.rank == 0:
        r1 = denoise(m1, inp["x0"], 8, sched, trajectory=True)
        errs = [float((a - b).norm() / b.norm()) for a, b in zip(r.trajectory, r1.trajectory)]
        print(os.environ.get("TAG", ""), sched.as_string(), ["%.1e" % e for e in errs], flush=True)
    dist.barrier()
m.close()
dist.destroy_process_group()
