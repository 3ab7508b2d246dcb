#!/usr/bin/env python
"""Per-shape kernel time of one full config-2 step (CUDA events per launch), any N:

    [torchrun --nproc-per-node P --master-addr 127.0.0.1] scripts/profile_shapes.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import SINGLE_DIT_2B, build_model, ops  # noqa: E402
from paper_2505_10584_b200.parallel import Ulysses, init_from_env  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
sp = None
if world > 1:
    init_from_env("nccl")
    sp = Ulysses()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
cfg, grid = SINGLE_DIT_2B, (5, 30, 52)
W = init_weights(cfg, seed=0, device="cuda")
inp = synthetic_inputs(cfg, grid, device="cuda")
model = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"])
del W
model.reset(inp["x0"], 30)
for _ in range(2):
    model.step("full", True)
torch.cuda.synchronize()
prof = ops.KernelProfiler(timing=True)
ops.set_profiler(prof)
model.step("full", True)
ops.set_profiler(None)
rows = prof.by_launch()
if sp is None or sp.rank == 0:
    tot = sum(v["ms"] for v in rows.values())
    print(f"P={world}: one full step, {tot:.2f} ms of kernels")
    for (name, work), v in sorted(rows.items(), key=lambda kv: -kv[1]["ms"]):
        rate = f"{work * v['launches'] / (v['ms'] / 1e3) / 1e12:8.1f} TFLOP/s" if "gemm" in name or "attention" in name else ""
        print(f"  {name:34s} work {work / 1e9:9.3f} G x{v['launches']:3d}  {v['ms']:8.3f} ms {100 * v['ms'] / tot:5.1f}% {rate}")
if sp:
    import torch.distributed as dist
    dist.barrier()
    os._exit(0)
