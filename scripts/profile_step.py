#!/usr/bin/env python
"""One full + one cached denoise step of the config-2 model, bracketed by
cudaProfilerStart/Stop — the launch list the bench's kernel shares come from.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import SINGLE_DIT_2B, build_model, plan_cache  # noqa: E402
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs  # noqa: E402


def main():
    cfg, grid = SINGLE_DIT_2B, (5, 30, 52)
    W = init_weights(cfg, seed=0, device="cuda")
    inp = synthetic_inputs(cfg, grid, device="cuda")
    model = build_model(cfg, weights=W).prepare(grid, inp["text"])
    del W
    model.reset(inp["x0"], 30, cache_mode=plan_cache(30).mode)
    for mode in ("full", "cached"):  # warm (one-time attribute setup, L2, clocks)
        model.step(mode, True)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    model.step("full", True)
    model.step("cached", True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one full + one cached step")


if __name__ == "__main__":
    main()
