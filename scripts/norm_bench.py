#!/usr/bin/env python
"""LayerNorm+modulate microbenchmark at the in-model shapes (config 2 full / Ulysses shards,
MM-DiT 720p shard).  Two timings per shape:

* ``single``: one launch between CUDA events after an L2 flush (includes launch latency);
* ``graph``: 24 launches captured in one CUDA graph over 8 rotating x/y buffer sets
  (> L2 in total), so consecutive launches overlap their prologues like in the model.

Bytes per launch = rows·H·(4 + 2) (f32 in, bf16 out).  ``--ncu rows H``: two launches of one
shape and nothing else (for ``ncu -k regex:norm_mod_row -s 1 -c 1``).
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"


def once(rows, H):
    x = torch.randn(rows, H, device=dev)
    y = torch.empty(rows, H, device=dev, dtype=torch.bfloat16)
    sh, sc = torch.randn(H, device=dev), torch.randn(H, device=dev)
    for _ in range(2):
        ops.norm_modulate(x, sh, sc, y)
    torch.cuda.synchronize()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--ncu":
        once(int(sys.argv[2]), int(sys.argv[3]))
        return
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = []
    for rows, H in ((7800, 2048), (3900, 2048), (1950, 2048), (975, 2048), (15106, 3072), (25696, 3072),
                    (7800 + 256, 1024)):
        nb = 8
        xs = [torch.randn(rows, H, device=dev) for _ in range(nb)]
        ys = [torch.empty(rows, H, device=dev, dtype=torch.bfloat16) for _ in range(nb)]
        sh, sc = torch.randn(H, device=dev), torch.randn(H, device=dev)
        for i in range(nb):
            ops.norm_modulate(xs[i], sh, sc, ys[i])
        torch.cuda.synchronize()
        ts = []
        for it in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.norm_modulate(xs[it % nb], sh, sc, ys[it % nb])
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        single = sorted(ts)[len(ts) // 2]
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                for i in range(24):
                    ops.norm_modulate(xs[i % nb], sh, sc, ys[i % nb])
        g.replay()
        torch.cuda.synchronize()
        gt = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            gt.append(e0.elapsed_time(e1) / 24)
        graph = sorted(gt)[len(gt) // 2]
        byt = rows * H * 6
        rec = {"rows": rows, "hidden": H,
               "single_us": single * 1e3, "single_gbs": byt / single / 1e6,
               "graph_us": graph * 1e3, "graph_gbs": byt / graph / 1e6}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del xs, ys, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
