#!/usr/bin/env python
"""Our tcgen05 GEMM (plain bf16 epilogue) vs cuBLAS (torch.matmul, bf16 out) at the config-2 and
MM-DiT projection shapes, both timed in a CUDA graph of 8 launches over 4 rotating A buffers."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

bf = torch.bfloat16


def graph_time(fn, n=8):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            for i in range(n):
                fn(i)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n)
    return sorted(ts)[3]


for m, n, k in ((7800, 6144, 2048), (7800, 2048, 2048), (7800, 8192, 2048), (7800, 2048, 8192), (1950, 6144, 2048),
                (1950, 2048, 2048), (975, 8192, 2048), (25696, 9216, 3072), (25696, 3072, 3072),
                (25696, 12288, 3072), (25696, 3072, 12288), (8192, 8192, 8192)):
    A = [torch.randn(m, k, device="cuda").to(bf) for _ in range(4)]
    w = (torch.randn(n, k, device="cuda") * 0.02).to(bf)
    O = [torch.empty(m, n, device="cuda", dtype=bf) for _ in range(4)]
    ours = graph_time(lambda i: ops.gemm(A[i % 4], w, O[i % 4]))
    wt = w.t()
    cub = graph_time(lambda i: torch.matmul(A[i % 4], wt, out=O[i % 4]))
    f = 2.0 * m * n * k
    print(json.dumps({"m": m, "n": n, "k": k, "ours_us": ours * 1e3, "cublas_us": cub * 1e3,
                      "ours_tflops": f / ours / 1e9, "cublas_tflops": f / cub / 1e9}), flush=True)
    del A, O
    torch.cuda.empty_cache()
