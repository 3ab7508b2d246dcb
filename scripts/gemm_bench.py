#!/usr/bin/env python
"""GEMM microbenchmark at the config-2 block shapes per Ulysses shard (M = 7800/P), timed in a
CUDA graph (8 back-to-back launches over 4 rotating operand sets, so launch gaps are hidden
like in the model).  AQB_GEMM_VARIANT forces a tile variant (read once per process)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402

dev = "cuda"
bf = torch.bfloat16


def case_once(name, m, n, k):
    """One warm-up + one launch (for ncu -k regex:gemm -s 1 -c 1)."""
    case(name, m, n, k, graph=False)


def case(name, m, n, k, graph=True):
    nb = 4
    A = [torch.randn(m, k, device=dev).to(bf) for _ in range(nb)]
    w = (torch.randn(n, k, device=dev) * 0.02).to(bf)
    b = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev)
    d = 128
    cos = torch.randn(m, d // 2, device=dev)
    sin = torch.randn(m, d // 2, device=dev)
    qw = torch.ones(d, device=dev)
    if name in ("proj", "xproj", "fc2"):
        O = [torch.randn(m, n, device=dev) for _ in range(nb)]
    else:
        O = [torch.empty(m, n, device=dev, dtype=bf) for _ in range(nb)]
    aux = [torch.empty(m, n, device=dev, dtype=bf) for _ in range(nb)]

    def launch(i):
        a, o = A[i % nb], O[i % nb]
        if name == "qkv":
            ops.gemm_qknorm_rope(a, w, o, n // 3, 2, qw, qw, 1e-6, bias=b, cos=cos, sin=sin, rope_rows=m)
        elif name == "xq":
            ops.gemm_qknorm_rope(a, w, o, n, 1, qw, None, 1e-6, bias=b)
        elif name == "proj":
            ops.gemm(a, w, o, bias=b, gate=g, epilogue="gate_res", aux=aux[i % nb])
        elif name in ("xproj", "fc2"):
            ops.gemm(a, w, o, bias=b, gate=g if name == "fc2" else None, epilogue="gate_res")
        elif name == "fc1":
            ops.gemm(a, w, o, bias=b, epilogue="gelu")

    for i in range(nb):
        launch(i)
    torch.cuda.synchronize()
    if not graph:
        return None
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr):
            for i in range(8):
                launch(i)
    gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 8)
    ms = sorted(ts)[len(ts) // 2]
    return {"name": name, "m": m, "n": n, "k": k, "variant": os.environ.get("AQB_GEMM_VARIANT", "auto"),
            "us": ms * 1e3, "tflops": 2.0 * m * n * k / ms / 1e9}


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--ncu":  # one launch of one case: --ncu name m n k
        name, m, n, k = sys.argv[2], *map(int, sys.argv[3:6])
        case_once(name, m, n, k)
        return
    ms = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["7800", "3900", "1950", "975"])]
    for m in ms:
        for name, n, k in (("qkv", 6144, 2048), ("proj", 2048, 2048), ("xq", 2048, 2048), ("xproj", 2048, 2048),
                           ("fc1", 8192, 2048), ("fc2", 2048, 8192)):
            print(json.dumps(case(name, m, n, k)), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
