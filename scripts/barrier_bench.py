#!/usr/bin/env python
"""aqb_peer_barrier round trip across P GPUs (CUDA events, max over ranks), eager and graph-captured."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402
from paper_2505_10584_b200.parallel import SIGNAL_BYTES, PeerBuffers, Ulysses, init_from_env  # noqa: E402

init_from_env("nccl")
sp = Ulysses(exchange="p2p")
peer = PeerBuffers(sp, {"sig": SIGNAL_BYTES}, "cuda")
sig = peer.ptrs("sig")
epoch = torch.zeros(1, device="cuda", dtype=torch.int32)
status = torch.zeros(1, device="cuda", dtype=torch.int32)
n = 200


def run():
    for _ in range(n):
        ops.peer_barrier(sig, sp.rank, epoch, status)


for mode in ("eager", "graph"):
    if mode == "graph":
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run()  # warm
        torch.cuda.synchronize()
        dist.barrier()
        with torch.cuda.graph(g):
            run()
        fn = g.replay
    else:
        fn = run
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    us = torch.tensor([e0.elapsed_time(e1) * 1e3 / n], device="cuda")
    dist.all_reduce(us, op=dist.ReduceOp.MAX)
    if sp.rank == 0:
        print(json.dumps({"P": sp.P, "mode": mode, "us_per_barrier": float(us), "status": int(status.item())}),
              flush=True)
    dist.barrier()
peer.close()
dist.destroy_process_group()
