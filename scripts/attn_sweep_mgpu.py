#!/usr/bin/env python
"""BASELINE config 5 at P GPUs: joint attention, 24 heads x head_dim 128, bf16, S = 4k..128k.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 scripts/attn_sweep_mgpu.py

Each rank holds the Ulysses-received input (all S rows, its 24/P heads — in the model the
QKV-projection epilogue delivers it) and runs the attention whose epilogue stores every
output row straight into the owning rank's O buffer over NVLink, then the peer barrier.
Timed with CUDA events after warm-up, max over ranks; TFLOP/s = 4·S²·128·24 / time (all
ranks together).  P = 1 runs the plain kernel.  One JSON line per S from rank 0.
"""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops  # noqa: E402
from paper_2505_10584_b200.parallel import SIGNAL_BYTES, PeerBuffers, Ulysses, init_from_env  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sp = None
    if world > 1:
        init_from_env("nccl")
        sp = Ulysses(exchange="p2p")
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    P = sp.P if sp else 1
    rank = sp.rank if sp else 0
    A, D = 24, 128
    hl = A // P
    H = A * D
    for S in (4096, 8192, 16384, 32768, 65536, 131072):
        n = S // P
        g = torch.Generator(device="cuda").manual_seed(S + rank)
        qkv = torch.randn(S, 3, hl, D, device="cuda", generator=g).to(torch.bfloat16).view(S, -1)
        ws = torch.zeros(max(16, ops.attention_workspace_bytes(S, S, hl, D)), device="cuda", dtype=torch.uint8)
        if sp:
            peer = PeerBuffers(sp, {"o": n * H * 2, "sig": SIGNAL_BYTES}, "cuda")
            dst = peer.ptrs("o", rank * hl * D * 2)
            sig = peer.ptrs("sig")
            epoch = torch.zeros(1, device="cuda", dtype=torch.int32)
            status = torch.zeros(1, device="cuda", dtype=torch.int32)

            def step():
                ops.attention_scatter(qkv, qkv[:, hl * D:], qkv[:, 2 * hl * D:], dst, H, hl, D, n, S, workspace=ws)
                ops.peer_barrier(sig, rank, epoch, status)
        else:
            o = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)

            def step():
                ops.attention(qkv, qkv[:, H:], qkv[:, 2 * H:], o, A, D, workspace=ws)
        iters = max(2, min(20, int(2e5 // (S // 1024) ** 2) or 2))
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if sp:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
        if sp:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if rank == 0:
            fl = 4.0 * S * S * D * A
            print(json.dumps({"config": "config5", "S": S, "P": P, "heads_per_rank": hl, "ms": float(ms),
                              "tflops_total": fl / float(ms) / 1e9, "tflops_per_gpu": fl / float(ms) / 1e9 / P,
                              "exchange": "attention epilogue -> owners' O over NVLink + peer barrier" if sp else None}),
                  flush=True)
        if sp:
            if int(status.item()) != 0:
                raise RuntimeError("peer barrier timed out")
            peer.close()
        del qkv, ws
        torch.cuda.empty_cache()
    if sp:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
