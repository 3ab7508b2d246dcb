#!/usr/bin/env python
"""Multi-rank VAE tile blend worker (``tests/test_multirank_gpu.py``): every rank "decodes" its
round-robin tiles (``plan.tiles_of(rank)``, ``inference.py:189-226``) into peer memory and blends
all of them straight from their owners' buffers (``tiling.PeerTiles``); the result must equal the
1-GPU blend of the same tiles bit for bit.

    [AQB_OVERSUBSCRIBE=1] torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_vae_blend.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200.parallel import Ulysses, init_from_env, oversubscribed  # noqa: E402
from paper_2505_10584_b200.tiling import PeerTiles, blend_tiles, plan_vae_tiles  # noqa: E402

OUT = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
init_from_env("nccl")
sp = Ulysses(exchange="p2p")
ok = True
for latent, tile, ov in (((9, 40, 64), (5, 16, 24), (1, 4, 8)), ((33, 90, 160), (9, 32, 32), (2, 8, 8))):
    plan = plan_vae_tiles(latent, tile, ov, devices=sp.P)
    C = 8
    g = torch.Generator().manual_seed(0)
    vol = torch.randn(C, *latent, generator=g)
    decoded = []
    for t in plan.tiles:  # "decode" = cut + a tile-dependent perturbation, same on every rank
        (t0, h0, w0), (st, sh, sw) = t.start, t.size
        decoded.append(vol[:, t0:t0 + st, h0:h0 + sh, w0:w0 + sw] + 0.01 * (t0 + h0 + w0))
    pt = PeerTiles(plan, sp, C)
    for i in plan.tiles_of(sp.rank):
        pt.local_tile(i).copy_(decoded[i])
    torch.cuda.synchronize()
    dist.barrier()
    out = torch.empty(C, *latent, device="cuda")
    pt.blend(out)
    torch.cuda.synchronize()
    ref = torch.empty_like(out)
    blend_tiles(plan, [d.cuda() for d in decoded], ref)
    same = torch.equal(out, ref)
    ok &= same
    if sp.rank == 0:
        rec = json.dumps({"P": sp.P, "latent": latent, "tiles": len(plan.tiles), "bitwise_vs_1gpu": same,
                          "max_abs": float((out - ref).abs().max())})
        print(rec, flush=True)
        if OUT:
            with open(OUT, "a") as fh:
                fh.write(rec + "\n")
    dist.barrier()
    pt.close()
flag = torch.tensor([1 if ok else 0], device="cpu" if oversubscribed() else "cuda")
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
dist.destroy_process_group()
sys.exit(0 if int(flag) else 1)
