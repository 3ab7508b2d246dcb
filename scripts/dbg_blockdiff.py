import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2505_10584_b200 import DiTConfig, build_model, ops
from paper_2505_10584_b200.parallel import Ulysses, init_from_env
from paper_2505_10584_b200.weights import init_weights, synthetic_inputs
init_from_env("nccl")
sp = Ulysses(exchange=os.environ.get("X_EXCH", "p2p"))
cfg = DiTConfig("single-dit", hidden_size=1024, num_heads=8, num_single=4, text_dim=256, text_len=40)
grid = (3, 8, 16)
W = init_weights(cfg, seed=0); inp = synthetic_inputs(cfg, grid)


def trace(model, rows):
    snaps = []
    names = ["norm_modulate", "gemm", "gemm_qknorm_rope", "gemm_qknorm_rope_scatter", "attention", "attention_scatter"]
    orig = {k: getattr(ops, k) for k in names}

    def wrap(k):
        def f(*a, **kw):
            r = orig[k](*a, **kw)
            torch.cuda.synchronize()
            q = model.a2a_rcv.clone() if hasattr(model, "a2a_rcv") else model.qkv.view(model.qkv.shape[0], 3, 8, 128)[:, :, :4].clone()
            snaps.append((k, model.x[:rows].clone(), model.m[:rows].clone(), model.o[:rows].clone(), q))
            return r
        return f
    for k in names:
        setattr(ops, k, wrap(k))
    try:
        model.reset(inp["x0"], 8)
        model.step("full", True)
        torch.cuda.synchronize()
    finally:
        for k in names:
            setattr(ops, k, orig[k])
    return snaps


m = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"])
s2 = trace(m, 48)
if sp.rank == 0:
    m1 = build_model(cfg, weights=W).prepare(grid, inp["text"])
    s1 = trace(m1, 48)
    for i, (a, b) in enumerate(zip(s1, s2)):
        dx = float((a[1] - b[1]).abs().max()); dm = float((a[2].float() - b[2].float()).abs().max())
        do = (a[3].float() - b[3].float()).abs()
        bad = (do.amax(1) > 0).nonzero().flatten().tolist()
        badc = (do.amax(0) > 0).nonzero().flatten().tolist()
        dq = (a[4].float() - b[4].float()[:a[4].shape[0]]).abs()
        print(json.dumps({"i": i, "op1": a[0], "op2": b[0], "dx": dx, "dm": dm, "do": float(do.max()),
                          "dq": float(dq.max()), "dq_rows": (dq.flatten(1).amax(1) > 0).nonzero().flatten().tolist()[:10],
                          "q_shapes": [list(a[4].shape), list(b[4].shape)],
                          "o_bad_rows": bad[:20], "o_bad_cols": [badc[:3], badc[-3:], len(badc)]}), flush=True)
        if dx or dm:
            break
dist.barrier()
