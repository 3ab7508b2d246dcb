import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import ops
dev = "cuda"
case = sys.argv[1]
P, hl, d = (2, 4, 128) if case == "odd_tiles" else (4, 2, 128)
rpr, St = {"aligned": (256, 0), "text": (256, 128), "straddle": (300, 0), "straddle_text": (300, 40),
           "odd_tiles": (192, 0)}[case]
H = P * hl * d
sq = P * rpr + St
qkv = torch.randn(sq, 3, hl, d, device=dev).to(torch.bfloat16)
flat = qkv.view(sq, -1)
ref_o = torch.empty(sq, hl * d, device=dev, dtype=torch.bfloat16)
ops.attention(flat, flat[:, hl * d:], flat[:, 2 * hl * d:], ref_o, hl, d, splits=1)
outs = [torch.zeros(rpr + St, H, device=dev, dtype=torch.bfloat16) for _ in range(P)]
dst = [o.data_ptr() + hl * d * 2 for o in outs]
ops.attention_scatter(flat, flat[:, hl * d:], flat[:, 2 * hl * d:], dst, H, hl, d, rpr, P * rpr, splits=1)
torch.cuda.synchronize()
ok = all(torch.equal(outs[r][:rpr, hl * d:2 * hl * d], ref_o[r * rpr:(r + 1) * rpr]) for r in range(P))
print(case, "ok" if ok else "MISMATCH")
