import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2505_10584_b200 import ops
dev="cuda"
rows, heads, P = 500, 4, 2
hl, H = heads // P, heads * 128
a = torch.randn(rows, H, device=dev).to(torch.bfloat16)
w = (torch.randn(3 * H, H, device=dev) * 0.03).to(torch.bfloat16)
b = torch.randn(3 * H, device=dev) * 0.1
qw = torch.ones(128, device=dev); kw = torch.ones(128, device=dev)
cos = torch.ones(4*rows, 64, device=dev); sin = torch.zeros(4*rows, 64, device=dev)
case = sys.argv[1]
if case == "pack_norope":
    snd = torch.zeros(P, rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, snd, H, 2, qw, kw, 1e-6, bias=b, out_row_stride=3 * hl * 128, groups=P, group_stride=rows * 3 * hl * 128, hpg=hl)
elif case == "pack_rope":
    snd = torch.zeros(P, rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, snd, H, 2, qw, kw, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=rows, rope_rows=4*rows, out_row_stride=3 * hl * 128, groups=P, group_stride=rows * 3 * hl * 128, hpg=hl)
elif case == "local":
    loc = torch.zeros(rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, loc, H, 2, qw, kw, 1e-6, bias=b, out_row_stride=3 * hl * 128, groups=1, hpg=hl, g_base=1)
elif case == "nat_hpg2":
    out = torch.zeros(rows, 3*H, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, out, H, 2, qw, kw, 1e-6, bias=b, out_row_stride=3*H, groups=2, group_stride=2*128, hpg=2)
torch.cuda.synchronize()
print(case, "ok")
