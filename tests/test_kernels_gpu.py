"""Per-kernel numerics on the B200, through the C-ABI (libaqb.so).

Each CUDA kernel is compared with a plain fp32 PyTorch statement of the same
op (the oracle's functions where one exists).  Tolerances are written next to
each assert; bf16 outputs are checked by relative L2 error.
"""

import math

import pytest
import torch

from oracle import dit_oracle as ref
from paper_2505_10584_b200 import ops

pytestmark = pytest.mark.gpu
dev = "cuda"


def rel_l2(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (7800, 2048, 2048), (300, 384, 200), (33, 32, 32),
                                   (1000, 6144, 2048), (257, 128, 4096),
                                   # half-width tail units (pair kernel) in the last partial wave
                                   (7800, 6144, 2048), (1950, 8192, 2048), (1000, 6144, 512)])
def test_gemm_bf16_matches_fp32(m, n, k):
    g = torch.Generator(device=dev).manual_seed(m + n + k)
    a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(n, device=dev, generator=g)
    out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    ops.gemm(a, w, out, bias=bias)
    exp = a.float() @ w.float().t() + bias
    assert rel_l2(out, exp) < 8e-3  # bf16 output rounding (~2^-9) dominates


@pytest.mark.parametrize("epi", ["gelu", "gate_res", "f32", "euler"])
def test_gemm_epilogues(epi):
    m, n, k = 777, 512, 384
    g = torch.Generator(device=dev).manual_seed(7)
    a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(n, device=dev, generator=g)
    acc = a.float() @ w.float().t() + bias
    if epi == "gelu":
        out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
        ops.gemm(a, w, out, bias=bias, epilogue="gelu")
        assert rel_l2(out, torch.nn.functional.gelu(acc, approximate="tanh")) < 8e-3
    elif epi == "gate_res":
        res = torch.randn(m, n, device=dev, generator=g)
        gate = torch.randn(n, device=dev, generator=g)
        exp = res + gate * acc
        ops.gemm(a, w, res, bias=bias, gate=gate, epilogue="gate_res")
        assert rel_l2(res, exp) < 1e-5  # fp32 epilogue, fp32 accumulation
    elif epi == "f32":
        out = torch.empty(m, n, device=dev)
        ops.gemm(a, w, out, bias=bias, epilogue="f32")
        assert rel_l2(out, acc) < 1e-5
    else:
        x = torch.randn(m, n, device=dev, generator=g)
        aux = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
        alpha = torch.tensor([0.125], device=dev)
        exp = x + 0.125 * acc
        ops.gemm(a, w, x, bias=bias, epilogue="euler", alpha=alpha, aux=aux)
        assert rel_l2(x, exp) < 1e-5
        assert rel_l2(aux, exp) < 8e-3


@pytest.mark.parametrize("m,n,k", [(777, 512, 384), (7800, 2048, 2048), (975, 2048, 8192), (300, 96, 64)])
def test_gemm_gate_res_with_bf16_copy(m, n, k):
    """gate*residual epilogue that also TMA-stores bf16(new residual) (the next projection's A)."""
    g = torch.Generator(device=dev).manual_seed(m + n)
    a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(n, device=dev, generator=g)
    gate = torch.randn(n, device=dev, generator=g)
    res = torch.randn(m, n, device=dev, generator=g)
    exp = res + gate * (a.float() @ w.float().t() + bias)
    aux = torch.full((m, n + 8), 7.0, device=dev, dtype=torch.bfloat16)[:, :n]
    ops.gemm(a, w, res, bias=bias, gate=gate, epilogue="gate_res", aux=aux)
    assert rel_l2(res, exp) < 1e-5
    assert torch.equal(aux, res.to(torch.bfloat16))  # exactly the rounded new residual


def test_gemm_run_flag_skips():
    a = torch.ones(128, 64, device=dev, dtype=torch.bfloat16)
    w = torch.ones(64, 64, device=dev, dtype=torch.bfloat16)
    out = torch.zeros(128, 64, device=dev)
    flag = torch.tensor([0], device=dev, dtype=torch.int32)
    ops.gemm(a, w, out, epilogue="f32", run_flag=flag, run_if=1)
    assert float(out.abs().sum()) == 0.0
    ops.gemm(a, w, out, epilogue="f32", run_flag=flag, run_if=0)
    assert torch.allclose(out, torch.full_like(out, 64.0))


def _attn_ref(q, k, v):
    # q [Sq, A, D] fp32 on CPU
    return ref.attention(q.float().cpu(), k.float().cpu(), v.float().cpu())


@pytest.mark.parametrize("sq,skv,heads,d", [(256, 256, 2, 128), (300, 300, 3, 128), (7800 // 8, 7800 // 8, 2, 128),
                                           (129, 16, 4, 128), (512, 4096, 1, 128), (200, 200, 4, 64),
                                           (48, 48, 4, 32), (32, 16, 4, 32)])
def test_attention_packed_qkv(sq, skv, heads, d):
    """Q/K/V read in place from a [S, 3, A, D] QKV buffer (self-attn layout)."""
    g = torch.Generator(device=dev).manual_seed(sq * 7 + skv)
    qkv = torch.randn(max(sq, skv), 3, heads, d, device=dev, generator=g).to(torch.bfloat16)
    q = qkv[:sq, 0]
    k = qkv[:skv, 1]
    v = qkv[:skv, 2]
    o = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    flat = qkv.view(qkv.shape[0], -1)
    ops.attention(flat[:sq, 0:], flat[:skv, heads * d:], flat[:skv, 2 * heads * d:], o, heads, d)
    exp = _attn_ref(q, k, v)
    assert rel_l2(o, exp) < 1e-2  # bf16 P and output rounding


def test_attention_large_logits_rescale():
    """Scores with a large dynamic range exercise the lazy O rescale path."""
    sq, skv, heads, d = 256, 1024, 2, 128
    g = torch.Generator(device=dev).manual_seed(11)
    q = (torch.randn(sq, heads, d, device=dev, generator=g) * 3).to(torch.bfloat16)
    k = (torch.randn(skv, heads, d, device=dev, generator=g) * 3).to(torch.bfloat16)
    # make later key tiles dominate so the running max keeps growing
    k[768:] *= 2
    v = torch.randn(skv, heads, d, device=dev, generator=g).to(torch.bfloat16)
    o = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    ops.attention(q.view(sq, -1), k.view(skv, -1), v.view(skv, -1), o, heads, d)
    assert rel_l2(o, _attn_ref(q, k, v)) < 1e-2


@pytest.mark.parametrize("hidden,kind", [(128, 0), (2048, 0), (3072, 0), (2048, 1), (4096, 0), (1024, 2), (3072, 1)])
def test_norm_modulate(hidden, kind):
    rows = 1000
    g = torch.Generator(device=dev).manual_seed(hidden)
    x = torch.randn(rows, hidden, device=dev, generator=g) * 3 + 1
    shift = torch.randn(hidden, device=dev, generator=g)
    scale = torch.randn(hidden, device=dev, generator=g) * 0.5
    out = torch.empty(rows, hidden, device=dev, dtype=torch.bfloat16)
    ops.norm_modulate(x, shift, scale, out, eps=1e-6, kind=kind)
    if kind == 0:
        exp = ref.modulate(x.cpu(), shift.cpu(), scale.cpu(), 1e-6)
    elif kind == 2:
        exp = x.cpu() * (1 + scale.cpu()) + shift.cpu()
    else:
        exp = x.cpu() * torch.rsqrt(x.cpu().pow(2).mean(-1, keepdim=True) + 1e-6) * (1 + scale.cpu()) + shift.cpu()
    assert rel_l2(out, exp) < 5e-3


@pytest.mark.parametrize("rows,hidden", [(513, 256), (975, 2048), (301, 3072)])
def test_norm_modulate_probe(rows, hidden):
    """warp-per-row (hidden < 1024) and CTA-per-row (wide rows) variants."""
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn(rows, hidden, device=dev, generator=g)
    prev = torch.randn(rows, hidden, device=dev, generator=g)
    prev0 = prev.clone()
    partials = torch.empty(2 * rows, device=dev)
    out = torch.empty(rows, hidden, device=dev, dtype=torch.bfloat16)
    ops.norm_modulate(x, None, None, out, probe_prev=prev, probe_partials=partials)
    m = ref.layer_norm(x.cpu(), 1e-6)
    sums = torch.empty(2, device=dev)
    ops.rel_l1_reduce(partials, rows, sums)
    exp_d = (m - prev0.cpu()).abs().sum()
    exp_p = prev0.cpu().abs().sum()
    assert abs(float(sums[0]) - float(exp_d)) / float(exp_d) < 1e-5
    assert abs(float(sums[1]) - float(exp_p)) / float(exp_p) < 1e-5
    assert rel_l2(prev, m) < 1e-6


@pytest.mark.parametrize("d", [32, 64, 128])
def test_qk_norm_rope_inplace(d):
    heads, grid = 3, (2, 4, 6)
    S = grid[0] * grid[1] * grid[2]
    St = 5  # trailing text rows: no rope
    rows = S + St
    dims = (d - 2 * ((d - (d // 4) // 2 * 2) // 2 // 2 * 2), (d - (d // 4) // 2 * 2) // 2 // 2 * 2,
            (d - (d // 4) // 2 * 2) // 2 // 2 * 2)
    ang = ref.rope_angles(grid, dims, 1000.0)
    cos = torch.cos(ang).float().to(dev)
    sin = torch.sin(ang).float().to(dev)
    g = torch.Generator(device=dev).manual_seed(d)
    qkv = torch.randn(rows, 3, heads, d, device=dev, generator=g).to(torch.bfloat16)
    qw = 1 + 0.1 * torch.randn(d, device=dev, generator=g)
    kw = 1 + 0.1 * torch.randn(d, device=dev, generator=g)
    src = qkv.clone()
    ops.qk_norm_rope(qkv.view(rows, -1), heads, d, qw, kw, 1e-6, cos, sin, 0, S)
    x = src.float().cpu()
    q = ref.rms_norm(x[:, 0], qw.cpu(), 1e-6)
    k = ref.rms_norm(x[:, 1], kw.cpu(), 1e-6)
    q = torch.cat([ref.apply_rope(q[:S], ang), q[S:]])
    k = torch.cat([ref.apply_rope(k[:S], ang), k[S:]])
    assert rel_l2(qkv[:, 0], q) < 5e-3
    assert rel_l2(qkv[:, 1], k) < 5e-3
    assert torch.equal(qkv[:, 2], src[:, 2])


def test_gemv_and_timestep_features():
    n, k = 777, 256
    g = torch.Generator(device=dev).manual_seed(5)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.1).to(torch.bfloat16)
    b = torch.randn(n, device=dev, generator=g)
    add = torch.randn(n, device=dev, generator=g)
    x = torch.randn(k, device=dev, generator=g)
    y = torch.empty(n, device=dev)
    ops.gemv(w, x, y, bias=b, add=add, in_silu=True)
    exp = w.float().cpu() @ torch.nn.functional.silu(x.cpu()) + b.cpu() + add.cpu()
    assert rel_l2(y, exp) < 1e-5
    t = torch.tensor([0.37], device=dev)
    ops.gemv(w, None, y, bias=b, t=t)
    exp = w.float().cpu() @ ref.timestep_features(0.37, k) + b.cpu()
    assert rel_l2(y, exp) < 1e-4


def test_patchify_roundtrip():
    C, grid, patch = 8, (3, 4, 5), (1, 2, 2)
    lat = torch.randn(C, 3, 8, 10, device=dev)
    S = 3 * 4 * 5
    tok = torch.empty(S, 32, device=dev)
    tokb = torch.empty(S, 32, device=dev, dtype=torch.bfloat16)
    ops.patchify(lat, tok, tokb, grid, patch)
    assert torch.equal(tok.cpu(), ref.patchify(lat.cpu(), patch))
    back = torch.empty_like(lat)
    ops.unpatchify(tok, back, grid, patch)
    assert torch.equal(back, lat)


def test_cache_decide_matches_policy():
    from paper_2505_10584_b200.schedule import RelL1Policy

    pol = RelL1Policy(threshold=0.15, warmup=2)
    rels = [0.0, 0.3, 0.05, 0.05, 0.07, 0.01, 0.2, 0.02, 0.03, 0.04]
    state = torch.zeros(4, dtype=torch.int32, device=dev)
    flags = torch.zeros(len(rels), dtype=torch.int32, device=dev)
    relo = torch.zeros(len(rels), device=dev)
    sums = torch.empty(2, device=dev)
    acc, exp_flags = 0.0, []
    for i, r in enumerate(rels):
        sums.copy_(torch.tensor([r * 1000.0, 1000.0]))
        ops.cache_decide(sums, state, pol.threshold, pol.warmup, len(rels), pol.force_last, flags, relo)
        full, acc = pol.decide(i + 1, len(rels), acc, r)
        exp_flags.append(int(full))
    assert flags.cpu().tolist() == exp_flags


def test_heads_to_seq():
    P, rows, w = 4, 37, 64
    src = torch.randn(P, rows, w, device=dev).to(torch.bfloat16)
    dst = torch.empty(rows, P * w, device=dev, dtype=torch.bfloat16)
    ops.heads_to_seq(src, rows, P, w, dst)
    assert torch.equal(dst, src.permute(1, 0, 2).reshape(rows, P * w))


def _qkv_ref(a, w, b, qw, kw, heads, rope_rows, cos, sin, row0=0):
    """fp32 statement: projection, per-head RMSNorm on q/k, RoPE on rows < rope_rows."""
    x = (a.float() @ w.float().t() + b).cpu().view(a.shape[0], 3, heads, 128)
    q = ref.rms_norm(x[:, 0], qw.cpu(), 1e-6)
    k = ref.rms_norm(x[:, 1], kw.cpu(), 1e-6)
    ang = torch.atan2(sin.cpu(), cos.cpu()).double()
    n = max(0, min(a.shape[0], rope_rows - row0))
    if n:
        q = torch.cat([ref.apply_rope(q[:n], ang[row0:row0 + n]), q[n:]])
        k = torch.cat([ref.apply_rope(k[:n], ang[row0:row0 + n]), k[n:]])
    return torch.stack([q, k, x[:, 2]], dim=1)  # [rows, 3, heads, 128]


@pytest.mark.parametrize("rows,heads", [(300, 2), (1000, 4), (7800, 16), (1000, 16)])
def test_gemm_qknorm_rope_natural_layout(rows, heads):
    g = torch.Generator(device=dev).manual_seed(rows)
    H = heads * 128
    a = torch.randn(rows, H, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(3 * H, H, device=dev, generator=g) * 0.03).to(torch.bfloat16)
    b = torch.randn(3 * H, device=dev, generator=g) * 0.1
    qw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    kw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    ang = torch.rand(rows, 64, device=dev, generator=g) * 6.28
    cos, sin = torch.cos(ang), torch.sin(ang)
    rope_rows = rows - 7  # last rows (text-like) unrotated
    out = torch.empty(rows, 3 * H, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, out, H, 2, qw, kw, 1e-6, bias=b, cos=cos, sin=sin, rope_rows=rope_rows)
    exp = _qkv_ref(a, w, b, qw, kw, heads, rope_rows, cos, sin)
    assert rel_l2(out.view(rows, 3, heads, 128), exp) < 6e-3


def test_gemm_qknorm_rope_ulysses_pack_and_local_heads():
    """Packed all-to-all send layout [P, rows, 3, hl, 128] and a local-heads-only (g_base) store."""
    rows, heads, P = 500, 4, 2
    hl, H = heads // P, heads * 128
    g = torch.Generator(device=dev).manual_seed(9)
    a = torch.randn(rows, H, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(3 * H, H, device=dev, generator=g) * 0.03).to(torch.bfloat16)
    b = torch.randn(3 * H, device=dev, generator=g) * 0.1
    qw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    kw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    ang = torch.rand(4 * rows, 64, device=dev, generator=g) * 6.28
    cos, sin = torch.cos(ang), torch.sin(ang)
    row0 = rows  # this rank's first global token
    snd = torch.zeros(P, rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, snd, H, 2, qw, kw, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=row0,
                         rope_rows=4 * rows, out_row_stride=3 * hl * 128, groups=P, group_stride=rows * 3 * hl * 128,
                         hpg=hl)
    exp = _qkv_ref(a, w, b, qw, kw, heads, 4 * rows, cos, sin, row0=row0)  # [rows, 3, heads, 128]
    got = snd.permute(1, 2, 0, 3, 4).reshape(rows, 3, heads, 128)
    assert rel_l2(got, exp) < 6e-3
    # local heads only (group 1 of 2), no rope: other heads are dropped
    loc = torch.zeros(rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, loc, H, 2, qw, kw, 1e-6, bias=b, out_row_stride=3 * hl * 128, groups=1, hpg=hl, g_base=1)
    exp2 = _qkv_ref(a, w, b, qw, kw, heads, 0, cos, sin)
    assert rel_l2(loc, exp2[:, :, hl:]) < 6e-3


def test_gemm_qknorm_rope_scatter_equals_pack():
    """The peer-scatter epilogue (one TMA map per destination rank) writes exactly what the
    packed all-to-all layout holds; destinations are local buffers standing in for peers."""
    rows, heads, P = 700, 8, 4
    hl, H = heads // P, heads * 128
    rs = 3 * hl * 128
    g = torch.Generator(device=dev).manual_seed(21)
    a = torch.randn(rows, H, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(3 * H, H, device=dev, generator=g) * 0.03).to(torch.bfloat16)
    b = torch.randn(3 * H, device=dev, generator=g) * 0.1
    qw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    kw = 1 + 0.1 * torch.randn(128, device=dev, generator=g)
    ang = torch.rand(P * rows, 64, device=dev, generator=g) * 6.28
    cos, sin = torch.cos(ang), torch.sin(ang)
    rank = 2
    snd = torch.zeros(P, rows, 3, hl, 128, device=dev, dtype=torch.bfloat16)
    ops.gemm_qknorm_rope(a, w, snd, H, 2, qw, kw, 1e-6, bias=b, cos=cos, sin=sin, rope_row0=rank * rows,
                         rope_rows=P * rows, out_row_stride=rs, groups=P, group_stride=rows * rs, hpg=hl)
    rcv = [torch.full((P * rows + 5, 3, hl, 128), 7.0, device=dev, dtype=torch.bfloat16) for _ in range(P)]
    dst = [r.data_ptr() + rank * rows * rs * 2 for r in rcv]
    ops.gemm_qknorm_rope_scatter(a, w, dst, H, 2, qw, kw, 1e-6, rs, hl, bias=b, cos=cos, sin=sin,
                                 rope_row0=rank * rows, rope_rows=P * rows)
    for r in range(P):
        assert torch.equal(rcv[r][rank * rows:(rank + 1) * rows], snd[r])
        assert bool((rcv[r][:rank * rows] == 7).all()) and bool((rcv[r][(rank + 1) * rows:] == 7).all())


@pytest.mark.parametrize("sq,skv,heads,d,splits", [(7800 // 8 * 8 + 256, 8056, 2, 128, 0), (1000, 3000, 2, 128, 3),
                                                   (300, 1000, 3, 128, 5), (200, 600, 4, 64, 2),
                                                   (96, 400, 4, 32, 4), (257, 129, 1, 128, 2),
                                                   (7800, 7800, 16, 128, 0), (25696, 25696, 6, 128, 0)])
def test_attention_split_kv(sq, skv, heads, d, splits):
    """Split-KV partials + combine equal the single-pass kernel (within bf16 rounding)."""
    g = torch.Generator(device=dev).manual_seed(sq + skv + splits)
    q = torch.randn(sq, heads * d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(skv, heads * d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(skv, heads * d, device=dev, generator=g).to(torch.bfloat16)
    o1 = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    ops.attention(q, k, v, o1, heads, d, splits=1)
    ws = torch.zeros(ops.attention_workspace_bytes(sq, skv, heads, d, splits or None), device=dev, dtype=torch.uint8)
    o2 = torch.empty_like(o1)
    ops.attention(q, k, v, o2, heads, d, splits=splits, workspace=ws)
    exp = _attn_ref(q.view(sq, heads, d), k.view(skv, heads, d), v.view(skv, heads, d))
    assert rel_l2(o2, exp) < 1e-2
    assert rel_l2(o2, o1) < 8e-3


@pytest.mark.parametrize("sq,skv,heads,d,g", [(7800, 256, 16, 128, None), (3000, 77, 3, 128, 3),
                                               (1000, 300, 2, 64, 2), (2100, 256, 2, 128, 5), (129, 16, 4, 128, 2),
                                               (4000, 256, 1, 128, 16)])
def test_attention_multi_block_ctas(sq, skv, heads, d, g, monkeypatch):
    """Short KV: CTAs that run several 256-query blocks with K/V resident give bit-identical
    outputs to one block per CTA (same per-tile math), and match the oracle."""
    gen = torch.Generator(device=dev).manual_seed(sq + 3 * skv)
    q = torch.randn(sq, heads * d, device=dev, generator=gen).to(torch.bfloat16)
    k = torch.randn(skv, heads * d, device=dev, generator=gen).to(torch.bfloat16)
    v = torch.randn(skv, heads * d, device=dev, generator=gen).to(torch.bfloat16)
    monkeypatch.setenv("AQB_ATTN_PAIRS", "1")
    o1 = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    ops.attention(q, k, v, o1, heads, d)
    if g is None:
        monkeypatch.delenv("AQB_ATTN_PAIRS")
        from paper_2505_10584_b200 import _native
        assert _native.query("aqb_attention_pairs_per_cta", sq, skv, heads, d) > 1
    else:
        monkeypatch.setenv("AQB_ATTN_PAIRS", str(g))
    o2 = torch.full_like(o1, 7.0)
    ops.attention(q, k, v, o2, heads, d)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    exp = _attn_ref(q.view(sq, heads, d), k.view(skv, heads, d), v.view(skv, heads, d))
    assert rel_l2(o2, exp) < 1e-2


@pytest.mark.parametrize("g,P,rpr,St,hl", [(3, 4, 300, 40, 2), (2, 2, 1000, 256, 4), (4, 4, 1950, 256, 4)])
def test_attention_scatter_multi_block(g, P, rpr, St, hl, monkeypatch):
    """Cross-attention (256 text K/V rows) through the scatter epilogue with several query
    blocks per CTA: every rank's rows equal the local one-block-per-CTA result."""
    d, skv = 128, 256
    H = P * hl * d
    sq = P * rpr + St
    gen = torch.Generator(device=dev).manual_seed(17 + g)
    q = torch.randn(sq, hl * d, device=dev, generator=gen).to(torch.bfloat16)
    kv = torch.randn(skv, 2, hl * d, device=dev, generator=gen).to(torch.bfloat16).view(skv, -1)
    monkeypatch.setenv("AQB_ATTN_PAIRS", "1")
    ref_o = torch.empty(sq, hl * d, device=dev, dtype=torch.bfloat16)
    ops.attention(q, kv, kv[:, hl * d:], ref_o, hl, d, splits=1)  # the general kernel, like the scatter
    monkeypatch.setenv("AQB_ATTN_PAIRS", str(g))
    outs = [torch.zeros(rpr + St, H, device=dev, dtype=torch.bfloat16) for _ in range(P)]
    rank = P - 1
    ops.attention_scatter(q, kv, kv[:, hl * d:], [o.data_ptr() + rank * hl * d * 2 for o in outs], H, hl, d, rpr,
                          P * rpr)
    torch.cuda.synchronize()
    cols = slice(rank * hl * d, (rank + 1) * hl * d)
    for r in range(P):
        assert torch.equal(outs[r][:rpr, cols], ref_o[r * rpr:(r + 1) * rpr])
        if St:
            assert torch.equal(outs[r][rpr:, cols], ref_o[P * rpr:])
        assert float(outs[r][:, :rank * hl * d].abs().sum()) == 0.0


def _native_splits(sq, skv, heads, d):
    from paper_2505_10584_b200 import _native
    return _native.query("aqb_attention_splits", sq, skv, heads, d)


def test_attention_auto_splits_for_few_heads():
    """Ulysses at 8 GPUs leaves 2 heads per rank: the planner must split KV to fill the SMs."""
    assert _native_splits(8056, 8056, 2, 128) >= 2
    assert _native_splits(119056, 119056, 24, 128) == 1
    assert _native_splits(7800, 256, 16, 128) == 1


def test_attention_tail_plan():
    """Config 2 (16 heads x 31 blocks of 256 queries = 496 tiles on 148 SMs): three whole waves,
    the 52-tile tail split over KV so the last wave is not a third full; a Ulysses shard of 8 or
    4 heads (248 / 124 tiles) splits too, with a long first part and short tails that fill the SMs
    the long parts leave idle (uneven split, merged in-kernel)."""
    from paper_2505_10584_b200 import _native
    assert _native.query("aqb_attention_whole_tiles", 7800, 7800, 16, 128) == 3 * 148
    assert _native_splits(7800, 7800, 16, 128) >= 2
    assert _native.query("aqb_attention_whole_tiles", 7800, 7800, 8, 128) % 148 == 0
    assert _native_splits(7800, 7800, 8, 128) >= 2
    assert ops.attention_workspace_bytes(7800, 7800, 8, 128) > 0


@pytest.mark.parametrize("heads", [16, 8, 4, 2])
def test_attention_planned_splits_match_single_pass(heads):
    """The planner's split (possibly uneven parts, launched split-major) equals the one-pass kernel
    within bf16 rounding, bit-identically twice in a row, and matches fp32 attention."""
    sq = skv = 7800
    d = 128
    g = torch.Generator(device=dev).manual_seed(heads)
    q = torch.randn(sq, heads * d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(skv, heads * d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(skv, heads * d, device=dev, generator=g).to(torch.bfloat16)
    ws = torch.zeros(max(16, ops.attention_workspace_bytes(sq, skv, heads, d)), device=dev, dtype=torch.uint8)
    o1 = torch.empty(sq, heads * d, device=dev, dtype=torch.bfloat16)
    ops.attention(q, k, v, o1, heads, d, splits=1)
    o2, o3 = torch.empty_like(o1), torch.empty_like(o1)
    ops.attention(q, k, v, o2, heads, d, workspace=ws)
    ops.attention(q, k, v, o3, heads, d, workspace=ws)
    assert torch.equal(o2, o3)
    assert rel_l2(o2, o1) < 8e-3
    sel = slice(0, 1000)  # fp32 reference on a row subset
    exp = _attn_ref(q[sel].view(-1, heads, d), k.view(skv, heads, d), v.view(skv, heads, d))
    assert rel_l2(o2[sel], exp) < 1e-2


@pytest.mark.parametrize("splits,P,rpr,St,hl", [(1, 4, 300, 40, 2), (3, 4, 300, 40, 2), (1, 2, 192, 0, 4),
                                                (1, 2, 256, 24, 4), (0, 2, 3900, 0, 16), (0, 4, 1950, 256, 16)])
def test_attention_scatter_rows_to_owners(splits, P, rpr, St, hl):
    """Scatter epilogue: video row r -> rank r // rpr, text rows -> every rank (local stand-ins for peers).
    (2, 192, 0): the last CTA's second Q tile lies wholly past the sequence end (regression)."""
    d = 128
    H = P * hl * d
    sq = P * rpr + St
    g = torch.Generator(device=dev).manual_seed(5 + splits)
    qkv = torch.randn(sq, 3, hl, d, device=dev, generator=g).to(torch.bfloat16)
    flat = qkv.view(sq, -1)
    ref_o = torch.empty(sq, hl * d, device=dev, dtype=torch.bfloat16)
    wsb = ops.attention_workspace_bytes(sq, sq, hl, d, splits or None)
    ops.attention(flat, flat[:, hl * d:], flat[:, 2 * hl * d:], ref_o, hl, d, splits=splits,
                  workspace=torch.zeros(wsb, device=dev, dtype=torch.uint8))
    outs = [torch.zeros(rpr + St, H, device=dev, dtype=torch.bfloat16) for _ in range(P)]
    rank = 1
    dst = [o.data_ptr() + rank * hl * d * 2 for o in outs]
    torch.cuda.synchronize()
    ws = torch.zeros(wsb, device=dev, dtype=torch.uint8)
    ops.attention_scatter(flat, flat[:, hl * d:], flat[:, 2 * hl * d:], dst, H, hl, d, rpr, P * rpr, splits=splits,
                          workspace=ws)
    cols = slice(rank * hl * d, (rank + 1) * hl * d)
    for r in range(P):
        assert torch.equal(outs[r][:rpr, cols], ref_o[r * rpr:(r + 1) * rpr])
        if St:
            assert torch.equal(outs[r][rpr:, cols], ref_o[P * rpr:])
        assert float(outs[r][:, :rank * hl * d].abs().sum()) == 0.0  # other ranks' head columns untouched


def test_peer_barrier_single_rank_payload():
    """nranks=1: the barrier advances the epoch and returns the payload (sum over one rank)."""
    import ctypes
    from paper_2505_10584_b200 import _native

    ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(64)
    _native.call("aqb_peer_alloc", 512, ctypes.addressof(ptr), ctypes.addressof(h))
    try:
        epoch = torch.zeros(1, device=dev, dtype=torch.int32)
        status = torch.zeros(1, device=dev, dtype=torch.int32)
        pay = torch.tensor([1.5, -2.25], device=dev)
        for i in range(3):
            ops.peer_barrier([ptr.value], 0, epoch, status, payload=pay, pay_out=pay)
        torch.cuda.synchronize()
        assert int(epoch) == 3 and int(status) == 0
        assert pay.tolist() == [1.5, -2.25]
    finally:
        _native.call("aqb_peer_free", ptr.value)


# ------------------------------------------------------------------ TP-SP kernels
@pytest.mark.parametrize("rows,hidden,kind", [(300, 2048, 0), (257, 512, 2), (975, 3072, 0)])
def test_norm_modulate_gather_writes_every_destination(rows, hidden, kind):
    """The fused all-gather: the same rows, bit-identical to norm_modulate, at an offset in each output."""
    g = torch.Generator(device=dev).manual_seed(rows)
    x = torch.randn(rows, hidden, device=dev, generator=g)
    sh = torch.randn(hidden, device=dev, generator=g) if kind == 0 else None
    sc = torch.randn(hidden, device=dev, generator=g) if kind == 0 else None
    ref_o = torch.empty(rows, hidden, device=dev, dtype=torch.bfloat16)
    ops.norm_modulate(x, sh, sc, ref_o, kind=kind)
    P, rank = 3, 1
    outs = [torch.full((P * rows, hidden), 7.0, device=dev, dtype=torch.bfloat16) for _ in range(P)]
    ops.norm_modulate_gather(x, sh, sc, [o.data_ptr() + rank * rows * hidden * 2 for o in outs], hidden, kind=kind)
    for o in outs:
        assert torch.equal(o[rank * rows:(rank + 1) * rows], ref_o)
        assert bool((o[:rank * rows] == 7).all()) and bool((o[(rank + 1) * rows:] == 7).all())


@pytest.mark.parametrize("rpr,n,k", [(300, 2048, 256), (1950, 2048, 1024), (128, 512, 64), (975, 1024, 2048)])
def test_gemm_gate_add_scatter_reduces_into_row_owners(rpr, n, k):
    """The fused reduce-scatter: row i of gate*(A W^T + b) is added into rank i // rpr's residual
    (blocks inside one rank by TMA reduce-add, rank-straddling blocks by red.v4); two partials sum."""
    P = 3
    m = P * rpr
    g = torch.Generator(device=dev).manual_seed(rpr + n)
    res = [torch.randn(rpr, n, device=dev, generator=g) for _ in range(P)]
    exp = torch.cat(res).clone()
    gate = torch.randn(n, device=dev, generator=g)
    bias = torch.randn(n, device=dev, generator=g)
    for part in range(2):  # two ranks' partials of a row-parallel projection
        a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn(n, k, device=dev, generator=g) * 0.05).to(torch.bfloat16)
        b = bias if part == 0 else None
        exp += gate * (a.float() @ w.float().t() + (b if b is not None else 0))
        ops.gemm_gate_add_scatter(a, w, [r.data_ptr() for r in res], n, rpr, bias=b, gate=gate)
    assert rel_l2(torch.cat(res), exp) < 1e-5


def test_gate_bcast_and_rank_ordered_slot_sum():
    """MM-DiT TP-SP text-row all-reduce: gate*partial into every rank's slot, then x += slots in
    rank order (bitwise the same sum on every rank)."""
    P, rows, cols = 3, 24, 512
    g = torch.Generator(device=dev).manual_seed(11)
    parts = [torch.randn(rows, cols, device=dev, generator=g) for _ in range(P)]
    gate = torch.randn(cols, device=dev, generator=g)
    slots = [torch.zeros(P, rows, cols, device=dev) for _ in range(P)]  # one slot buffer per "rank"
    for r in range(P):  # rank r writes its slot r on every rank
        ops.gate_bcast(parts[r], gate, [s[r].data_ptr() for s in slots], cols)
    x0 = torch.randn(rows, cols, device=dev, generator=g)
    xs = [x0.clone() for _ in range(P)]
    for r in range(P):
        ops.sum_slots(xs[r], slots[r])
    exp = x0.clone()
    for r in range(P):
        exp = exp + gate * parts[r]
    for r in range(P):
        assert torch.equal(xs[r], xs[0])  # replicated rows stay identical
    assert rel_l2(xs[0], exp) < 1e-6
    flag = torch.zeros(1, device=dev, dtype=torch.int32)  # gated off: untouched
    y = x0.clone()
    ops.sum_slots(y, slots[0], run_flag=flag, run_if=1)
    assert torch.equal(y, x0)
