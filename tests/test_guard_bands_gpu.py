"""Out-of-bounds-write checks for every kernel class (compute-sanitizer is closed on this GPU pool:
runs under it left GPUs needing a reset).

Every output (and in-place operand) lives in the middle of a larger allocation whose guard bands
hold a NaN bit pattern; after the launch the bands must be bit-for-bit unchanged, and the result
must equal the same launch on a plain (unguarded) tensor — so a kernel that writes past a ragged
edge (partial M/N tiles, the last KV block, split-KV partials, TMA boxes clipped at the tensor
end, the Ulysses pack layout) is caught.  Shapes are ragged on purpose.  Two launches of each op
must also agree bit for bit (no write races between CTAs on the output).
"""

import pytest
import torch

from paper_2505_10584_b200 import ops

pytestmark = pytest.mark.gpu
dev = "cuda"
bf = torch.bfloat16
GUARD = 8192  # elements each side (16-32 KB)
SENT = {bf: -1, torch.float32: -1, torch.uint8: 0xA5}  # 0xFFFF / 0xFFFFFFFF: NaN patterns


def guarded(shape, dtype, init=None):
    n = 1
    for d in shape:
        n *= d
    itype = {bf: torch.int16, torch.float32: torch.int32, torch.uint8: torch.uint8}[dtype]
    raw = torch.full((2 * GUARD + n,), SENT[dtype], dtype=itype, device=dev)
    t = raw[GUARD:GUARD + n].view(dtype).view(*shape)
    if init is not None:
        t.copy_(init)
    return raw, t


def intact(raw):
    s = SENT[torch.uint8] if raw.dtype == torch.uint8 else -1
    return bool((raw[:GUARD] == s).all() and (raw[-GUARD:] == s).all())


def g(*shape, dt=torch.float32, seed=0, scale=1.0):
    gen = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(*shape, device=dev, generator=gen) * scale).to(dt)


@pytest.mark.parametrize("m,n,k", [(33, 48, 64), (300, 400, 200), (1000, 2048, 512), (257, 6144, 128)])
@pytest.mark.parametrize("epi", ["bf16", "gelu", "f32", "gate_res", "gate_res_aux", "euler"])
def test_gemm_epilogues_stay_in_bounds(m, n, k, epi):
    a, w, b, gate = g(m, k, dt=bf, seed=1), g(n, k, dt=bf, seed=2, scale=0.05), g(n, seed=3), g(n, seed=4)
    out_dt = bf if epi in ("bf16", "gelu") else torch.float32
    init = g(m, n, seed=5) if epi in ("gate_res", "gate_res_aux", "euler") else None
    raw, out = guarded((m, n), out_dt, init)
    plain = init.clone() if init is not None else torch.empty(m, n, device=dev, dtype=out_dt)
    kw = {}
    if epi.startswith("gate_res"):
        kw = dict(gate=gate, epilogue="gate_res")
    elif epi == "euler":
        kw = dict(epilogue="euler", alpha=torch.full((1,), 0.1, device=dev))
    else:
        kw = dict(epilogue=epi)
    raw_aux = aux = None
    if epi in ("gate_res_aux", "euler"):
        raw_aux, aux = guarded((m, n), bf)
        kw["aux"] = aux
    ops.gemm(a, w, out, bias=b, **kw)
    if "aux" in kw:
        kw["aux"] = torch.empty(m, n, device=dev, dtype=bf)
    ops.gemm(a, w, plain, bias=b, **kw)
    assert intact(raw)
    if raw_aux is not None:
        assert intact(raw_aux) and torch.equal(aux, kw["aux"])
    assert torch.equal(out, plain)


@pytest.mark.parametrize("rows,heads", [(129, 2), (384, 8), (1000, 3)])
def test_gemm_qknorm_rope_stays_in_bounds(rows, heads):
    d, k = 128, 256
    a, w = g(rows, k, dt=bf, seed=1), g(3 * heads * d, k, dt=bf, seed=2, scale=0.05)
    cos, sin, qw = g(rows, d // 2, seed=3), g(rows, d // 2, seed=4), g(d, seed=5)
    raw, out = guarded((rows, 3 * heads * d), bf)
    ops.gemm_qknorm_rope(a, w, out, heads * d, 2, qw, qw, 1e-6, bias=g(3 * heads * d, seed=6), cos=cos, sin=sin,
                         rope_rows=rows)
    assert intact(raw)
    assert torch.isfinite(out.float()).all()


@pytest.mark.parametrize("sq,skv,heads,splits", [(300, 300, 2, 0), (129, 16, 4, 0), (700, 256, 3, 0),
                                                 (1000, 1100, 1, 3), (2000, 2000, 1, 0)])
def test_attention_stays_in_bounds(sq, skv, heads, splits):
    d = 128
    q, k, v = g(sq, heads * d, dt=bf, seed=1), g(skv, heads * d, dt=bf, seed=2), g(skv, heads * d, dt=bf, seed=3)
    nws = max(16, ops.attention_workspace_bytes(sq, skv, heads, d, splits or None))
    raw_ws, ws = guarded((nws,), torch.uint8, torch.zeros(nws, dtype=torch.uint8, device=dev))  # counters start 0
    raw, o = guarded((sq, heads * d), bf)
    ops.attention(q, k, v, o, heads, d, splits=splits, workspace=ws)
    o2 = torch.empty(sq, heads * d, device=dev, dtype=bf)
    ops.attention(q, k, v, o2, heads, d, splits=splits,
                  workspace=torch.empty(nws, device=dev, dtype=torch.uint8))
    assert intact(raw) and intact(raw_ws)
    assert torch.equal(o, o2)


@pytest.mark.parametrize("rows,hidden", [(257, 2048), (33, 3072), (100, 1024), (70, 256), (1, 4096)])
def test_norm_modulate_stays_in_bounds(rows, hidden):
    x = g(rows, hidden)
    raw, y = guarded((rows, hidden), bf)
    raw_p, prev = guarded((rows, hidden), torch.float32, g(rows, hidden, seed=7))
    raw_s, part = guarded((2 * rows,), torch.float32)
    ops.norm_modulate(x, g(hidden, seed=1), g(hidden, seed=2), y, probe_prev=prev, probe_partials=part)
    assert intact(raw) and intact(raw_p) and intact(raw_s)


def test_qk_norm_gemv_cache_patchify_stay_in_bounds():
    rows, heads, d = 77, 3, 64
    raw, qkv = guarded((rows, 3 * heads * d), bf, g(rows, 3 * heads * d, dt=bf))
    ops.qk_norm_rope(qkv, heads, d, g(d, seed=1), g(d, seed=2), 1e-6, g(rows, d // 2), g(rows, d // 2), 0, rows)
    assert intact(raw)
    n, kk = 6 * 256, 256
    raw, out = guarded((n,), torch.float32)
    ops.gemv(g(n, kk, dt=bf, scale=0.05), g(kk), out, bias=g(n))
    assert intact(raw)
    raw_x, x = guarded((50, 256), torch.float32, g(50, 256))
    raw_o, off = guarded((50, 256), torch.float32, g(50, 256, seed=3))
    for mode in (0, 1, 2):
        ops.cache_offset(x, off, mode)
    assert intact(raw_x) and intact(raw_o)
    lat = g(8, 5, 12, 20)
    raw_t, tok = guarded((5 * 6 * 10, 32), torch.float32)
    raw_b, tokb = guarded((5 * 6 * 10, 32), bf)
    ops.patchify(lat, tok, tokb, (5, 6, 10), (1, 2, 2))
    raw_l, back = guarded((8, 5, 12, 20), torch.float32)
    ops.unpatchify(tok, back, (5, 6, 10), (1, 2, 2))
    assert intact(raw_t) and intact(raw_b) and intact(raw_l)
    assert torch.equal(back, lat)


def test_fp32_validation_kernels_stay_in_bounds():
    m, n, k = 77, 100, 96
    raw, out = guarded((m, n), torch.float32)
    ops.gemm(g(m, k), g(n, k, dt=bf, scale=0.05), out, bias=g(n), epilogue="f32")
    assert intact(raw)
    sq, skv, heads, d = 45, 70, 2, 64
    raw, o = guarded((sq, heads * d), torch.float32)
    ops.attention(g(sq, heads * d), g(skv, heads * d, seed=2), g(skv, heads * d, seed=3), o, heads, d)
    assert intact(raw)
