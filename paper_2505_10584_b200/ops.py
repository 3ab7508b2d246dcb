"""Torch-facing wrappers over the C-ABI (``include/aqb.h``).

Each wrapper validates device / dtype / layout, then passes raw pointers and
the *current* CUDA stream to libaqb.so (so calls are stream-ordered and CUDA
graph capturable).  Nothing here computes on the CPU and there is no
fallback path: a missing library or a non-CUDA tensor raises.
"""

from __future__ import annotations

import os

import torch

from . import _native
from .errors import NativeError

EPI = {"bf16": 0, "gelu": 1, "gate_res": 2, "f32": 3, "euler": 4}
BF16, F32 = torch.bfloat16, torch.float32


def _stream():
    return torch.cuda.current_stream().cuda_stream


class KernelProfiler:
    """Optional per-launch CUDA-event timing / counting (bench.py).

    When installed with :func:`set_profiler`, every kernel launch is
    bracketed by CUDA events on the launching (current) stream and recorded
    as ``(kind, start, end, work)`` where ``work`` is FLOPs for tensor-core
    kernels and algorithmic HBM bytes for the memory-bound ones.  With
    ``timing=False`` launches are only counted.
    """

    def __init__(self, timing: bool = True):
        self.timing = timing
        self.records = []
        self.count = 0

    def by_launch(self):
        """Per (C-ABI entry, work) group — i.e. per shape — launches, ms and work."""
        torch.cuda.synchronize()
        out = {}
        for _kind, e0, e1, work, name in self.records:
            d = out.setdefault((name, work), {"launches": 0, "ms": 0.0})
            d["launches"] += 1
            d["ms"] += e0.elapsed_time(e1)
        return out

    def summary(self):
        """Per kind: launches, ms (0 without timing) and algorithmic work."""
        torch.cuda.synchronize()
        out = {}
        for kind, e0, e1, work, _name in self.records:
            d = out.setdefault(kind, {"launches": 0, "ms": 0.0, "work": 0.0})
            d["launches"] += 1
            d["ms"] += e0.elapsed_time(e1) if e0 is not None else 0.0
            d["work"] += work
        return out


# kernel symbol -> kind (the KernelProfiler kinds), for CUPTI traces of libaqb kernels
KERNEL_KINDS = (("gemm", ("gemm",)), ("attention", ("attn_", "attention_kernel")), ("norm_modulate", ("norm_mod",)),
                ("qk_norm_rope", ("qk_norm_rope",)), ("gemv", ("gemv",)), ("cache_offset", ("cache_offset",)),
                ("peer", ("barrier_kernel",)),
                ("layout", ("patchify", "heads_to_seq", "blend_kernel", "window_kernel")))


def kernel_kind(symbol: str) -> str | None:
    """The kind of a libaqb kernel symbol (None: not one of ours)."""
    if "aqb::" not in symbol:
        return None
    for kind, keys in KERNEL_KINDS:
        if any(k in symbol for k in keys):
            return kind
    return "small"


def trace_kernels(fn) -> dict:
    """Run ``fn`` under the CUDA activity tracer (torch.profiler / CUPTI) with programmatic
    dependent launch off, and return per kind ``{"launches", "ms"}`` of the libaqb kernels it
    launched — device execution time of each kernel, free of event/launch gaps (with PDL on,
    a dependent kernel's span would include its wait for the predecessor)."""
    from torch.profiler import ProfilerActivity, profile

    prev = set_pdl(False)
    try:
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
    finally:
        set_pdl(prev)
    out = {}
    for ev in prof.key_averages():
        kind = kernel_kind(ev.key)
        if kind is None:
            continue
        us = getattr(ev, "device_time_total", None)
        if us is None:
            us = ev.cuda_time_total
        d = out.setdefault(kind, {"launches": 0, "ms": 0.0})
        d["launches"] += ev.count
        d["ms"] += us / 1e3
    return out


def set_pdl(on: bool) -> bool:
    """Programmatic dependent launch on/off for subsequent launches; returns the previous state."""
    return bool(_native.query("aqb_set_pdl", 1 if on else 0))


_PROF: KernelProfiler | None = None


def set_profiler(p: KernelProfiler | None):
    global _PROF
    _PROF = p


_SYNC_DEBUG = bool(os.environ.get("AQB_SYNC_DEBUG"))


def _run(kind, work, name, *args):
    prof = _PROF
    if _SYNC_DEBUG:  # debugging aid: fail at the launch that faults, naming it
        _native.call(name, *args)
        try:
            torch.cuda.synchronize()
        except Exception as e:
            raise NativeError(f"{name} faulted: {e}") from e
        return
    if prof is None:
        _native.call(name, *args)
        return
    prof.count += 1
    if not prof.timing:
        _native.call(name, *args)
        prof.records.append((kind, None, None, float(work), name))
        return
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.call(name, *args)
    e1.record()
    prof.records.append((kind, e0, e1, float(work), name))


def _p(t):
    return None if t is None else t.data_ptr()


def _need(t, dtype, name):
    if not t.is_cuda:
        raise NativeError(f"{name}: tensor must be on a CUDA device (no CPU fallback)")
    if t.dtype != dtype:
        raise NativeError(f"{name}: expected {dtype}, got {t.dtype}")
    if t.stride(-1) != 1:
        raise NativeError(f"{name}: innermost dim must be contiguous")


def norm_modulate(x, shift, scale, out, eps=1e-6, kind=0, probe_prev=None, probe_partials=None,
                  run_flag=None, run_if=1):
    """out = norm(x)·(1+scale)+shift, row-wise over the last dim (out bf16, or f32 in fp32 validation mode)."""
    _need(x, F32, "norm_modulate.x")
    f32 = out.dtype == F32
    _need(out, F32 if f32 else BF16, "norm_modulate.out")
    rows, hidden = x.shape
    _run("norm_modulate", rows * hidden * (4 + out.element_size()) + (8 * rows * hidden if probe_prev is not None else 0),
         "aqb_norm_modulate_f32" if f32 else "aqb_norm_modulate", _p(x), x.stride(0), _p(shift), _p(scale), _p(out),
         out.stride(0), rows, hidden, float(eps), int(kind), _p(probe_prev), _p(probe_partials), _p(run_flag),
         int(run_if), _stream())
    return out


def norm_modulate_gather(x, shift, scale, outs, ldy, eps=1e-6, kind=0, probe_prev=None, probe_partials=None,
                         run_flag=None, run_if=1):
    """norm_modulate whose rows are stored into every address in ``outs`` (device pointers with
    stride ``ldy``, bf16): the TP-SP all-gather done by the producing kernel's own stores."""
    _need(x, F32, "norm_modulate_gather.x")
    rows, hidden = x.shape
    _run("norm_modulate", rows * hidden * (4 + 2 * len(outs)) + (8 * rows * hidden if probe_prev is not None else 0),
         "aqb_norm_modulate_gather", _p(x), x.stride(0), _p(shift), _p(scale), _native.ptr_array(outs), len(outs),
         int(ldy), rows, hidden, float(eps), int(kind), _p(probe_prev), _p(probe_partials), _p(run_flag),
         int(run_if), _stream())


def gate_bcast(src, gate, dsts, ldd, run_flag=None, run_if=1):
    """gate * src (f32 [rows, cols]) stored into every device address in ``dsts`` (row stride ``ldd``)."""
    _need(src, F32, "gate_bcast.src")
    rows, cols = src.shape
    _run("small", rows * cols * 4 * (1 + len(dsts)), "aqb_gate_bcast", _p(src), src.stride(0), _p(gate),
         _native.ptr_array(dsts), len(dsts), int(ldd), rows, cols, _p(run_flag), int(run_if), _stream())


def sum_slots(x, slots, run_flag=None, run_if=1):
    """x += sum_k slots[k] in slot order (x f32 [rows, cols], slots f32 [P, rows, cols])."""
    _need(x, F32, "sum_slots.x")
    _need(slots, F32, "sum_slots.slots")
    rows, cols = x.shape
    _run("small", rows * cols * 4 * (2 + slots.shape[0]), "aqb_sum_slots", _p(x), x.stride(0), _p(slots),
         slots.shape[0], slots.stride(0), slots.stride(1), rows, cols, _p(run_flag), int(run_if), _stream())


def gemm_gate_add_scatter(a, w, peer_out, ldo, rows_per_rank, bias=None, gate=None, run_flag=None, run_if=1):
    """Row-parallel projection partial, gate * (a @ w.T + bias) reduce-added into the residual
    (f32, stride ``ldo``) of the rank owning each row (``peer_out[r]``): the TP-SP reduce-scatter
    fused into the GEMM epilogue."""
    _need(a, BF16, "gemm_gate_add_scatter.a")
    _need(w, BF16, "gemm_gate_add_scatter.w")
    m, k = a.shape
    n = w.shape[0]
    if w.shape[1] != k:
        raise NativeError(f"gemm_gate_add_scatter: K mismatch {k} vs {w.shape[1]}")
    _run("gemm", 2.0 * m * n * k, "aqb_gemm_gate_add_scatter", _p(a), a.stride(0), _p(w), w.stride(0),
         _native.ptr_array(peer_out), len(peer_out), int(ldo), int(rows_per_rank), m, n, k, _p(bias), _p(gate),
         _p(run_flag), int(run_if), _stream())


def gemm(a, w, out, bias=None, gate=None, epilogue="bf16", alpha=None, aux=None, run_flag=None, run_if=1):
    """out = epilogue(a @ w.T + bias) on tcgen05 (a [M,K] bf16, w [N,K] bf16).

    fp32 validation mode: ``a`` f32 selects the SIMT fp32 kernel (out/aux f32)."""
    _need(w, BF16, "gemm.w")
    m, k = a.shape
    n, k2 = w.shape
    if k2 != k:
        raise NativeError(f"gemm: K mismatch {k} vs {k2}")
    e = EPI[epilogue]
    f32 = a.dtype == F32
    _need(a, F32 if f32 else BF16, "gemm.a")
    _need(out, F32 if (f32 or e not in (0, 1)) else BF16, "gemm.out")
    if out.shape[0] != m or out.shape[1] < n:
        raise NativeError(f"gemm: out shape {tuple(out.shape)} vs ({m},{n})")
    _run("gemm", 2.0 * m * n * k, "aqb_gemm_f32" if f32 else "aqb_gemm_bf16", _p(a), a.stride(0), _p(w), w.stride(0),
         _p(out), out.stride(0), m, n, k, _p(bias), _p(gate), e, _p(alpha), _p(aux),
         aux.stride(0) if aux is not None else 0, _p(run_flag), int(run_if), _stream())
    return out


def gemm_qknorm_rope(a, w, out, part_width, norm_parts, q_w, k_w, eps, bias=None, cos=None, sin=None, rope_row0=0,
                     rope_rows=0, out_row_stride=None, groups=1, group_stride=0, hpg=None, g_base=0, run_flag=None,
                     run_if=1):
    """QKV projection with QK-RMSNorm + 3D RoPE (+ Ulysses pack) fused in the epilogue (head_dim 128)."""
    _need(a, BF16, "gemm_qknorm_rope.a")
    _need(w, BF16, "gemm_qknorm_rope.w")
    _need(out, BF16, "gemm_qknorm_rope.out")
    m, k = a.shape
    n = w.shape[0]
    hpg = part_width // 128 if hpg is None else hpg
    if out_row_stride is None:
        out_row_stride = out.stride(0)
    _run("gemm", 2.0 * m * n * k, "aqb_gemm_qknorm_rope", _p(a), a.stride(0), _p(w), w.stride(0), m, n, k, _p(bias),
         int(part_width), int(norm_parts), _p(q_w), _p(k_w), float(eps), _p(cos), _p(sin), int(rope_row0),
         int(rope_rows), _p(out), int(out_row_stride), int(groups), int(group_stride), int(hpg), int(g_base),
         _p(run_flag), int(run_if), _stream())
    return out


def qk_norm_rope(src, heads, head_dim, q_w, k_w, eps, cos=None, sin=None, rope_row0=0, rope_rows=0,
                 dst=None, head_begin=0, head_count=None, hpg=None, dst_group_stride=0, dst_row_stride=None,
                 dst_which_stride=None, parts=3, norm_parts=2, run_flag=None, run_if=1):
    """QK-RMSNorm + 3D RoPE over a [rows, parts, heads, D] buffer (optionally repacked into dst).

    bf16, or f32 (fp32 validation mode) — src and dst share the dtype."""
    f32 = src.dtype == F32
    _need(src, F32 if f32 else BF16, "qk_norm_rope.src")
    rows = src.shape[0]
    head_count = heads if head_count is None else head_count
    hpg = head_count if hpg is None else hpg
    if dst is None:
        dst = src
    if dst_row_stride is None:
        dst_row_stride = dst.stride(0)
    if dst_which_stride is None:
        dst_which_stride = heads * head_dim
    if dst.dtype != src.dtype:
        raise NativeError("qk_norm_rope: src and dst dtypes differ")
    _run("qk_norm_rope", 2 * rows * head_count * head_dim * parts * src.element_size(),
         "aqb_qk_norm_rope_f32" if f32 else "aqb_qk_norm_rope", _p(src), src.stride(0), rows, heads, head_begin, head_count, head_dim,
                 _p(q_w), _p(k_w), float(eps), _p(cos), _p(sin), int(rope_row0), int(rope_rows), _p(dst),
                 int(dst_group_stride), int(dst_row_stride), int(dst_which_stride), int(hpg), int(parts),
                 int(norm_parts), _p(run_flag), int(run_if), _stream())
    return dst


def attention_workspace_bytes(seq_q, seq_kv, heads, head_dim, splits=None):
    """Workspace the split-KV path needs (0 when one pass is best)."""
    if splits is None:
        return int(_native.query("aqb_attention_auto_workspace_bytes", seq_q, seq_kv, heads, head_dim))
    return int(_native.query("aqb_attention_workspace_bytes", seq_q, heads, head_dim, splits))


def attention(q, k, v, o, heads, head_dim, q_head_stride=None, k_head_stride=None, v_head_stride=None,
              o_head_stride=None, scale=None, splits=0, workspace=None, run_flag=None, run_if=1):
    """Non-causal flash attention; q/k/v/o are 2-D row views [seq, ld] (head h at column h*head_stride).

    ``splits``: 0 = automatic split-KV (uses ``workspace`` when given, a uint8
    CUDA tensor), 1 = single pass."""
    f32 = q.dtype == F32
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (o, "o")):
        _need(t, F32 if f32 else BF16, f"attention.{nm}")
    hs = lambda x: head_dim if x is None else x  # noqa: E731
    scale = head_dim ** -0.5 if scale is None else scale
    if f32:  # fp32 validation mode
        _run("attention", 4.0 * q.shape[0] * k.shape[0] * head_dim * heads, "aqb_attention_f32", _p(q), q.stride(0),
             hs(q_head_stride), _p(k), k.stride(0), hs(k_head_stride), _p(v), v.stride(0), hs(v_head_stride), _p(o),
             o.stride(0), hs(o_head_stride), q.shape[0], k.shape[0], heads, head_dim, float(scale), _p(run_flag),
             int(run_if), _stream())
        return o
    ws, wsb = (_p(workspace), workspace.numel()) if workspace is not None else (None, 0)
    _run("attention", 4.0 * q.shape[0] * k.shape[0] * head_dim * heads, "aqb_attention_fwd", _p(q), q.stride(0),
         hs(q_head_stride), _p(k), k.stride(0), hs(k_head_stride), _p(v), v.stride(0), hs(v_head_stride), _p(o),
         o.stride(0), hs(o_head_stride), q.shape[0], k.shape[0], heads, head_dim, float(scale), int(splits), ws, wsb,
         _p(run_flag), int(run_if), _stream())
    return o


def attention_scatter(q, k, v, peer_o, ldo, heads, head_dim, rows_per_rank, text_row0, scale=None, splits=0,
                      workspace=None, run_flag=None, run_if=1):
    """Attention whose epilogue stores each output row into the owning rank's O buffer (peer memory)."""
    for t, nm in ((q, "q"), (k, "k"), (v, "v")):
        _need(t, BF16, f"attention_scatter.{nm}")
    scale = head_dim ** -0.5 if scale is None else scale
    ws, wsb = (_p(workspace), workspace.numel()) if workspace is not None else (None, 0)
    _run("attention", 4.0 * q.shape[0] * k.shape[0] * head_dim * heads, "aqb_attention_fwd_scatter", _p(q),
         q.stride(0), head_dim, _p(k), k.stride(0), head_dim, _p(v), v.stride(0), head_dim,
         _native.ptr_array(peer_o), len(peer_o), int(ldo), head_dim, int(rows_per_rank), int(text_row0), q.shape[0],
         k.shape[0], heads, head_dim, float(scale), int(splits), ws, wsb, _p(run_flag), int(run_if), _stream())


def gemm_qknorm_rope_scatter(a, w, peer_out, part_width, norm_parts, q_w, k_w, eps, out_row_stride, hpg, bias=None,
                             cos=None, sin=None, rope_row0=0, rope_rows=0, run_flag=None, run_if=1):
    """QKV projection + QK-RMSNorm + 3D RoPE whose epilogue stores head group g into rank g's buffer."""
    _need(a, BF16, "gemm_qknorm_rope_scatter.a")
    _need(w, BF16, "gemm_qknorm_rope_scatter.w")
    m, k = a.shape
    n = w.shape[0]
    _run("gemm", 2.0 * m * n * k, "aqb_gemm_qknorm_rope_scatter", _p(a), a.stride(0), _p(w), w.stride(0), m, n, k,
         _p(bias), int(part_width), int(norm_parts), _p(q_w), _p(k_w), float(eps), _p(cos), _p(sin), int(rope_row0),
         int(rope_rows), _native.ptr_array(peer_out), len(peer_out), int(out_row_stride), int(hpg), _p(run_flag),
         int(run_if), _stream())


def peer_barrier(peer_signal, rank, epoch, status, payload=None, pay_out=None, run_flag=None, run_if=1):
    """Stream-ordered barrier over peer memory (optionally summing a few floats in rank order)."""
    npay = 0 if payload is None else payload.numel()
    _run("peer", 0, "aqb_peer_barrier", _native.ptr_array(peer_signal), int(rank), len(peer_signal), _p(epoch),
         _p(payload), npay, _p(pay_out), _p(status), _p(run_flag), int(run_if), _stream())


def gemv(w, x, out, bias=None, add=None, in_silu=False, t=None):
    """out[f32] = w @ in(x) + bias + add  (x f32, or timestep features of device scalar t)."""
    _need(w, BF16, "gemv.w")
    n, k = w.shape
    _run("gemv", 2 * n * k, "aqb_gemv", _p(w), _p(x), _p(t), _p(bias), _p(add), _p(out), n, k, int(bool(in_silu)), _stream())
    return out


def add_bcast(out, a, b):
    _run("small", 12 * b.numel(), "aqb_add_bcast", _p(out), _p(a), a.numel(), _p(b), b.numel(), _stream())
    return out


def rel_l1_reduce(partials, rows, sums):
    _run("small", 8 * rows, "aqb_rel_l1_reduce", _p(partials), rows, _p(sums), _stream())


def cache_decide(sums, state, threshold, warmup, total_steps, force_last, flags_out, rel_out):
    _run("small", 0, "aqb_cache_decide", _p(sums), _p(state), float(threshold), int(warmup), int(total_steps),
                 int(bool(force_last)), _p(flags_out), _p(rel_out), _stream())


def cache_offset(x, off, mode, run_flag=None, run_if=1):
    rows, hidden = off.shape
    _run("cache_offset", (8 if mode == 0 else 12) * rows * hidden, "aqb_cache_offset", _p(x), x.stride(0), _p(off), rows, hidden, int(mode), _p(run_flag),
                 int(run_if), _stream())


def step_scalars(ts, dts, idx, cur, advance=False):
    _run("small", 0, "aqb_step_scalars", _p(ts), _p(dts), _p(idx), _p(cur), int(bool(advance)), _stream())


def patchify(lat, tok, tok_bf16, grid, patch, frame_offset=0):
    """tokens <- latent frames [frame_offset, frame_offset + T*pt) of lat [C, Tl, H, W]."""
    C, Tl = lat.shape[0], lat.shape[1]
    _run("layout", 10 * tok.numel(), "aqb_patchify", _p(lat), _p(tok), _p(tok_bf16), C, grid[0], grid[1], grid[2],
         patch[0], patch[1], patch[2], Tl, int(frame_offset), _stream())


def unpatchify(tok, lat, grid, patch, frame_offset=0):
    C, Tl = lat.shape[0], lat.shape[1]
    _run("layout", 8 * tok.numel(), "aqb_unpatchify", _p(tok), _p(lat), C, grid[0], grid[1], grid[2], patch[0],
         patch[1], patch[2], Tl, int(frame_offset), _stream())


def heads_to_seq(src, rows, P, width, dst, run_flag=None, run_if=1):
    _run("layout", 4 * rows * P * width, "aqb_heads_to_seq", _p(src), rows, P, width, _p(dst), dst.stride(0), _p(run_flag), int(run_if),
                 _stream())


def tile_blend(ptrs, starts, counts, tile, overlap, latent, out):
    """VAE tile blend (``aqb_tile_blend``); ptrs int64 / starts int32 device tensors."""
    _need(out, F32, "tile_blend.out")
    C = out.shape[0]
    _run("layout", 8.0 * out.numel(), "aqb_tile_blend", _p(ptrs), _p(starts), *[int(c) for c in counts],
         *[int(x) for x in tile], *[int(x) for x in overlap], *[int(x) for x in latent], C, _p(out), _stream())
    return out


def window_average(ptrs, starts, nclips, n, n_prime, out):
    """Temporal MultiDiffusion Eq. 3 (``aqb_window_average``); out f32 [C, n', H, W]."""
    _need(out, F32, "window_average.out")
    C = out.shape[0]
    hw = out[0, 0].numel()
    _run("layout", 4.0 * out.numel() * (1 + n * nclips / n_prime), "aqb_window_average", _p(ptrs), _p(starts),
         int(nclips), int(n), int(n_prime), C, hw, _p(out), _stream())
    return out
