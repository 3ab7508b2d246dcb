"""Single-DiT and MM-DiT denoise step on hand-written sm_100a kernels.

Model construction mirrors the paper's two families (``PAPER.md:15-17,103,
106``); every tensor op of a step is a libaqb.so kernel launched on the
current stream (see ``ops.py``):

Single-DiT block (AdaLN-single, PixArt layout)::

    m   = norm_modulate(x, shift1, scale1)                  [HBM-bound]
    qkv = gemm(m, Wqkv) (+bias)                             [tcgen05]
    qkv = qk_norm_rope(qkv)  (in place / Ulysses pack)      [HBM-bound]
    o   = attention(q, k, v)  (3D full, non-causal)         [tcgen05 + TMEM]
    x  += gate1 * gemm(o, Wproj)                            [tcgen05, gate·residual epilogue]
    x  += gemm(attention(qk_norm(gemm(x, Wq)), textK, textV), Wxproj)
    x  += gate2 * gemm(gelu(gemm(norm_modulate(x), W1)), W2)

MM-DiT runs the video and text streams as two row ranges of one residual
buffer ``x = [video; text]``, so the joint attention over the concatenated
sequence needs no concat copy; dual blocks use per-stream weights, single
blocks one weight set over all rows.

Diffusion cache (``dit-layer-cache``): the front
``ceil(fraction·L)`` blocks always run; on a full step the rear blocks'
offset ``x_out - x_in`` (video rows) is stored, on a cached step it is added
instead of running them.  ``mode='dynamic'`` takes the decision on device
(rel-L1 probe fused into block 0's norm kernel) and gates the rear kernels
with a device flag — no host round-trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .config import DiTConfig
from .errors import ConfigError
from .parallel import SIGNAL_BYTES, PeerBuffers, Ulysses, exchange_offsets, tp_shard
from .schedule import front_block_count
from .weights import init_weights

BF16, F32 = torch.bfloat16, torch.float32
PRECISIONS = ("bf16", "fp32")


def rope_tables(grid, dims, theta, device):
    """cos/sin [S, D/2] of the 3D RoPE (interleaved pairs, t|h|w channel split).

    Setup-time table (once per geometry); the per-step rotation runs in
    ``aqb_qk_norm_rope``.  Computed in float64 then rounded to fp32.
    """
    T, H, W = grid
    tt, hh, ww = torch.meshgrid(torch.arange(T, device=device), torch.arange(H, device=device),
                                torch.arange(W, device=device), indexing="ij")
    pos = [tt.reshape(-1).double(), hh.reshape(-1).double(), ww.reshape(-1).double()]
    ang = []
    for p, d in zip(pos, dims):
        j = torch.arange(0, d, 2, dtype=torch.float64, device=device)
        ang.append(p[:, None] * (theta ** (-j / d))[None, :])
    ang = torch.cat(ang, dim=1)
    return torch.cos(ang).float().contiguous(), torch.sin(ang).float().contiguous()


@dataclass
class _Geometry:
    grid: tuple
    Sv: int        # video tokens (global)
    Sv_loc: int    # video tokens on this rank
    St: int        # text tokens (MM-DiT joint rows; 0 for Single-DiT)
    rows: int      # rows of the residual buffer on this rank


class DiTModel:
    """Executable DiT (either family) bound to one GPU / one Ulysses rank."""

    def __init__(self, cfg: DiTConfig, weights: dict | None = None, seed: int = 0, device="cuda",
                 sp: Ulysses | None = None, cached_cost_fraction: float = 0.25, precision: str = "bf16"):
        """``precision``: ``"bf16"`` (the product path: bf16 activations, tcgen05 kernels) or
        ``"fp32"`` (validation mode, north_star <= 1e-4: fp32 activations, SIMT kernels; 1 GPU)."""
        if not torch.cuda.is_available():
            raise ConfigError("a CUDA device is required (no CPU fallback)", "device")
        if precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {PRECISIONS}", "model.precision")
        if precision == "fp32" and sp is not None and sp.P > 1:
            raise ConfigError("fp32 validation mode runs on one GPU", "model.precision")
        self.precision = precision
        self.fp32 = precision == "fp32"
        self.act = F32 if self.fp32 else BF16
        self.cfg = cfg
        self.device = torch.device(device)
        self.sp = sp
        if weights is None:
            weights = init_weights(cfg, seed=seed, device=self.device)
        self.W = {k: v.to(self.device).contiguous() for k, v in weights.items()}
        self.n_front = front_block_count(cfg.num_layers, cached_cost_fraction)
        self._stack_modulation()
        self.geo = None

    # ------------------------------------------------------------------ setup
    def _stack_modulation(self):
        cfg, W, H = self.cfg, self.W, self.cfg.hidden_size
        if cfg.family == "single-dit":
            self.tables = torch.stack([W[f"blocks.{i}.table"] for i in range(cfg.num_single)]).contiguous()
            return
        names = []
        for i in range(cfg.num_dual):
            names += [f"dual.{i}.img.mod", f"dual.{i}.txt.mod"]
        names += [f"single.{i}.mod" for i in range(cfg.num_single)]
        names += ["final.mod"]
        self.mod_names = names
        self.mod_w = torch.cat([W[f"{n}.w"] for n in names]).contiguous()
        self.mod_b = torch.cat([W[f"{n}.b"] for n in names]).contiguous()
        off, self.mod_off = 0, {}
        for n in names:
            self.mod_off[n] = off
            off += W[f"{n}.b"].numel()
        for n in names:  # the stacked copy is the only one kept
            del W[f"{n}.w"]

    def prepare(self, grid, text: torch.Tensor, pooled: torch.Tensor | None = None):
        """Bind geometry + conditioning; allocate the step workspace."""
        cfg, dev = self.cfg, self.device
        self._text, self._pooled = text, pooled
        grid = tuple(int(g) for g in grid)
        Sv = grid[0] * grid[1] * grid[2]
        P = 1 if self.sp is None else self.sp.P
        if self.sp is not None:
            self.sp.check(cfg.num_heads, Sv)
        Sv_loc = Sv // P
        St = cfg.text_len if cfg.family == "mm-dit" else 0
        if text.shape != (cfg.text_len, cfg.text_dim):
            raise ConfigError(f"text must be [{cfg.text_len}, {cfg.text_dim}]", "inputs.text")
        self.geo = _Geometry(grid, Sv, Sv_loc, St, Sv_loc + St)
        H, F, A, D = cfg.hidden_size, cfg.ffn_dim, cfg.num_heads, cfg.head_dim
        rows = self.geo.rows
        e = lambda *s, dt=self.act: torch.empty(*s, device=dev, dtype=dt)  # noqa: E731
        self.x = e(rows, H, dt=F32)
        self.m = e(rows, H)
        self.qkv = e(rows, 3 * H)
        self.o = e(rows, H)
        self.h = e(rows, F)
        self.lat = e(Sv_loc, cfg.patch_dim, dt=F32)
        self.lat_bf = e(Sv_loc, cfg.patch_dim)
        self.off = e(Sv_loc, H, dt=F32)
        self.cos, self.sin = rope_tables(grid, cfg.rope_dims, cfg.rope_theta, dev)
        # per-step scalars (t, dt) live on device so one captured step replays for every step
        self.idx = torch.zeros(1, device=dev, dtype=torch.int32)
        self.cur = torch.zeros(2, device=dev, dtype=F32)
        # cache probe / decision state
        self.prev = torch.zeros(Sv_loc, H, device=dev, dtype=F32)
        self.partials = e(2 * Sv_loc, dt=F32)
        self.sums = e(2, dt=F32)
        self.cstate = torch.zeros(4, device=dev, dtype=torch.int32)
        self.flag = self.cstate[1:2]
        t_bf = text.to(dev, F32).to(self.act).contiguous()
        W = self.W
        if cfg.family == "single-dit":
            self.t0 = e(H, dt=F32)
            self.th = e(H, dt=F32)
            self.tmod = e(6 * H, dt=F32)
            self.mods = e(cfg.num_single, 6 * H, dt=F32)
            self.fmods = e(2 * H, dt=F32)
            self.xq = e(Sv_loc, H)
            # step-independent cross-attention K/V of the text, once per call (K RMS-normed)
            self.text_kv = []
            heads = A // P if self._tp() else A  # TP-SP: this rank's heads
            for i in range(cfg.num_single):
                kv = e(cfg.text_len, 2 * heads * D)
                ops.gemm(t_bf, W[f"blocks.{i}.xkv.w"], kv, bias=W[f"blocks.{i}.xkv.b"])
                ops.qk_norm_rope(kv, heads, D, W[f"blocks.{i}.xk_norm"], None, cfg.qk_norm_eps, parts=2,
                                 norm_parts=1)
                self.text_kv.append(kv)
        else:
            if pooled is None or pooled.shape != (cfg.pooled_dim,):
                raise ConfigError(f"pooled must be [{cfg.pooled_dim}]", "inputs.pooled")
            self.th = e(H, dt=F32)
            self.vec = e(H, dt=F32)
            self.pe = e(H, dt=F32)
            pl = pooled.to(dev, F32).contiguous()
            ops.gemv(W["p_emb.fc1.w"], pl, self.th, bias=W["p_emb.fc1.b"])
            ops.gemv(W["p_emb.fc2.w"], self.th, self.pe, bias=W["p_emb.fc2.b"], in_silu=True)
            self.allmods = e(self.mod_w.shape[0], dt=F32)
            self.txt0 = e(St, H, dt=F32)
            ops.gemm(t_bf, W["txt_in.w"], self.txt0, bias=W["txt_in.b"], epilogue="f32")
        self.peer = None
        self.ocache = self.xocache = None
        self.cache_mode = "dit-layer-cache"
        hl = A // P
        self.hl = hl
        if self._tp():
            self._prepare_tp()
        elif self.sp is not None and P > 1:
            if self.sp.exchange == "p2p" and D == 128:
                # symmetric buffers: attention input (all heads of this rank's group, full
                # sequence) and the residual-row-major attention output
                rs = 3 * hl * D
                self.peer = PeerBuffers(self.sp, {"rcv": (Sv + St) * rs * 2, "o": rows * H * 2,
                                                  "sig": SIGNAL_BYTES}, dev)
                self.a2a_rcv = self.peer.local("rcv", (Sv + St, 3, hl, D), BF16)
                self.o = self.peer.local("o", (rows, H), BF16)
                off = exchange_offsets(self.sp.rank, P, Sv_loc, hl, D, H)
                self.qkv_dst = self.peer.ptrs("rcv", off["qkv"])
                self.o_dst = self.peer.ptrs("o", off["o"])
                self.sig = self.peer.ptrs("sig")
                self.epoch = torch.zeros(1, device=dev, dtype=torch.int32)
                self.peer_status = torch.zeros(1, device=dev, dtype=torch.int32)
            else:
                self.a2a_snd = e(P, Sv_loc, 3, hl, D)
                self.a2a_rcv = e(Sv + St, 3, hl, D)
                self.oh = e(Sv + St, hl * D)
                self.ob = e(P, Sv_loc, hl * D)
                if St:
                    self.tg = e(P, St, hl * D)
        # split-KV workspace for the attention launches of this geometry
        need = ops.attention_workspace_bytes(Sv + St if P > 1 else rows, Sv + St, hl, D)
        if cfg.family == "single-dit":
            xq_rows, xheads = (Sv, hl) if self._tp() else (Sv_loc, A)
            need = max(need, ops.attention_workspace_bytes(xq_rows, cfg.text_len, xheads, D))
        self.attn_ws = torch.zeros(max(need, 16), device=dev, dtype=torch.uint8)  # split counters start at 0
        return self

    def _tp(self) -> bool:
        return self.sp is not None and getattr(self.sp, "tensor_parallel", False)

    def _prepare_tp(self):
        raise ConfigError("TP-SP needs a TP model class (build_model with a TensorSP group)", "parallel.tp")

    def _barrier(self, flag=None, run_if=1, payload=None):
        ops.peer_barrier(self.sig, self.sp.rank, self.epoch, self.peer_status, payload=payload,
                         pay_out=payload, run_flag=flag, run_if=run_if)

    def peer_ok(self) -> bool:
        """False if a peer barrier timed out (a rank never arrived) since prepare()."""
        return self.peer is None or int(self.peer_status.item()) == 0

    def close(self):
        """Release the symmetric peer buffers (collective under a multi-rank group; drop any
        CUDA graph that captured this model first — it holds their addresses)."""
        for name in ("peer_ocache", "peer"):
            pb = self.__dict__.pop(name, None)
            if pb is not None:
                pb.close()
        self.peer = None

    # ------------------------------------------------------------- primitives
    def _mod(self, name):
        H = self.cfg.hidden_size
        if self.cfg.family == "single-dit":
            i = name
            row = self.mods[i]
            return [row[k * H:(k + 1) * H] for k in range(6)]
        o = self.mod_off[name]
        n = 2 if name == "final.mod" else 6
        return [self.allmods[o + k * H:o + (k + 1) * H] for k in range(n)]

    def _qkv_attention(self, pi, pt, flag, run_if):
        """QKV projection(s) + QK-RMSNorm + 3D RoPE + joint self-attention -> self._ob
        (``self.o``, or this block's attention-cache slot).

        ``pi``: weight prefix of the video stream (rows [0, Sv_loc)); ``pt``:
        prefix of the text rows [Sv_loc, rows) (MM-DiT; == pi for single
        blocks) or None (Single-DiT).  head_dim 128 uses the fused
        GEMM+norm+RoPE(+pack) kernel; other head dims run GEMM then
        ``aqb_qk_norm_rope``.  P > 1 (Ulysses): the projection epilogue writes
        the all-to-all send layout, text rows go straight into the receive
        buffer's tail (local heads), attention runs over A/P heads and full
        sequence, then the all-to-all back + head->sequence repack.
        """
        cfg, g, W = self.cfg, self.geo, self.W
        A, D, H, eps = cfg.num_heads, cfg.head_dim, cfg.hidden_size, cfg.qk_norm_eps
        n, R, St = g.Sv_loc, g.rows, g.St
        fused = D == 128 and not self.fp32
        m, qkv = self.m, self.qkv
        wi, bi = W[f"{pi}.qkv.w"], W[f"{pi}.qkv.b"]
        if pt is not None:
            wt, bt = W[f"{pt}.qkv.w"], W[f"{pt}.qkv.b"]
        if self.sp is None or self.sp.P == 1:
            if fused:
                if pt == pi or pt is None:
                    ops.gemm_qknorm_rope(m, wi, qkv, H, 2, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, bias=bi,
                                         cos=self.cos, sin=self.sin, rope_rows=g.Sv, run_flag=flag, run_if=run_if)
                else:
                    ops.gemm_qknorm_rope(m[:n], wi, qkv[:n], H, 2, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, bias=bi,
                                         cos=self.cos, sin=self.sin, rope_rows=g.Sv, run_flag=flag, run_if=run_if)
                    ops.gemm_qknorm_rope(m[n:], wt, qkv[n:], H, 2, W[f"{pt}.q_norm"], W[f"{pt}.k_norm"], eps, bias=bt,
                                         run_flag=flag, run_if=run_if)
            else:
                if pt == pi or pt is None:
                    ops.gemm(m, wi, qkv, bias=bi, run_flag=flag, run_if=run_if)
                else:
                    ops.gemm(m[:n], wi, qkv[:n], bias=bi, run_flag=flag, run_if=run_if)
                    ops.gemm(m[n:], wt, qkv[n:], bias=bt, run_flag=flag, run_if=run_if)
                ops.qk_norm_rope(qkv[:n], A, D, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, self.cos, self.sin, 0, g.Sv,
                                 run_flag=flag, run_if=run_if)
                if St:
                    ops.qk_norm_rope(qkv[n:], A, D, W[f"{pt}.q_norm"], W[f"{pt}.k_norm"], eps, run_flag=flag,
                                     run_if=run_if)
            ops.attention(qkv, qkv[:, H:], qkv[:, 2 * H:], self._ob, A, D, workspace=self.attn_ws, run_flag=flag,
                          run_if=run_if)
            return
        sp, P, hl = self.sp, self.sp.P, self.hl
        rcv = self.a2a_rcv
        rs = 3 * hl * D  # row stride of the packed layouts
        if self.peer is not None:
            # fused exchange: QKV epilogue -> owners' input buffers, attention epilogue -> owners' O rows
            ops.gemm_qknorm_rope_scatter(m[:n], wi, self.qkv_dst, H, 2, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, rs,
                                         hl, bias=bi, cos=self.cos, sin=self.sin, rope_row0=sp.rank * n,
                                         rope_rows=g.Sv, run_flag=flag, run_if=run_if)
            if St:
                ops.gemm_qknorm_rope(m[n:], wt, rcv[g.Sv:].view(St, -1), H, 2, W[f"{pt}.q_norm"], W[f"{pt}.k_norm"],
                                     eps, bias=bt, out_row_stride=rs, groups=1, hpg=hl, g_base=sp.rank,
                                     run_flag=flag, run_if=run_if)
            self._barrier(flag, run_if)
            q = rcv.view(g.Sv + St, -1)
            ops.attention_scatter(q, q[:, hl * D:], q[:, 2 * hl * D:], self._odst, H, hl, D, n, g.Sv,
                                  workspace=self.attn_ws, run_flag=flag, run_if=run_if)
            self._barrier(flag, run_if)
            return
        snd = self.a2a_snd
        if fused:
            ops.gemm_qknorm_rope(m[:n], wi, snd, H, 2, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, bias=bi,
                                 cos=self.cos, sin=self.sin, rope_row0=sp.rank * n, rope_rows=g.Sv, out_row_stride=rs,
                                 groups=P, group_stride=n * rs, hpg=hl, run_flag=flag, run_if=run_if)
        else:
            ops.gemm(m[:n], wi, qkv[:n], bias=bi, run_flag=flag, run_if=run_if)
            ops.qk_norm_rope(qkv[:n], A, D, W[f"{pi}.q_norm"], W[f"{pi}.k_norm"], eps, self.cos, self.sin,
                             sp.rank * n, g.Sv, dst=snd, hpg=hl, dst_group_stride=n * rs, dst_row_stride=rs,
                             dst_which_stride=hl * D, run_flag=flag, run_if=run_if)
        sp.all_to_all(rcv[:g.Sv].view(-1), snd.view(-1))
        if St:
            tail = rcv[g.Sv:].view(St, -1)
            if fused:
                ops.gemm_qknorm_rope(m[n:], wt, tail, H, 2, W[f"{pt}.q_norm"], W[f"{pt}.k_norm"], eps, bias=bt,
                                     out_row_stride=rs, groups=1, hpg=hl, g_base=sp.rank, run_flag=flag,
                                     run_if=run_if)
            else:
                ops.gemm(m[n:], wt, qkv[n:], bias=bt, run_flag=flag, run_if=run_if)
                ops.qk_norm_rope(qkv[n:], A, D, W[f"{pt}.q_norm"], W[f"{pt}.k_norm"], eps, dst=tail,
                                 head_begin=sp.rank * hl, head_count=hl, hpg=hl, dst_row_stride=rs,
                                 dst_which_stride=hl * D, run_flag=flag, run_if=run_if)
        q = rcv.view(g.Sv + St, -1)
        ops.attention(q, q[:, hl * D:], q[:, 2 * hl * D:], self.oh, hl, D, workspace=self.attn_ws, run_flag=flag,
                      run_if=run_if)
        sp.all_to_all(self.ob.view(-1), self.oh[:g.Sv].reshape(-1))
        ops.heads_to_seq(self.ob, n, P, hl * D, self._ob[:n], run_flag=flag, run_if=run_if)
        if St:
            sp.all_gather(self.tg.view(-1), self.oh[g.Sv:].reshape(-1))
            ops.heads_to_seq(self.tg, St, P, hl * D, self._ob[n:], run_flag=flag, run_if=run_if)

    def _mlp(self, p, r0, r1, mods, flag, run_if):
        """x += gate2 * fc2(gelu(fc1(norm_mod(x, shift2, scale2))))  on rows [r0, r1)."""
        W, eps = self.W, self.cfg.norm_eps
        x, m, h = self.x[r0:r1], self.m[r0:r1], self.h[r0:r1]
        ops.norm_modulate(x, mods[3], mods[4], m, eps, run_flag=flag, run_if=run_if)
        ops.gemm(m, W[f"{p}.fc1.w"], h, bias=W[f"{p}.fc1.b"], epilogue="gelu", run_flag=flag, run_if=run_if)
        ops.gemm(h, W[f"{p}.fc2.w"], x, bias=W[f"{p}.fc2.b"], gate=mods[5], epilogue="gate_res", run_flag=flag,
                 run_if=run_if)

    # ----------------------------------------------------------------- blocks
    def _single_dit_block(self, i, flag, run_if, probe, ag):
        cfg, g, W = self.cfg, self.geo, self.W
        A, D, H, eps = cfg.num_heads, cfg.head_dim, cfg.hidden_size, cfg.norm_eps
        p = f"blocks.{i}"
        mods = self._mod(i)
        n = g.Sv_loc
        askip, aflag, arun = ag
        ops.norm_modulate(self.x, mods[0], mods[1], self.m, eps, probe_prev=self.prev if probe else None,
                          probe_partials=self.partials if probe else None, run_flag=flag, run_if=run_if)
        if probe:
            self._decide()
        if not askip:
            self._qkv_attention(p, None, aflag, arun)
        # the out-projection also writes bf16(x): the cross-attention q projection's input
        # (no norm before cross-attention, PixArt-α) without a separate cast pass
        ops.gemm(self._ob, W[f"{p}.proj.w"], self.x, bias=W[f"{p}.proj.b"], gate=mods[2], epilogue="gate_res",
                 aux=self.m, run_flag=flag, run_if=run_if)
        # cross-attention to the text; K/V precomputed per call
        xo = self._xo
        if not askip:
            if D == 128 and not self.fp32:  # q projection with the QK-RMSNorm fused in its epilogue
                ops.gemm_qknorm_rope(self.m, W[f"{p}.xq.w"], self.xq, H, 1, W[f"{p}.xq_norm"], None,
                                     cfg.qk_norm_eps, bias=W[f"{p}.xq.b"], run_flag=aflag, run_if=arun)
            else:
                ops.gemm(self.m, W[f"{p}.xq.w"], self.xq, bias=W[f"{p}.xq.b"], run_flag=aflag, run_if=arun)
                ops.qk_norm_rope(self.xq, A, D, W[f"{p}.xq_norm"], None, cfg.qk_norm_eps, parts=1, norm_parts=1,
                                 run_flag=aflag, run_if=arun)
            kv = self.text_kv[i]
            ops.attention(self.xq, kv, kv[:, H:], xo, A, D, workspace=self.attn_ws, run_flag=aflag, run_if=arun)
        ops.gemm(xo, W[f"{p}.xproj.w"], self.x, bias=W[f"{p}.xproj.b"], epilogue="gate_res", run_flag=flag,
                 run_if=run_if)
        self._mlp(p, 0, n, mods, flag, run_if)

    def _mm_dual_block(self, i, flag, run_if, probe, ag):
        cfg, g, W, eps = self.cfg, self.geo, self.W, self.cfg.norm_eps
        n, R = g.Sv_loc, g.rows
        pi, pt = f"dual.{i}.img", f"dual.{i}.txt"
        mi, mt = self._mod(f"{pi}.mod"), self._mod(f"{pt}.mod")
        askip, aflag, arun = ag
        if probe or not askip:
            ops.norm_modulate(self.x[:n], mi[0], mi[1], self.m[:n], eps, probe_prev=self.prev if probe else None,
                              probe_partials=self.partials if probe else None,
                              run_flag=flag if probe else aflag, run_if=run_if if probe else arun)
        if probe:
            self._decide()
        if not askip:
            ops.norm_modulate(self.x[n:], mt[0], mt[1], self.m[n:], eps, run_flag=aflag, run_if=arun)
            self._qkv_attention(pi, pt, aflag, arun)
        o = self._ob
        ops.gemm(o[:n], W[f"{pi}.proj.w"], self.x[:n], bias=W[f"{pi}.proj.b"], gate=mi[2], epilogue="gate_res",
                 run_flag=flag, run_if=run_if)
        ops.gemm(o[n:], W[f"{pt}.proj.w"], self.x[n:], bias=W[f"{pt}.proj.b"], gate=mt[2], epilogue="gate_res",
                 run_flag=flag, run_if=run_if)
        self._mlp(pi, 0, n, mi, flag, run_if)
        self._mlp(pt, n, R, mt, flag, run_if)

    def _mm_single_block(self, i, flag, run_if, probe, ag):
        cfg, g, W, eps = self.cfg, self.geo, self.W, self.cfg.norm_eps
        n, R = g.Sv_loc, g.rows
        p = f"single.{i}"
        md = self._mod(f"{p}.mod")
        askip, aflag, arun = ag
        if probe:
            ops.norm_modulate(self.x[:n], md[0], md[1], self.m[:n], eps, probe_prev=self.prev,
                              probe_partials=self.partials, run_flag=flag, run_if=run_if)
            self._decide()
            if not askip:
                ops.norm_modulate(self.x[n:], md[0], md[1], self.m[n:], eps, run_flag=aflag, run_if=arun)
        elif not askip:
            ops.norm_modulate(self.x, md[0], md[1], self.m, eps, run_flag=aflag, run_if=arun)
        if not askip:
            self._qkv_attention(p, p, aflag, arun)
        ops.gemm(self._ob, W[f"{p}.proj.w"], self.x, bias=W[f"{p}.proj.b"], gate=md[2], epilogue="gate_res",
                 run_flag=flag, run_if=run_if)
        self._mlp(p, 0, R, md, flag, run_if)

    def _block(self, i, flag, run_if, probe, ag=None):
        """Block i; ``ag`` = (skip, flag, run_if) of its attention part (attention-cache mode),
        default: same gate as the block."""
        cfg = self.cfg
        if ag is None:
            ag = (False, flag, run_if)
        self._bind_attention_output(i)
        if cfg.family == "single-dit":
            return self._single_dit_block(i, flag, run_if, probe, ag)
        if i < cfg.num_dual:
            return self._mm_dual_block(i, flag, run_if, probe, ag)
        return self._mm_single_block(i - cfg.num_dual, flag, run_if, probe, ag)

    def _bind_attention_output(self, i):
        """Where block i's attention output lives: the shared ``o`` buffer, or (attention-cache
        mode) block i's cache slot, which a cached step reads instead of recomputing."""
        if self.cache_mode == "attention-cache":
            self._ob = self.ocache[i]
            self._xo = self.xocache[i] if self.xocache is not None else None
            if self.peer is not None:
                g, H = self.geo, self.cfg.hidden_size
                self._odst = self.peer_ocache.ptrs("ocache", (i * g.rows * H + self.sp.rank * self.hl *
                                                               self.cfg.head_dim) * 2)
        else:
            self._ob, self._xo = self.o, self.o
            if self.peer is not None:
                self._odst = self.o_dst

    def _alloc_attention_cache(self):
        """Per-block attention-output slots [L, rows, H] (+ Single-DiT cross-attention [L, Sv_loc, H]).
        Under the p2p Ulysses exchange the slots are peer memory (collective allocation)."""
        if self.ocache is not None:
            return
        cfg, g, L, H = self.cfg, self.geo, self.cfg.num_layers, self.cfg.hidden_size
        if self.peer is not None:
            self.peer_ocache = PeerBuffers(self.sp, {"ocache": L * g.rows * H * 2}, self.device)
            self.ocache = self.peer_ocache.local("ocache", (L, g.rows, H), BF16)
        else:
            self.ocache = torch.zeros(L, g.rows, H, device=self.device, dtype=self.act)
        if cfg.family == "single-dit":
            self.xocache = torch.zeros(L, g.Sv_loc, H, device=self.device, dtype=self.act)

    # ------------------------------------------------------------------ steps
    def reset(self, x0: torch.Tensor, num_steps: int, policy=None, cache_mode: str = "dit-layer-cache",
              frame_offset: int | None = None, cached_cost_fraction: float | None = None):
        """Load the initial latent [C, T, H, W] and the Euler grid t_i = i/N.

        ``cache_mode``: ``dit-layer-cache`` (rear-block offset reuse) or
        ``attention-cache`` (per-block attention-output reuse).
        ``cached_cost_fraction``: the schedule's cost of a cached step (``inference.py:77``);
        under ``dit-layer-cache`` a cached step runs the front ``ceil(fraction·L)`` blocks, so
        the split follows the schedule the caller passes (default: the constructor's).
        ``frame_offset``: ``x0`` is a longer latent and this model's clip starts at that
        latent frame (temporal MultiDiffusion)."""
        cfg, g = self.cfg, self.geo
        if g is None:
            raise ConfigError("call prepare() first", "model")
        if cache_mode not in ("dit-layer-cache", "attention-cache"):
            raise ConfigError("unknown cache mode", "cache.mode")
        self.cache_mode = cache_mode
        if cached_cost_fraction is not None:
            self.n_front = front_block_count(cfg.num_layers, cached_cost_fraction)
        if cache_mode == "attention-cache":
            self._alloc_attention_cache()
        C = cfg.latent_channels
        pt, ph, pw = cfg.patch
        exp = (C, g.grid[0] * pt, g.grid[1] * ph, g.grid[2] * pw)
        shape = tuple(x0.shape)
        if frame_offset is None:
            if shape != exp:
                raise ConfigError(f"latent must be {exp}, got {shape}", "inputs.x0")
        elif (len(shape) != 4 or shape[0] != C or shape[2:] != exp[2:] or frame_offset < 0
              or frame_offset + exp[1] > shape[1]):
            raise ConfigError(f"clip {exp} at frame {frame_offset} does not fit latent {shape}", "inputs.x0")
        dev = self.device
        self.load_latent(x0.to(dev, F32, non_blocking=True).contiguous(), frame_offset or 0)
        if getattr(self, "num_steps", None) != num_steps:
            # (re)allocate the per-step tables; captured CUDA graphs hold their addresses,
            # so a new step count starts a new graph generation
            self.num_steps = num_steps
            self.ts = torch.empty(num_steps, device=dev, dtype=F32)
            self.dts = torch.empty(num_steps, device=dev, dtype=F32)
            self.flags_out = torch.empty(num_steps, device=dev, dtype=torch.int32)
            self.rels_out = torch.empty(num_steps, device=dev, dtype=F32)
            self.generation = getattr(self, "generation", 0) + 1
        self.ts.copy_(torch.arange(num_steps, device=dev, dtype=torch.float64).div(num_steps))
        self.dts.fill_(1.0 / num_steps)
        self.flags_out.zero_()
        self.rels_out.zero_()
        self.idx.zero_()
        self.cstate.zero_()
        self.prev.zero_()
        self.policy = policy

    def load_latent(self, lat: torch.Tensor, frame_offset: int = 0):
        """Set the denoise state from latent frames [frame_offset, +T*pt) of ``lat`` (f32
        [C, Tl, H, W] on this device) — one patchify kernel (+ this rank's token slice)."""
        cfg, g = self.cfg, self.geo
        if self.sp is None or self.sp.P == 1:
            ops.patchify(lat, self.lat, self.lat_bf if not self.fp32 else None, g.grid, cfg.patch, frame_offset)
            if self.fp32:
                self.lat_bf.copy_(self.lat)
            return
        full_tok = torch.empty(g.Sv, cfg.patch_dim, device=self.device, dtype=F32)
        ops.patchify(lat, full_tok, None, g.grid, cfg.patch, frame_offset)
        r = self.sp.rank
        self.lat.copy_(full_tok[r * g.Sv_loc:(r + 1) * g.Sv_loc])
        self.lat_bf.copy_(self.lat)

    def fork(self):
        """A second denoise context sharing this model's weights (its own activations, cache
        state and step tables) — one per temporal-MultiDiffusion clip."""
        import copy

        if self.geo is None:
            raise ConfigError("call prepare() first", "model")
        twin = copy.copy(self)
        for a in ("num_steps", "ts", "dts", "flags_out", "rels_out", "peer_ocache"):
            twin.__dict__.pop(a, None)
        twin.generation = 0
        return twin.prepare(self.geo.grid, self._text, self._pooled)

    def _decide(self):
        pol = self.policy
        ops.rel_l1_reduce(self.partials, self.geo.Sv_loc, self.sums)
        if self.peer is not None:
            self._barrier(payload=self.sums)  # sums over ranks, rank order, identical everywhere
        elif self.sp is not None and self.sp.P > 1:
            self.sp.all_reduce_sum(self.sums)
        ops.cache_decide(self.sums, self.cstate, pol.threshold, pol.warmup, self.num_steps, pol.force_last,
                         self.flags_out, self.rels_out)

    def _embed(self):
        cfg, W, g = self.cfg, self.W, self.geo
        ops.step_scalars(self.ts, self.dts, self.idx, self.cur)
        t = self.cur[0:1]
        ops.gemv(W["t_emb.fc1.w"], None, self.th, bias=W["t_emb.fc1.b"], t=t)
        if cfg.family == "single-dit":
            ops.gemv(W["t_emb.fc2.w"], self.th, self.t0, bias=W["t_emb.fc2.b"], in_silu=True)
            ops.gemv(W["t_block.w"], self.t0, self.tmod, bias=W["t_block.b"], in_silu=True)
            ops.add_bcast(self.mods.view(-1), self.tmod, self.tables.view(-1))
            ops.add_bcast(self.fmods, self.t0, W["final.table"])
        else:
            ops.gemv(W["t_emb.fc2.w"], self.th, self.vec, bias=W["t_emb.fc2.b"], add=self.pe, in_silu=True)
            self._adaln_gemv()
        n = g.Sv_loc
        ops.gemm(self.lat_bf, W["x_emb.w"], self.x[:n], bias=W["x_emb.b"], epilogue="f32")
        if g.St:
            self.x[n:].copy_(self.txt0)

    def _adaln_gemv(self):
        """Every block's AdaLN-zero modulation (MM-DiT) in one GEMV over the stacked regressors."""
        ops.gemv(self.mod_w, self.vec, self.allmods, bias=self.mod_b, in_silu=True)

    def _final(self):
        cfg, W, g = self.cfg, self.W, self.geo
        n, H = g.Sv_loc, cfg.hidden_size
        if cfg.family == "single-dit":
            shift, scale = self.fmods[:H], self.fmods[H:]
        else:
            shift, scale = self._mod("final.mod")
        ops.norm_modulate(self.x[:n], shift, scale, self.m[:n], cfg.norm_eps)
        ops.gemm(self.m[:n], W["final.w"], self.lat, bias=W["final.b"], epilogue="euler", alpha=self.cur[1:2],
                 aux=self.lat_bf)
        ops.step_scalars(self.ts, self.dts, self.idx, self.cur, advance=True)

    def step(self, mode: str = "full", use_cache: bool = True):
        """Issue one denoise step (velocity + Euler update) on the current stream.

        mode: ``full`` | ``cached`` (host-decided, static schedule) |
        ``dynamic`` (device-decided with the rel-L1 policy set in reset()).
        ``use_cache=False`` skips the offset bookkeeping (schedule without cached steps).
        """
        cfg = self.cfg
        L, nf = cfg.num_layers, self.n_front
        dyn = mode == "dynamic"
        flag = self.flag if dyn else None
        if self.cache_mode == "attention-cache":
            # every block runs; only its attention part is skipped (static) or gated (dynamic)
            self._embed()
            ag = (mode == "cached", flag, 1)
            for i in range(L):
                self._block(i, None, 1, probe=(dyn and i == 0), ag=ag)
            self._final()
            return
        xi = self.x[:self.geo.Sv_loc]
        self._embed()
        cache = use_cache and nf < L
        for i in range(L):
            if i == nf and cache:
                if mode == "cached":
                    ops.cache_offset(xi, self.off, 2)
                    break
                if dyn:
                    ops.cache_offset(xi, self.off, 2, run_flag=flag, run_if=0)
                ops.cache_offset(xi, self.off, 0, run_flag=flag, run_if=1)
            rear = i >= nf
            self._block(i, flag if (dyn and rear) else None, 1, probe=(dyn and i == 0))
        if cache and mode != "cached":
            ops.cache_offset(xi, self.off, 1, run_flag=flag, run_if=1)
        self._final()

    def latent(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """Current latent [C, T, H, W] (gathered over Ulysses ranks), optionally into ``out``."""
        cfg, g = self.cfg, self.geo
        tok = self.lat
        if self.sp is not None and self.sp.P > 1:
            full = torch.empty(g.Sv, cfg.patch_dim, device=self.device, dtype=F32)
            self.sp.all_gather(full.view(-1), self.lat.view(-1))
            tok = full
        pt, ph, pw = cfg.patch
        if out is None:
            out = torch.empty(cfg.latent_channels, g.grid[0] * pt, g.grid[1] * ph, g.grid[2] * pw,
                              device=self.device, dtype=F32)
        ops.unpatchify(tok, out, g.grid, cfg.patch)
        return out


class SingleDiT(DiTModel):
    """Aquarius Single-DiT (2B): AdaLN-single + cross-attention."""

    def __init__(self, cfg: DiTConfig, **kw):
        if cfg.family != "single-dit":
            raise ConfigError("SingleDiT needs a single-dit config", "model.family")
        super().__init__(cfg, **kw)


class MMDiT(DiTModel):
    """Aquarius Multimodal-DiT (13.4B): dual-stream then joint blocks."""

    def __init__(self, cfg: DiTConfig, **kw):
        if cfg.family != "mm-dit":
            raise ConfigError("MMDiT needs an mm-dit config", "model.family")
        super().__init__(cfg, **kw)


class _TensorParallel:
    """TP-SP machinery shared by both families (:class:`~paper_2505_10584_b200.parallel.TensorSP`).

    Weights are sharded at construction (:func:`~paper_2505_10584_b200.parallel.tp_shard`):
    QKV / FFN1 (and Single-DiT's cross-attention q and text K/V) by output rows — this
    rank's A/P heads and F/P hidden columns — and the out / FFN2 (/ cross-out) projections
    by input columns, their bias on rank 0 only.  AdaLN, timestep / pooled MLPs, patch
    embed and final layer are replicated.  Each sub-layer is

      AG(LN+mod of this rank's video rows) -> column-parallel GEMM(s) on all rows
      [-> attention over the local heads]  -> row-parallel GEMM -> RS into x

    with the all-gather stored by the LN kernel into every rank (``aqb_norm_modulate_gather``),
    the reduce-scatter reduce-added by the GEMM epilogue into the owners' rows
    (``aqb_gemm_gate_add_scatter``), and an ``aqb_peer_barrier`` after each.  The video
    rows' reduce-scatter sums f32 partials at the owner in arrival order, so a run is
    reproducible to rounding, not bitwise (unlike the Ulysses path).
    """

    def _tp_setup(self, cfg, sp, kw):
        if sp is None or not getattr(sp, "tensor_parallel", False):
            raise ConfigError("a TP-SP model needs a TensorSP group", "parallel.tp")
        if kw.get("precision", "bf16") != "bf16":
            raise ConfigError("TP-SP runs the bf16 product path", "model.precision")
        if cfg.head_dim != 128:
            raise ConfigError("TP-SP needs head_dim 128 (fused QK-norm epilogue)", "parallel.tp")

    def _tp_shard(self):
        self.W = tp_shard(self.W, self.cfg, self.sp.P, self.sp.rank)
        torch.cuda.empty_cache()

    def _embed(self):
        super()._embed()
        if self.cache_mode == "attention-cache":
            # a cached step's block 0 starts with a reduce-scatter into the peers' residual
            # rows, with no all-gather (and its barrier) before it: without this barrier a
            # rank could add into a peer's x before the peer has finished reading the last
            # step's x (final layer) and re-embedding it (patch-embed GEMM overwrites x)
            self._barrier()

    def _bind_attention_output(self, i):
        """Block i's local-head attention outputs (full sequence): the shared buffers, or under
        ``attention-cache`` block i's slots, which a cached step feeds to the row-parallel
        projections instead of recomputing QKV + attention."""
        if self.cache_mode == "attention-cache":
            self._o_tp = self.ocache[i]
            self._xo_tp = self.xocache[i] if self.xocache is not None else None
        else:
            self._o_tp = self.o_full
            self._xo_tp = getattr(self, "xo_full", None)

    def _alloc_attention_cache(self):
        """Per-block slots of this rank's heads over the full sequence: [L, S_v + S_t, A/P·D]
        (+ Single-DiT cross-attention [L, S_v, A/P·D]); rank-local, no peer memory."""
        if self.ocache is not None:
            return
        cfg, g, L = self.cfg, self.geo, self.cfg.num_layers
        hd = self.hl * cfg.head_dim
        self.ocache = torch.zeros(L, g.Sv + g.St, hd, device=self.device, dtype=BF16)
        if cfg.family == "single-dit":
            self.xocache = torch.zeros(L, g.Sv, hd, device=self.device, dtype=BF16)

    def _rs(self, a, name, gate, flag, run_if, barrier=True):
        """Row-parallel projection of video rows: this rank's partial reduce-added into the
        owners' residual rows."""
        W = self.W
        ops.gemm_gate_add_scatter(a, W[f"{name}.w"], self.x_dst, self.cfg.hidden_size, self.geo.Sv_loc,
                                  bias=W[f"{name}.b"], gate=gate, run_flag=flag, run_if=run_if)
        if barrier:
            self._barrier(flag, run_if)

    def _ag(self, shift, scale, kind, flag, run_if, probe=False, local=None):
        """Sequence-parallel LN + modulation (or cast, kind 2) of this rank's video rows into
        every rank's ``mg``; ``local`` = (shift, scale) of the replicated text rows, normalised
        in place by each rank (MM-DiT)."""
        n, H = self.geo.Sv_loc, self.cfg.hidden_size
        ops.norm_modulate_gather(self.x[:n], shift, scale, self.mg_dst, H, self.cfg.norm_eps, kind=kind,
                                 probe_prev=self.prev if probe else None,
                                 probe_partials=self.partials if probe else None, run_flag=flag, run_if=run_if)
        if local is not None:
            ops.norm_modulate(self.x[n:], local[0], local[1], self.mg[self.geo.Sv:], self.cfg.norm_eps,
                              run_flag=flag, run_if=run_if)
        if probe:
            self._decide()  # its barrier (carrying the rel-L1 sums) also completes the gather
        else:
            self._barrier(flag, run_if)

    def _tp_peer(self, extra: dict):
        """Symmetric buffers: the gathered modulated input ``mg`` (every rank stores its video
        rows into every copy) and the residual ``x`` (every rank reduce-adds its partials into
        the owner's rows), + ``extra``."""
        cfg, g, dev = self.cfg, self.geo, self.device
        H = cfg.hidden_size
        self.sp.check(cfg.num_heads, g.Sv, cfg.ffn_dim)
        S, n, St = g.Sv, g.Sv_loc, g.St
        sizes = {"mg": (S + St) * H * 2, "x": (n + St) * H * 4, "sig": SIGNAL_BYTES}
        sizes.update(extra)
        self.peer = PeerBuffers(self.sp, sizes, dev)
        self.mg = self.peer.local("mg", (S + St, H), BF16)
        self.x = self.peer.local("x", (n + St, H), F32)
        self.mg_dst = self.peer.ptrs("mg", self.sp.rank * n * H * 2)
        self.x_dst = self.peer.ptrs("x")
        self.sig = self.peer.ptrs("sig")
        self.epoch = torch.zeros(1, device=dev, dtype=torch.int32)
        self.peer_status = torch.zeros(1, device=dev, dtype=torch.int32)
        e = lambda *s_, dt=BF16: torch.empty(*s_, device=dev, dtype=dt)  # noqa: E731
        hd = self.hl * cfg.head_dim
        self.qkv_full = e(S + St, 3 * hd)
        self.o_full = e(S + St, hd)
        self.h_full = e(S + St, cfg.ffn_dim // self.sp.P)
        self.h = self.h[:0]  # the unsharded buffers are unused under TP
        self.qkv = self.qkv[:0]
        return e


class SingleDiTTP(_TensorParallel, SingleDiT):
    """Single-DiT under TP-SP.  Per block, six sub-steps each end in a peer barrier:

      AG(LN+mod(x))  -> QKV(local heads, all rows) -> attention -> proj  -> RS into x
      AG(bf16 x)     -> q(local heads) -> cross-attention to text -> proj -> RS into x
      AG(LN+mod(x))  -> FFN1(local columns, GeLU) -> FFN2 -> RS into x
    """

    def __init__(self, cfg: DiTConfig, sp=None, **kw):
        self._tp_setup(cfg, sp, kw)
        super().__init__(cfg, sp=sp, **kw)
        self._tp_shard()

    def _prepare_tp(self):
        e = self._tp_peer({})
        hd = self.hl * self.cfg.head_dim
        self.xq_full = e(self.geo.Sv, hd)
        self.xo_full = e(self.geo.Sv, hd)

    def _single_dit_block(self, i, flag, run_if, probe, ag):
        cfg, g, W = self.cfg, self.geo, self.W
        D, eps, hl = cfg.head_dim, cfg.qk_norm_eps, self.hl
        hd = hl * D
        p = f"blocks.{i}"
        mods = self._mod(i)
        S = g.Sv
        askip, aflag, arun = ag  # attention-cache: skip (static) / gate (dynamic) the attention parts
        # self-attention: local heads over the whole sequence
        if probe:
            self._ag(mods[0], mods[1], 0, flag, run_if, probe=True)
        elif not askip:
            self._ag(mods[0], mods[1], 0, aflag, arun)
        if not askip:
            ops.gemm_qknorm_rope(self.mg, W[f"{p}.qkv.w"], self.qkv_full, hd, 2, W[f"{p}.q_norm"], W[f"{p}.k_norm"],
                                 eps, bias=W[f"{p}.qkv.b"], cos=self.cos, sin=self.sin, rope_row0=0, rope_rows=S,
                                 run_flag=aflag, run_if=arun)
            q = self.qkv_full
            ops.attention(q, q[:, hd:], q[:, 2 * hd:], self._o_tp, hl, D, workspace=self.attn_ws, run_flag=aflag,
                          run_if=arun)
        self._rs(self._o_tp, f"{p}.proj", mods[2], flag, run_if)
        # cross-attention to the text (no norm before it, PixArt-alpha): gather bf16(x)
        if not askip:
            self._ag(None, None, 2, aflag, arun)
            ops.gemm_qknorm_rope(self.mg, W[f"{p}.xq.w"], self.xq_full, hd, 1, W[f"{p}.xq_norm"], None, eps,
                                 bias=W[f"{p}.xq.b"], run_flag=aflag, run_if=arun)
            kv = self.text_kv[i]
            ops.attention(self.xq_full, kv, kv[:, hd:], self._xo_tp, hl, D, workspace=self.attn_ws, run_flag=aflag,
                          run_if=arun)
        self._rs(self._xo_tp, f"{p}.xproj", None, flag, run_if)
        # MLP: F/P hidden columns per rank
        self._ag(mods[3], mods[4], 0, flag, run_if)
        ops.gemm(self.mg, W[f"{p}.fc1.w"], self.h_full, bias=W[f"{p}.fc1.b"], epilogue="gelu", run_flag=flag,
                 run_if=run_if)
        self._rs(self.h_full, f"{p}.fc2", mods[5], flag, run_if)


class MMDiTTP(_TensorParallel, MMDiT):
    """MM-DiT under TP-SP — the paper's own inference layout for the 13.4B model
    (``PAPER.md:191,197,320``).  Video rows are sequence-sharded as for Single-DiT; the
    256 text rows are replicated on every rank (their LN runs locally, their
    row-parallel projections are all-reduced deterministically: gate·partial into every
    rank's slot, then a rank-ordered sum).  Dual blocks use the per-stream weights on the
    two row ranges; joint attention runs over video + text rows for the local heads.
    Per block, four sub-steps each end in a peer barrier (AG → QKV → attention → RS, AG →
    FFN1 → FFN2 → RS)."""

    def __init__(self, cfg: DiTConfig, sp=None, **kw):
        self._tp_setup(cfg, sp, kw)
        super().__init__(cfg, sp=sp, **kw)
        self._tp_shard()
        # AdaLN regressors column-parallel: this rank keeps 1/P of the stacked
        # [sum 6H, H] output rows (~4.5B parameters at 13.4B dims) and all-gathers the
        # modulation vectors each step
        P, r = sp.P, sp.rank
        self.mod_rows = self.mod_w.shape[0]
        if self.mod_rows % (4 * P):
            raise ConfigError(f"AdaLN rows {self.mod_rows} not divisible into {P} float4 shards", "parallel.tp")
        per = self.mod_rows // P
        self.mod_w = self.mod_w[r * per:(r + 1) * per].contiguous()
        self.mod_b = self.mod_b[r * per:(r + 1) * per].contiguous()
        torch.cuda.empty_cache()

    def _prepare_tp(self):
        g, H = self.geo, self.cfg.hidden_size
        P, St = self.sp.P, g.St
        per = self.mod_rows // P
        e = self._tp_peer({"tslot": P * St * H * 4, "mods": self.mod_rows * 4})
        self.tslot = self.peer.local("tslot", (P, St, H), F32)
        self.tslot_dst = self.peer.ptrs("tslot", self.sp.rank * St * H * 4)
        self.tpart = e(St, H, dt=F32)
        self.allmods = self.peer.local("mods", (self.mod_rows,), F32)
        self.mods_dst = self.peer.ptrs("mods", self.sp.rank * per * 4)
        self.mods_part = e(1, per, dt=F32)

    def _adaln_gemv(self):
        """This rank's slice of the AdaLN outputs, stored into every rank's ``allmods``: the
        all-gather of the column-parallel AdaLN Linear.  The first barrier keeps a rank from
        overwriting a peer's vectors while the peer still reads the previous step's (its final
        layer runs after the last block barrier); the second publishes the new ones."""
        self._barrier()
        ops.gemv(self.mod_w, self.vec, self.mods_part.view(-1), bias=self.mod_b, in_silu=True)
        ops.gate_bcast(self.mods_part, None, self.mods_dst, self.mods_part.shape[1])
        self._barrier()

    def _text_rs(self, a, name, gate, flag, run_if):
        """Row-parallel projection of the replicated text rows: f32 partial, gate·partial into
        this rank's slot on every rank (the barrier follows in the caller)."""
        W = self.W
        ops.gemm(a, W[f"{name}.w"], self.tpart, bias=W[f"{name}.b"], epilogue="f32", run_flag=flag, run_if=run_if)
        ops.gate_bcast(self.tpart, gate, self.tslot_dst, self.cfg.hidden_size, run_flag=flag, run_if=run_if)

    def _tp_block(self, pv, pt, mv, mt, flag, run_if, probe, ag):
        cfg, g, W = self.cfg, self.geo, self.W
        D, eps, hl = cfg.head_dim, cfg.qk_norm_eps, self.hl
        hd = hl * D
        S, n = g.Sv, g.Sv_loc
        askip, aflag, arun = ag  # attention-cache: skip (static) / gate (dynamic) the attention part
        # joint attention over video + text rows, local heads
        if probe:
            self._ag(mv[0], mv[1], 0, flag, run_if, probe=True, local=(mt[0], mt[1]))
        elif not askip:
            self._ag(mv[0], mv[1], 0, aflag, arun, local=(mt[0], mt[1]))
        if not askip:
            if pv == pt:
                ops.gemm_qknorm_rope(self.mg, W[f"{pv}.qkv.w"], self.qkv_full, hd, 2, W[f"{pv}.q_norm"],
                                     W[f"{pv}.k_norm"], eps, bias=W[f"{pv}.qkv.b"], cos=self.cos, sin=self.sin,
                                     rope_row0=0, rope_rows=S, run_flag=aflag, run_if=arun)
            else:
                ops.gemm_qknorm_rope(self.mg[:S], W[f"{pv}.qkv.w"], self.qkv_full[:S], hd, 2, W[f"{pv}.q_norm"],
                                     W[f"{pv}.k_norm"], eps, bias=W[f"{pv}.qkv.b"], cos=self.cos, sin=self.sin,
                                     rope_row0=0, rope_rows=S, run_flag=aflag, run_if=arun)
                ops.gemm_qknorm_rope(self.mg[S:], W[f"{pt}.qkv.w"], self.qkv_full[S:], hd, 2, W[f"{pt}.q_norm"],
                                     W[f"{pt}.k_norm"], eps, bias=W[f"{pt}.qkv.b"], run_flag=aflag, run_if=arun)
            q = self.qkv_full
            ops.attention(q, q[:, hd:], q[:, 2 * hd:], self._o_tp, hl, D, workspace=self.attn_ws, run_flag=aflag,
                          run_if=arun)
        self._rs(self._o_tp[:S], f"{pv}.proj", mv[2], flag, run_if, barrier=False)
        self._text_rs(self._o_tp[S:], f"{pt}.proj", mt[2], flag, run_if)
        self._barrier(flag, run_if)
        ops.sum_slots(self.x[n:], self.tslot, run_flag=flag, run_if=run_if)
        # MLP
        self._ag(mv[3], mv[4], 0, flag, run_if, local=(mt[3], mt[4]))
        if pv == pt:
            ops.gemm(self.mg, W[f"{pv}.fc1.w"], self.h_full, bias=W[f"{pv}.fc1.b"], epilogue="gelu", run_flag=flag,
                     run_if=run_if)
        else:
            ops.gemm(self.mg[:S], W[f"{pv}.fc1.w"], self.h_full[:S], bias=W[f"{pv}.fc1.b"], epilogue="gelu",
                     run_flag=flag, run_if=run_if)
            ops.gemm(self.mg[S:], W[f"{pt}.fc1.w"], self.h_full[S:], bias=W[f"{pt}.fc1.b"], epilogue="gelu",
                     run_flag=flag, run_if=run_if)
        self._rs(self.h_full[:S], f"{pv}.fc2", mv[5], flag, run_if, barrier=False)
        self._text_rs(self.h_full[S:], f"{pt}.fc2", mt[5], flag, run_if)
        self._barrier(flag, run_if)
        ops.sum_slots(self.x[n:], self.tslot, run_flag=flag, run_if=run_if)

    def _mm_dual_block(self, i, flag, run_if, probe, ag):
        pi, pt = f"dual.{i}.img", f"dual.{i}.txt"
        self._tp_block(pi, pt, self._mod(f"{pi}.mod"), self._mod(f"{pt}.mod"), flag, run_if, probe, ag)

    def _mm_single_block(self, i, flag, run_if, probe, ag):
        p = f"single.{i}"
        md = self._mod(f"{p}.mod")
        self._tp_block(p, p, md, md, flag, run_if, probe, ag)


def build_model(cfg: DiTConfig, **kw) -> DiTModel:
    sp = kw.get("sp")
    if sp is not None and getattr(sp, "tensor_parallel", False):
        return (SingleDiTTP if cfg.family == "single-dit" else MMDiTTP)(cfg, **kw)
    return (SingleDiT if cfg.family == "single-dit" else MMDiT)(cfg, **kw)
