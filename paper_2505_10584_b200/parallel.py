"""Ulysses sequence parallelism (one process per GPU, NCCL over NVLink).

The north_star's multi-GPU path: video tokens are sharded S_v/P per rank for
every token-wise op; around attention an all-to-all swaps the sequence shard
for a head shard (A/P heads over the full sequence) and back
(``PAPER.md:193`` describes the same exchange as the paper's CP for >200k
tokens; the reference only costs it, ``comm.py:65-96``).  Text tokens are
replicated on every rank (their head slice is taken locally; their
attention output is all-gathered).  The rel-L1 cache decision all-reduces two
scalars so every rank takes the same branch.

Two exchange implementations:

* ``p2p`` (default): no collective on the data path.  :class:`PeerBuffers`
  allocates the attention-input and attention-output buffers in libaqb and
  maps every rank's copy into every process (CUDA IPC over NVLink/NVSwitch);
  the QKV-GEMM epilogue stores each head group straight into its owner's
  input buffer, the attention epilogue stores each output row straight into
  its owner's O buffer, and a device barrier kernel (``aqb_peer_barrier``)
  orders them.  The rel-L1 sums ride on that barrier.
* ``nccl``: ``all_to_all_single`` / ``all_gather`` between a packing epilogue
  and ``aqb_heads_to_seq`` (kept as the measured baseline).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import _native
from .errors import ConfigError, NativeError


EXCHANGES = ("p2p", "nccl")
PEER_MAX_RANKS = 8          # one NVSwitch box
IPC_HANDLE_BYTES = 64       # AQB_IPC_HANDLE_BYTES
SIGNAL_BYTES = 512          # AQB_PEER_SIGNAL_BYTES


class Ulysses:
    """Sequence-parallel group context (``P`` ranks, this rank ``rank``)."""

    tensor_parallel = False

    def __init__(self, group=None, exchange: str | None = None):
        if not dist.is_initialized():
            raise ConfigError("torch.distributed is not initialised", "parallel.group")
        self.group = group if group is not None else dist.group.WORLD
        self.P = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if exchange is None:
            exchange = os.environ.get("AQB_ULYSSES", "p2p")
        if exchange not in EXCHANGES:
            raise ConfigError(f"exchange must be one of {EXCHANGES}", "parallel.exchange")
        if exchange == "p2p" and self.P > PEER_MAX_RANKS:
            raise ConfigError(f"p2p exchange supports up to {PEER_MAX_RANKS} ranks", "parallel.exchange")
        self.exchange = exchange

    def check(self, num_heads: int, video_tokens: int):
        if num_heads % self.P:
            raise ConfigError(f"num_heads {num_heads} not divisible by {self.P} ranks", "parallel.ulysses")
        if video_tokens % self.P:
            raise ConfigError(f"video tokens {video_tokens} not divisible by {self.P} ranks", "parallel.ulysses")

    def _host_staged(self, t: torch.Tensor) -> bool:
        # gloo (the oversubscribed correctness mode) only reduces/gathers host tensors
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor):
        if self._host_staged(out):
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), group=self.group)
            out.copy_(o)
            return
        dist.all_to_all_single(out, inp, group=self.group)

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        if self._host_staged(out):
            parts = [torch.empty_like(inp, device="cpu") for _ in range(self.P)]
            dist.all_gather(parts, inp.cpu(), group=self.group)
            out.copy_(torch.cat(parts).view_as(out))
            return
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce_sum(self, t: torch.Tensor):
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            return
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)


class TensorSP(Ulysses):
    """TP-SP group (the paper's intra-node inference parallelism, ``PAPER.md:191,197,320``;
    the reference only costs it, ``comm.py:28-53``).

    Megatron-style tensor parallelism with sequence-parallel norms: the residual
    stream stays sharded by video rows (S_v/P per rank, as under Ulysses); each
    rank holds A/P heads of the QKV / cross-attention projections and F/P columns of
    FFN1 (column-parallel) and the matching input columns of the out / FFN2
    projections (row-parallel).  Per sub-layer: the sequence-parallel LayerNorm +
    modulation stores its rows into every rank's gathered input (the all-gather is
    the kernel's own NVLink stores, ``aqb_norm_modulate_gather``); the column-parallel
    GEMM and attention run on the full sequence for the local heads; the row-parallel
    GEMM's epilogue reduce-adds its partial straight into the owning rank's residual
    rows (the reduce-scatter, ``aqb_gemm_gate_add_scatter``).  ``aqb_peer_barrier``
    orders the steps.  No collective runs on the data path.  MM-DiT text rows (replicated on
    every rank) are all-reduced deterministically: each rank stores gate·partial into its
    slot of every rank's slot buffer (``aqb_gate_bcast``) and every rank sums the slots in
    rank order (``aqb_sum_slots``).
    """

    tensor_parallel = True

    def __init__(self, group=None):
        super().__init__(group, exchange="p2p")

    def check(self, num_heads: int, video_tokens: int, ffn_dim: int | None = None):
        super().check(num_heads, video_tokens)
        if ffn_dim is not None and ffn_dim % (8 * self.P):
            raise ConfigError(f"ffn_dim {ffn_dim} not divisible into {self.P} x 8-column shards", "parallel.tp")


def _tp_rows(t, parts, width, P, rank):
    """Rows [k*width*P + rank*width, +width) of each of ``parts`` parts (column-parallel slice)."""
    return torch.cat([t[k * width * P + rank * width:k * width * P + (rank + 1) * width]
                      for k in range(parts)]).contiguous()


def _tp_stream(out: dict, W: dict, p: str, P: int, rank: int, hd: int, fl: int, cross: bool = False):
    """Slice one attention+MLP stream ``p``: qkv / fc1 (and Single-DiT's xq / xkv) by output
    rows, proj / fc2 (and xproj) by input columns with the bias on rank 0 only."""
    col_parallel = [("qkv", 3, hd), ("fc1", 1, fl)] + ([("xq", 1, hd), ("xkv", 2, hd)] if cross else [])
    row_parallel = [("proj", hd), ("fc2", fl)] + ([("xproj", hd)] if cross else [])
    for name, parts, width in col_parallel:
        out[f"{p}.{name}.w"] = _tp_rows(W[f"{p}.{name}.w"], parts, width, P, rank)
        out[f"{p}.{name}.b"] = _tp_rows(W[f"{p}.{name}.b"], parts, width, P, rank)
    for name, width in row_parallel:
        out[f"{p}.{name}.w"] = W[f"{p}.{name}.w"][:, rank * width:(rank + 1) * width].contiguous()
        out[f"{p}.{name}.b"] = W[f"{p}.{name}.b"] if rank == 0 else None


def tp_shard(W: dict, cfg, P: int, rank: int) -> dict:
    """This rank's TP-SP slice of a weight dict (other entries shared, not copied).

    Column-parallel (output rows): ``qkv`` (q, k, v parts: heads [rank*A/P, (rank+1)*A/P)),
    ``fc1`` (hidden columns [rank*F/P, ...)), Single-DiT's ``xq`` and ``xkv`` (k, v parts).
    Row-parallel (input columns): ``proj``, ``fc2``, ``xproj``; their bias only on rank 0
    (``None`` elsewhere: the reduce adds it once).  MM-DiT: every dual-block stream
    (``dual.i.img`` / ``dual.i.txt``) and every single block."""
    if cfg.num_heads % P or cfg.ffn_dim % P:
        raise ConfigError(f"heads {cfg.num_heads} / ffn {cfg.ffn_dim} not divisible by {P}", "parallel.tp")
    if not 0 <= rank < P:
        raise ConfigError(f"rank {rank} outside [0, {P})", "parallel.rank")
    hd = (cfg.num_heads // P) * cfg.head_dim
    fl = cfg.ffn_dim // P
    out = dict(W)
    if cfg.family == "single-dit":
        for i in range(cfg.num_single):
            _tp_stream(out, W, f"blocks.{i}", P, rank, hd, fl, cross=True)
    else:
        for i in range(cfg.num_dual):
            for st in ("img", "txt"):
                _tp_stream(out, W, f"dual.{i}.{st}", P, rank, hd, fl)
        for i in range(cfg.num_single):
            _tp_stream(out, W, f"single.{i}", P, rank, hd, fl)
    return out


def tp_shard_single_dit(W: dict, cfg, P: int, rank: int) -> dict:
    """:func:`tp_shard` for a Single-DiT (kept for callers of the first TP-SP release)."""
    return tp_shard(W, cfg, P, rank)


def oversubscribed() -> bool:
    """``AQB_OVERSUBSCRIBE=1``: more ranks than GPUs (e.g. P=8 on 2 GPUs), a correctness-only mode.

    Ranks share GPUs round-robin and the process group is gloo (NCCL refuses two ranks
    on one device).  The fused p2p exchange is unchanged — CUDA IPC maps a peer's
    buffer whether it lives on another GPU or on the same one — so the P-rank data
    path (head/row partition, scatter maps, barrier, split-KV choice) runs exactly as on
    P GPUs, only time-sliced."""
    return os.environ.get("AQB_OVERSUBSCRIBE", "0") == "1"


def local_device_index() -> int:
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if oversubscribed() and torch.cuda.is_available():
        return local % torch.cuda.device_count()
    return local


def init_from_env(backend: str | None = None):
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous)."""
    if dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if oversubscribed():
        backend = "gloo"
    if torch.cuda.is_available():
        torch.cuda.set_device(local_device_index())
    dist.init_process_group(backend=backend)


def exchange_offsets(rank: int, P: int, rows_per_rank: int, heads_per_rank: int, head_dim: int, hidden: int,
                     elem_bytes: int = 2) -> dict:
    """Byte offsets this rank adds to every peer's base pointer for the fused exchange.

    * ``qkv``: into each peer's attention input ``[S_v + S_t, 3, A/P, D]`` — this rank's
      video rows start at row ``rank * S_v/P`` (row stride ``3·(A/P)·D``);
    * ``o``: into each peer's attention output ``[S_v/P + S_t, H]`` — this rank's heads
      are columns ``[rank·(A/P)·D, (rank+1)·(A/P)·D)``.
    """
    if not 0 <= rank < P:
        raise ConfigError(f"rank {rank} outside [0, {P})", "parallel.rank")
    row = 3 * heads_per_rank * head_dim
    if heads_per_rank * head_dim * P != hidden:
        raise ConfigError("hidden != P * heads_per_rank * head_dim", "parallel.ulysses")
    return {"qkv": rank * rows_per_rank * row * elem_bytes, "o": rank * heads_per_rank * head_dim * elem_bytes}


class _DeviceBytes:
    """``__cuda_array_interface__`` view of a libaqb allocation (so torch can wrap it)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerBuffers:
    """Named symmetric buffers: same sizes on every rank, every rank's copy mapped in every process.

    ``local(name, shape, dtype)`` is this rank's buffer as a torch tensor;
    ``ptrs(name, offset)`` the device addresses of all ranks' copies (+ a byte
    offset), in rank order, for the scatter epilogues and the barrier.
    Collective: every rank must construct it with the same ``sizes``.
    """

    def __init__(self, sp: Ulysses, sizes: dict, device):
        import ctypes

        self.sp, self.device = sp, torch.device(device)
        self._own, self._opened, self._nbytes = {}, [], dict(sizes)
        handles = {}
        for name, nbytes in sizes.items():
            nbytes = max(int(nbytes), 16)
            ptr = ctypes.c_void_p()
            h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
            _native.call("aqb_peer_alloc", nbytes, ctypes.addressof(ptr), ctypes.addressof(h))
            self._own[name] = int(ptr.value)
            handles[name] = h.raw
        gathered = [None] * sp.P
        dist.all_gather_object(gathered, handles, group=sp.group)
        self._all = {}
        for name in sizes:
            row = []
            for r in range(sp.P):
                if r == sp.rank:
                    row.append(self._own[name])
                    continue
                ptr = ctypes.c_void_p()
                hb = ctypes.create_string_buffer(gathered[r][name], IPC_HANDLE_BYTES)
                _native.call("aqb_peer_open", ctypes.addressof(hb), ctypes.addressof(ptr))
                row.append(int(ptr.value))
                self._opened.append(int(ptr.value))
            self._all[name] = row

    def local(self, name: str, shape, dtype) -> torch.Tensor:
        n = 1
        for d in shape:
            n *= int(d)
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        if nbytes > self._nbytes[name]:
            raise NativeError(f"peer buffer {name}: {nbytes} B requested, {self._nbytes[name]} allocated")
        raw = torch.as_tensor(_DeviceBytes(self._own[name], nbytes), device=self.device)
        return raw.view(dtype).view(*shape)

    def ptrs(self, name: str, offset_bytes: int = 0) -> list:
        return [p + int(offset_bytes) for p in self._all[name]]

    def close(self):
        """Unmap peers and free this rank's buffers (collective).

        Drain this rank's queued kernels first (its scatter epilogues and barrier signals
        store into the peers' buffers), then the host barrier: once every rank has passed
        it, no kernel anywhere can still write into the memory freed below (with gloo the
        barrier is host-only, so the device drain must come before it)."""
        if not self._own and not self._opened:
            return
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        dist.barrier(group=self.sp.group)
        for p in self._opened:
            _native.call("aqb_peer_close", p)
        for p in self._own.values():
            _native.call("aqb_peer_free", p)
        self._opened, self._own = [], {}
