"""Ulysses sequence parallelism (one process per GPU, NCCL over NVLink).

The north_star's multi-GPU path: video tokens are sharded S_v/P per rank for
every token-wise op; around attention an all-to-all swaps the sequence shard
for a head shard (A/P heads over the full sequence) and back
(``PAPER.md:193`` describes the same exchange as the paper's CP for >200k
tokens; the reference only costs it, ``comm.py:65-96``).  Text tokens are
replicated on every rank (their head slice is taken locally; their
attention output is all-gathered).  The rel-L1 cache decision all-reduces two
scalars so every rank takes the same branch.

This module only wraps ``torch.distributed``; the packing into the
all-to-all layout is fused into the QK-norm/RoPE kernel and the unpacking is
the ``aqb_heads_to_seq`` kernel.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .errors import ConfigError


class Ulysses:
    """Sequence-parallel group context (``P`` ranks, this rank ``rank``)."""

    def __init__(self, group=None):
        if not dist.is_initialized():
            raise ConfigError("torch.distributed is not initialised", "parallel.group")
        self.group = group if group is not None else dist.group.WORLD
        self.P = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)

    def check(self, num_heads: int, video_tokens: int):
        if num_heads % self.P:
            raise ConfigError(f"num_heads {num_heads} not divisible by {self.P} ranks", "parallel.ulysses")
        if video_tokens % self.P:
            raise ConfigError(f"video tokens {video_tokens} not divisible by {self.P} ranks", "parallel.ulysses")

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor):
        dist.all_to_all_single(out, inp, group=self.group)

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce_sum(self, t: torch.Tensor):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)


def init_from_env(backend: str | None = None):
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous)."""
    if dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend=backend)
