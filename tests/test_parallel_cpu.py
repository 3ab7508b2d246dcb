"""Multi-rank host logic of the Ulysses path on CPU: world_size-2 ``gloo`` process
groups (no GPU).  Covers the group wrapper (validation, the rel-L1 all-reduce), the
peer-buffer rendezvous (IPC handles gathered and opened in rank order; the native
calls are stubbed — they need a GPU) and the scatter offset arithmetic."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_10584_b200.errors import ConfigError
from paper_2505_10584_b200.parallel import exchange_offsets


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_10584_b200 import _native, parallel

        sp = parallel.Ulysses(exchange="p2p")
        out = {"P": sp.P, "rank": sp.rank}
        try:
            sp.check(num_heads=24, video_tokens=7801)
        except ConfigError as e:
            out["check_path"] = e.path
        sp.check(num_heads=16, video_tokens=7800)
        t = torch.tensor([1.5 * (rank + 1), float(rank)])
        sp.all_reduce_sum(t)
        out["sums"] = t.tolist()
        # peer rendezvous with stubbed native calls: "addresses" encode (rank, buffer)
        import ctypes

        calls = []

        def fake_call(name, *args):
            calls.append(name)
            if name == "aqb_peer_alloc":
                nbytes, pptr, phandle = args
                ptr = (rank + 1) << 32 | nbytes
                ctypes.c_void_p.from_address(pptr).value = ptr
                ctypes.memmove(phandle, ptr.to_bytes(8, "little") + bytes(56), 64)
            elif name == "aqb_peer_open":
                phandle, pptr = args
                raw = ctypes.string_at(phandle, 8)
                ctypes.c_void_p.from_address(pptr).value = int.from_bytes(raw, "little") + 7  # mapped alias
            elif name in ("aqb_peer_close", "aqb_peer_free"):
                pass
            else:
                raise AssertionError(name)

        _native_call = _native.call
        _native.call = fake_call
        try:
            pb = parallel.PeerBuffers(sp, {"rcv": 4096, "o": 1024}, "cpu")
            out["rcv"] = pb.ptrs("rcv", 16)
            out["o"] = pb.ptrs("o")
            pb.close()
        finally:
            _native.call = _native_call
        out["calls"] = sorted(set(calls))
        q.put(out)
    except BaseException as e:  # surface worker failures to the test immediately
        q.put({"rank": rank, "error": repr(e)})
        raise
    finally:
        dist.destroy_process_group()


def test_ulysses_host_logic_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda d: d["rank"])
    assert not any("error" in d for d in res), res
    for r, d in enumerate(res):
        assert d["P"] == 2 and d["check_path"] == "parallel.ulysses"
        assert d["sums"] == [1.5 + 3.0, 1.0]  # identical on both ranks
        # every rank sees every rank's buffer in rank order: own pointer as allocated,
        # peers' through the opened alias (+7 in the stub), plus the requested offset
        own = [(q + 1) << 32 | 4096 for q in range(2)]
        assert d["rcv"] == [(own[q] if q == r else own[q] + 7) + 16 for q in range(2)]
        assert d["calls"] == ["aqb_peer_alloc", "aqb_peer_close", "aqb_peer_free", "aqb_peer_open"]


def test_exchange_offsets():
    # 8 ranks, 7800 video tokens -> 975 rows each, 16 heads -> 2 per rank, D=128, H=2048
    off = exchange_offsets(3, 8, 975, 2, 128, 2048)
    assert off["qkv"] == 3 * 975 * (3 * 2 * 128) * 2
    assert off["o"] == 3 * 2 * 128 * 2
    with pytest.raises(ConfigError):
        exchange_offsets(8, 8, 975, 2, 128, 2048)
    with pytest.raises(ConfigError):
        exchange_offsets(0, 8, 975, 3, 128, 2048)


@pytest.mark.parametrize("P", [2, 4])
def test_tp_shards_recombine_to_the_full_block(P):
    """TP-SP weight slices: column-parallel outputs concatenate (per q/k/v part) and row-parallel
    partials sum (bias once, rank 0) to the unsharded projections."""
    from paper_2505_10584_b200.config import DiTConfig
    from paper_2505_10584_b200.parallel import tp_shard_single_dit
    from paper_2505_10584_b200.weights import init_weights

    cfg = DiTConfig("single-dit", hidden_size=512, num_heads=4, num_single=1, text_dim=64, text_len=8)
    W = init_weights(cfg, seed=3)
    shards = [tp_shard_single_dit(W, cfg, P, r) for r in range(P)]
    g = torch.Generator().manual_seed(0)
    H, F = cfg.hidden_size, cfg.ffn_dim
    x = torch.randn(5, H, generator=g)
    p = "blocks.0"
    full = x @ W[f"{p}.qkv.w"].float().t() + W[f"{p}.qkv.b"]
    parts = [x @ s[f"{p}.qkv.w"].float().t() + s[f"{p}.qkv.b"] for s in shards]
    hd = H // P
    for k in range(3):  # q, k, v: rank r owns columns [k*H + r*hd, +hd)
        got = torch.cat([pr[:, k * hd:(k + 1) * hd] for pr in parts], dim=1)
        assert torch.allclose(got, full[:, k * H:(k + 1) * H], atol=1e-5)
    h = torch.randn(5, F, generator=g)
    exp = h @ W[f"{p}.fc2.w"].float().t() + W[f"{p}.fc2.b"]
    fl = F // P
    got = sum(h[:, r * fl:(r + 1) * fl] @ s[f"{p}.fc2.w"].float().t() + (s[f"{p}.fc2.b"] if s[f"{p}.fc2.b"] is not None
                                                                         else 0) for r, s in enumerate(shards))
    assert torch.allclose(got, exp, atol=1e-4)
    assert all(s[f"{p}.proj.b"] is None for s in shards[1:]) and shards[0][f"{p}.proj.b"] is W[f"{p}.proj.b"]
    kv = [s[f"{p}.xkv.w"] for s in shards]
    assert torch.equal(torch.cat([k_[:hd] for k_ in kv]), W[f"{p}.xkv.w"][:H])
    assert torch.equal(torch.cat([k_[hd:] for k_ in kv]), W[f"{p}.xkv.w"][H:])
    assert shards[1]["t_block.w"] is W["t_block.w"]  # replicated entries are shared


def test_tp_shard_validates():
    from paper_2505_10584_b200.config import DiTConfig
    from paper_2505_10584_b200.parallel import tp_shard_single_dit

    cfg = DiTConfig("single-dit", hidden_size=384, num_heads=3, num_single=1, text_dim=64, text_len=8)
    with pytest.raises(ConfigError) as e:
        tp_shard_single_dit({}, cfg, 2, 0)
    assert e.value.path == "parallel.tp"
