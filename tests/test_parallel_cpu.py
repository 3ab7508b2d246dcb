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
