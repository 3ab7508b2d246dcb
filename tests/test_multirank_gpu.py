"""Multi-rank parity the driver runs: P = 2, 4, 8 ranks on the GPUs of the box
(``AQB_OVERSUBSCRIBE=1``: ranks share GPUs round-robin when there are fewer GPUs than ranks —
the p2p exchange is unchanged, CUDA IPC maps a same-GPU buffer like a peer's).

Ulysses (fused p2p exchange) and TP-SP, Single-DiT and MM-DiT (incl. 24 heads -> 3 per rank at
P = 8), each under a static ``plan_cache``, a rel-L1 policy that really skips (threshold from the
oracle's probe), the attention cache, and the rel-L1 policy over the attention cache.  The worker
is ``tests/mp_parity.py``; every case line must say ok, with cached steps on every rank.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("parallel", ["ulysses", "tp"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_multirank_parity(parallel, P, tmp_path):
    out = tmp_path / "cases.jsonl"
    env = dict(os.environ, AQB_OVERSUBSCRIBE="1", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_parity.py"),
           "--parallel", parallel, "--out", str(out)]
    n_cases = 4
    if P == 2:  # P = 4 and 8 run every model; P = 2 keeps one per family (GPU-test time budget)
        cmd += ["--cases", "single,mm"]
        n_cases = 2
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    lines = [json.loads(x) for x in out.read_text().splitlines()] if out.exists() else []
    bad = [x for x in lines if not x["ok"]]
    assert r.returncode == 0 and lines and not bad, (r.returncode, bad, r.stdout[-3000:], r.stderr[-3000:])
    assert len(lines) == 4 * n_cases  # models x 4 cache policies
    for x in lines:
        assert len(x["schedule_per_rank"]) == P
        assert all(s == x["schedule_oracle"] for s in x["schedule_per_rank"])
        assert "c" in x["schedule_oracle"]  # cached steps on every rank, every policy


@pytest.mark.parametrize("P", [2, 4])
def test_multirank_vae_tile_blend(P, tmp_path):
    """Multi-GPU VAE blend (PeerTiles): each rank's tiles read from its peer memory blend to the
    same bits as the 1-GPU blend (the worker exits 1 otherwise)."""
    out = tmp_path / "blend.jsonl"
    env = dict(os.environ, AQB_OVERSUBSCRIBE="1", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_vae_blend.py"),
           "--out", str(out)]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in out.read_text().splitlines()] if out.exists() else []
    assert r.returncode == 0 and len(lines) == 2, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert all(x["bitwise_vs_1gpu"] for x in lines)
