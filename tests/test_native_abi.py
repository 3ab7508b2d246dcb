"""The C-ABI library loads and exports every symbol include/aqb.h declares (CPU, no compute)."""

import ctypes
import os
import subprocess

import pytest

from paper_2505_10584_b200 import _native
from paper_2505_10584_b200.build import LIB, build


@pytest.fixture(scope="module")
def lib_path():
    if not os.path.exists(LIB):
        build()
    return LIB


def test_header_symbols_exported(lib_path):
    syms = _native.header_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a ctypes signature in the binding
    assert set(syms) == set(_native.SIGNATURES)


def test_abi_version_and_error_string(lib_path):
    lib = _native.load()
    assert lib.aqb_abi_version() == 1
    assert isinstance(lib.aqb_last_error(), bytes)


def test_invalid_args_fail_loudly_without_gpu(lib_path):
    """Argument validation runs before any CUDA call: a bad call returns AQB_EINVAL."""
    lib = _native.load()
    rc = lib.aqb_gemm_bf16(None, 0, None, 0, None, 0, 0, 0, 0, None, None, 0, None, None, 0, None, 1, None)
    assert rc == -1
    assert b"null pointer" in lib.aqb_last_error()
    rc = lib.aqb_attention_fwd(1, 8, 8, 1, 8, 8, 1, 8, 8, 1, 8, 8, 16, 16, 1, 48, 1.0, None, 1, None)
    assert rc == -1 and b"head_dim" in lib.aqb_last_error()


def test_ops_refuse_cpu_tensors():
    import torch

    from paper_2505_10584_b200 import ops
    from paper_2505_10584_b200.errors import NativeError

    a = torch.zeros(4, 8, dtype=torch.bfloat16)
    with pytest.raises(NativeError, match="CUDA"):
        ops.gemm(a, a, torch.zeros(4, 4, dtype=torch.bfloat16))


def test_sass_is_blackwell_native(lib_path):
    """tcgen05 MMA, TMEM loads and TMA loads are present in the shipped cubin."""
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG"):
        assert mnem in out, mnem
    assert "HMMA" not in out.replace("UTCHMMA", "")
