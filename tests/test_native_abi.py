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
    assert lib.aqb_abi_version() == 2
    assert isinstance(lib.aqb_last_error(), bytes)


def test_invalid_args_fail_loudly_without_gpu(lib_path):
    """Argument validation runs before any CUDA call: a bad call returns AQB_EINVAL."""
    lib = _native.load()
    rc = lib.aqb_gemm_bf16(None, 0, None, 0, None, 0, 0, 0, 0, None, None, 0, None, None, 0, None, 1, None)
    assert rc == -1
    assert b"null pointer" in lib.aqb_last_error()
    rc = lib.aqb_attention_fwd(1, 8, 8, 1, 8, 8, 1, 8, 8, 1, 8, 8, 16, 16, 1, 48, 1.0, 0, None, 0, None, 1, None)
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


def test_attention_split_planner_and_workspace_without_gpu(lib_path):
    """Host-side split-KV planner (SM count falls back to 148 without a GPU) and workspace sizing."""
    lib = _native.load()
    assert lib.aqb_attention_splits(8056, 8056, 2, 128) >= 2       # 2 heads x 32 tiles << 148 SMs
    assert lib.aqb_attention_splits(119056, 119056, 24, 128) == 1  # 10k CTAs: no split
    assert lib.aqb_attention_workspace_bytes(1000, 4, 128, 1) == 0
    rows = 3 * (4 * 4) * 256  # splits x (heads x 256-query tiles) x 256 rows, compact partial layout
    assert lib.aqb_attention_workspace_bytes(1000, 4, 128, 3) == ((rows + 63) // 64 * 64 + rows * 128) * 4
    # wave-quantisation tail (config 2: 16 heads x 31 tiles = 496 on 148 SMs): 3 whole waves + split tail
    assert lib.aqb_attention_whole_tiles(7800, 7800, 16, 128) == 444
    out = (ctypes.c_int32 * 5)()
    assert lib.aqb_attention_plan(7800, 7800, 16, 128, out) == 0
    n_whole, splits, first, per, major = list(out)
    assert (n_whole, major) == (444, 1) and splits >= 2 and first >= per  # long first part, split-major
    assert first + (splits - 1) * per >= 61 > first + (splits - 2) * per   # the parts cover the 61 KV blocks
    tail_rows = (496 - 444) * splits * 256
    assert lib.aqb_attention_auto_workspace_bytes(7800, 7800, 16, 128) == ((tail_rows + 63) // 64 * 64 +
                                                                          tail_rows * 128) * 4
    assert lib.aqb_attention_whole_tiles(7800, 7800, 4, 128) == 124  # 124 tiles: splitting does not pay
    assert lib.aqb_attention_auto_workspace_bytes(7800, 7800, 4, 128) == 0


def test_peer_barrier_validates_before_launch(lib_path):
    lib = _native.load()
    assert lib.aqb_peer_barrier(None, 0, 2, None, None, 0, None, None, None, 1, None) == -1
    arr = _native.ptr_array([16, 32])
    assert lib.aqb_peer_barrier(arr, 2, 2, 64, None, 0, None, None, None, 1, None) == -1  # rank out of range
    assert lib.aqb_peer_barrier(arr, 0, 9, 64, None, 0, None, None, None, 1, None) == -1  # > 8 ranks


def test_gemm_trace_is_a_measurement_build_only(lib_path):
    """aqb_gemm_trace: NULL (off) always succeeds; a buffer is refused unless the library was built
    with -DAQB_GEMM_TRACE (the shipped build has no per-k-block stamp checks)."""
    if "AQB_GEMM_TRACE" in os.environ.get("AQB_BUILD_DEFINES", ""):
        pytest.skip("trace build")
    lib = _native.load()
    assert lib.aqb_gemm_trace(None) == 0
    assert lib.aqb_gemm_trace(ctypes.c_void_p(4096)) == -1
    assert b"AQB_GEMM_TRACE" in lib.aqb_last_error()


def test_kernel_kind_mapping_of_trace_symbols():
    """bench's CUPTI table groups libaqb kernels by symbol; foreign kernels (torch) are ignored."""
    from paper_2505_10584_b200.ops import kernel_kind

    assert kernel_kind("void aqb::gemm::gemm2_kernel<256, 4, 2>(CUtensorMap_st, ...)") == "gemm"
    assert kernel_kind("void aqb::attn::attn_fwd_kernel<128, 82u>(CUtensorMap_st, ...)") == "attention"
    assert kernel_kind("void aqb::attn::attn_short_kernel<82u>(CUtensorMap_st, ...)") == "attention"
    assert kernel_kind("void aqb::attn::attn_combine_kernel(aqb::attn::Params)") == "attention"
    assert kernel_kind("void aqb::norm_mod_row_kernel<4, 4, __nv_bfloat16>(float const*, ...)") == "norm_modulate"
    assert kernel_kind("aqb::peer::barrier_kernel(aqb::peer::BarrierArgs)") == "peer"
    assert kernel_kind("void aqb::step_scalars_kernel(float const*, ...)") == "small"
    assert kernel_kind("void at::native::vectorized_elementwise_kernel<4, ...>") is None


def test_bench_arms_share_the_config():
    """The reference arm and ours print the same config dict (the driver compares them)."""
    import bench

    assert bench.config_dict() == bench.config_dict()
    assert bench.config_dict()["seq_len"] == 7800
