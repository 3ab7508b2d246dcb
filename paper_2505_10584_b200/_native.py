"""ctypes binding of libaqb.so — the only way the product reaches the GPU.

There is no CPU fallback: if the library is missing or fails to load, every
op raises.  Signatures mirror ``include/aqb.h`` exactly.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaqb.so")

c_int, c_int32, c_int64, c_float, c_void_p = ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
c_char_p = ctypes.c_char_p

P = c_void_p  # every pointer is passed as an integer address
SIGNATURES = {
    "aqb_abi_version": (c_int, []),
    "aqb_build_id": (c_char_p, []),
    "aqb_last_error": (c_char_p, []),
    "aqb_sm_count": (c_int, []),
    "aqb_set_pdl": (c_int, [c_int]),
    "aqb_attention_trace": (c_int, [P]),
    "aqb_gemm_trace": (c_int, [P]),
    "aqb_attention_plan": (c_int, [c_int64, c_int64, c_int32, c_int32, P]),
    "aqb_norm_modulate": (c_int, [P, c_int64, P, P, P, c_int64, c_int64, c_int32, c_float, c_int32, P, P, P, c_int32, P]),
    "aqb_gate_bcast": (c_int, [P, c_int64, P, P, c_int32, c_int64, c_int64, c_int64, P, c_int32, P]),
    "aqb_sum_slots": (c_int, [P, c_int64, P, c_int32, c_int64, c_int64, c_int64, c_int64, P, c_int32, P]),
    "aqb_norm_modulate_gather": (c_int, [P, c_int64, P, P, P, c_int32, c_int64, c_int64, c_int32, c_float, c_int32, P,
                                         P, P, c_int32, P]),
    "aqb_gemm_gate_add_scatter": (c_int, [P, c_int64, P, c_int64, P, c_int32, c_int64, c_int64, c_int64, c_int64,
                                          c_int64, P, P, P, c_int32, P]),
    "aqb_gemm_bf16": (c_int, [P, c_int64, P, c_int64, P, c_int64, c_int64, c_int64, c_int64, P, P, c_int32, P, P,
                              c_int64, P, c_int32, P]),
    "aqb_gemm_qknorm_rope": (c_int, [P, c_int64, P, c_int64, c_int64, c_int64, c_int64, P, c_int32, c_int32, P, P,
                                     c_float, P, P, c_int64, c_int64, P, c_int64, c_int32, c_int64, c_int32, c_int32,
                                     P, c_int32, P]),
    "aqb_qk_norm_rope": (c_int, [P, c_int64, c_int64, c_int32, c_int32, c_int32, c_int32, P, P, c_float, P, P, c_int64,
                                 c_int64, P, c_int64, c_int64, c_int64, c_int32, c_int32, c_int32, P, c_int32, P]),
    "aqb_attention_fwd": (c_int, [P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64, c_int64,
                                  c_int64, c_int64, c_int32, c_int32, c_float, c_int32, P, c_int64, P, c_int32, P]),
    "aqb_attention_splits": (c_int, [c_int64, c_int64, c_int32, c_int32]),
    "aqb_attention_workspace_bytes": (c_int64, [c_int64, c_int32, c_int32, c_int32]),
    "aqb_attention_whole_tiles": (c_int, [c_int64, c_int64, c_int32, c_int32]),
    "aqb_attention_pairs_per_cta": (c_int, [c_int64, c_int64, c_int32, c_int32]),
    "aqb_attention_auto_workspace_bytes": (c_int64, [c_int64, c_int64, c_int32, c_int32]),
    "aqb_attention_fwd_scatter": (c_int, [P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64, c_int64, P, c_int32,
                                          c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int32, c_int32,
                                          c_float, c_int32, P, c_int64, P, c_int32, P]),
    "aqb_gemm_qknorm_rope_scatter": (c_int, [P, c_int64, P, c_int64, c_int64, c_int64, c_int64, P, c_int32, c_int32,
                                             P, P, c_float, P, P, c_int64, c_int64, P, c_int32, c_int64, c_int32, P,
                                             c_int32, P]),
    "aqb_norm_modulate_f32": (c_int, [P, c_int64, P, P, P, c_int64, c_int64, c_int32, c_float, c_int32, P, P, P,
                                      c_int32, P]),
    "aqb_qk_norm_rope_f32": (c_int, [P, c_int64, c_int64, c_int32, c_int32, c_int32, c_int32, P, P, c_float, P, P,
                                     c_int64, c_int64, P, c_int64, c_int64, c_int64, c_int32, c_int32, c_int32, P,
                                     c_int32, P]),
    "aqb_gemm_f32": (c_int, [P, c_int64, P, c_int64, P, c_int64, c_int64, c_int64, c_int64, P, P, c_int32, P, P,
                             c_int64, P, c_int32, P]),
    "aqb_attention_f32": (c_int, [P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64, c_int64, P, c_int64,
                                  c_int64, c_int64, c_int64, c_int32, c_int32, c_float, P, c_int32, P]),
    "aqb_tile_blend": (c_int, [P, P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                               c_int32, c_int32, c_int32, c_int32, P, P]),
    "aqb_window_average": (c_int, [P, P, c_int32, c_int32, c_int32, c_int32, c_int64, P, P]),
    "aqb_peer_alloc": (c_int, [c_int64, P, P]),
    "aqb_peer_open": (c_int, [P, P]),
    "aqb_peer_close": (c_int, [P]),
    "aqb_peer_free": (c_int, [P]),
    "aqb_peer_can_access": (c_int, [c_int32, c_int32]),
    "aqb_peer_barrier": (c_int, [P, c_int32, c_int32, P, P, c_int32, P, P, P, c_int32, P]),
    "aqb_gemv": (c_int, [P, P, P, P, P, P, c_int64, c_int64, c_int32, P]),
    "aqb_add_bcast": (c_int, [P, P, c_int64, P, c_int64, P]),
    "aqb_rel_l1_reduce": (c_int, [P, c_int64, P, P]),
    "aqb_cache_decide": (c_int, [P, P, c_float, c_int32, c_int32, c_int32, P, P, P]),
    "aqb_cache_offset": (c_int, [P, c_int64, P, c_int64, c_int32, c_int32, P, c_int32, P]),
    "aqb_step_scalars": (c_int, [P, P, P, P, c_int32, P]),
    "aqb_patchify": (c_int, [P, P, P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                             P]),
    "aqb_unpatchify": (c_int, [P, P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                               P]),
    "aqb_heads_to_seq": (c_int, [P, c_int64, c_int32, c_int32, P, c_int64, P, c_int32, P]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every ``aqb_*`` function declared in include/aqb.h (for the ABI test)."""
    import re

    path = os.path.join(os.path.dirname(_HERE), "include", "aqb.h")
    with open(path) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(aqb_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load (once) and type the library; raise NativeError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"{LIB_PATH} not built — run `python -m paper_2505_10584_b200.build` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    from .build import header_hash

    built = lib.aqb_build_id().decode()
    if built != header_hash():
        raise NativeError(f"{LIB_PATH} was built from a different include/aqb.h ({built[:12]} vs "
                          f"{header_hash()[:12]}) — rebuild with `python -m paper_2505_10584_b200.build --force`")
    _lib = lib
    return lib


def query(name: str, *args):
    """Call a pure host-side query (returns its value; no status code)."""
    return getattr(load(), name)(*args)


def ptr_array(ptrs):
    """HOST array of device pointers (``void* const*`` arguments)."""
    return (c_void_p * len(ptrs))(*[int(p) for p in ptrs])


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.aqb_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")
