"""ctypes binding of the C ABI in include/wheelsieve/gpu.h.

The shared library is built in-tree (paper_2310_17746_b200/libwheelsieve_cuda.so,
by ``__graft_entry__.build()`` / ``make -C paper_2310_17746_b200/csrc``).  There
is no fallback: if it is missing or cannot be loaded, importing this module
raises, and every call on a machine without an sm_100 GPU raises
``Error(Errc.NoDevice)``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwheelsieve_cuda.so")

# Every symbol include/wheelsieve/gpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ws_opts_default", "ws_status_name", "ws_ctx_create", "ws_ctx_destroy", "ws_last_error",
    "ws_ctx_stream", "ws_last_timing", "ws_count_range", "ws_enumerate_range",
    "ws_count_intervals", "ws_prime_count_bound", "ws_partition", "ws_start_offsets",
    "ws_isqrt", "ws_version", "ws_base_primes", "ws_sieve_segment", "ws_store_range",
    "ws_read_back", "ws_verify_store", "ws_count_ranges", "ws_nccl_unique_id",
    "ws_ctx_num_devices", "ws_ctx_num_shards", "ws_ctx_device", "ws_ctx_device_stream",
    "ws_device_timing", "ws_ctx_comm_info", "ws_combine_checks", "ws_enumerate_shards",
    "ws_store_open", "ws_store_append", "ws_store_set_frontier", "ws_store_flush",
    "ws_store_durable_count", "ws_store_last_error", "ws_store_close",
)

WS_WANT_CHECKS = 0x1
WS_OUT_DEVICE = 0x2
WS_FRESH_BASE = 0x4

u64 = C.c_uint64
u32 = C.c_uint32
P64 = C.POINTER(C.c_uint64)
P32 = C.POINTER(C.c_uint32)


WS_MAX_DEVICES = 16
WS_NCCL_ID_BYTES = 128


class WsOpts(C.Structure):
    _fields_ = [("struct_size", u32), ("segment_slots", u32), ("device", C.c_int32),
                ("n_devices", u32), ("device_ids", C.c_int32 * WS_MAX_DEVICES),
                ("world", u32), ("rank", u32), ("nccl_id", C.c_uint8 * WS_NCCL_ID_BYTES)]


class WsChecks(C.Structure):
    _fields_ = [("count", u64), ("sum", u64), ("xor_", u64), ("largest", u64)]


class WsTiming(C.Structure):
    _fields_ = [("base_ms", C.c_double), ("sieve_ms", C.c_double), ("total_ms", C.c_double),
                ("launches", u64), ("segments", u64), ("base_primes", u64),
                ("h2d_bytes", u64), ("d2h_bytes", u64)]


def _preload_nccl() -> None:
    """libwheelsieve_cuda.so links libnccl.so.2.  If PyTorch's bundled NCCL
    (nvidia-nccl wheel, newer than the system's) is installed, load it first:
    whichever libnccl.so.2 enters the process first serves every later user
    of that soname, and torch needs its own (newer) symbols."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        so = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(so):
            C.CDLL(so, mode=C.RTLD_GLOBAL)
            return


def _load(path: str = LIB_PATH) -> C.CDLL:
    _preload_nccl()
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(path)
    vp = C.c_void_p
    sig = {
        "ws_opts_default": (None, [C.POINTER(WsOpts)]),
        "ws_status_name": (C.c_char_p, [C.c_int]),
        "ws_ctx_create": (C.c_int, [C.POINTER(WsOpts), C.POINTER(vp)]),
        "ws_ctx_destroy": (None, [vp]),
        "ws_last_error": (C.c_char_p, [vp]),
        "ws_ctx_stream": (vp, [vp]),
        "ws_last_timing": (C.c_int, [vp, C.POINTER(WsTiming)]),
        "ws_count_range": (C.c_int, [vp, u64, u64, u32, C.POINTER(WsChecks), vp, u64, P64]),
        "ws_enumerate_range": (C.c_int, [vp, u64, u64, u32, vp, u64, P64, C.POINTER(WsChecks)]),
        "ws_count_intervals": (C.c_int, [vp, vp, u64, u64, u32, vp, vp, vp]),
        "ws_prime_count_bound": (u64, [u64, u64]),
        "ws_partition": (C.c_int, [u64, u64, u32, u32, u32, P64, P64]),
        "ws_start_offsets": (C.c_int, [u64, u64, P64, P64]),
        "ws_isqrt": (u64, [u64]),
        "ws_base_primes": (C.c_int, [vp, u64, u32, vp, u64, P64]),
        "ws_sieve_segment": (C.c_int, [vp, u64, u64, u32, vp, vp]),
        "ws_store_range": (C.c_int, [vp, u64, u64, C.c_char_p, u32, u64, P64]),
        "ws_read_back": (C.c_int, [C.c_char_p, u64, u64, vp, u64, P64]),
        "ws_verify_store": (C.c_int, [C.c_char_p]),
        "ws_version": (C.c_char_p, []),
        "ws_count_ranges": (C.c_int, [vp, vp, vp, u64, u32, vp]),
        "ws_nccl_unique_id": (C.c_int, [vp]),
        "ws_ctx_num_devices": (u32, [vp]),
        "ws_ctx_num_shards": (u32, [vp]),
        "ws_ctx_device": (C.c_int32, [vp, u32]),
        "ws_ctx_device_stream": (vp, [vp, u32]),
        "ws_device_timing": (C.c_int, [vp, u32, C.POINTER(WsTiming)]),
        "ws_ctx_comm_info": (C.c_int, [vp, u32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "ws_combine_checks": (C.c_int, [vp, u64, C.POINTER(WsChecks)]),
        "ws_enumerate_shards": (C.c_int, [vp, u64, u64, u32, vp, vp, vp, C.POINTER(WsChecks)]),
        "ws_store_open": (C.c_int, [C.c_char_p, u32, u64, C.POINTER(vp)]),
        "ws_store_append": (C.c_int, [vp, vp, u64]),
        "ws_store_set_frontier": (C.c_int, [vp, u64]),
        "ws_store_flush": (C.c_int, [vp]),
        "ws_store_durable_count": (u64, [vp]),
        "ws_store_last_error": (C.c_char_p, [vp]),
        "ws_store_close": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
