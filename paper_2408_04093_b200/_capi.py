"""ctypes binding of the C-ABI in include/treedec_b200.h.

The library is the product: there is no Python or CPU fallback. Loading
fails loudly when libtreedec_b200.so is missing or when no CUDA device is
visible at call time.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtreedec_b200.so")

TD_OK, TD_EINVAL, TD_EDOMAIN, TD_ECUDA, TD_ENCCL, TD_ESTATE = range(6)
TD_F64, TD_F32, TD_BF16 = 0, 1, 2
TD_TREE_BINARY, TD_RING_ALLREDUCE, TD_HIERARCHICAL = 0, 1, 2
TD_HOST_IO, TD_TIME_KERNELS, TD_BF16_OUT, TD_TIME_PHASES, TD_P2P, TD_DEBUG_TS, TD_DETERMINISTIC = 1, 2, 4, 8, 16, 32, 64
TD_PINNED_IO = 128
TD_DYNAMIC = 256
TD_GRAPH = 512
TD_NCCL_DEVICE = 1024

# Every symbol include/treedec_b200.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "td_version", "td_last_error", "td_seeded_fill", "td_set_deterministic", "td_decode_workspace_bytes",
    "td_decode_partial", "td_combine_partials", "td_partial_to_numerator", "td_combine_pair",
    "td_finalize", "td_create", "td_destroy", "td_stream", "td_comm_unique_id", "td_comm_init",
    "td_comm_info", "td_p2p_handle", "td_p2p_open", "td_p2p_status", "td_kv_place", "td_kv_generate", "td_kv_info", "td_kv_pointers",
    "td_kv_append", "td_kv_reserve",
    "td_energy_workspace_bytes", "td_energy_partial", "td_energy_combine", "td_energy_grad_combine",
    "td_energy_forward", "td_energy_grad", "td_calibration_info",
    "td_tree_decode", "td_ring_decode", "td_local_partial", "td_output_bf16", "td_kernel_time",
    "td_reset_kernel_timer", "td_phase_times", "td_debug_stamps", "td_last_launch_stats", "td_memory_bytes",
    "td_group_create", "td_group_destroy", "td_group_context", "td_group_p2p_open", "td_group_tree_decode",
]


class TreeDecError(RuntimeError):
    """Base class; status code in .status."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class InvalidArgument(TreeDecError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(TreeDecError, ArithmeticError):
    """std::domain_error in the reference."""


_lib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_fp = ctypes.POINTER(ctypes.c_float)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    # torch first: its libnccl.so.2 (and libcudart) are then the ones this
    # library binds to at run time (td_capi.cu resolves NCCL with dlopen).
    import torch  # noqa: F401
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.td_version.restype = ctypes.c_int
    L.td_last_error.restype = ctypes.c_char_p
    L.td_seeded_fill.argtypes = [ctypes.c_int, _vp, ctypes.c_uint64, ctypes.c_double, _i64, _i64, _i64, _i64, _i64, _vp]
    L.td_set_deterministic.argtypes = [ctypes.c_int]
    L.td_decode_workspace_bytes.argtypes = [ctypes.c_int, _i64, _i64, _i64, _i64, _i64, ctypes.POINTER(ctypes.c_size_t)]
    L.td_decode_partial.argtypes = [ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_double,
                                    _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
    L.td_combine_partials.argtypes = [ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _vp]
    L.td_partial_to_numerator.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _vp]
    L.td_combine_pair.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]
    L.td_finalize.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp]
    L.td_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
    L.td_destroy.argtypes = [_vp]
    L.td_stream.argtypes = [_vp, ctypes.POINTER(_vp)]
    L.td_comm_unique_id.argtypes = [ctypes.c_char_p]
    L.td_comm_init.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    L.td_comm_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    L.td_p2p_handle.argtypes = [_vp, _i64, _i64, ctypes.c_char_p]
    L.td_p2p_open.argtypes = [_vp, ctypes.c_char_p]
    L.td_p2p_status.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
    L.td_kv_place.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, ctypes.c_int]
    L.td_kv_generate.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_double]
    L.td_kv_info.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_size_t)]
    L.td_kv_pointers.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
    L.td_kv_append.argtypes = [_vp, _vp, _vp, ctypes.c_int]
    L.td_kv_reserve.argtypes = [_vp, _i64]
    L.td_energy_workspace_bytes.argtypes = [ctypes.c_int] + [_i64] * 5 + [ctypes.POINTER(ctypes.c_size_t)]
    L.td_energy_partial.argtypes = [ctypes.c_int] + [_vp] * 4 + [_i64] * 5 + [_vp] * 4 + [ctypes.c_size_t, _vp]
    L.td_energy_combine.argtypes = [ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp, _vp]
    L.td_energy_grad_combine.argtypes = [ctypes.c_int] + [_vp] * 4 + [_i64, _i64, _vp, _vp]
    L.td_energy_forward.argtypes = [_vp, _vp, _vp, _i64, _vp, _vp, _vp, ctypes.c_int]
    L.td_energy_grad.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, ctypes.c_int]
    L.td_calibration_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    L.td_tree_decode.argtypes = [_vp, _vp, _i64, ctypes.c_double, ctypes.c_int, _vp, ctypes.c_int]
    L.td_ring_decode.argtypes = [_vp, _vp, _i64, ctypes.c_double, _vp, ctypes.c_int]
    L.td_local_partial.argtypes = [_vp, _vp, _i64, ctypes.c_double, _vp, _vp, _vp, ctypes.c_int]
    L.td_output_bf16.argtypes = [_vp, ctypes.POINTER(_vp)]
    L.td_kernel_time.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    L.td_reset_kernel_timer.argtypes = [_vp]
    L.td_debug_stamps.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.td_phase_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                 ctypes.POINTER(ctypes.c_int)]
    L.td_last_launch_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int)]
    L.td_memory_bytes.argtypes = [_vp, ctypes.POINTER(ctypes.c_size_t)]
    L.td_group_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(_vp)]
    L.td_group_destroy.argtypes = [_vp]
    L.td_group_context.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp)]
    L.td_group_p2p_open.argtypes = [_vp, _i64, _i64]
    L.td_group_tree_decode.argtypes = [_vp, _vp, _i64, ctypes.c_double, ctypes.c_int, _vp, ctypes.c_int]
    for name in EXPORTS:
        fn = getattr(L, name)
        if fn.restype is ctypes.c_int or name not in ("td_last_error",):
            if name != "td_last_error":
                fn.restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == TD_OK:
        return
    msg = lib().td_last_error().decode(errors="replace")
    if rc == TD_EINVAL:
        raise InvalidArgument(rc, msg)
    if rc == TD_EDOMAIN:
        raise DomainError(rc, msg)
    raise TreeDecError(rc, msg)
