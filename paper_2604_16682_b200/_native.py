"""Loader for the in-tree CUDA library (the C ABI of include/agentsim_b200.h).

There is no CPU fallback: every entry point requires the sm_100a library and
a CUDA device, and fails loudly otherwise.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _abi
from ._build import LIB_PATH

_LIB: C.CDLL | None = None


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (no CPU fallback exists)."""


def _declare(lib: C.CDLL) -> None:
    vp, i32, i64, f64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
    sig = {
        "asb_abi_version": (C.c_int, []),
        "asb_struct_sizes": (C.c_int, [vp]),
        "asb_workspace_bytes": (sz, [i32, i64, i64]),
        "asb_run_scenarios": (C.c_int, [vp, i32, i32, _abi.AsbTracePool, _abi.AsbTablePool, _abi.AsbOutputs,
                                        i64, i64, vp, sz, vp]),
        "asb_scenario_stats": (C.c_int, [vp, i32, _abi.AsbOutputs, vp, vp, sz, vp]),
        "asb_reduce_stats": (C.c_int, [vp, vp, i32, vp, vp]),
        "asb_select_level_batch": (C.c_int, [vp, vp, vp, vp, vp, i64, vp]),
        "asb_service_time_batch": (C.c_int, [vp, vp, vp, vp, vp, vp, f64, f64, vp, i64, vp]),
        "asb_assign_batch": (C.c_int, [vp, vp, i32, i64, f64, i32, vp, i64, vp]),
        "asb_reassign_batch": (C.c_int, [vp, vp, i32, vp, vp, i32, f64, i32, i32, vp, i64, vp]),
        "asb_min_throughput_batch": (C.c_int, [vp, vp, vp, i64, i32, vp, vp, vp]),
        "asb_regime_classify": (C.c_int, [vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """The loaded CUDA library (raises NativeUnavailable when not built)."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("ASB_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 engine has no CPU fallback)"
            )
        handle = C.CDLL(path)
        _declare(handle)
        _LIB = handle
    return _LIB


def device(dev=None):
    """A CUDA device for the engine; raises NativeUnavailable without one."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("agentsim_b200 requires a CUDA (sm_100a) device; there is no CPU fallback")
    lib()
    d = torch.device(dev) if dev is not None else torch.device("cuda", torch.cuda.current_device())
    if d.type != "cuda":
        raise NativeUnavailable(f"agentsim_b200 runs on CUDA devices only, got {d}")
    return d


def stream_handle(dev) -> int:
    import torch

    return torch.cuda.current_stream(dev).cuda_stream


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed with status {rc}")
