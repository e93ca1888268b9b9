"""ctypes binding of the C ABI in include/hps_leaf.h (libhps_leaf.so).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
Loading fails loudly: there is no CPU implementation behind these symbols.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeUnavailableError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libhps_leaf.so")
# diagnostics: HPS_LIB points at an alternative in-tree build (tuning variants)
LIB_PATH = os.environ.get("HPS_LIB", LIB_PATH)

EXPORTS = (
    "hps_abi_version", "hps_last_error", "hps_device_count", "hps_plan_create",
    "hps_plan_destroy", "hps_plan_info", "hps_leaf_dtn", "hps_leaf_dtn_host",
    "hps_leaf_reduce_load", "hps_leaf_interior_solve", "hps_leaf_solution_operator",
    "hps_plan_set_profile", "hps_plan_create_legendre", "hps_leaf_apply",
    "hps_interface_scatter", "hps_leaf_factors", "hps_plan_release", "hps_plan_workspace",
)
ABI_VERSION = 2

_lib = None

_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int


def _sig(lib):
    lib.hps_abi_version.restype = _I
    lib.hps_last_error.restype = ctypes.c_char_p
    lib.hps_device_count.restype = _I
    lib.hps_plan_create.argtypes = [ctypes.POINTER(_P), _I, _I, _I, _I, _I, _P, _P, _P, _P, _I,
                                    ctypes.c_size_t]
    lib.hps_plan_create_legendre.argtypes = [ctypes.POINTER(_P), _I, _I, _I, _I, _I, _I, _P, _P, _P,
                                             _P, _P, _I, _P, _I, ctypes.c_size_t]
    lib.hps_leaf_apply.argtypes = [_P, _I, _P, _P, _P, _P, _P]
    lib.hps_plan_destroy.argtypes = [_P]
    lib.hps_plan_info.argtypes = [_P] + [ctypes.POINTER(_I)] * 4 + [ctypes.POINTER(ctypes.c_size_t)] * 2
    lib.hps_leaf_dtn.argtypes = [_P, _I, _P, _P, _P, _P]
    lib.hps_leaf_dtn_host.argtypes = [_P, _I, _P, _P, _P, _I]
    lib.hps_leaf_reduce_load.argtypes = [_P, _I, _P, _P, _P, _P, _P, _P]
    lib.hps_leaf_interior_solve.argtypes = [_P, _I, _P, _P, _P, _P, _P, _P]
    lib.hps_leaf_solution_operator.argtypes = [_P, _I, _P, _P, _P, _P]
    lib.hps_leaf_factors.argtypes = [_P, _I, _P, _P, _P, _P, _P]
    lib.hps_plan_release.argtypes = [_P]
    lib.hps_plan_workspace.argtypes = [_P, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(_I)]
    lib.hps_plan_set_profile.argtypes = [_P, _P]
    lib.hps_interface_scatter.argtypes = [_I, _P, ctypes.c_longlong, ctypes.c_longlong,
                                          ctypes.c_longlong, _I, _P, _P, _P, _P]
    for name in EXPORTS:
        if name not in ("hps_abi_version", "hps_last_error", "hps_device_count"):
            getattr(lib, name).restype = _I


def load():
    """Return the loaded library, raising NativeUnavailableError if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailableError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeUnavailableError(f"cannot load {LIB_PATH}: {exc}") from exc
        _sig(lib)
        if lib.hps_abi_version() != ABI_VERSION:
            raise NativeUnavailableError("libhps_leaf.so ABI version mismatch; rebuild")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("hps native call failed: " + load().hps_last_error().decode())
