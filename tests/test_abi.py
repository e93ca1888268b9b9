"""The C-ABI library loads and exports every symbol of include/hps_leaf.h.

No compute call is made without a GPU; on a CPU-only host the plan entry
point must fail loudly (there is no CPU fallback behind the ABI).
"""

import ctypes
import os
import re

import pytest

from paper_2503_04033_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hps_leaf.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hps_\w+)\s*\(", text, re.M)))


def test_library_exports_header_symbols():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_native.EXPORTS)
    assert lib.hps_abi_version() == _native.ABI_VERSION


def test_library_is_sm100a_cubin():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_no_cpu_fallback():
    lib = _native.load()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    assert lib.hps_device_count() == 0
    plan = ctypes.c_void_p()
    rc = lib.hps_plan_create(ctypes.byref(plan), 0, 3, 6, 0, 1, None, None, None, None, 0, 0)
    assert rc != 0 and not plan.value
    assert lib.hps_last_error()
    from paper_2503_04033_b200.engine import LeafEngine
    from paper_2503_04033_b200.errors import NativeUnavailableError
    from paper_2503_04033_b200.local_ops import LeafTemplate
    with pytest.raises(NativeUnavailableError):
        LeafEngine(LeafTemplate((1.0, 1.0, 1.0), 6, "drop", False), False, True)


def test_interface_scatter_argument_errors():
    """hps_interface_scatter validates sizes and pointers before touching the
    device (same error convention as the other entry points), and an empty job
    list is a no-op."""
    lib = _native.load()
    assert lib.hps_interface_scatter(0, None, 0, 0, 0, 5, None, None, None, None) != 0
    assert b"bad sizes" in lib.hps_last_error()
    assert lib.hps_interface_scatter(0, None, 4, 16, 0, -1, None, None, None, None) != 0
    assert lib.hps_interface_scatter(0, None, 4, 16, 0, 3, None, None, None, None) != 0
    assert b"null pointer" in lib.hps_last_error()
    assert lib.hps_interface_scatter(0, None, 4, 16, 0, 0, None, None, None, None) == 0


def test_no_cpu_fallback_for_device_assembly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2503_04033_b200.assembly import DeviceAssembler, InterfacePattern
    from paper_2503_04033_b200.geometry import DomainBox, MeshConfig, build_discretization
    pat = InterfacePattern(build_discretization(DomainBox((0.0, 0.0), (1.0, 1.0)), MeshConfig((2, 2), 6)))
    with pytest.raises(Exception):
        DeviceAssembler(pat, 0)
