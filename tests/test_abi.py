"""The C-ABI library exists, loads, and exports every symbol include/tvs_b200.h declares."""
import ctypes
import re
from pathlib import Path

from paper_2006_10004_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "tvs_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(tvs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_api():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.tvs_abi_version() == 2


def test_invalid_arguments_report_errors_without_gpu_work():
    lib = _native.load()
    plan = ctypes.c_void_p()
    assert lib.tvs_plan_create(0, 2, 64, 5, 1, ctypes.byref(plan)) == _native.TVS_E_INVALID
    assert b"depth" in lib.tvs_last_error()
    assert lib.tvs_plan_create(0, 17, 96, 5, 1, ctypes.byref(plan)) == _native.TVS_E_UNSUPPORTED
    assert lib.tvs_plan_create(0, 17, 64, 5, 1, None) == _native.TVS_E_INVALID
    assert lib.tvs_forward(None, None, None, None, 1, 1, 1, 0, -1, None) == _native.TVS_E_INVALID
    assert lib.tvs_forward_checked(None, None, None, None, None, 1, 1, 1, 0, -1, None) == _native.TVS_E_INVALID
    assert lib.tvs_plan_destroy(None) == 0
    assert lib.tvs_plan_set_option(None, b"stack", 1) == _native.TVS_E_INVALID
    assert lib.tvs_plan_sync(None, None) == _native.TVS_E_INVALID
    assert lib.tvs_last_used_stack(None) == 0
