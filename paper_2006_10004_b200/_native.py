"""ctypes binding of libtvsb200.so (include/tvs_b200.h).

The library is the product: there is no Python or CPU fallback.  Loading it
fails loudly if the .so is missing (run ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtvsb200.so"


def _lib_path() -> Path:
    """The product library, or a diagnostics build named by TVS_LIB (e.g.
    libtvsb200_trace.so from build.py --trace), read when the library loads."""
    return Path(os.environ["TVS_LIB"]).resolve() if os.environ.get("TVS_LIB") else LIB_PATH

TVS_OK = 0
TVS_E_INVALID = -1
TVS_E_UNSUPPORTED = -2
TVS_E_CUDA = -3
TVS_E_STATE = -4
TVS_E_NUMERIC = -5

MODE_FP32 = 0
MODE_FAST = 1

EXPORTS = (
    "tvs_abi_version",
    "tvs_last_error",
    "tvs_plan_create",
    "tvs_plan_create_ex",
    "tvs_plan_set_weights",
    "tvs_plan_set_option",
    "tvs_plan_sync",
    "tvs_forward",
    "tvs_forward_checked",
    "tvs_forward_host",
    "tvs_last_launch_count",
    "tvs_last_used_stack",
    "tvs_profile_enable",
    "tvs_profile_read",
    "tvs_profile_span",
    "tvs_plan_destroy",
    "tvs_band_stats",
    "tvs_tvflow_workspace_bytes",
    "tvs_tvflow_analyze",
    "tvs_train_create",
    "tvs_train_forward",
    "tvs_train_backward",
    "tvs_train_set_option",
    "tvs_train_destroy",
    "tvs_loss_sums",
    "tvs_loss_grad",
)

_lock = threading.Lock()
_lib = None


class TVSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libtvsb200 error {code}: {msg}")
        self.code = code


def load() -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Raises if the library is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _lib_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: the TVSpecNET B200 path has no CPU fallback; "
                "build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(path))
        P = ctypes.c_void_p
        i = ctypes.c_int
        lib.tvs_abi_version.restype = i
        lib.tvs_abi_version.argtypes = []
        lib.tvs_last_error.restype = ctypes.c_char_p
        lib.tvs_last_error.argtypes = []
        lib.tvs_plan_create.restype = i
        lib.tvs_plan_create.argtypes = [i, i, i, i, i, ctypes.POINTER(P)]
        lib.tvs_plan_create_ex.restype = i
        lib.tvs_plan_create_ex.argtypes = [i, i, i, i, i, i, ctypes.POINTER(P)]
        lib.tvs_plan_set_weights.restype = i
        lib.tvs_plan_set_weights.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), i, P]
        lib.tvs_plan_set_option.restype = i
        lib.tvs_plan_set_option.argtypes = [P, ctypes.c_char_p, ctypes.c_longlong]
        lib.tvs_plan_sync.restype = i
        lib.tvs_plan_sync.argtypes = [P, P]
        lib.tvs_last_used_stack.restype = i
        lib.tvs_last_used_stack.argtypes = [P]
        lib.tvs_forward.restype = i
        lib.tvs_forward.argtypes = [P, P, P, P, i, i, i, i, i, P]
        if hasattr(lib, "tvs_forward_checked"):  # (absent only in older diagnostics builds, TVS_LIB)
            lib.tvs_forward_checked.restype = i
            lib.tvs_forward_checked.argtypes = [P, P, P, P, P, i, i, i, i, i, P]
        lib.tvs_forward_host.restype = i
        lib.tvs_forward_host.argtypes = [P, P, P, P, i, i, i, P]
        lib.tvs_last_launch_count.restype = i
        lib.tvs_last_launch_count.argtypes = [P]
        lib.tvs_profile_enable.restype = i
        lib.tvs_profile_enable.argtypes = [P, i]
        lib.tvs_profile_read.restype = i
        lib.tvs_profile_read.argtypes = [P, i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong),
                                         ctypes.POINTER(ctypes.c_double)]
        lib.tvs_profile_span.restype = i
        lib.tvs_profile_span.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong), i]
        lib.tvs_band_stats.restype = i
        lib.tvs_band_stats.argtypes = [P, P, i, i, i, P, P, P]
        lib.tvs_tvflow_workspace_bytes.restype = ctypes.c_size_t
        lib.tvs_tvflow_workspace_bytes.argtypes = [i, i, i]
        d = ctypes.c_double
        lib.tvs_tvflow_analyze.restype = i
        lib.tvs_tvflow_analyze.argtypes = [P, i, i, i, d, i, P, i, i, d, d, d, i, P, P, P, P, P, P]
        lib.tvs_train_create.restype = i
        lib.tvs_train_create.argtypes = [i, i, i, ctypes.POINTER(P)]
        PP = ctypes.POINTER(P)
        lib.tvs_train_forward.restype = i
        lib.tvs_train_forward.argtypes = [P, PP, PP, PP, PP, ctypes.c_float, P, P, P, P, i, i, i, P]
        lib.tvs_train_backward.restype = i
        lib.tvs_train_backward.argtypes = [P, P, PP, PP, PP, PP, P]
        lib.tvs_train_set_option.restype = i
        lib.tvs_train_set_option.argtypes = [P, ctypes.c_char_p, ctypes.c_int]
        lib.tvs_train_destroy.restype = i
        lib.tvs_train_destroy.argtypes = [P]
        lib.tvs_loss_sums.restype = i
        lib.tvs_loss_sums.argtypes = [P, P, P, P, i, i, i, i, i, ctypes.c_float, P, P, P]
        lib.tvs_loss_grad.restype = i
        lib.tvs_loss_grad.argtypes = [P, P, P, P, i, i, i, i, i, ctypes.c_float, P, P, P, P]
        lib.tvs_plan_destroy.restype = i
        lib.tvs_plan_destroy.argtypes = [P]
        _lib = lib
        return lib


def check(code: int) -> None:
    if code != TVS_OK:
        msg = load().tvs_last_error().decode(errors="replace")
        if code == TVS_E_INVALID:
            raise ValueError(msg)
        if code == TVS_E_NUMERIC:
            raise FloatingPointError(f"libtvsb200: {msg}")
        raise TVSError(code, msg)


class Plan:
    """RAII owner of one ``tvs_plan`` (one device, one architecture, one mode)."""

    def __init__(self, device: int, depth: int, channels: int, out_bands: int, mode: int, unshuffle: int = 1):
        self.lib = load()
        self.handle = ctypes.c_void_p()
        check(self.lib.tvs_plan_create_ex(device, depth, channels, out_bands, mode, unshuffle,
                                          ctypes.byref(self.handle)))
        self.device, self.depth, self.channels, self.out_bands, self.mode = device, depth, channels, out_bands, mode
        self.unshuffle = unshuffle

    def set_weights(self, w_ptrs, scale_ptrs, shift_ptrs, stream: int) -> None:
        """Device pointers per layer; scale_ptrs entries may be 0 (= no BatchNorm)."""
        n = len(w_ptrs)
        W = (ctypes.c_void_p * n)(*w_ptrs)
        S = (ctypes.c_void_p * n)(*[p or None for p in scale_ptrs])
        Bv = (ctypes.c_void_p * n)(*shift_ptrs)
        check(self.lib.tvs_plan_set_weights(self.handle, W, S, Bv, n, ctypes.c_void_p(stream)))

    def set_option(self, name: str, value: int) -> None:
        """Plan option (include/tvs_b200.h tvs_plan_set_option)."""
        check(self.lib.tvs_plan_set_option(self.handle, name.encode(), int(value)))

    def sync(self, stream: int) -> None:
        """Synchronise `stream` and raise any deferred forward failure."""
        check(self.lib.tvs_plan_sync(self.handle, ctypes.c_void_p(stream)))

    def last_used_stack(self) -> bool:
        return bool(self.lib.tvs_last_used_stack(self.handle))

    def forward(self, x_ptr, bands_ptr, closure_ptr, B, H, W, row0, rows, stream: int) -> None:
        check(
            self.lib.tvs_forward(
                self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(bands_ptr),
                ctypes.c_void_p(closure_ptr) if closure_ptr else None,
                B, H, W, row0, rows, ctypes.c_void_p(stream),
            )
        )

    def forward_checked(self, x_ptr, bands_ptr, closure_ptr, recon_ptr, B, H, W, row0, rows, stream: int) -> None:
        """tvs_forward_checked: the forward plus the fused band-sum
        reconstruction check sums (recon: device float64 (B, 2))."""
        check(
            self.lib.tvs_forward_checked(
                self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(bands_ptr), ctypes.c_void_p(closure_ptr),
                ctypes.c_void_p(recon_ptr), B, H, W, row0, rows, ctypes.c_void_p(stream),
            )
        )

    def forward_host(self, x_ptr, bands_ptr, closure_ptr, B, H, W, stream: int) -> None:
        check(
            self.lib.tvs_forward_host(
                self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(bands_ptr),
                ctypes.c_void_p(closure_ptr) if closure_ptr else None, B, H, W, ctypes.c_void_p(stream),
            )
        )

    def last_launch_count(self) -> int:
        return int(self.lib.tvs_last_launch_count(self.handle))

    def profile_enable(self, on: bool) -> None:
        check(self.lib.tvs_profile_enable(self.handle, 1 if on else 0))

    def profile_read(self, kind: int) -> tuple[float, int, float]:
        """(device ms, launches, algorithmic FLOPs) for kind 0 conv0, 1 hidden, 2 head."""
        ms, n, fl = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        check(self.lib.tvs_profile_read(self.handle, kind, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl)))
        return ms.value, n.value, fl.value

    def profile_span(self, reset: bool = True) -> tuple[float, int]:
        """(device ms, launches) of the hidden-layer kernels since the last
        reset, measured inside the kernels (plan option "span")."""
        ms, n = ctypes.c_double(), ctypes.c_longlong()
        check(self.lib.tvs_profile_span(self.handle, ctypes.byref(ms), ctypes.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def close(self) -> None:
        if self.handle and self.handle.value:
            self.lib.tvs_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptrs(seq):
    return (ctypes.c_void_p * len(seq))(*[p or None for p in seq])


class TrainPlan:
    """RAII owner of one ``tvs_train`` (training step on one device)."""

    def __init__(self, device: int, depth: int, out_bands: int):
        self.lib = load()
        self.handle = ctypes.c_void_p()
        check(self.lib.tvs_train_create(device, depth, out_bands, ctypes.byref(self.handle)))
        self.device, self.depth, self.out_bands = device, depth, out_bands

    def forward(self, w, bias, gamma, beta, eps, x, out, mean, var, B, H, W, stream: int) -> None:
        check(self.lib.tvs_train_forward(self.handle, _ptrs(w), _ptrs(bias), _ptrs(gamma), _ptrs(beta),
                                         ctypes.c_float(eps), ctypes.c_void_p(x), ctypes.c_void_p(out),
                                         ctypes.c_void_p(mean), ctypes.c_void_p(var), B, H, W,
                                         ctypes.c_void_p(stream)))

    def backward(self, g_out, dw, dbias, dgamma, dbeta, stream: int) -> None:
        check(self.lib.tvs_train_backward(self.handle, ctypes.c_void_p(g_out), _ptrs(dw), _ptrs(dbias),
                                          _ptrs(dgamma), _ptrs(dbeta), ctypes.c_void_p(stream)))

    def set_option(self, name: str, value: int) -> None:
        check(self.lib.tvs_train_set_option(self.handle, name.encode(), int(value)))

    def close(self) -> None:
        if self.handle and self.handle.value:
            self.lib.tvs_train_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
