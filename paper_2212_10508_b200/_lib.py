"""ctypes binding of libparalangevin_b200.so (the C ABI in include/paralangevin_b200.h).

Device memory and streams come from PyTorch (plumbing); every computation is
a call into the CUDA library.  There is no CPU fallback: if the library or a
CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import sys as _sys
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libparalangevin_b200.so")

PL_OK, PL_EARG, PL_EBLOWUP, PL_EPOT, PL_ECUDA = 0, 2, 3, 4, 5

_lib = None
_lock = threading.Lock()

vp = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32
dbl = C.c_double
u64 = C.c_uint64
pd = C.POINTER(C.c_double)
pi64 = C.POINTER(C.c_int64)
pi32 = C.POINTER(C.c_int32)

# name -> (restype, argtypes)
SIGNATURES = {
    "pl_version": (C.c_int, []),
    "pl_last_error": (C.c_char_p, []),
    "pl_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "pl_ctx_set_stream": (C.c_int, [vp, vp]),
    "pl_ctx_synchronize": (C.c_int, [vp]),
    "pl_ctx_destroy": (C.c_int, [vp]),
    "pl_derive_seeds": (C.c_int, [vp, u64, i64, vp]),
    "pl_gaussian_streams": (C.c_int, [vp, vp, i64, i64, vp]),
    "pl_pot_free": (C.c_int, [vp, C.POINTER(vp)]),
    "pl_pot_harmonic": (C.c_int, [vp, i64, pd, C.POINTER(vp)]),
    "pl_pot_double_well": (C.c_int, [vp, i64, pd, pd, C.POINTER(vp)]),
    "pl_pot_lj": (C.c_int, [vp, dbl, dbl, C.c_int, C.c_int, C.POINTER(vp)]),
    "pl_pot_perturbed": (C.c_int, [vp, vp, vp, dbl, C.POINTER(vp)]),
    "pl_pot_eam": (C.c_int, [vp, C.c_int, pd, dbl, C.c_int, dbl, pd, pd, C.c_int, dbl, pd,
                             C.POINTER(vp)]),
    "pl_pot_snap": (C.c_int, [vp, C.c_int, pd, C.c_int, dbl, dbl, dbl, C.c_int, dbl, pd,
                              C.c_int, C.POINTER(vp)]),
    "pl_pot_destroy": (C.c_int, [vp]),
    "pl_snap_bispectrum": (C.c_int, [vp, vp, i64, vp, vp]),
    "pl_snap_info": (C.c_int, [vp, pi32, pd]),
    "pl_pot_flops": (C.c_double, [vp]),
    "pl_neighbours": (C.c_int, [vp, vp, i64, vp, C.c_int, vp, vp]),
    "pl_compute": (C.c_int, [vp, vp, i64, i64, vp, vp, vp, vp]),
    "pl_propagate_windows": (C.c_int, [vp, vp, i64, i64, C.c_int, vp, vp, vp, pd, vp, dbl, dbl,
                                       dbl, vp, vp, vp]),
    "pl_propagate_windows_moments": (C.c_int, [vp, vp, i64, i64, C.c_int, vp, vp, vp, pd, vp, dbl, dbl,
                                               dbl, vp, vp, vp, vp, vp]),
    "pl_minimize": (C.c_int, [vp, vp, i64, i64, vp, dbl, i64, pi32, pi64, pd]),
    "pl_sweep": (C.c_int, [vp, vp, i64, C.c_int, i64, i64, C.c_int, vp, vp, vp, vp, vp, vp, vp,
                           vp, pd, vp, dbl, dbl, dbl, dbl, pd, vp, pi64, pi32]),
    "pl_sub": (C.c_int, [vp, i64, vp, vp, vp]),
    "pl_sweep_batch": (C.c_int, [vp, vp, i64, C.c_int, i64, C.c_int, pi32, pi64, pi64, pi32, C.c_int, vp, vp,
                                 vp, vp, vp, vp, vp, pd, vp, dbl, dbl, dbl, dbl, pd, pi64, vp]),
    "pl_bootstrap": (C.c_int, [vp, vp, i64, C.c_int, i64, i64, vp, vp, vp, vp, vp, pd, vp, dbl, dbl, dbl,
                               pi64, pi32]),
    "pl_sia_sites": (C.c_int, [vp, i64, C.c_int, C.c_int, dbl, vp, vp]),
    "pl_prof_begin": (C.c_int, [vp]),
    "pl_prof_end": (C.c_int, [vp, C.c_int, pd, pi64]),
    "pl_fp64_peak": (C.c_int, [vp, pd]),
    "pl_ctx_set_spec": (C.c_int, [vp, C.c_int]),
    "pl_ctx_enable_progress": (C.c_int, [vp, C.POINTER(C.c_void_p)]),
    "pl_sweep_path": (C.c_int, [vp]),
    "pl_pot_overflow_async": (C.c_int, [vp, vp, vp]),
    "pl_dmma_peak": (C.c_int, [vp, pd]),
    "pl_yi_timing": (C.c_int, [vp]),
}


class LibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or a CUDA call failed."""


class CallError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code
        self.message = message


def load():
    """Load (building first if the .so is missing or stale) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = LIB_PATH
        variant = os.environ.get("PL_LIB_VARIANT")  # A/B builds (build.py --variant), never built here
        if variant:
            path = os.path.join(HERE, f"libparalangevin_b200_{variant}.so")
        elif not os.path.exists(LIB_PATH) or os.environ.get("PL_REBUILD"):
            from . import build as _build
            _build.build()
        try:
            lib = C.CDLL(path)
        except OSError as exc:  # no silent fallback
            raise LibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != PL_OK:
        msg = _lib.pl_last_error().decode(errors="replace")
        raise CallError(rc, msg)


def exported_symbols():
    return list(SIGNATURES)


# ---------------------------------------------------------------- context
class Context:
    """One library context per (device, thread); stream = torch's current stream."""

    def __init__(self, device: int):
        lib = load()
        self.device = device
        self.handle = vp()
        check(lib.pl_ctx_create(device, None, C.byref(self.handle)))

    def bind_stream(self):
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(_lib.pl_ctx_set_stream(self.handle, vp(s)))
        return self.handle

    def __del__(self):
        # at interpreter shutdown the CUDA runtime may already be gone: leave it to the driver
        try:
            if _sys.is_finalizing():
                return
            if _lib is not None and self.handle:
                _lib.pl_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx_local = threading.local()


def context(device: int | None = None) -> Context:
    import torch
    if not torch.cuda.is_available():
        raise LibraryError("paralangevin_b200 needs a CUDA device (none visible); "
                           "there is no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    cache = getattr(_ctx_local, "ctxs", None)
    if cache is None:
        cache = _ctx_local.ctxs = {}
    if device not in cache:
        cache[device] = Context(device)
    ctx = cache[device]
    ctx.bind_stream()
    return ctx


def ptr(t) -> vp:
    """Device pointer of a contiguous torch tensor (or NULL for None)."""
    if t is None:
        return vp(0)
    assert t.is_contiguous(), "tensor must be contiguous"
    return vp(t.data_ptr())


def dptr(arr) -> pd:
    """Host pointer of a contiguous float64 numpy array."""
    return arr.ctypes.data_as(pd)
