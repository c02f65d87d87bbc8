"""ctypes binding of libskc.so (the C ABI in include/skc.h).

This is the package's only route to compute: every public function of
engine/svfilter/optim calls one of the `skc_*` entry points below on device
memory.  The reference gates its compiled path with `_fastpath.HAVE_NUMBA`
(svfilter.py:18, 189-190); here `HAVE_CUDA` plays that role, except that there
is no CPU fallback -- without the library or a CUDA device the product raises
`NativeUnavailable` instead of computing something else.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libskc.so"

SKC_OK, SKC_EBADARG, SKC_ENONFINITE, SKC_ETRUNC, SKC_ECUDA, SKC_EDEGENERATE, SKC_ENOTTAKEN = 0, 1, 2, 3, 4, 5, 6
SKC_F32, SKC_F16, SKC_F64 = 0, 1, 2
SKC_ZERO, SKC_CLAMP = 0, 1
SKC_HWC, SKC_CHW = 0, 1
LOSS_IDS = {"charbonnier": 0, "l1": 1, "l2": 2}
WN_IDS = {"none": 0, "sum": 1, "sofm": 2}
FIT_HDR = 8

# Symbols declared in include/skc.h (checked by tests/test_abi.py).
EXPORTS = (
    "skc_version", "skc_last_error", "skc_release_scratch", "skc_max_taps", "skc_layer_fwd", "skc_layer_fwd_ex", "skc_relayout", "skc_chain_is_fused", "skc_chain_relayouts", "skc_chain_mid_dtype", "skc_layer_plan", "skc_sparse_compile_check", "skc_layer_pair_fwd", "skc_pair_compile_check", "skc_set_jit_mode", "skc_jit_wait",
    "skc_chain_fwd",
    "skc_sv_fwd", "skc_sv_grid_fwd", "skc_ir_batch", "skc_ir_energies", "skc_backward_batch", "skc_fit_init", "skc_fit_run",
    "skc_adam_step", "skc_pst_run", "skc_bilinear_sample", "skc_sv_ground_truth",
)


class NativeUnavailable(RuntimeError):
    """libskc.so or a CUDA device is missing: the product path cannot run."""


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class FitCfg(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int),
        ("lr_start", ctypes.c_float),
        ("lr_end", ctypes.c_float),
        ("beta1", ctypes.c_float),
        ("beta2", ctypes.c_float),
        ("eps", ctypes.c_float),
        ("weight_norm", ctypes.c_int),
        ("kws", ctypes.c_int),
        ("loss_kind", ctypes.c_int),
        ("loss_eps", ctypes.c_float),
    ]


class PstCfg(ctypes.Structure):
    _fields_ = [
        ("chains", ctypes.c_int),
        ("iterations", ctypes.c_int),
        ("swap_interval", ctypes.c_int),
        ("sum_normalize", ctypes.c_int),
        ("t_max", ctypes.c_double),
        ("t_min", ctypes.c_double),
        ("sigma_offset", ctypes.c_double),
        ("sigma_weight", ctypes.c_double),
        ("seed", ctypes.c_ulonglong),
        ("loss_kind", ctypes.c_int),
        ("loss_eps", ctypes.c_float),
    ]


_lib = None
_load_error = None

_vp = ctypes.c_void_p
_i = ctypes.c_int
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def _declare(lib):
    lib.skc_version.restype = _i
    lib.skc_last_error.restype = ctypes.c_char_p
    lib.skc_max_taps.restype = _i
    lib.skc_layer_fwd.argtypes = [_vp, _i, _vp, _i, _i, _i, _i, _i, _dp, _i, _i, _vp]
    lib.skc_layer_fwd_ex.argtypes = [_vp, _i, _i, _vp, _i, _i, _i, _i, _i, _i, _dp, _i, _i, _vp]
    lib.skc_relayout.argtypes = [_vp, _i, _i, _vp, _i, _i, _i, _i, _i, _i, _vp]
    lib.skc_chain_is_fused.argtypes = [_dp, _ip, _i, _i, _i, _i, _i]
    lib.skc_chain_relayouts.argtypes = [_dp, _ip, _i, _i, _i, _i, _i, _i]
    lib.skc_chain_mid_dtype.argtypes = [_ip, _i, _i, _i]
    lib.skc_sparse_compile_check.argtypes = [_dp, _i, _i, _i, _i, _i]
    lib.skc_layer_pair_fwd.argtypes = [_vp, _vp, _i, _i, _i, _i, _dp, _i, _dp, _i, _i, _vp]
    lib.skc_pair_compile_check.argtypes = [_dp, _i, _dp, _i]
    lib.skc_set_jit_mode.argtypes = [_i]
    lib.skc_jit_wait.argtypes = []
    lib.skc_layer_plan.argtypes = [_dp, _i, _i, _i, _i, _i, _ip, _ip]
    lib.skc_chain_fwd.argtypes = [_vp, _i, _vp, _i, _i, _i, _i, _i, _dp, _ip, _i, _i, _vp]
    lib.skc_sv_fwd.argtypes = [_vp, _i, _vp, _i, _i, _i, _i, _vp, _dp, _i, _dp, _i, _ip, _i, _i,
                               _vp]
    lib.skc_sv_grid_fwd.argtypes = [_vp, _vp, _i, _i, _i, _vp, _dp, _i, _dp, _i, _dp, _i, _ip, _i, _i, _vp]
    lib.skc_ir_batch.argtypes = [_vp, _i, _ip, _i, _i, _i, _vp, _vp]
    lib.skc_ir_energies.argtypes = [_vp, _i, _ip, _i, _i, _i, _vp, _i, _i, ctypes.c_float, _vp, _vp]
    lib.skc_backward_batch.argtypes = [_vp, _i, _ip, _i, _i, _vp, _i, _i, _i, ctypes.c_float,
                                       _vp, _vp, _vp, _vp]
    lib.skc_fit_init.argtypes = [_vp, _vp, _i, _ip, _i, _i, _i, ctypes.POINTER(FitCfg), _vp, _vp]
    lib.skc_fit_run.argtypes = [_vp, _i, _ip, _i, _i, _vp, _i, ctypes.POINTER(FitCfg), _vp, _vp,
                                _vp]
    lib.skc_adam_step.argtypes = [_vp, _vp, _vp, _vp, _ip, _i, _i, ctypes.POINTER(FitCfg),
                                  ctypes.c_float, _vp, _vp]
    lib.skc_pst_run.argtypes = [_vp, _ip, _i, _i, _i, _vp, _i, ctypes.POINTER(PstCfg), _vp, _dp, _vp, _dp,
                                _dp, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong), _vp]
    lib.skc_bilinear_sample.argtypes = [_vp, _i, _i, _i, _i, _vp, _vp, _vp, ctypes.c_longlong, ctypes.c_longlong,
                                        _vp, _vp]
    lib.skc_sv_ground_truth.argtypes = [_vp, _i, _i, _i, _vp, _vp, _i, _i, _vp, _vp]
    for name in EXPORTS[2:]:
        getattr(lib, name).restype = _i


def load_library():
    """Load libskc.so (no device needed).  Raises NativeUnavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        _load_error = f"{LIB_PATH} not built (run __graft_entry__.build())"
        raise NativeUnavailable(_load_error)
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        _load_error = str(exc)
        raise NativeUnavailable(_load_error) from exc
    try:
        _declare(lib)
    except AttributeError as exc:
        _load_error = f"{LIB_PATH} is stale ({exc}); rebuild with __graft_entry__.build()"
        raise NativeUnavailable(_load_error) from exc
    _lib = lib
    return lib


def _device_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def have_cuda() -> bool:
    try:
        load_library()
    except NativeUnavailable:
        return False
    return _device_ok()


def __getattr__(name):
    # HAVE_CUDA is resolved on first access, not at import: importing the
    # package (e.g. for its synthetic-input recipes) must not map libskc.so
    if name == "HAVE_CUDA":
        return have_cuda()
    raise AttributeError(name)


def lib():
    """The library, asserting a usable CUDA device (fails loudly otherwise)."""
    l = load_library()
    if not _device_ok():
        raise NativeUnavailable("no CUDA device: the sm_100a path cannot run here")
    return l


def last_error() -> str:
    return (load_library().skc_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc != SKC_OK:
        raise NativeError(rc, f"{what}: {last_error()}" if what else last_error())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dbl(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def ints(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def fit_cfg(steps, lr_start, lr_end, beta1, beta2, eps, weight_norm, kws, loss_kind, loss_eps):
    return FitCfg(int(steps), float(lr_start), float(lr_end), float(beta1), float(beta2), float(eps),
                  WN_IDS[weight_norm], int(bool(kws)), LOSS_IDS[loss_kind], float(loss_eps))


def release_scratch() -> None:
    """Return the library's cached scratch blocks to the driver (skc_release_scratch)."""
    import torch
    torch.cuda.synchronize()
    check(load_library().skc_release_scratch(), "release_scratch")


def set_jit_mode(sync: bool) -> None:
    """Generated-stencil compiles: True = synchronous on first use (every call
    of a layer runs the same kernel), False = background (default; the tap /
    dense kernels serve a layer until its kernel is ready)."""
    check(load_library().skc_set_jit_mode(1 if sync else 0), "set_jit_mode")


def jit_wait() -> None:
    """Block until every background stencil compile has finished."""
    check(load_library().skc_jit_wait(), "jit_wait")
