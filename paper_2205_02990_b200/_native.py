"""Loader for the in-tree C-ABI library `_hbs_b200.so` (include/hbs_b200.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises NativeError.  Build it with `python __graft_entry__.py` or
`make -C paper_2205_02990_b200/csrc`.
"""

import ctypes
import os

from .errors import ConfigurationError, DimensionError, IllConditionedProbeError, NativeError

# HBS_B200_LIB overrides the path (development builds of kernel variants)
LIB_PATH = os.environ.get("HBS_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_hbs_b200.so")

HBS_OK = 0
HBS_ERR_DIMENSION = 1
HBS_ERR_CONFIGURATION = 2
HBS_ERR_ILL_CONDITIONED = 3
HBS_ERR_CUDA = 4
HBS_ERR_WORKSPACE = 5
HBS_ERR_UNSUPPORTED = 6

# Every symbol declared in include/hbs_b200.h, with its ctypes signature.
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_PP = ctypes.POINTER(ctypes.c_void_p)
SIGNATURES = {
    "hbs_b200_version": ([], ctypes.c_char_p),
    "hbs_level_workspace_bytes": ([_I64, _I, _I, _I, ctypes.POINTER(_SZ)], _I),
    "hbs_compress_level": ([_I64, _P, _P, _I, _I, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                            _P, _SZ, _P, _P], _I),
    "hbs_compress_level_profiled": ([_I64, _P, _P, _I, _I, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                     _P, _P, _SZ, _P, _P, ctypes.POINTER(ctypes.c_float)], _I),
    "hbs_launch_counter": ([], ctypes.c_ulonglong),
    "hbs_level_hint": ([ctypes.c_int], None),
    "hbs_probe_qr_scratch_bytes": ([_I64, _I, _I, ctypes.POINTER(_SZ)], _I),
    "hbs_basis_qr_scratch_bytes": ([_I64, _I, _I, ctypes.POINTER(_SZ)], _I),
    "hbs_basis_qr": ([_I64, _P, _P, _I, _I, _P, _P, _P, _P], _I),
    "hbs_gram_probe_factor": ([_I64, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P], _I),
    "hbs_basis_orth": ([_I64, _P, _P, _I, _I, _P, _P, _P, _P, _P], _I),
    "hbs_probe_qr": ([_I64, _P, _P, _I, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "hbs_root_workspace_bytes": ([_I, _I, ctypes.POINTER(_SZ)], _I),
    "hbs_compress_root": ([_P, _P, _I, _I, _D, _P, _P, _P, _P, _SZ, _P, _P], _I),
    "hbs_apply_workspace_bytes": ([_I, _I, _I64, ctypes.POINTER(_SZ)], _I),
    "hbs_apply": ([_I, _I, _I64, _I64, _PP, _PP, _PP, _PP, _PP, _P, _P, _P, _I, _P, _SZ, _P], _I),
    "hbs_apply_up": ([_I, _I, _I, _I64, _P, _PP, _PP, _PP, _P, _PP, _P], _I),
    "hbs_apply_root": ([_I, _I64, _P, _I, _P, _P, _P], _I),
    "hbs_apply_down": ([_I, _I, _I, _I64, _P, _PP, _PP, _I, _PP, _PP, _I, _PP, _PP, _P, _P, _P], _I),
    "hbs_dense_apply": ([_I64, _I64, _P, _P, _P, _I, _P], _I),
    "hbs_fill_log_kernel": ([_I64, _I64, _I64, _P, _P], _I),
}

_lib = None


def lib():
    """The loaded library (loads on first use; raises NativeError if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"CUDA extension {LIB_PATH} is not built; run `python __graft_entry__.py build` "
                "(there is no CPU fallback)")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (args, res) in SIGNATURES.items():
            if not hasattr(handle, name):
                raise NativeError(f"{LIB_PATH} does not export {name}")
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == HBS_OK:
        return
    if rc == HBS_ERR_DIMENSION:
        raise DimensionError(f"{what}: invalid dimensions")
    if rc == HBS_ERR_CONFIGURATION:
        raise ConfigurationError(f"{what}: probe count leaves nullity below the rank")
    if rc == HBS_ERR_ILL_CONDITIONED:
        raise IllConditionedProbeError(f"{what}: ill-conditioned probe block")
    names = {HBS_ERR_CUDA: "CUDA launch error", HBS_ERR_WORKSPACE: "workspace too small",
             HBS_ERR_UNSUPPORTED: "unsupported size"}
    raise NativeError(f"{what}: {names.get(rc, 'error')} (code {rc})")


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else t.data_ptr()


def ptr_array(values):
    arr = (ctypes.c_void_p * len(values))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr
