"""ctypes binding of the sm_100a library (include/d2ip_b200.h).

The shared object is built in-tree by `build_ext.py` (or
`__graft_entry__.build()`). There is no fallback: if it is missing or fails to
load, every compute call raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import NativeLibraryError

LIB_PATH = Path(__file__).resolve().parent / "_d2ip_b200.so"
ABI_VERSION = 4
ARCH_CONFIG_RESUNET = 0  # D2IP_ARCH_* (include/d2ip_b200.h)
ARCH_FAST_RESUNET = 1

PREC = {"fp32": 0, "tf32": 1, "bf16": 2}
NORM = {"l2sq": 0, "l2": 1}

E_ARG = -1


class Act(C.Structure):
    """d2ip_act: NDHWC activation view."""

    _fields_ = [
        ("ptr", C.c_void_p),
        ("d", C.c_int),
        ("h", C.c_int),
        ("w", C.c_int),
        ("c", C.c_int),
        ("cstride", C.c_int),
        ("bstride", C.c_longlong),
        ("bf16", C.c_void_p),  # optional bf16 twin (same element layout); NULL = none
    ]


class NetDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int),
        ("R", C.c_int),
        ("C", C.c_int),
        ("P", C.c_int),
        ("levels", C.c_int),
        ("channels", C.c_int * 8),
        ("in_channels", C.c_int),
        ("negative_slope", C.c_float),
        ("M", C.c_int),
        ("V", C.c_int),
        ("Vp", C.c_int),
        ("n_rhs", C.c_int),
        ("j_shared", C.c_int),
        ("data_norm", C.c_int),
        ("lo", C.c_float),
        ("hi", C.c_float),
        ("lr", C.c_float),
        ("beta1", C.c_float),
        ("beta2", C.c_float),
        ("eps", C.c_float),
        ("precision", C.c_int),
        ("lambda_tv", C.c_float),
        ("lambda_s", C.c_float),
        ("lambda_t", C.c_float),
        ("tv_eps", C.c_float),
        ("max_history", C.c_int),
        ("max_iters", C.c_int),
        ("arch", C.c_int),
        ("depthwise", C.c_int),
        ("n_dil", C.c_int),
        ("dil", C.c_int * 8),
    ]


class Bindings(C.Structure):
    _fields_ = [
        ("theta", C.c_void_p),
        ("grad", C.c_void_p),
        ("adam_m", C.c_void_p),
        ("adam_v", C.c_void_p),
        ("z", C.c_void_p),
        ("J", C.c_void_p),
        ("vox_of_col", C.c_void_p),
        ("col_of_vox", C.c_void_p),
        ("dv", C.c_void_p),
        ("history", C.c_void_p),
        ("mapped", C.c_void_p),
        ("sig", C.c_void_p),
        ("trace", C.c_void_p),
        ("status", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


_SIGS = {
    "d2ip_abi_version": (C.c_int, []),
    "d2ip_last_error": (C.c_char_p, []),
    "d2ip_last_variant": (C.c_char_p, []),
    "d2ip_trace_begin": (C.c_int, []),
    "d2ip_trace_dump": (C.c_int, [C.c_char_p, C.c_size_t]),
    "d2ip_set_wgrad_variant": (C.c_int, [C.c_int]),
    "d2ip_get_wgrad_variant": (C.c_int, []),
    "d2ip_assemble_sensitivity": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                            C.c_double, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "d2ip_conv3d_ws_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "d2ip_conv3d_fwd": (C.c_int, [Act, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_int, Act, C.c_int,
                                  C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "d2ip_conv3d_dgrad": (C.c_int, [Act, C.c_void_p, C.c_longlong, C.c_int, C.c_int, Act, C.c_int, C.c_int,
                                    C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "d2ip_conv3d_wgrad_ws_bytes": (C.c_size_t, [Act, Act, C.c_int, C.c_int]),
    "d2ip_conv3d_wgrad": (C.c_int, [Act, Act, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_size_t,
                                    C.c_int, C.c_int, C.c_void_p]),
    "d2ip_norm_act_fwd": (C.c_int, [Act, C.c_void_p, C.c_void_p, C.c_longlong, Act, C.c_int, C.c_float, Act,
                                    C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "d2ip_norm_act_bwd_ws_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "d2ip_norm_act_bwd": (C.c_int, [Act, Act, C.c_int, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_longlong, Act, Act, C.c_void_p, C.c_longlong, C.c_void_p, C.c_size_t,
                                    C.c_int, C.c_void_p]),
    "d2ip_upsample2x_fwd": (C.c_int, [Act, Act, C.c_int, C.c_void_p]),
    "d2ip_upsample2x_bwd": (C.c_int, [Act, Act, C.c_int, C.c_int, C.c_void_p]),
    "d2ip_jac_nseg": (C.c_int, [C.c_int]),
    "d2ip_jac_fwd": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_int, C.c_int, C.c_void_p,
                               C.c_int, C.c_int, C.c_void_p]),
    "d2ip_jac_adj_ws_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "d2ip_jac_adj": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_longlong,
                               C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "d2ip_adam": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_float, C.c_float,
                            C.c_float, C.c_float, C.c_void_p, C.c_void_p]),
    "d2ip_tv4d_ws_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    "d2ip_tv4d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                            C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "d2ip_project_f64": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "d2ip_engine_create": (C.c_int, [C.POINTER(NetDesc), C.POINTER(C.c_void_p)]),
    "d2ip_engine_destroy": (None, [C.c_void_p]),
    "d2ip_engine_param_count": (C.c_longlong, [C.c_void_p]),
    "d2ip_engine_workspace_bytes": (C.c_size_t, [C.c_void_p]),
    "d2ip_engine_bind": (C.c_int, [C.c_void_p, C.POINTER(Bindings)]),
    "d2ip_engine_set_history": (C.c_int, [C.c_void_p, C.c_int]),
    "d2ip_engine_reset_frame": (C.c_int, [C.c_void_p, C.c_void_p]),
    "d2ip_engine_step": (C.c_int, [C.c_void_p, C.c_void_p]),
    "d2ip_engine_run": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "d2ip_engine_forward": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "d2ip_engine_grads": (C.c_int, [C.c_void_p, C.c_void_p]),
    "d2ip_engine_grads_graph": (C.c_int, [C.c_void_p, C.c_void_p]),
    "d2ip_engine_predict": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "d2ip_engine_adam": (C.c_int, [C.c_void_p, C.c_void_p]),
    "d2ip_engine_launches_per_iter": (C.c_int, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib():
    """Load (once) and return the ctypes library; raise if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH.name} is not built; run `python build_ext.py` (no CPU fallback exists)"
            )
        try:
            h = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise NativeLibraryError(f"failed to load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        if h.d2ip_abi_version() != ABI_VERSION:
            raise NativeLibraryError("ABI version mismatch; rebuild the extension")
        _lib = h
        return h


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().d2ip_last_error().decode(errors="replace")
    if rc == E_ARG:
        raise ValueError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def act(t, d, h, w, c, cstride=None, offset=0, bstride=None) -> Act:
    """Act view over a CUDA tensor laid out [B][d][h][w][cstride]."""
    cs = c if cstride is None else cstride
    a = Act()
    a.ptr = t.data_ptr() + offset * t.element_size() if t is not None else None
    a.d, a.h, a.w, a.c, a.cstride = d, h, w, c, cs
    a.bstride = d * h * w * cs if bstride is None else bstride
    return a


def null_act() -> Act:
    return Act()
