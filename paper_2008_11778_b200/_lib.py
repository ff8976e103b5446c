"""ctypes binding of libseisgpu.so (C ABI in include/seisgpu.h).

The library is loaded with ``ctypes.CDLL`` (releases the GIL during calls) on
first use.  There is no fallback: if the shared object is missing or no CUDA
device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .model import StabilityError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libseisgpu.so")

SG_OK, SG_ERR_ARG, SG_ERR_STABILITY, SG_ERR_EMPTY = 0, 1, 2, 3
SG_ERR_CUDA, SG_ERR_OOM, SG_ERR_MODEL, SG_ERR_STATE = 4, 5, 6, 7
SG_F32, SG_F64 = 4, 8
SG_RECON_FULL, SG_RECON_CHECKPOINT, SG_RECON_AUTO, SG_RECON_BOUNDARY = 0, 1, 2, 3
SG_BUILD_EXPERIMENTAL = 1


class EmptyWindowError(Exception):
    """Operation requires at least one stored column (seisopt/optim/qr.py:18-19)."""


class ModelError(ValueError):
    """Model is not positive and finite (seisopt/gradients.py:312-331)."""


class SeisGpuError(RuntimeError):
    """CUDA / resource failure inside libseisgpu."""


class SgDesc(C.Structure):
    _fields_ = [
        ("nz", C.c_int32), ("nx", C.c_int32),
        ("pad_top", C.c_int32), ("pad_bottom", C.c_int32),
        ("pad_left", C.c_int32), ("pad_right", C.c_int32),
        ("nt", C.c_int32), ("n_shots", C.c_int32), ("n_rec", C.c_int32),
        ("dtype", C.c_int32), ("order", C.c_int32), ("recon", C.c_int32),
        ("batch", C.c_int32), ("checkpoint_every", C.c_int32), ("device", C.c_int32),
        ("use_graphs", C.c_int32), ("group", C.c_int32), ("step_mode", C.c_int32),
        ("chains", C.c_int32), ("resident", C.c_int32),
        ("dx", C.c_double), ("dz", C.c_double), ("dt", C.c_double),
        ("cfl_safety", C.c_double), ("mem_budget_bytes", C.c_double),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)

# symbol -> (restype, argtypes); every symbol declared in include/seisgpu.h
SIGNATURES = {
    "sg_last_error": (C.c_char_p, []),
    "sg_version": (C.c_int, []),
    "sg_build_flags": (C.c_int, []),
    "sg_create": (C.c_int, [C.POINTER(SgDesc), C.POINTER(_P)]),
    "sg_destroy": (C.c_int, [_P]),
    "sg_set_stream": (C.c_int, [_P, _P]),
    "sg_set_sponge": (C.c_int, [_P, _DP, _DP]),
    "sg_set_geometry": (C.c_int, [_P, _IP, _IP, _DP, _IP, _IP, _DP, _D]),
    "sg_set_wavelet": (C.c_int, [_P, _DP]),
    "sg_set_model": (C.c_int, [_P, _P, _I32]),
    "sg_fwi_synthetic": (C.c_int, [_P, _I32, _I32, _P]),
    "sg_fwi_misfit": (C.c_int, [_P, _I32, _I32, _P, _DP]),
    "sg_fwi_gradient": (C.c_int, [_P, _I32, _I32, _P, _DP, _P, _I32]),
    "sg_born_cache": (C.c_int, [_P, _I32, _I32, _I32]),
    "sg_born_cached": (C.c_int, [_P, _IP, _IP]),
    "sg_born_forward": (C.c_int, [_P, _I32, _I32, _P, _P]),
    "sg_born_adjoint": (C.c_int, [_P, _I32, _I32, _P, _P, _I32]),
    "sg_lsrtm_gradient": (C.c_int, [_P, _I32, _I32, _P, _P, _DP, _P, _I32]),
    "sg_lsrtm_misfit": (C.c_int, [_P, _I32, _I32, _P, _P, _DP]),
    "sg_forward_history": (C.c_int, [_P, _I32, _P, _P]),
    "sg_adjoint_history": (C.c_int, [_P, _P, _P]),
    "sg_query": (C.c_int, [_P, _IP, _IP, _DP]),
    "sg_chains": (C.c_int, [_P, C.c_int32]),
    "sg_resident_plan": (C.c_int, [_P, _IP]),
    "sg_time_step_kernel": (C.c_int, [_P, _I32, _I32, _I32, C.POINTER(C.c_float)]),
    "sg_phase_times": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "sg_launch_count": (C.c_int64, []),
    "sg_last_nonfinite": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "sg_redzone_check": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64), _I32]),
    "sg_aa_create": (C.c_int, [_I64, _I32, _I32, _I32, C.POINTER(_P)]),
    "sg_aa_destroy": (C.c_int, [_P]),
    "sg_aa_set_stream": (C.c_int, [_P, _P]),
    "sg_aa_set_reducer": (C.c_int, [_P, _P, _P]),
    "sg_aa_clear": (C.c_int, [_P]),
    "sg_aa_push": (C.c_int, [_P, _P, _P]),
    "sg_aa_m_k": (C.c_int, [_P]),
    "sg_aa_weights": (C.c_int, [_P, _DP, _DP, _DP, _IP]),
    "sg_aa_step": (C.c_int, [_P, _D, _DP, _DP, _P]),
    "sg_aa_fk_norm": (C.c_int, [_P, _DP]),
    "sg_aa_set_qr": (C.c_int, [_P, _I32]),
    "sg_aa_qr_info": (C.c_int, [_P, _IP, C.POINTER(C.c_int64)]),
    "sg_vec_axpby": (C.c_int, [_I64, _I32, _D, _P, _D, _P, _P, _P]),
    "sg_vec_lerp": (C.c_int, [_I64, _I32, _P, _P, _D, _P, _P]),
    "sg_vec_blend_dots": (C.c_int, [_I64, _I32, _P, _P, _P, _P, _DP, _P]),
    "sg_vec_stats": (C.c_int, [_I64, _I32, _P, _DP, _P]),
    "sg_vec_multi_dot": (C.c_int, [_I64, _I32, _I32, C.POINTER(_P), _P, _DP, _P]),
    "sg_vec_multi_axpy": (C.c_int, [_I64, _I32, _I32, _DP, C.POINTER(_P), _P, _P, _P]),
}

# sg_reduce_fn: int (*)(double* buf, int32_t n, void* ctx)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int32, C.c_void_p)

_lock = threading.Lock()
_lib = None


def load(path: str | None = None):
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or os.environ.get("SG_LIB") or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"libseisgpu.so not built at {p}; run `python -m paper_2008_11778_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def redzone_check(poke=False):
    """(corrupted guard bytes, guarded allocations) of the SG_REDZONE=1 mode
    (include/seisgpu.h sg_redzone_check); allocations == 0: the mode is off."""
    bad, n = C.c_int64(), C.c_int64()
    check(load().sg_redzone_check(C.byref(bad), C.byref(n), 1 if poke else 0), "redzone_check")
    return bad.value, n.value


def last_error() -> str:
    return load().sg_last_error().decode(errors="replace")


def check(rc: int, what: str = ""):
    """Map a C return code onto the reference's exception types."""
    if rc == SG_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == SG_ERR_ARG:
        raise ValueError(msg)
    if rc == SG_ERR_STABILITY:
        raise StabilityError(msg)
    if rc == SG_ERR_EMPTY:
        raise EmptyWindowError(msg)
    if rc == SG_ERR_MODEL:
        raise ModelError(msg)
    raise SeisGpuError(f"[code {rc}] {msg}")


def experimental_kernels() -> bool:
    """Whether the opt-in two-step / cluster-resident kernels are compiled in
    (build with defines=("SG_EXPERIMENTAL=1",))."""
    return bool(load().sg_build_flags() & SG_BUILD_EXPERIMENTAL)


def launch_count() -> int:
    return int(load().sg_launch_count())


def dptr(t) -> C.c_void_p:
    """Device pointer of a contiguous torch CUDA tensor."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def hptr_d(a):
    return a.ctypes.data_as(_DP)


def hptr_i(a):
    return a.ctypes.data_as(_IP)
