"""Inner products and linear combinations of N-vectors for the Krylov and
quasi-Newton loops.

CUDA tensors go through libseisgpu's fused vector kernels
(``sg_vec_multi_dot`` / ``sg_vec_multi_axpy``, csrc/sg_aa.cu): one pass over
k vectors with fp64 accumulation, only the k scalars reach the host.  They
replace the reference's ``np.dot`` / ``x -= a * y`` on host arrays
(seisopt/krylov.py:77-94, :189; seisopt/optim/quasi_newton.py:24-54,
seisopt/optim/linesearch.py:49-66).

Host (CPU) tensors -- a problem whose vectors live on the host, e.g. the
quadratic test problems -- are combined with torch on the host in fp64, like
the reference does with NumPy; device vectors never take that path, and a
missing library raises.
"""

from __future__ import annotations

import ctypes as C

from . import _lib

MAX_K = 32  # sg_vec_multi_* take at most this many vectors per pass


def _torch():
    import torch
    return torch


def _dt(t):
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.SG_F32
    if t.dtype == torch.float64:
        return _lib.SG_F64
    raise ValueError("vectors must be float32 or float64")


def _stream(t):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _flat(t):
    t = t.reshape(-1)
    return t if t.is_contiguous() else t.contiguous()


def dots(xs, y):
    """([<x_i, y> for x_i in xs], <y, y>) in one pass over the vectors."""
    y = _flat(y)
    xs = [_flat(x) for x in xs]
    if not y.is_cuda:
        yd = y.double()
        return [float(x.double().dot(yd)) for x in xs], float(yd.dot(yd))
    out_d, yy = [], 0.0
    lib = _lib.load()
    for c0 in range(0, max(1, len(xs)), MAX_K):
        chunk = xs[c0:c0 + MAX_K]
        k = len(chunk)
        ptrs = (C.c_void_p * max(k, 1))(*[x.data_ptr() for x in chunk])
        out = (C.c_double * (k + 1))()
        for x in chunk:
            if x.device != y.device or x.dtype != y.dtype or x.numel() != y.numel():
                raise ValueError("vectors must share device, dtype and length")
        _lib.check(lib.sg_vec_multi_dot(y.numel(), _dt(y), k, ptrs, _lib.dptr(y), out,
                                        _stream(y)), "vec_multi_dot")
        out_d += [out[i] for i in range(k)]
        yy = out[k]
    return out_d, yy


def dot(x, y):
    return dots([x], y)[0][0]


def norm(x):
    return dots([], x)[1] ** 0.5


def axpy(coefs, xs, y=None, out=None):
    """out = y + sum_i coefs[i] xs[i] (y None: the plain combination); fp64
    per element, accumulated in the order y, x_0, x_1, ...  ``out`` may be y."""
    torch = _torch()
    xs = [_flat(x) for x in xs]
    ref = y if y is not None else xs[0]
    ref = _flat(ref)
    if out is None:
        out = torch.empty_like(ref)
    if not ref.is_cuda:
        acc = ref.double().clone() if y is not None else torch.zeros_like(ref, dtype=torch.float64)
        for c, x in zip(coefs, xs):
            acc += float(c) * x.double()
        out.reshape(-1).copy_(acc)
        return out
    lib = _lib.load()
    o = out.reshape(-1)
    base = None if y is None else _flat(y)
    for c0 in range(0, max(1, len(xs)), MAX_K):
        chunk = xs[c0:c0 + MAX_K]
        cs = [float(c) for c in coefs[c0:c0 + MAX_K]]
        k = len(chunk)
        ptrs = (C.c_void_p * max(k, 1))(*[x.data_ptr() for x in chunk])
        cf = (C.c_double * max(k, 1))(*cs)
        yp = C.c_void_p(0) if base is None else _lib.dptr(base)
        _lib.check(lib.sg_vec_multi_axpy(o.numel(), _dt(o), k, cf, ptrs, yp, _lib.dptr(o),
                                         _stream(o)), "vec_multi_axpy")
        base = o  # later chunks accumulate onto the partial result
    return out


def scale(c, x, out=None):
    return axpy([c], [x], None, out)
