"""Drop-in replacements of lbwind._kernels (/root/reference/pkg/src/lbwind/
_kernels.py:304-445) on host arrays, running the sm_100a kernels through
liblbw (copy in, one kernel, copy out).  Same signatures and in-place
semantics; the float64 ghosted block layout (nx+2, ny+2, nz+2, ncomp).
The time step itself does not use these: it keeps state on the device
(paper_2402_13171_b200.sim).
"""

import numpy as np

from . import _lib


def _c(a, ncomp):
    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.shape[-1] != ncomp:
        raise ValueError(f"expected a C-contiguous float64 array with last axis {ncomp}")
    return a


def _dims(f):
    return tuple(int(s) - 2 for s in f.shape[:3])


def collide_bgk_block(f, force, macro, omega, dt, mode=_lib.MODE_EXACT):
    lib = _lib.require_gpu()
    _c(f, 27), _c(force, 3), _c(macro, 4)
    _lib.check(lib.lbw_collide_bgk_block(_lib.ptr(f), _lib.ptr(force), _lib.ptr(macro),
                                         *_dims(f), float(omega), float(dt), mode))


def collide_cumulant_block(f, force, macro, omega, w3, w4, w5, w6, dt, mode=_lib.MODE_EXACT):
    lib = _lib.require_gpu()
    _c(f, 27), _c(force, 3), _c(macro, 4)
    _lib.check(lib.lbw_collide_cumulant_block(
        _lib.ptr(f), _lib.ptr(force), _lib.ptr(macro), *_dims(f), float(omega), float(w3),
        float(w4), float(w5), float(w6), float(dt), mode))


def moments_block(f, force, macro, dt):
    lib = _lib.require_gpu()
    _c(f, 27), _c(force, 3), _c(macro, 4)
    _lib.check(lib.lbw_moments_block(_lib.ptr(f), _lib.ptr(force), _lib.ptr(macro),
                                     *_dims(f), float(dt)))


def stream_pull_block(fsrc, fdst):
    lib = _lib.require_gpu()
    _c(fsrc, 27), _c(fdst, 27)
    if fsrc.shape != fdst.shape:
        raise ValueError("fsrc and fdst shapes differ")
    _lib.check(lib.lbw_stream_pull_block(_lib.ptr(fsrc), _lib.ptr(fdst), *_dims(fsrc)))


def collide_bgk_batch(f2, F2, macro2, omega, dt, mode=_lib.MODE_EXACT):
    lib = _lib.require_gpu()
    _c(f2, 27), _c(F2, 3), _c(macro2, 4)
    _lib.check(lib.lbw_collide_bgk_batch(_lib.ptr(f2), _lib.ptr(F2), _lib.ptr(macro2),
                                         f2.shape[0], float(omega), float(dt), mode))


def collide_cumulant_batch(f2, F2, macro2, omega, w3, w4, w5, w6, dt, mode=_lib.MODE_EXACT):
    lib = _lib.require_gpu()
    _c(f2, 27), _c(F2, 3), _c(macro2, 4)
    _lib.check(lib.lbw_collide_cumulant_batch(
        _lib.ptr(f2), _lib.ptr(F2), _lib.ptr(macro2), f2.shape[0], float(omega), float(w3),
        float(w4), float(w5), float(w6), float(dt), mode))


def warm_up(dtypes=(np.float64,)):
    """Kernels are compiled ahead of time (sm_100a cubins in liblbw.so);
    this only loads the library and creates the CUDA context."""
    _lib.require_gpu()
