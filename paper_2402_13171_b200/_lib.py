"""ctypes binding of liblbw.so (include/lbw.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2402_13171_b200/csrc``).  There is no fallback: every entry point of
this package that computes goes through the sm_100a kernels, and a missing
library or missing GPU raises instead of silently running on the CPU.
"""

import ctypes
import os
import threading

from .errors import ConfigError

LIB_PATH = os.environ.get("LBW_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "liblbw.so")   # LBW_LIB: A/B builds of the library

ABI_VERSION = 2
LBW_PREC_DOUBLE = 0
LBW_PREC_SINGLE = 1
WALL_KINDS = {"none": 0, "no_slip": 1, "free_slip": 2}

LBW_OK = 0
LBW_EINVAL = -1
LBW_ECUDA = -2
LBW_ENONFINITE = -3
LBW_ESTATE = -4
LBW_ENOMEM = -5
LBW_ECOMM = -6

OP_BGK = 0
OP_CUMULANT = 1
MODE_EXACT = 0
MODE_FAST = 1
BC_PERIODIC = 0
BC_INFLOW_OUTFLOW = 1

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i32_p = ctypes.POINTER(ctypes.c_int32)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)


class DomainDesc(ctypes.Structure):
    _fields_ = [
        ("cells", ctypes.c_int64 * 3),
        ("slab_x0", ctypes.c_int64),
        ("slab_nx", ctypes.c_int64),
        ("periodic", ctypes.c_int32 * 3),
        ("op", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("boundary", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("omega", ctypes.c_double),
        ("rates", ctypes.c_double * 4),
        ("u_in", ctypes.c_double * 3),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("feq_in_given", ctypes.c_int32),
        ("feq_in", ctypes.c_double * 27),
        ("precision", ctypes.c_int32),
        ("walls", ctypes.c_int32 * 4),
        ("reserved32", ctypes.c_int32),
        ("reserved", ctypes.c_int64 * 5),
    ]


class AlmDesc(ctypes.Structure):
    _fields_ = [
        ("n_points", ctypes.c_int32),
        ("chord", _c_double_p),
        ("element_length", _c_double_p),
        ("twist", _c_double_p),
        ("polar_index", _c_i32_p),
        ("n_polars", ctypes.c_int32),
        ("polar_offset", _c_i32_p),
        ("polar_rows", _c_i32_p),
        ("polar_alpha", _c_double_p),
        ("polar_cl", _c_double_p),
        ("polar_cd", _c_double_p),
        ("velocity_scale", ctypes.c_double),
        ("rho_ref", ctypes.c_double),
        ("force_dt2", ctypes.c_double),
        ("force_den", ctypes.c_double),
        ("point_ring", _c_i32_p),
        ("area", _c_double_p),
        ("n_rings", ctypes.c_int32),
        ("ring_first", _c_i32_p),
        ("ring_count", _c_i32_p),
        ("ring_ct", _c_double_p),
        ("spread_kernel", ctypes.c_int32),
        ("reserved32", ctypes.c_int32),
        ("spread_epsilon", ctypes.c_double),
        ("reserved", ctypes.c_int64 * 6),
    ]


class KinDesc(ctypes.Structure):
    _fields_ = [
        ("n_components", ctypes.c_int32),
        ("parent", _c_i32_p),
        ("rel_p", _c_double_p),
        ("rel_T", _c_double_p),
        ("axis", _c_double_p),
        ("rate", _c_double_p),
        ("step_rotation", _c_double_p),
        ("spin", _c_double_p),
        ("line_first", _c_i32_p),
        ("line_count", _c_i32_p),
        ("offsets", _c_double_p),
        ("orientations", _c_double_p),
        ("local_frames", _c_double_p),
        ("dx", ctypes.c_double),
        ("advance_first", ctypes.c_int32),
        ("is_disk", _c_i32_p),
        ("disk_center", _c_double_p),
        ("reserved", ctypes.c_int64 * 8),
    ]


# name -> (restype, argtypes); exactly the declarations of include/lbw.h
_VP = ctypes.c_void_p
_I = ctypes.c_int
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
SIGNATURES = {
    "lbw_abi_version": (_I, []),
    "lbw_last_error": (ctypes.c_char_p, []),
    "lbw_device_count": (_I, []),
    "lbw_kernel_launches": (_I64, []),
    "lbw_collide_cumulant_batch": (_I, [_VP, _VP, _VP, _I64, _D, _D, _D, _D, _D, _D, _I]),
    "lbw_collide_bgk_batch": (_I, [_VP, _VP, _VP, _I64, _D, _D, _I]),
    "lbw_collide_cumulant_block": (_I, [_VP, _VP, _VP, _I64, _I64, _I64, _D, _D, _D, _D, _D,
                                        _D, _I]),
    "lbw_collide_bgk_block": (_I, [_VP, _VP, _VP, _I64, _I64, _I64, _D, _D, _I]),
    "lbw_moments_block": (_I, [_VP, _VP, _VP, _I64, _I64, _I64, _D]),
    "lbw_stream_pull_block": (_I, [_VP, _VP, _I64, _I64, _I64]),
    "lbw_domain_create": (_I, [ctypes.POINTER(DomainDesc), ctypes.POINTER(_VP)]),
    "lbw_domain_destroy": (_I, [_VP]),
    "lbw_domain_stream": (_I, [_VP, ctypes.POINTER(_VP)]),
    "lbw_domain_device_bytes": (_I64, [_VP]),
    "lbw_domain_upload_pdf": (_I, [_VP, _VP]),
    "lbw_domain_download_pdf": (_I, [_VP, _VP]),
    "lbw_domain_upload_pdf_device": (_I, [_VP, _VP]),
    "lbw_domain_fill_uniform": (_I, [_VP, _VP]),
    "lbw_domain_init_modes": (_I, [_VP, _D, _VP, _I32, _VP, _I32]),
    "lbw_domain_set_force": (_I, [_VP, _VP]),
    "lbw_domain_download_force": (_I, [_VP, _VP]),
    "lbw_domain_set_macro": (_I, [_VP, _VP, _VP]),
    "lbw_domain_download_macro": (_I, [_VP, _VP]),
    "lbw_domain_recompute_moments": (_I, [_VP, _VP]),
    "lbw_domain_step": (_I, [_VP, _I32]),
    "lbw_domain_step_index": (_I64, [_VP]),
    "lbw_domain_set_step_index": (_I, [_VP, _I64]),
    "lbw_domain_poll_nonfinite": (_I, [_VP, _I, _c_i64_p, _c_i64_p, _c_i32_p]),
    "lbw_domain_hold_collided": (_I, [_VP]),
    "lbw_domain_sync": (_I, [_VP]),
    "lbw_domain_sweep_timing": (_I, [_VP, _I]),
    "lbw_domain_sweep_time": (_I, [_VP, _c_double_p, _c_i64_p]),
    "lbw_alm_configure": (_I, [_VP, ctypes.POINTER(AlmDesc)]),
    "lbw_alm_configure_kinematics": (_I, [_VP, ctypes.POINTER(KinDesc)]),
    "lbw_alm_download_kinematics": (_I, [_VP, _VP, _VP, _VP]),
    "lbw_alm_kinematics_step": (_I64, [_VP]),
    "lbw_alm_set_kinematics": (_I, [_VP, _VP]),
    "lbw_alm_get": (_I, [_VP, _VP, _VP, _VP]),
    "lbw_alm_record_loads": (_I, [_VP, _I64]),
    "lbw_alm_read_loads": (_I, [_VP, _VP, _I64, _VP, _VP]),
    "lbw_alm_clamp_flags": (_I, [_VP, _c_i32_p]),
    "lbw_peer_blob_bytes": (_I64, []),
    "lbw_domain_export_handle": (_I, [_VP, _VP, _c_i64_p]),
    "lbw_domain_import_peers": (_I, [_VP, _VP, _VP]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    """liblbw.so is not built (run __graft_entry__.build())."""


def load():
    """Load liblbw.so once; raise LibraryMissing if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lbw_abi_version() != ABI_VERSION:
            raise LibraryMissing("liblbw.so ABI version mismatch")
        _lib = lib
        return lib


def last_error():
    return load().lbw_last_error().decode(errors="replace")


def check(rc, what=""):
    """Map an lbw status code onto the reference's exception classes."""
    if rc == LBW_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == LBW_EINVAL:
        raise ConfigError(msg)
    if rc == LBW_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"liblbw error {rc}: {msg}")


def require_gpu():
    lib = load()
    if lib.lbw_device_count() < 1:
        raise RuntimeError(
            "no CUDA device visible: this package runs its kernels on a B200 "
            "(there is no CPU fallback)")
    return lib


def ptr(a):
    """Raw pointer of a C-contiguous numpy array (None for None)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def dptr(a):
    """ctypes double* of a C-contiguous float64 array."""
    return a.ctypes.data_as(_c_double_p)


def iptr(a):
    """ctypes int32* of a C-contiguous int32 array."""
    return a.ctypes.data_as(_c_i32_p)


def kernel_launches():
    return int(load().lbw_kernel_launches())
