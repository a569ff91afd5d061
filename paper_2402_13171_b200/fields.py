"""Host view of one device-resident slab (the PdfField surface of
lbwind.fields, fields.py:22-67).

The populations live on the GPU as two [x+1][27][y][z] buffers of the run's
storage dtype (fp64, or fp32 with ``precision: single``; arithmetic is fp64
either way, _kernels.py:5-7); this object exposes the reference's accessors
on demand, as arrays of that dtype:

    interior        (nx,ny,nz,27)  f_n, the post-stream state between steps
    interior_force  (nx,ny,nz,3)   the force of the latest collide (or the
                                   user-set body force)
    interior_macro  (nx,ny,nz,4)   (rho, u) the next actuator step samples

Reading downloads a fresh copy.  The returned arrays write through: any
item assignment (``fld.interior[...] = x``, ``fld.interior_force[..., 0] =
F``, augmented assignment) uploads the whole array back, so the
reference's in-place idioms keep working on device state.
"""

import numpy as np

from . import _lib
from .collision import equilibrium_pdf, product_equilibrium


class _WriteThrough(np.ndarray):
    """ndarray whose item assignment pushes the root array to the device."""

    def __array_finalize__(self, obj):
        self._push = getattr(obj, "_push", None)
        self._root = getattr(obj, "_root", None)

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        if self._push is not None:
            self._push(self._root)


def _write_through(arr, push):
    out = arr.view(_WriteThrough)
    out._push = push
    out._root = out
    return out


def fourier_modes(cells, u0, intensity=0.05, n_modes=32, seed=2402):
    """(n_modes, 7) table (kx, ky, kz, ax, ay, az, phase) of a seeded
    "turbulent-like" velocity perturbation for DeviceField.initialize_modes
    (u = U e_x + du, du a random Fourier field at ~5 %
    intensity).  Wavenumbers are whole periods of the domain (1..4 per
    axis), amplitudes are perpendicular to k (divergence free) and scaled
    so the rms of |du| is intensity * |u0|."""
    rng = np.random.default_rng(seed)
    L = np.asarray(cells, dtype=np.float64)
    out = np.zeros((n_modes, 7))
    for m in range(n_modes):
        k = 2.0 * np.pi * rng.integers(1, 5, 3) * rng.choice([-1, 1], 3) / L
        a = rng.normal(size=3)
        a -= (a @ k) / (k @ k) * k
        out[m, 0:3], out[m, 3:6], out[m, 6] = k, a, rng.uniform(0.0, 2.0 * np.pi)
    rms = np.sqrt(0.5 * np.sum(out[:, 3:6] ** 2))
    out[:, 3:6] *= intensity * np.linalg.norm(u0) / rms
    return out


class DeviceField:
    def __init__(self, sim, size, origin, block_id=0):
        self._sim = sim
        self.size = tuple(int(s) for s in size)
        self.origin = tuple(int(o) for o in origin)
        self.block_id = int(block_id)
        self.dtype = np.dtype(sim.cfg.dtype)

    def _stored(self, out):
        # device values of a single-precision field are fp32-representable:
        # the cast is exact
        return out if self.dtype == np.float64 else out.astype(self.dtype)

    # -- device handle
    @property
    def _d(self):
        return self._sim._domain

    def cell_count(self):
        nx, ny, nz = self.size
        return nx * ny * nz

    # -- populations
    def download_pdf(self):
        out = np.empty(self.size + (27,))
        _lib.check(_lib.load().lbw_domain_download_pdf(self._d, _lib.ptr(out)), "download")
        return self._stored(out)

    def upload_pdf(self, f):
        f = np.ascontiguousarray(np.broadcast_to(np.asarray(f, dtype=np.float64),
                                                 self.size + (27,)))
        _lib.check(_lib.load().lbw_domain_upload_pdf(self._d, _lib.ptr(f)), "upload")

    @property
    def interior(self):
        return _write_through(self.download_pdf(), lambda a: self.upload_pdf(np.asarray(a)))

    @interior.setter
    def interior(self, value):
        self.upload_pdf(value)

    @property
    def f(self):
        """Snapshot of PdfField.f (fields.py:32): the populations with a
        zero one-cell ghost ring (ghosts live only inside the device sweep)."""
        nx, ny, nz = self.size
        out = np.zeros((nx + 2, ny + 2, nz + 2, 27), self.dtype)
        out[1:-1, 1:-1, 1:-1] = self.download_pdf()
        return out

    # -- force
    def download_force(self):
        out = np.empty(self.size + (3,))
        _lib.check(_lib.load().lbw_domain_download_force(self._d, _lib.ptr(out)), "force")
        return self._stored(out)

    def set_force(self, force):
        if force is None:
            _lib.check(_lib.load().lbw_domain_set_force(self._d, None), "force")
            return
        force = np.ascontiguousarray(np.broadcast_to(np.asarray(force, dtype=np.float64),
                                                     self.size + (3,)))
        _lib.check(_lib.load().lbw_domain_set_force(self._d, _lib.ptr(force)), "force")

    @property
    def interior_force(self):
        return _write_through(self.download_force(), lambda a: self.set_force(np.asarray(a)))

    @interior_force.setter
    def interior_force(self, value):
        self.set_force(value)

    # -- macro
    def download_macro(self):
        out = np.empty(self.size + (4,))
        _lib.check(_lib.load().lbw_domain_download_macro(self._d, _lib.ptr(out)), "macro")
        return self._stored(out)

    def set_macro(self, macro):
        macro = np.ascontiguousarray(np.broadcast_to(np.asarray(macro, dtype=np.float64),
                                                     self.size + (4,)))
        _lib.check(_lib.load().lbw_domain_set_macro(self._d, _lib.ptr(macro), None), "macro")

    @property
    def interior_macro(self):
        return _write_through(self.download_macro(), lambda a: self.set_macro(np.asarray(a)))

    @interior_macro.setter
    def interior_macro(self, value):
        self.set_macro(value)

    def initialize_modes(self, rho, u0, modes, product=False):
        """initialize_equilibrium with u(x) = u0 + sum_m a_m sin(k_m.x + phi_m)
        evaluated on the device (no lattice-sized host array; fourier_modes)."""
        modes = np.ascontiguousarray(np.asarray(modes, dtype=np.float64).reshape(-1, 7))
        u0 = np.ascontiguousarray(np.asarray(u0, dtype=np.float64).reshape(3))
        _lib.check(_lib.load().lbw_domain_init_modes(self._d, float(rho), _lib.ptr(u0),
                                                     modes.shape[0], _lib.ptr(modes),
                                                     int(bool(product))), "init")

    def initialize_equilibrium(self, rho, u, product=False):
        """Interior populations at equilibrium of (rho, u); the sampled macro
        becomes exactly (rho, u) and the force field is cleared
        (fields.py:54-67).  rho scalar or (nx,ny,nz); u (3,) or (nx,ny,nz,3)."""
        n = self.size
        rho_arr = np.broadcast_to(np.asarray(rho, np.float64), n)
        u_arr = np.broadcast_to(np.asarray(u, np.float64), n + (3,))
        uniform = np.ndim(rho) == 0 and np.shape(u) == (3,)
        self.set_force(None)
        lib = _lib.load()
        if uniform:
            # one cell's equilibrium, evaluated by the same numpy expression,
            # replicated on the device (no lattice-sized host array)
            one = np.ascontiguousarray((product_equilibrium if product else equilibrium_pdf)(
                np.asarray(rho, np.float64), np.asarray(u, np.float64)), dtype=np.float64)
            _lib.check(lib.lbw_domain_fill_uniform(self._d, _lib.ptr(one)), "init")
        else:
            self.upload_pdf((product_equilibrium if product else equilibrium_pdf)(rho_arr, u_arr))
        if uniform:
            u4 = np.array([float(rho), *np.asarray(u, np.float64)])
            _lib.check(lib.lbw_domain_set_macro(self._d, None, _lib.ptr(u4)), "macro")
        else:
            m = np.empty(n + (4,))
            m[..., 0] = rho_arr
            m[..., 1:4] = u_arr
            self.set_macro(m)


class PdfField:
    """Host block storage of the reference (fields.py:22-67): f, f_next,
    force, macro as (nx+2, ny+2, nz+2, ncomp) arrays with a ghost ring.  Its
    collide / stream (collide_field, stream below) run the sm_100a block
    kernels through liblbw; the device-resident time step (Simulation) does
    not use this class."""

    def __init__(self, size, dtype=np.float64, origin=(0, 0, 0), block_id=0):
        nx, ny, nz = (int(s) for s in size)
        if min(nx, ny, nz) < 1:
            raise ValueError("block size must be positive")
        self.size = (nx, ny, nz)
        self.dtype = np.dtype(dtype)
        self.origin = tuple(int(o) for o in origin)
        self.block_id = int(block_id)
        shape = (nx + 2, ny + 2, nz + 2)
        self.f = np.zeros(shape + (27,), self.dtype)
        self.f_next = np.zeros(shape + (27,), self.dtype)
        self.force = np.zeros(shape + (3,), self.dtype)
        self.macro = np.zeros(shape + (4,), self.dtype)
        self.macro[..., 0] = 1.0

    @property
    def interior(self):
        return self.f[1:-1, 1:-1, 1:-1, :]

    @property
    def interior_macro(self):
        return self.macro[1:-1, 1:-1, 1:-1, :]

    @property
    def interior_force(self):
        return self.force[1:-1, 1:-1, 1:-1, :]

    def cell_count(self):
        nx, ny, nz = self.size
        return nx * ny * nz

    def initialize_equilibrium(self, rho, u, product=False):
        n = self.size
        rho_arr = np.broadcast_to(np.asarray(rho, np.float64), n)
        u_arr = np.broadcast_to(np.asarray(u, np.float64), n + (3,))
        eq = product_equilibrium(rho_arr, u_arr) if product else equilibrium_pdf(rho_arr, u_arr)
        self.interior[...] = eq
        self.interior_macro[..., 0] = rho_arr
        self.interior_macro[..., 1:4] = u_arr
        self.force[...] = 0.0


def _as64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def collide_field(field, cfg, dt=1.0):
    """Collide every interior cell of a PdfField in place and refresh its
    macro (fields.py:70-83) with the block kernels of liblbw.  float32 fields
    are widened exactly and rounded back on store, as the reference's
    kernels do (_kernels.py:5-7)."""
    from . import kernels
    cfg.validate()
    f, force, macro = _as64(field.f), _as64(field.force), _as64(field.macro)
    if cfg.operator == "bgk":
        kernels.collide_bgk_block(f, force, macro, float(cfg.omega), float(dt))
    else:
        w3, w4, w5, w6 = (float(r) for r in cfg.higher_order_rates)
        kernels.collide_cumulant_block(f, force, macro, float(cfg.omega), w3, w4, w5, w6,
                                       float(dt))
    if f is not field.f:
        field.f[...] = f
    if macro is not field.macro:
        field.macro[...] = macro
    return field


def stream(field):
    """Pull streaming into f_next and swap (fields.py:86-94); the ghost ring
    of f must be filled."""
    from . import kernels
    src = _as64(field.f)
    dst = _as64(field.f_next)
    kernels.stream_pull_block(src, dst)
    if dst is not field.f_next:
        field.f_next[...] = dst
    field.f, field.f_next = field.f_next, field.f
    return field
