"""CPU oracle for the lbwind time step — TEST INFRASTRUCTURE, NOT PRODUCT.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or as
the timed CPU baseline.  The product package (paper_2402_13171_b200) never
imports it.

Layers:
  * liboracle.so (oracle/lbw_oracle.c): bit-exact C restatement of the
    numba kernels (_kernels.py:44-397) plus the single-block ghost refresh
    (halo.py:92-104) and the inflow/outflow boundary (halo.py:144-160).
  * numpy restatement of the actuator-line path on one block: trilinear
    sampling (actuator.py:70-93), angle of attack / blade element force
    (actuator.py:117-146, sim.py:210-235), polar lookup (polars.py:65-80),
    point routing with periodic images (actuator.py:284-341) and Roma
    spreading in global-id order (actuator.py:100-110, 190-247).
  * OracleSim: Simulation.step (sim.py:264-300) for a single block, driven
    with per-step actuator kinematics supplied by the caller.

Parity status: pinned.  tests/test_oracle.py checks every layer against
golden vectors produced by the reference itself (tests/golden/).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

# stencil.py:15-44
C = np.array([(cx, cy, cz) for cx in (-1, 0, 1) for cy in (-1, 0, 1) for cz in (-1, 0, 1)],
             dtype=np.int64)
_CLASS_W = {0: 8.0 / 27.0, 1: 2.0 / 27.0, 2: 1.0 / 54.0, 3: 1.0 / 216.0}
W = np.array([_CLASS_W[int(np.sum(c * c))] for c in C])
CS2 = 1.0 / 3.0

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp, i64, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        L.orc_collide_batch.argtypes = [ctypes.c_int, vp, vp, vp, i64, d, d, d, d, d, d]
        L.orc_collide_block.argtypes = [ctypes.c_int, vp, vp, vp, i64, i64, i64, d, d, d, d,
                                        d, d]
        L.orc_moments_block.argtypes = [vp, vp, vp, i64, i64, i64, d]
        L.orc_stream_pull_block.argtypes = [vp, vp, i64, i64, i64]
        L.orc_fill_ghosts.argtypes = [vp, i64, i64, i64, ctypes.c_int, vp]
        L.orc_apply_walls.argtypes = [vp, i64, i64, i64, vp, vp]
        L.orc_apply_inflow_outflow.argtypes = [vp, i64, i64, i64, vp]
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_threads.restype = None
        for fn in (L.orc_collide_batch, L.orc_collide_block, L.orc_moments_block,
                   L.orc_stream_pull_block, L.orc_fill_ghosts, L.orc_apply_inflow_outflow):
            fn.restype = None
        _lib = L
    return _lib


def set_threads(n):
    """OpenMP threads of the oracle's loops (the CPU-baseline timing leg)."""
    lib().orc_set_threads(int(n))


def _p(a):
    assert a.flags["C_CONTIGUOUS"] and a.dtype == np.float64
    return ctypes.c_void_p(a.ctypes.data)


# ------------------------------------------------------------ kernel layer

def collide_batch(op, f2, F2, omega, rates=(1.0, 1.0, 1.0, 1.0), dt=1.0):
    """(f', macro) of collide_{bgk,cumulant}_batch (_kernels.py:400-427)."""
    f2 = np.ascontiguousarray(f2, dtype=np.float64).copy()
    F2 = np.ascontiguousarray(np.broadcast_to(F2, (f2.shape[0], 3)), dtype=np.float64)
    m2 = np.zeros((f2.shape[0], 4))
    lib().orc_collide_batch(1 if op == "cumulant" else 0, _p(f2), _p(F2), _p(m2),
                            f2.shape[0], omega, *rates, dt)
    return f2, m2


def collide_block(op, f, force, macro, omega, rates=(1.0, 1.0, 1.0, 1.0), dt=1.0):
    nx, ny, nz = (s - 2 for s in f.shape[:3])
    lib().orc_collide_block(1 if op == "cumulant" else 0, _p(f), _p(force), _p(macro),
                            nx, ny, nz, omega, *rates, dt)


def moments_block(f, force, macro, dt=1.0):
    nx, ny, nz = (s - 2 for s in f.shape[:3])
    lib().orc_moments_block(_p(f), _p(force), _p(macro), nx, ny, nz, dt)


def stream_pull_block(fsrc, fdst):
    nx, ny, nz = (s - 2 for s in fsrc.shape[:3])
    lib().orc_stream_pull_block(_p(fsrc), _p(fdst), nx, ny, nz)


def fill_ghosts(a, periodic):
    nx, ny, nz = (s - 2 for s in a.shape[:3])
    per = np.asarray([int(bool(p)) for p in periodic], dtype=np.int32)
    lib().orc_fill_ghosts(_p(a), nx, ny, nz, a.shape[3], ctypes.c_void_p(per.ctypes.data))


# -------------------------------------------------------------- equilibria

def equilibrium_pdf(rho, u):
    """collision.py:54-67"""
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    cu = u @ C.T.astype(np.float64)
    usq = np.sum(u * u, axis=-1)[..., None]
    return W * rho[..., None] * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq)


def product_equilibrium(rho, u):
    """collision.py:70-100"""
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)

    def g(uc):
        return np.stack([0.5 * (uc * uc - uc + CS2), 1.0 - uc * uc - CS2,
                         0.5 * (uc * uc + uc + CS2)], axis=-1)

    gx, gy, gz = g(u[..., 0]), g(u[..., 1]), g(u[..., 2])
    return (rho[..., None] * gx[..., C[:, 0] + 1] * gy[..., C[:, 1] + 1]
            * gz[..., C[:, 2] + 1])


# --------------------------------------------------------------- actuator

def roma(r):
    """actuator.py:100-110 (scalar)"""
    a = abs(float(r))
    if a <= 0.5:
        return (1.0 + np.sqrt(1.0 - 3.0 * a ** 2)) / 3.0
    if a <= 1.5:
        return (5.0 - 3.0 * a - np.sqrt(1.0 - 3.0 * (1.0 - a) ** 2)) / 6.0
    return 0.0


def interpolate(macro, x_lat):
    """actuator.py:70-93 on a single ghosted block at origin 0."""
    x = np.asarray(x_lat, dtype=np.float64)
    j0 = np.floor(x - 0.5).astype(np.int64)
    t = x - 0.5 - j0
    lx, ly, lz = j0 + 1
    cube = macro[lx:lx + 2, ly:ly + 2, lz:lz + 2, :]
    wx = np.array([1.0 - t[0], t[0]])
    wy = np.array([1.0 - t[1], t[1]])
    wz = np.array([1.0 - t[2], t[2]])
    w = wx[:, None, None] * wy[None, :, None] * wz[None, None, :]
    vals = np.einsum("xyz,xyzc->c", w, cube)
    return float(vals[0]), vals[1:4].copy()


def polar_lookup(alpha_tab, cl_tab, cd_tab, a):
    """polars.py:65-80 (the warning is the host's business)"""
    clamped = a < alpha_tab[0] or a > alpha_tab[-1]
    if clamped:
        a = min(max(a, alpha_tab[0]), alpha_tab[-1])
    return float(np.interp(a, alpha_tab, cl_tab)), float(np.interp(a, alpha_tab, cd_tab)), clamped


def blade_force(kin_row, rho_lat, u_lat, chord, elen, twist, polar, vscale, rho_ref):
    """angle_of_attack + blade_element_force (actuator.py:117-146) as driven
    by sim.py:218-235.  Returns the force ON THE BLADE (N)."""
    if polar is None:
        return np.zeros(3)
    vel, ec, en, es = kin_row[3:6], kin_row[6:9], kin_row[9:12], kin_row[12:15]
    u_rel = u_lat * vscale - vel
    u_plane = u_rel - (u_rel @ es) * es
    speed = float(np.linalg.norm(u_plane))
    if speed < 1e-12:
        return np.zeros(3)
    phi = float(np.arctan2(u_plane @ en, u_plane @ ec))
    alpha = phi - twist
    e_d = u_plane / speed
    e_l = np.cross(es, e_d)
    cl, cd, _ = polar_lookup(*polar, alpha)
    rho = rho_lat * rho_ref
    if not rho > 0.0:
        raise ValueError(f"density must be positive, got {rho}")
    scale = 0.5 * rho * speed * speed * chord * elen
    return scale * (cl * np.asarray(e_l) + cd * np.asarray(e_d))


def disk_forces(ct, axis_world, rho_samples, u_samples, areas, rings, sectors):
    """actuator_disk_forces (actuator.py:149-183): per-ring momentum theory,
    force on the FLUID per sample."""
    axis = np.asarray(axis_world, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    forces = np.zeros((rings * sectors, 3))
    u_ax = np.asarray(u_samples) @ axis
    for j in range(rings):
        sl = slice(j * sectors, (j + 1) * sectors)
        if ct[j] == 0.0:
            continue
        a = (1.0 - np.sqrt(1.0 - ct[j])) / 2.0
        ring_area = areas[sl].sum()
        u_d = float((u_ax[sl] * areas[sl]).sum() / ring_area)
        rho = float((rho_samples[sl] * areas[sl]).sum() / ring_area)
        u_inf = u_d / (1.0 - a)
        thrust = 0.5 * rho * u_inf * u_inf * ct[j] * ring_area
        direction = -np.sign(u_d) if u_d != 0.0 else 0.0
        forces[sl] = direction * (thrust / ring_area) * areas[sl][:, None] * axis[None, :]
    return forces


def _support_box(pos, halo=1):
    lo = np.empty(3, dtype=np.int64)
    hi = np.empty(3, dtype=np.int64)
    for k in range(3):
        n0 = int(np.floor(pos[k]))
        j0 = int(np.floor(pos[k] - 0.5))
        lo[k] = min(n0 - halo, j0)
        hi[k] = max(n0 + halo, j0 + 1)
    return lo, hi


def axis_weights(x, kernel="roma", eps=0.0):
    """Deposit cells and weights along one axis: the reference's 3-point
    Roma kernel (actuator.py:190-195), or the Gaussian extension
    exp(-(r/eps)^2) over |r| <= 3 eps, normalised over that support."""
    if kernel == "roma":
        n0 = int(np.floor(x))
        return [(n0 - 1 + q, roma(r)) for q, r in
                enumerate((x - (n0 - 0.5), x - (n0 + 0.5), x - (n0 + 1.5)))]
    R = 3.0 * eps
    jlo, jhi = int(np.ceil(x - 0.5 - R)), int(np.floor(x - 0.5 + R))
    e = [np.exp(-((x - (j + 0.5)) / eps) ** 2) for j in range(jlo, jhi + 1)]
    inv = 1.0 / sum(e)
    return [(j, v * inv) for j, v in zip(range(jlo, jhi + 1), e)]


def route_single_block(records, dims, periodic, halo=1):
    """mark_and_exchange_points (actuator.py:297-341) for a 1x1x1 block grid:
    the block receives its own records plus an image, shifted by -wrap*L,
    for every periodic neighbour offset its support box touches."""
    gd = np.asarray(dims, dtype=np.float64)
    out = []
    imgs = []
    for gid, pos, force in records:
        out.append((gid, pos, force))
        lo, hi = _support_box(pos, halo)
        for ox in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for oz in (-1, 0, 1):
                    off = (ox, oy, oz)
                    if off == (0, 0, 0):
                        continue
                    if any(o != 0 and not periodic[k] for k, o in enumerate(off)):
                        continue
                    hit = all(not (hi[k] < off[k] * dims[k] or lo[k] > off[k] * dims[k] + dims[k] - 1)
                              for k in range(3))
                    if hit:
                        imgs.append((gid, pos - np.asarray(off, dtype=np.float64) * gd, force))
    out.extend(imgs)
    out.sort(key=lambda r: r[0])
    return out


def _identity(a):
    return a


def round_f32(a):
    """Value a float32 array stores for `a` (numpy assignment rounds to
    nearest even)."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def spread(records, force, dims, dt2, den, rnd=_identity, kernel="roma", eps=0.0):
    """spread_forces (actuator.py:204-247) into a ghosted block at origin 0.
    rnd models the storage dtype of `force`: `+=` on a float32 array rounds
    after every addition."""
    nx, ny, nz = dims
    for gid, pos, f_newton in records:
        f_lat = np.asarray(f_newton, dtype=np.float64) * dt2 / den
        cells, ws = [], []
        for k in range(3):
            cw = axis_weights(pos[k], kernel, eps)
            cells.append([c for c, _ in cw])
            ws.append([w for _, w in cw])
        for i in range(len(cells[0])):
            lx = cells[0][i]
            if not 0 <= lx < nx or ws[0][i] == 0.0:
                continue
            for j in range(len(cells[1])):
                ly = cells[1][j]
                if not 0 <= ly < ny or ws[1][j] == 0.0:
                    continue
                wxy = ws[0][i] * ws[1][j]
                for k in range(len(cells[2])):
                    lz = cells[2][k]
                    if not 0 <= lz < nz or ws[2][k] == 0.0:
                        continue
                    force[lx + 1, ly + 1, lz + 1, :] = rnd(
                        force[lx + 1, ly + 1, lz + 1, :] + (wxy * ws[2][k]) * f_lat)


# ------------------------------------------------------------ single block

class OracleSim:
    """Simulation.step (sim.py:264-300) on one block, CPU, bit-exact LBM.

    points: dict with chord, element_length, twist (P,), polar (list of
    (alpha, cl, cd) tuples or None per point), vscale, rho_ref, dt2, den.
    step(kin) takes the (P,15) kinematics of this step (lattice position,
    velocity, e_chord, e_normal, e_span) from the caller.
    dtype float32 models ``precision: single``: every array keeps fp64
    arithmetic but holds float32-representable values, rounded wherever the
    reference stores into its float32 fields (_kernels.py:5-7, 342-353).
    """

    def __init__(self, cells, periodic=(True, True, True), op="cumulant", omega=1.0,
                 rates=(1.0, 1.0, 1.0, 1.0), boundary="periodic", u_in=(0.0, 0.0, 0.0),
                 points=None, dtype=np.float64, walls=(0, 0, 0, 0)):
        self.dims = tuple(int(c) for c in cells)
        self.rnd = round_f32 if np.dtype(dtype) == np.float32 else _identity
        # y_lo, y_hi, z_lo, z_hi: 0 none, 1 no-slip, 2 free-slip (extension)
        self.walls = np.ascontiguousarray(walls, dtype=np.int32)
        nx, ny, nz = self.dims
        shape = (nx + 2, ny + 2, nz + 2)
        self.periodic = tuple(bool(p) for p in periodic)
        self.op, self.omega, self.rates = op, float(omega), tuple(float(r) for r in rates)
        self.boundary = boundary
        self.u_in = np.asarray(u_in, dtype=np.float64)
        self.f = np.zeros(shape + (27,))
        self.f_next = np.zeros(shape + (27,))
        self.force = np.zeros(shape + (3,))
        self.macro = np.zeros(shape + (4,))
        self.macro[..., 0] = 1.0
        self.points = points
        self.step_index = 0
        self.samples = None
        self.blade = None

    @property
    def interior(self):
        return self.f[1:-1, 1:-1, 1:-1]

    def initialize_equilibrium(self, rho, u, product):
        """fields.py:54-67"""
        n = self.dims
        rho_arr = np.broadcast_to(np.asarray(rho, np.float64), n)
        u_arr = np.broadcast_to(np.asarray(u, np.float64), n + (3,))
        eq = product_equilibrium(rho_arr, u_arr) if product else equilibrium_pdf(rho_arr, u_arr)
        self.f[1:-1, 1:-1, 1:-1] = self.rnd(eq)
        self.macro[1:-1, 1:-1, 1:-1, 0] = self.rnd(rho_arr)
        self.macro[1:-1, 1:-1, 1:-1, 1:4] = self.rnd(u_arr)
        self.force[...] = 0.0

    def _actuators(self, kin, blade=None):
        pts = self.points
        P = kin.shape[0]
        fill_ghosts(self.macro, self.periodic)   # exchange_macro_halos (sim.py:273-274)
        self.samples = np.zeros((P, 4))
        self.blade = np.zeros((P, 3))
        records = []
        for p in range(P):
            rho, u = interpolate(self.macro, kin[p, 0:3])
            self.samples[p, 0] = rho
            self.samples[p, 1:] = u
            self.blade[p] = blade_force(kin[p], rho, u, pts["chord"][p],
                                        pts["element_length"][p], pts["twist"][p],
                                        pts["polar"][p], pts["vscale"], pts["rho_ref"])
        # disks: sim.py:236-244 (samples in physical units, axis = centre +x,
        # carried in the kinematics' e_chord slot)
        for first, rings, sectors, ct in pts.get("disks", ()):
            sl = slice(first, first + rings * sectors)
            f = disk_forces(ct, kin[first, 6:9], self.samples[sl, 0] * pts["rho_ref"],
                            self.samples[sl, 1:] * pts["vscale"], pts["area"][sl], rings, sectors)
            self.blade[sl] = -f
        # blade: forces from elsewhere (the device's), spread in place of the
        # oracle's own -- the LBM + spreading path then has identical inputs
        self.blade_own = self.blade.copy()
        if blade is not None:
            self.blade = np.array(blade, dtype=np.float64)
        for p in range(P):
            records.append((p, kin[p, 0:3].copy(), -self.blade[p]))
        kernel, eps = pts.get("spreading", ("roma", 0.0))
        halo = 1 if kernel == "roma" else int(np.ceil(3.0 * eps)) + 1
        routed = route_single_block(records, self.dims, self.periodic, halo)
        self.force[...] = 0.0
        spread(routed, self.force, self.dims, pts["dt2"], pts["den"], self.rnd, kernel, eps)

    def step(self, kin=None, blade=None):
        if self.points is not None:
            self._actuators(np.asarray(kin, dtype=np.float64), blade)
        collide_block(self.op, self.f, self.force, self.macro, self.omega, self.rates)
        if self.rnd is not _identity:
            self.f[...] = self.rnd(self.f)
            self.macro[...] = self.rnd(self.macro)
        m = self.macro[1:-1, 1:-1, 1:-1]
        if not np.all(np.isfinite(m)):
            bad = np.argwhere(~np.isfinite(m))[0]
            raise FloatingPointError((self.step_index, tuple(int(b) for b in bad[:3]),
                                      "density" if bad[3] == 0 else "velocity"))
        fill_ghosts(self.f, self.periodic)
        if self.boundary == "velocity_inflow_outflow":
            feq_in = np.ascontiguousarray(self.rnd(equilibrium_pdf(1.0, self.u_in)))
            nx, ny, nz = self.dims
            lib().orc_apply_inflow_outflow(_p(self.f), nx, ny, nz, _p(feq_in))
            self.macro[0, :, :, 0] = 1.0
            self.macro[0, :, :, 1:4] = self.rnd(self.u_in)
            self.force[0] = 0.0
            self.macro[-1] = self.macro[-2]
            self.force[-1] = self.force[-2]
        if self.walls.any():
            per = np.ascontiguousarray([int(p) for p in self.periodic], dtype=np.int32)
            nx, ny, nz = self.dims
            lib().orc_apply_walls(_p(self.f), nx, ny, nz, ctypes.c_void_p(self.walls.ctypes.data),
                                  ctypes.c_void_p(per.ctypes.data))
        stream_pull_block(self.f, self.f_next)
        self.f, self.f_next = self.f_next, self.f
        self.step_index += 1

    def recompute_moments(self):
        moments_block(self.f, self.force, self.macro)
        self.macro[...] = self.rnd(self.macro)
        return self.macro[1:-1, 1:-1, 1:-1].copy()
