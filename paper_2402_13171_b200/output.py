"""Probe CSVs, VTK field dumps and global gathers (lbwind.output,
/root/reference/pkg/src/lbwind/output.py:33-167).

Output ticks are off the timed loop: the macro field is recomputed on the
device (K3, the same arithmetic as moments_block), downloaded once per tick
and sampled on the host.  Values are written with repr() so files are
bit-identical whenever the state is.
"""

import os

import numpy as np

from .errors import ConfigError
from .turbine import LineSpec

AXIAL_HEADER = "x_m,u_axial_m_per_s"
RADIAL_HEADER = "y_m,u_axial_m_per_s"
BLADE_HEADER = "r_over_R,f_normal_N_per_m,f_tangential_N_per_m"


def ghosted_macro(sim, macro):
    """Interior macro (nx,ny,nz,4) -> ghosted array with the reference's ghost
    values: periodic wrap, inflow (1, u_in), outflow copy, (1,0,0,0) else."""
    nx, ny, nz = macro.shape[:3]
    g = np.zeros((nx + 2, ny + 2, nz + 2, 4))
    g[..., 0] = 1.0
    g[1:-1, 1:-1, 1:-1] = macro
    per = sim.grid.periodicity
    for axis in range(3):
        if not per[axis]:
            continue
        lo = [slice(None)] * 4
        hi = [slice(None)] * 4
        src_lo = [slice(None)] * 4
        src_hi = [slice(None)] * 4
        n = macro.shape[axis]
        lo[axis], src_lo[axis] = 0, n
        hi[axis], src_hi[axis] = n + 1, 1
        g[tuple(lo)] = g[tuple(src_lo)]
        g[tuple(hi)] = g[tuple(src_hi)]
    if sim.boundary.kind == "velocity_inflow_outflow" and sim.step_index > 0:
        g[0, :, :, 0] = 1.0
        g[0, :, :, 1:4] = sim.boundary.u_in_lat
        g[-1] = g[-2]
    return g


class CubeSource:
    """A sparse ghosted macro field: only the cells of given sampling cubes,
    keyed by ghosted global index (i, j, k) (interior cell x <-> i = x + 1).
    Multi-GPU output ticks gather just these cells to rank 0 instead of the
    whole lattice; cubes come out as the same (2,2,2,4) arrays a dense
    ghosted field gives, so the samples are bit-identical."""

    def __init__(self, cells):
        self.cells = cells

    def cube(self, lx, ly, lz):
        out = np.empty((2, 2, 2, 4))
        for a in range(2):
            for b in range(2):
                for c in range(2):
                    out[a, b, c] = self.cells[(lx + a, ly + b, lz + c)]
        return out


def _cube_origin(x_lat):
    x = np.asarray(x_lat, dtype=np.float64)
    j0 = np.floor(x - 0.5).astype(np.int64)
    return x, j0, x - 0.5 - j0


def interpolate(gmacro, x_lat):
    """Trilinear sample of a ghosted single-block macro (actuator.py:70-93);
    gmacro is a dense ghosted array or a CubeSource."""
    x, j0, t = _cube_origin(x_lat)
    lx, ly, lz = (int(v) for v in j0 + 1)
    if isinstance(gmacro, CubeSource):
        cube = gmacro.cube(lx, ly, lz)
    else:
        cube = gmacro[lx:lx + 2, ly:ly + 2, lz:lz + 2, :]
    wx = np.array([1.0 - t[0], t[0]])
    wy = np.array([1.0 - t[1], t[1]])
    wz = np.array([1.0 - t[2], t[2]])
    w = wx[:, None, None] * wy[None, :, None] * wz[None, None, :]
    vals = np.einsum("xyz,xyzc->c", w, cube)
    return float(vals[0]), vals[1:4].copy()


def _sample_velocity(sim, gmacro, pos_m):
    lat = np.asarray(pos_m, dtype=np.float64) / sim.units.dx
    L = np.asarray(sim.grid.global_dims, dtype=np.float64)
    periodic = np.asarray(sim.grid.periodicity, dtype=bool)
    lat = np.where(periodic, np.mod(lat, L), lat)
    sim.grid.owner_block_of_position(lat)
    _, u_lat = interpolate(gmacro, lat)
    return sim.units.velocity_to_physical(u_lat)


def _probe_lattice_positions(sim, probe):
    """Lattice positions (wrapped on periodic axes) a position probe samples,
    in the order probe_rows visits them."""
    Lx, Ly, Lz = sim.cfg.domain_length_m()
    if probe.kind == "axial_line":
        y0 = probe.y_m if probe.y_m is not None else 0.5 * Ly
        z0 = probe.z_m if probe.z_m is not None else 0.5 * Lz
        pos = [((i + 0.5) * Lx / probe.samples, y0, z0) for i in range(probe.samples)]
    elif probe.kind == "radial_profile":
        z0 = probe.z_m if probe.z_m is not None else 0.5 * Lz
        pos = [(probe.x_m, (j + 0.5) * Ly / probe.samples, z0) for j in range(probe.samples)]
    else:
        return []
    L = np.asarray(sim.grid.global_dims, dtype=np.float64)
    periodic = np.asarray(sim.grid.periodicity, dtype=bool)
    out = []
    for p in pos:
        lat = np.asarray(p, dtype=np.float64) / sim.units.dx
        out.append(np.where(periodic, np.mod(lat, L), lat))
    return out


def probe_cube_cells(sim):
    """Ghosted global indices of every cell the position probes' sampling
    cubes read (sorted)."""
    need = set()
    for probe in sim.cfg.probes:
        for lat in _probe_lattice_positions(sim, probe):
            _, j0, _ = _cube_origin(lat)
            lx, ly, lz = (int(v) for v in j0 + 1)
            for a in range(2):
                for b in range(2):
                    for c in range(2):
                        need.add((lx + a, ly + b, lz + c))
    return sorted(need)


def ghost_source(sim, key):
    """Where ghosted_macro takes cell `key` (ghosted global index) from:
    ("cell", (x, y, z)) of the interior, or ("const", 4-vector) -- the same
    periodic-wrap / inflow / outflow / (1,0,0,0) rules."""
    dims = tuple(sim.grid.global_dims)
    per = sim.grid.periodicity
    gi, gj, gk = key
    if sim.boundary.kind == "velocity_inflow_outflow" and sim.step_index > 0:
        if gi == 0:
            return "const", np.concatenate([[1.0], np.asarray(sim.boundary.u_in_lat, float)])
        if gi == dims[0] + 1:
            gi = dims[0]
    idx = []
    for axis, g in enumerate((gi, gj, gk)):
        i = g - 1
        if 0 <= i < dims[axis]:
            idx.append(i)
        elif per[axis]:
            idx.append(i % dims[axis])
        else:
            return "const", np.array([1.0, 0.0, 0.0, 0.0])
    return "cell", tuple(idx)


def probe_rows(sim, probe, gmacro=None):
    if gmacro is None:
        gmacro = ghosted_macro(sim, sim.fields[0].download_macro())
    Lx, Ly, Lz = sim.cfg.domain_length_m()
    if probe.kind == "axial_line":
        y0 = probe.y_m if probe.y_m is not None else 0.5 * Ly
        z0 = probe.z_m if probe.z_m is not None else 0.5 * Lz
        xs = [(i + 0.5) * Lx / probe.samples for i in range(probe.samples)]
        rows = np.array([[x, _sample_velocity(sim, gmacro, (x, y0, z0))[0]] for x in xs])
        return AXIAL_HEADER, rows.reshape(-1, 2)
    if probe.kind == "radial_profile":
        z0 = probe.z_m if probe.z_m is not None else 0.5 * Lz
        ys = [(j + 0.5) * Ly / probe.samples for j in range(probe.samples)]
        rows = np.array([[y, _sample_velocity(sim, gmacro, (probe.x_m, y, z0))[0]] for y in ys])
        return RADIAL_HEADER, rows.reshape(-1, 2)
    if probe.kind == "blade_loads":
        return BLADE_HEADER, blade_load_rows(sim, probe)
    raise ConfigError(f"unknown probe kind {probe.kind!r}")


def blade_load_rows(sim, probe):
    """Per-station force per unit span along the rotor axis and in-plane
    (output.py:69-99); also the source of thrust/power time series."""
    topo = sim.cfg.topologies[probe.turbine]
    comp = next((c for c in topo.components if isinstance(c.discretization, LineSpec)
                 and (not probe.component or c.name == probe.component)), None)
    if comp is None:
        raise ConfigError(f"probe {probe.name}: no actuator line {probe.component or ''!r} "
                          f"on turbine {probe.turbine}")
    sl = next(s for c, _, s in sim._line_groups if c is comp)
    spec = comp.discretization
    r = np.linalg.norm(spec.offsets, axis=1)
    r_max = r.max() or 1.0
    axis = comp.world_spin_axis
    axis = np.array([1.0, 0.0, 0.0]) if axis is None else np.asarray(axis)
    pts = sim.points[sl]
    rows = np.zeros((len(pts), 3))
    for i, p in enumerate(pts):
        tangent = np.cross(axis, p.e_span)
        nt = np.linalg.norm(tangent)
        tangent = p.e_chord if nt < 1e-9 else tangent / nt
        bf = p.blade_force
        rows[i] = (r[i] / r_max, (bf @ axis) / p.element_length,
                   (bf @ tangent) / p.element_length)
    return rows


def rotor_loads(sim, turbine=0):
    """(thrust N, torque N m, power W) of one turbine from the blade forces of
    the last step: thrust = sum F.a, torque = sum ((p - hub) x F).a,
    power = torque * rate.  (The reference has no thrust/power output; this
    is the time series the north star asks for, derived from blade_force.)"""
    topo = sim.cfg.topologies[turbine]
    thrust = torque = power = 0.0
    for comp, spec, sl in sim._line_groups:
        if comp not in topo.components:
            continue
        axis = comp.world_spin_axis
        if axis is None:
            continue
        axis = np.asarray(axis) / np.linalg.norm(axis)
        hub = None
        for c in topo.components:
            if c.rate != 0.0 and comp in _descendants(c):
                hub, rate = c.world.p, c.rate
        if hub is None:
            continue
        F = sim._alm_results()[2][sl]
        arm = sim._kin_view()[sl, 15:18] - hub   # world positions (m), unwrapped
        thrust += float(np.sum(F @ axis))
        tq = float(np.sum(np.cross(arm, F) @ axis))
        torque += tq
        power += tq * rate
    return thrust, torque, power


def _descendants(comp):
    out, stack = [], list(comp.children)
    while stack:
        c = stack.pop()
        out.append(c)
        stack.extend(c.children)
    return out


def write_probe_csv(path, header, rows):
    with open(path, "w") as fh:
        fh.write(header + "\n")
        for row in np.asarray(rows, dtype=np.float64):
            fh.write(",".join(repr(float(v)) for v in row) + "\n")
    return path


def gather_global_fields(sim):
    """(density kg/m^3, velocity m/s, force N) of this slab, physical units."""
    u = sim.units
    fld = sim.fields[0]
    m = fld.download_macro()
    return (u.density_to_physical(m[..., 0]), u.velocity_to_physical(m[..., 1:4]),
            u.force_to_physical(fld.download_force()))


def write_field_vtk(path, sim):
    rho, vel, frc = gather_global_fields(sim)
    nx, ny, nz = rho.shape
    dx = sim.units.dx
    per = ",".join(str(int(p)) for p in sim.cfg.periodicity)
    with open(path, "w") as fh:
        fh.write("# vtk DataFile Version 3.0\n")
        fh.write(f"{sim.cfg.name} step={sim.step_index} periodicity={per} dx={dx!r}\n")
        fh.write("ASCII\nDATASET STRUCTURED_POINTS\n")
        fh.write(f"DIMENSIONS {nx} {ny} {nz}\n")
        fh.write(f"ORIGIN {0.5 * dx!r} {0.5 * dx!r} {0.5 * dx!r}\n")
        fh.write(f"SPACING {dx!r} {dx!r} {dx!r}\n")
        fh.write(f"POINT_DATA {nx * ny * nz}\n")
        fh.write("SCALARS density double 1\nLOOKUP_TABLE default\n")
        fh.write("".join(repr(float(v)) + "\n" for v in rho.transpose(2, 1, 0).ravel()))
        for name, arr in (("velocity", vel), ("force", frc)):
            fh.write(f"VECTORS {name} double\n")
            flat = arr.transpose(2, 1, 0, 3).reshape(-1, 3)
            fh.write("".join(" ".join(repr(float(c)) for c in v) + "\n" for v in flat))
    return path


def probe_tick(sim, gmacro=None):
    """Probe CSVs (+ running averages) and the VTK dump of one output tick
    (sim.py:304-333).  gmacro: the sampled field (dense ghosted array or
    CubeSource); default: this simulation's macro, downloaded and ghosted."""
    cfg = sim.cfg
    if not (cfg.probes or cfg.vtk):
        return
    if not sim._macro_fresh:
        sim._recompute_moments()
    os.makedirs(cfg.output_dir, exist_ok=True)
    if gmacro is None and any(p.kind != "blade_loads" for p in cfg.probes):
        gmacro = ghosted_macro(sim, sim.fields[0].download_macro())
    for probe in cfg.probes:
        header, rows = probe_rows(sim, probe, gmacro)
        write_probe_csv(os.path.join(cfg.output_dir, f"{probe.name}_{sim.step_index:08d}.csv"),
                        header, rows)
        if probe.average_from_step is not None and sim.step_index >= probe.average_from_step:
            count, sums = sim._avg.get(probe.name, (0, 0.0))
            count += 1
            sums = sums + rows
            sim._avg[probe.name] = (count, sums)
            avg = rows.copy()
            avg[:, 1:] = sums[:, 1:] / count
            write_probe_csv(os.path.join(cfg.output_dir,
                                         f"{probe.name}_avg_{sim.step_index:08d}.csv"),
                            header, avg)
    if cfg.vtk:
        write_field_vtk(os.path.join(cfg.output_dir, f"{cfg.name}_{sim.step_index:08d}.vtk"), sim)
