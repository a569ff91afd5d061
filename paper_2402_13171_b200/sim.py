"""Time-stepping driver on the GPU (the Simulation surface of lbwind.sim,
/root/reference/pkg/src/lbwind/sim.py:56-400).

One Simulation owns one device-resident x-slab (the whole lattice on one
GPU, or slab ``rank`` of ``nranks`` in a multi-GPU run, see
paper_2402_13171_b200.parallel) plus the turbine topologies.  A step keeps
the reference's order (sim.py:5-21):

  host   refresh actuator kinematics for t = n dt (vectorised, bit-identical
         to refresh_points) and queue them (one async H2D)
  K4     sample the previous step's macro field, blade-element forces
  K5     zero last step's force rows, spread in ascending global id
  K1     fused pull-stream + collide + Guo, outer boundary folded into the
         pull, non-finite flag, edge planes pushed to the neighbour slabs
  host   advance the topologies by dt

Everything between the two host parts is queued on the domain's CUDA
stream; the only synchronisation per step is a non-blocking poll of the
non-finite flag.
"""

import json
import os

import numpy as np

from . import _lib
from .collision import CollisionConfig
from .errors import ConfigError, NumericalAbort
from .fields import DeviceField
from .halo import BoundarySpec
from .roofline import RunTimer, lbm_kernel_cost, lightspeed, measure_mlups, percent_table_row
from .turbine import DiskSpec, LineSpec

_EX = np.array([1.0, 0.0, 0.0])
KIN_COLS = 18   # lattice pos, velocity, e_chord, e_normal, e_span, position m


class BlockDescriptor:
    def __init__(self, id, block_index, origin, size, owner=0):
        self.id, self.block_index = id, tuple(block_index)
        self.origin, self.size = tuple(origin), tuple(size)
        self.owner, self.weight = owner, 1.0
        self.neighbors = {}


class SlabGrid:
    """The device decomposition: x-slabs, one per GPU.  Exposes the bits of
    lbwind.blocks.BlockGrid that callers read (blocks, global_dims,
    periodicity, counts, owner_block_of_position)."""

    def __init__(self, cells, periodicity, nranks, rank):
        self.global_dims = tuple(int(c) for c in cells)
        self.periodicity = tuple(bool(p) for p in periodicity)
        self.nranks, self.rank = int(nranks), int(rank)
        nx = self.global_dims[0]
        self.bounds = [(r * nx) // self.nranks for r in range(self.nranks + 1)]
        if any(self.bounds[r + 1] - self.bounds[r] < 1 for r in range(self.nranks)):
            raise ConfigError(f"{nx} x planes cannot be split over {nranks} GPUs")
        self.counts = (self.nranks, 1, 1)
        self.block_dims = (self.bounds[1] - self.bounds[0],) + self.global_dims[1:]
        x0, x1 = self.bounds[rank], self.bounds[rank + 1]
        self.blocks = [BlockDescriptor(rank, (rank, 0, 0), (x0, 0, 0),
                                       (x1 - x0,) + self.global_dims[1:], owner=rank)]

    def __len__(self):
        return len(self.blocks)

    def owner_block_of_position(self, pos):
        x = None
        for k in range(3):
            v = pos[k] % self.global_dims[k] if self.periodicity[k] else pos[k]
            if not 0.0 <= v < self.global_dims[k]:
                raise ConfigError(f"position component {pos[k]} outside the non-periodic domain")
            if k == 0:
                x = v
        return int(np.searchsorted(self.bounds, x, side="right") - 1)


class ActuatorPoint:
    """One actuator point (attribute surface of lbwind.actuator.ActuatorPoint,
    actuator.py:33-63).  Per-step state lives in the Simulation's arrays;
    attribute reads fetch device results lazily."""

    def __init__(self, sim, gid, chord=0.0, element_length=0.0, twist=0.0, polar=None,
                 area=0.0, disk=False):
        self._sim = sim
        self.global_id = int(gid)
        self.chord = float(chord)
        self.element_length = float(element_length)
        self.twist = float(twist)
        self.polar = polar
        self.area = float(area)
        self.owner_block = -1
        self.is_disk_sample = bool(disk)

    def _k(self, a, b):
        return self._sim._kin_view()[self.global_id, a:b].copy()

    def _frame(self, k):
        # disk samples keep the identity frame of the reference (actuator.py:50-55)
        return np.eye(3)[k].copy() if self.is_disk_sample else self._k(6 + 3 * k, 9 + 3 * k)

    position = property(lambda s: s._k(15, 18))
    position_lat = property(lambda s: s._k(0, 3))
    velocity = property(lambda s: s._k(3, 6))
    e_chord = property(lambda s: s._frame(0))
    e_normal = property(lambda s: s._frame(1))
    e_span = property(lambda s: s._frame(2))
    sampled_rho = property(lambda s: float(s._sim._alm_results()[0][s.global_id]))
    sampled_u = property(lambda s: s._sim._alm_results()[1][s.global_id].copy())
    blade_force = property(lambda s: s._sim._alm_results()[2][s.global_id].copy())
    fluid_force = property(lambda s: -s._sim._alm_results()[2][s.global_id])


class Simulation:
    """kinematics: "device" (default) advances the turbine trees on the GPU
    (no per-step host work or H2D; positions within 1e-13 of the reference,
    inside the actuator tolerance); "host" replays the reference's numpy
    kinematics bit for bit and uploads them each step (test_acceptance.py
    test_07 budget: host replay costs ~0.2 ms/step of Python)."""

    def __init__(self, cfg, rank=0, nranks=1, device=None, kinematics=None):
        self.cfg = cfg
        self.units = cfg.units
        if kinematics is None:
            kinematics = "device"
        if kinematics not in ("host", "device"):
            raise ConfigError(f"kinematics must be host or device, got {kinematics!r}")
        self.kinematics = kinematics
        lib = _lib.require_gpu()
        self.grid = SlabGrid(cfg.cells, cfg.periodicity, nranks, rank)
        desc = self.grid.blocks[0]
        self.collision = CollisionConfig(cfg.operator, self.units.omega,
                                         cfg.higher_order_rates).validate()
        wind_lat = self.units.velocity_to_lattice(np.asarray(cfg.wind, dtype=np.float64))
        self.boundary = BoundarySpec(cfg.boundary_kind, u_in_lat=wind_lat)
        self.device = cfg.device if device is None else int(device)
        self._domain = self._create_domain(lib, desc, rank, nranks)
        self.fields = [DeviceField(self, desc.size, desc.origin, desc.id)]
        self.fields[0].initialize_equilibrium(1.0, wind_lat,
                                              product=(cfg.operator == "cumulant"))
        self._build_points()
        self.timer = RunTimer(int(np.prod(cfg.cells)))
        self.step_index = 0
        self._macro_fresh = False
        self._avg = {}
        self._results = None
        self._warned = set()

    # ----------------------------------------------------------- setup
    def _create_domain(self, lib, desc, rank, nranks):
        cfg = self.cfg
        d = _lib.DomainDesc()
        for k in range(3):
            d.cells[k] = cfg.cells[k]
            d.periodic[k] = int(cfg.periodicity[k])
        d.slab_x0, d.slab_nx = desc.origin[0], desc.size[0]
        d.op = _lib.OP_CUMULANT if cfg.operator == "cumulant" else _lib.OP_BGK
        d.mode = _lib.MODE_FAST if cfg.arithmetic == "fast" else _lib.MODE_EXACT
        d.boundary = (_lib.BC_INFLOW_OUTFLOW if cfg.boundary_kind == "velocity_inflow_outflow"
                      else _lib.BC_PERIODIC)
        d.device = self.device
        d.omega = float(self.units.omega)
        for k in range(4):
            d.rates[k] = float(cfg.higher_order_rates[k])
        for k in range(3):
            d.u_in[k] = float(self.boundary.u_in_lat[k])
        d.rank, d.nranks = rank, nranks
        d.precision = _lib.LBW_PREC_SINGLE if cfg.precision == "single" else _lib.LBW_PREC_DOUBLE
        for k, code in enumerate(cfg.wall_codes()):
            d.walls[k] = code
        d.feq_in_given = 1
        feq = self.boundary.inflow_populations()
        for i in range(27):
            d.feq_in[i] = float(feq[i])
        handle = _lib.ctypes.c_void_p()
        _lib.check(lib.lbw_domain_create(_lib.ctypes.byref(d), _lib.ctypes.byref(handle)),
                   "domain")
        return handle

    def _build_points(self):
        """Global ids in topology -> component -> point order (sim.py:113-143)."""
        cfg = self.cfg
        self.points, self._line_groups, self._disk_groups = [], [], []
        polar_ids = sorted(cfg.polars)
        gid = 0
        for topo in cfg.topologies:
            for comp in topo.components:
                spec = comp.discretization
                if isinstance(spec, LineSpec):
                    start = gid
                    for pi in range(spec.n_points):
                        pid = spec.polar[pi]
                        self.points.append(ActuatorPoint(
                            self, gid, spec.chord[pi], spec.element_length[pi], spec.twist[pi],
                            cfg.polars.get(pid) if pid is not None else None))
                        gid += 1
                    self._line_groups.append((comp, spec, slice(start, gid)))
                elif isinstance(spec, DiskSpec):
                    offs, areas = spec.sample_offsets()
                    start = gid
                    for si in range(len(areas)):
                        self.points.append(ActuatorPoint(self, gid, area=areas[si], disk=True))
                        gid += 1
                    self._disk_groups.append((comp, spec, offs, areas, slice(start, gid)))
        P = len(self.points)
        self._kin = np.zeros((P, KIN_COLS))
        self._pos_m = np.zeros((P, 3))
        self._kin_stale = False
        self._topo_pending = False
        self._polar_list = []
        if P == 0:
            self.kinematics = "host"
            return
        # static point data + concatenated polar tables -> device
        index_of = {pid: k for k, pid in enumerate(polar_ids)}
        self._polar_list = [cfg.polars[pid] for pid in polar_ids]
        pidx = np.full(P, -1, dtype=np.int32)
        for p in self.points:
            if p.polar is not None:
                pidx[p.global_id] = index_of[p.polar.id]
        rows = np.array([t.alpha.size for t in self._polar_list] or [0], dtype=np.int32)
        offs = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int32)
        cat = (lambda attr: np.ascontiguousarray(np.concatenate(
            [getattr(t, attr) for t in self._polar_list]) if self._polar_list else np.zeros(1)))
        self._alm_static = dict(
            chord=np.array([p.chord for p in self.points]),
            elen=np.array([p.element_length for p in self.points]),
            twist=np.array([p.twist for p in self.points]), pidx=pidx, rows=rows, offs=offs,
            alpha=cat("alpha"), cl=cat("cl"), cd=cat("cd"))
        s = self._alm_static
        D = _lib.ctypes.POINTER(_lib.ctypes.c_double)
        I = _lib.ctypes.POINTER(_lib.ctypes.c_int32)
        a = _lib.AlmDesc()
        a.n_points = P
        a.chord = s["chord"].ctypes.data_as(D)
        a.element_length = s["elen"].ctypes.data_as(D)
        a.twist = s["twist"].ctypes.data_as(D)
        a.polar_index = s["pidx"].ctypes.data_as(I)
        a.n_polars = len(self._polar_list)
        a.polar_offset = s["offs"].ctypes.data_as(I)
        a.polar_rows = s["rows"].ctypes.data_as(I)
        a.polar_alpha = s["alpha"].ctypes.data_as(D)
        a.polar_cl = s["cl"].ctypes.data_as(D)
        a.polar_cd = s["cd"].ctypes.data_as(D)
        a.velocity_scale = self.units.velocity_scale
        a.rho_ref = self.units.rho_ref
        a.force_dt2 = self.units.force_dt2
        a.force_den = self.units.force_den
        a.spread_kernel = 1 if self.cfg.spread_kernel == "gaussian" else 0
        a.spread_epsilon = float(self.cfg.spread_epsilon)
        if self._disk_groups:
            # one ring = `sectors` consecutive samples (DiskSpec.sample_offsets)
            ring_first, ring_count, ring_ct = [], [], []
            point_ring = np.full(P, -1, dtype=np.int32)
            for comp, spec, offs, areas, sl in self._disk_groups:
                for j in range(spec.rings):
                    first = sl.start + j * spec.sectors
                    point_ring[first:first + spec.sectors] = len(ring_first)
                    ring_first.append(first)
                    ring_count.append(spec.sectors)
                    ring_ct.append(float(spec.thrust_coefficient[j]))
            s["point_ring"] = point_ring
            s["area"] = np.array([p.area for p in self.points])
            s["ring_first"] = np.array(ring_first, dtype=np.int32)
            s["ring_count"] = np.array(ring_count, dtype=np.int32)
            s["ring_ct"] = np.array(ring_ct, dtype=np.float64)
            a.point_ring = s["point_ring"].ctypes.data_as(I)
            a.area = s["area"].ctypes.data_as(D)
            a.n_rings = len(ring_first)
            a.ring_first = s["ring_first"].ctypes.data_as(I)
            a.ring_count = s["ring_count"].ctypes.data_as(I)
            a.ring_ct = s["ring_ct"].ctypes.data_as(D)
        _lib.check(_lib.load().lbw_alm_configure(self._domain, _lib.ctypes.byref(a)), "ALM")
        self._kin_stale = False
        self._topo_pending = False
        if self.kinematics == "device":
            self._configure_device_kinematics()

    def _flat_components(self):
        comps, parent = [], []
        for topo in self.cfg.topologies:
            base = len(comps)
            index = {id(c): base + k for k, c in enumerate(topo.components)}
            for c in topo.components:
                comps.append(c)
                parent.append(-1)
            for c in topo.components:
                for ch in c.children:
                    parent[index[id(ch)]] = index[id(c)]
        return comps, parent

    def _configure_device_kinematics(self):
        """Flatten the turbine trees for the device walk (lbw_kin_desc)."""
        from .turbine import rotation_matrix
        comps, parent = self._flat_components()
        C, P = len(comps), len(self.points)
        dt = self.units.dt
        first = {id(comp): sl.start for comp, spec, sl in self._line_groups}
        arr = {k: np.zeros(s) for k, s in (("rel_p", (C, 3)), ("rel_T", (C, 3, 3)),
                                            ("axis", (C, 3)), ("rate", (C,)),
                                            ("rstep", (C, 3, 3)), ("spin", (C, 3, 3)),
                                            ("off", (P, 3)), ("orient", (P, 3, 3)),
                                            ("lframe", (P, 3, 3)))}
        line_first = np.full(C, -1, dtype=np.int32)
        line_count = np.zeros(C, dtype=np.int32)
        is_disk = np.zeros(C, dtype=np.int32)
        disk_center = np.zeros((C, 12))
        disks = {id(comp): (spec, offs, sl) for comp, spec, offs, areas, sl in self._disk_groups}
        for c, comp in enumerate(comps):
            arr["rel_p"][c] = comp.relative.p
            arr["rel_T"][c] = comp.relative.T
            arr["rate"][c] = comp.rate
            arr["spin"][c] = comp.spin
            arr["rstep"][c] = np.eye(3)
            if comp.axis is not None:
                arr["axis"][c] = comp.axis
                if comp.rate != 0.0 and dt != 0.0:
                    arr["rstep"][c] = rotation_matrix(comp.axis, comp.rate * dt)
            if id(comp) in first:
                spec = comp.discretization
                g0 = first[id(comp)]
                line_first[c], line_count[c] = g0, spec.n_points
                arr["off"][g0:g0 + spec.n_points] = spec.offsets
                arr["orient"][g0:g0 + spec.n_points] = spec.orientations
                arr["lframe"][g0:g0 + spec.n_points] = spec.frames_local()
            if id(comp) in disks:
                spec, offs, sl = disks[id(comp)]
                line_first[c], line_count[c] = sl.start, sl.stop - sl.start
                is_disk[c] = 1
                disk_center[c, :3] = spec.center.p
                disk_center[c, 3:] = spec.center.T.ravel()
                arr["off"][sl] = offs
                arr["orient"][sl] = np.eye(3)
                arr["lframe"][sl] = np.eye(3)
        par = np.asarray(parent, dtype=np.int32)
        self._kin_arrays = (arr, line_first, line_count, par, is_disk, disk_center)
        k = _lib.KinDesc()
        k.n_components = C
        k.parent = _lib.iptr(par)
        k.rel_p, k.rel_T = _lib.dptr(arr["rel_p"]), _lib.dptr(arr["rel_T"])
        k.axis, k.rate = _lib.dptr(arr["axis"]), _lib.dptr(arr["rate"])
        k.step_rotation, k.spin = _lib.dptr(arr["rstep"]), _lib.dptr(arr["spin"])
        k.line_first, k.line_count = _lib.iptr(line_first), _lib.iptr(line_count)
        k.offsets, k.orientations = _lib.dptr(arr["off"]), _lib.dptr(arr["orient"])
        k.local_frames = _lib.dptr(arr["lframe"])
        k.dx = self.units.dx
        k.advance_first = 0
        k.is_disk = _lib.iptr(is_disk)
        k.disk_center = _lib.dptr(disk_center)
        _lib.check(_lib.load().lbw_alm_configure_kinematics(self._domain, _lib.ctypes.byref(k)),
                   "kinematics")
        self._flat = comps

    def _kin_view(self):
        """(P,15) kinematics of the latest step (downloaded in device mode)."""
        if self.kinematics == "device" and self._kin_stale and len(self.points):
            _lib.check(_lib.load().lbw_alm_download_kinematics(
                self._domain, _lib.ptr(self._kin), None, None), "kinematics")
            self._kin_stale = False
        return self._kin

    def sync_topologies(self):
        """Bring the host turbine objects to the device state: spins from the
        device, then the host walk advances them to t = step_index * dt, as
        the reference's per-step advance would have."""
        if self.kinematics != "device" or not self._topo_pending:
            return
        lib = _lib.load()
        spin = np.zeros((len(self._flat), 3, 3))
        _lib.check(lib.lbw_alm_download_kinematics(self._domain, None, _lib.ptr(spin), None),
                   "kinematics")
        behind = self.step_index - int(lib.lbw_alm_kinematics_step(self._domain))
        for c, comp in enumerate(self._flat):
            comp.spin = spin[c].copy()
        for topo in self.cfg.topologies:
            topo.advance(self.units.dt if behind > 0 else 0.0)
        self._topo_pending = False

    # ------------------------------------------------------- per step
    def refresh_points(self):
        """Positions, velocities and frames from the topology state
        (sim.py:167-191), stacked: identical doubles, O(1) numpy calls per
        line."""
        fill_kinematics(self._line_groups, self._disk_groups, self.grid, self.units.dx,
                        self._kin, self._pos_m)

    def _alm_results(self):
        if self._results is None:
            P = len(self.points)
            rho, u, blade = np.zeros(P), np.zeros((P, 3)), np.zeros((P, 3))
            if P:
                rc = _lib.load().lbw_alm_get(self._domain, _lib.ptr(rho), _lib.ptr(u),
                                             _lib.ptr(blade))
                if rc == _lib.LBW_EINVAL:
                    msg = _lib.last_error()
                    # owner_block_of_position (blocks.py:57-70) raises ConfigError;
                    # a non-positive density is blade_element_force's ValueError
                    raise (ConfigError if "outside" in msg or "spans" in msg else ValueError)(msg)
                _lib.check(rc, "ALM results")
            self._results = (rho, u, blade)
        return self._results

    def _poll(self, wait):
        step, field = _lib.ctypes.c_int64(), _lib.ctypes.c_int32()
        cell = (_lib.ctypes.c_int64 * 3)()
        rc = _lib.load().lbw_domain_poll_nonfinite(self._domain, int(wait),
                                                   _lib.ctypes.byref(step), cell,
                                                   _lib.ctypes.byref(field))
        if rc < 0:
            _lib.check(rc, "poll")
        if rc == 1:
            raise NumericalAbort(int(step.value), tuple(int(c) for c in cell),
                                 "density" if field.value == 0 else "velocity")

    def _abort_now(self):
        """run.abort: immediate -- wait for this step's collide and, when it
        produced a non-finite macro value, leave the state the reference
        leaves (sim.py:254-262, 281): the post-collision populations of the
        aborted step, not streamed, step_index not advanced."""
        try:
            self._poll(wait=True)
        except NumericalAbort:
            _lib.check(_lib.load().lbw_domain_hold_collided(self._domain), "abort")
            self._macro_fresh = False
            raise

    def _warn_clamps(self):
        if not self.points or not self._polar_list:
            return
        flags = np.zeros(len(self._polar_list), dtype=np.int32)
        _lib.check(_lib.load().lbw_alm_clamp_flags(
            self._domain, flags.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_int32))))
        for k in np.nonzero(flags)[0]:
            self._polar_list[k].warn_clamp()

    def step(self):
        lib = _lib.load()
        t = self.timer
        host_kin = self.kinematics == "host"
        if self.points and host_kin:
            t.start_phase("turbine")
            self.refresh_points()
            _lib.check(lib.lbw_alm_set_kinematics(self._domain, _lib.ptr(self._kin)), "ALM")
            t.stop_phase()
        t.start_phase("collide")
        _lib.check(lib.lbw_domain_step(self._domain, 1), "step")
        t.stop_phase()
        self._results = None
        if self.cfg.abort == "immediate":
            self._abort_now()
        else:
            self._poll(wait=False)
        if self.cfg.topologies:
            if host_kin or not self.points:
                t.start_phase("turbine")
                for topo in self.cfg.topologies:
                    topo.advance(self.units.dt)
                t.stop_phase()
            else:
                self._kin_stale = True
                self._topo_pending = True
        t.count_step()
        self.step_index += 1
        self._macro_fresh = False

    def advance(self, n):
        """n steps; with device kinematics (or no actuator points) they are
        queued by ONE native call (lbw_domain_step(n)) instead of n Python
        step() calls -- the same launches, no per-step host work.  A
        non-finite state aborts at the first offending step as step() does."""
        n = int(n)
        if n <= 0:
            return
        if (self.points and self.kinematics == "host") or self.cfg.abort == "immediate":
            for _ in range(n):
                self.step()
            return
        t = self.timer
        t.start_phase("collide")
        _lib.check(_lib.load().lbw_domain_step(self._domain, n), "step")
        t.stop_phase()
        self._results = None
        self._poll(wait=False)
        if self.cfg.topologies:
            if not self.points:
                t.start_phase("turbine")
                for _ in range(n):
                    for topo in self.cfg.topologies:
                        topo.advance(self.units.dt)
                t.stop_phase()
            else:
                self._kin_stale = True
                self._topo_pending = True
        t.count_step(n)
        self.step_index += n
        self._macro_fresh = False

    def record_loads(self, capacity=4096):
        """Start recording every step's blade forces (the thrust / power time
        series) device->host without synchronising the step loop."""
        if self.points:
            _lib.check(_lib.load().lbw_alm_record_loads(self._domain, int(capacity)), "loads")
        self._loads_cap = int(capacity)

    def read_loads(self):
        """(first_step, blade forces (n, P, 3)) of the steps executed since
        the last read (record_loads must be on)."""
        P = len(self.points)
        n_max = max(1, getattr(self, "_loads_cap", 0))
        out = np.empty((n_max, P, 3))
        first = _lib.ctypes.c_int64()
        n = _lib.ctypes.c_int64()
        if not P:
            return self.step_index, out[:0]
        _lib.check(_lib.load().lbw_alm_read_loads(self._domain, _lib.ptr(out), n_max,
                                                  _lib.ctypes.byref(first),
                                                  _lib.ctypes.byref(n)), "loads")
        return int(first.value), out[:n.value]

    def synchronize(self):
        _lib.check(_lib.load().lbw_domain_sync(self._domain), "sync")
        self._poll(wait=True)
        self._warn_clamps()
        self.sync_topologies()
        if self.points:
            self._results = None
            self._alm_results()   # raises for points that left the domain (device flags)

    # ---------------------------------------------------------- output
    def _recompute_moments(self):
        """moments of the current populations with the current force; they
        also become the next actuator sampling source (sim.py:160-165)."""
        self._poll(wait=True)
        _lib.check(_lib.load().lbw_domain_recompute_moments(self._domain, None), "moments")
        self._macro_fresh = True

    def _probe_tick(self):
        from . import output
        output.probe_tick(self)

    def run(self):
        cfg = self.cfg
        self.timer.start()
        remaining = cfg.steps
        while remaining > 0:
            n = remaining
            if cfg.cadence > 0:
                n = min(n, cfg.cadence - self.step_index % cfg.cadence)
            self.advance(n)
            remaining -= n
            if cfg.cadence > 0 and self.step_index % cfg.cadence == 0:
                self.synchronize()
                self.timer.stop()
                self._probe_tick()
                self.timer.start()
        self.synchronize()
        self.timer.stop()
        if cfg.cadence == 0 and (cfg.probes or cfg.vtk):
            self._probe_tick()
        report = self.report()
        self._write_report(report)
        return report

    def _write_report(self, report):
        os.makedirs(self.cfg.output_dir, exist_ok=True)
        with open(os.path.join(self.cfg.output_dir, "report.json"), "w") as fh:
            json.dump(report, fh, indent=2, sort_keys=True)

    def report(self):
        cfg = self.cfg
        cost = lbm_kernel_cost(precision_bytes=np.dtype(cfg.dtype).itemsize,
                               n_f=cfg.kernel_flops())
        u = self.units
        out = {"config": cfg.echo(),
               "units": {"dx_m": u.dx, "dt_s": u.dt, "u_lat": u.u_lat, "nu_lat": u.nu_lat,
                         "tau": u.tau, "omega": u.omega},
               "grid": {"cells": list(cfg.cells), "blocks": self.grid.nranks,
                        "block_dims": list(self.grid.block_dims), "workers": cfg.workers,
                        "actuator_points": len(self.points), "devices": self.grid.nranks},
               "kernel": dict(cost.to_dict(), operator=cfg.operator, precision=cfg.precision,
                              arithmetic=cfg.arithmetic),
               "performance": dict(self.timer.to_dict(),
                                   phase_fractions=self.timer.phase_fractions())}
        if self.timer.steps > 0 and self.timer.wall_seconds > 0.0:
            mlups, _ = measure_mlups(self.timer)
            out["performance"]["mlups"] = mlups
            if cfg.machine is not None:
                out["performance"].update(percent_table_row(mlups, cfg.machine, cost))
        if cfg.machine is not None:
            out["machine"] = cfg.machine.to_dict()
            ls = lightspeed(cfg.machine, cost)
            if ls is not None:
                out["machine"]["lightspeed"] = ls
        return out

    def close(self):
        if getattr(self, "_domain", None):
            _lib.load().lbw_domain_destroy(self._domain)
            self._domain = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_simulation(cfg):
    sim = Simulation(cfg)
    try:
        return sim.run()
    finally:
        sim.close()


def fill_kinematics(line_groups, disk_groups, grid, dx, kin, pos_m):
    """Host kinematics rows (P,18) of every actuator point from the current
    topology state (Simulation.refresh_points, sim.py:167-191)."""
    for comp, spec, sl in line_groups:
        frames = comp.point_frames_arr
        n = spec.n_points
        pos_m[sl] = comp.point_positions_arr
        kin[sl, 3:6] = comp.point_velocities
        for col, v in ((6, spec.chord_local), (9, spec.normal_local), (12, spec.span_local)):
            kin[sl, col:col + 3] = np.matmul(frames, np.broadcast_to(v, (n, 3))[:, :, None])[:, :, 0]
    for comp, spec, offs, areas, sl in disk_groups:
        # sim.py:182-187; the disk axis (centre frame +x) rides in e_chord
        cp, cT = comp.point_positions_arr[0], comp.point_frames_arr[0]
        pos_m[sl] = cp[None, :] + offs @ cT.T
        kin[sl, 3:6] = comp.point_velocities[0]
        kin[sl, 6:9] = cT @ _EX
        kin[sl, 9:15] = (0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    if line_groups or disk_groups:
        L = np.asarray(grid.global_dims, dtype=np.float64)
        periodic = np.asarray(grid.periodicity, dtype=bool)
        lat = pos_m / dx
        lat = np.where(periodic, np.mod(lat, L), lat)
        bad = (~periodic) & ((lat < 0.0) | (lat >= L))
        if np.any(bad):
            p, k = np.argwhere(bad)[0]
            raise ConfigError(f"position component {lat[p, k]} outside the non-periodic domain")
        kin[:, 0:3] = lat
        kin[:, 15:18] = pos_m


def point_groups(cfg):
    """(point metadata, line groups, disk groups) in global-id order
    (topology -> component -> point, sim.py:113-143).  Metadata rows are
    dicts with chord, element_length, twist, polar, area, disk."""
    meta, lines, disks = [], [], []
    for topo in cfg.topologies:
        for comp in topo.components:
            spec = comp.discretization
            if isinstance(spec, LineSpec):
                start = len(meta)
                for pi in range(spec.n_points):
                    pid = spec.polar[pi]
                    meta.append(dict(chord=spec.chord[pi], element_length=spec.element_length[pi],
                                     twist=spec.twist[pi], area=0.0, disk=False,
                                     polar=cfg.polars.get(pid) if pid is not None else None))
                lines.append((comp, spec, slice(start, len(meta))))
            elif isinstance(spec, DiskSpec):
                offs, areas = spec.sample_offsets()
                start = len(meta)
                for si in range(len(areas)):
                    meta.append(dict(chord=0.0, element_length=0.0, twist=0.0, area=areas[si],
                                     disk=True, polar=None))
                disks.append((comp, spec, offs, areas, slice(start, len(meta))))
    return meta, lines, disks


class HostKinematics:
    """The host half of a Simulation's actuator path without a device:
    per-step kinematics rows of a configuration (used to drive the CPU
    oracle with the same actuator motion)."""

    def __init__(self, cfg):
        self.cfg, self.units = cfg, cfg.units
        self.grid = SlabGrid(cfg.cells, cfg.periodicity, 1, 0)
        wind_lat = cfg.units.velocity_to_lattice(np.asarray(cfg.wind, dtype=np.float64))
        self.boundary = BoundarySpec(cfg.boundary_kind, u_in_lat=wind_lat)
        meta, self._line_groups, self._disk_groups = point_groups(cfg)
        self.points = [type("PointMeta", (), m)() for m in meta]
        self._kin = np.zeros((len(meta), KIN_COLS))
        self._pos_m = np.zeros((len(meta), 3))

    def refresh(self):
        fill_kinematics(self._line_groups, self._disk_groups, self.grid, self.units.dx,
                        self._kin, self._pos_m)
        return self._kin.copy()

    def advance(self):
        for topo in self.cfg.topologies:
            topo.advance(self.units.dt)
