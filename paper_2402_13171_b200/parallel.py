"""Multi-GPU x-slab decomposition (one process per GPU, torchrun).

Each rank owns planes [bounds[r], bounds[r+1]) of the global x extent
(SlabGrid).  Neighbour slabs are linked once at setup: the ranks exchange
opaque liblbw handle blobs (CUDA IPC handles) through torch.distributed
and from then on every step runs without host communication —

  * the sweep kernel stores the nine outgoing direction planes of its first
    and last x plane straight into the neighbours' ghost planes (NVLink),
  * actuator sampling cubes that straddle a slab face are completed by the
    neighbour's stores into this rank's cube buffer,
  * steps are ordered by GPU-side waits on counters the neighbours write.

Results are bit-identical to the single-GPU run: every cell is computed by
exactly one rank with the same arithmetic, and every actuator point's force
is evaluated from the same cube values in the same order on each rank that
needs it.

torch.distributed is plumbing only (rendezvous, handle exchange, the
non-finite consensus at synchronisation points).
"""

import ctypes

import numpy as np

from . import _lib
from .errors import NumericalAbort
from .sim import SlabGrid, Simulation


def slab_neighbours(rank, nranks, periodic_x):
    """(lo, hi) neighbour ranks of slab `rank`; -1 across a non-periodic face."""
    lo = rank - 1 if rank > 0 else (nranks - 1 if periodic_x and nranks > 1 else -1)
    hi = rank + 1 if rank < nranks - 1 else (0 if periodic_x and nranks > 1 else -1)
    return lo, hi


def first_nonfinite(reports):
    """Consensus over per-rank non-finite reports [(step, cell, field) or
    None]: the earliest step, then the first cell in C order — the cell the
    single-block reference reports (sim.py:254-262)."""
    hits = [r for r in reports if r is not None]
    if not hits:
        return None
    return min(hits, key=lambda r: (r[0], tuple(r[1])))


def _dist():
    import torch.distributed as dist
    return dist


def exchange_neighbour_blobs(blob, rank, nranks, periodic_x, group=None):
    """Every rank publishes its handle blob; returns the (lo, hi) neighbours'
    blobs (None across a non-periodic face)."""
    blobs = [None] * nranks
    _dist().all_gather_object(blobs, blob, group=group)
    lo, hi = slab_neighbours(rank, nranks, periodic_x)
    return (blobs[lo] if lo >= 0 else None), (blobs[hi] if hi >= 0 else None)


def gather_probe_cells(sim, macro, x0, rank, nranks, group=None):
    """The cells of the position probes' sampling cubes, each sent by the
    rank owning it (macro: this rank's slab, first global plane x0), merged
    with the constant ghost values on rank 0 into an output.CubeSource
    (None on the other ranks)."""
    from . import output
    keys = output.probe_cube_cells(sim)
    mine = {}
    for key in keys:
        kind, src = output.ghost_source(sim, key)
        if kind == "cell" and x0 <= src[0] < x0 + macro.shape[0]:
            mine[key] = np.array(macro[src[0] - x0, src[1], src[2]])
    parts = [None] * nranks if rank == 0 else None
    _dist().gather_object(mine, parts, dst=0, group=group)
    if rank != 0:
        return None
    cells = {}
    for part in parts:
        cells.update(part)
    for key in keys:
        kind, src = output.ghost_source(sim, key)
        if kind == "const":
            cells[key] = src
    return output.CubeSource(cells)


class SlabSimulation(Simulation):
    """Simulation of one x-slab, linked to its neighbours on other GPUs."""

    def __init__(self, cfg, rank, nranks, device=None, group=None, kinematics=None):
        super().__init__(cfg, rank=rank, nranks=nranks, device=device, kinematics=kinematics)
        self.rank, self.nranks, self._group = int(rank), int(nranks), group
        self._pending_abort = None
        self._link()

    def _link(self):
        dist = _dist()
        lib = _lib.load()
        n = int(lib.lbw_peer_blob_bytes())
        buf = (ctypes.c_char * n)()
        size = ctypes.c_int64(n)
        _lib.check(lib.lbw_domain_export_handle(self._domain, buf, ctypes.byref(size)), "export")
        lo, hi = exchange_neighbour_blobs(bytes(buf[:size.value]), self.rank, self.nranks,
                                          self.cfg.periodicity[0], self._group)
        lo_b = ctypes.create_string_buffer(lo, len(lo)) if lo is not None else None
        hi_b = ctypes.create_string_buffer(hi, len(hi)) if hi is not None else None
        _lib.check(lib.lbw_domain_import_peers(self._domain, lo_b, hi_b), "import peers")
        dist.barrier(group=self._group)

    # non-finite flags: recorded per rank while stepping, agreed on collectively
    def _poll(self, wait):
        try:
            super()._poll(wait)
        except NumericalAbort as e:
            if self._pending_abort is None:
                self._pending_abort = (e.step, e.cell, e.field)

    def synchronize(self):
        super().synchronize()
        reports = [None] * self.nranks
        _dist().all_gather_object(reports, self._pending_abort, group=self._group)
        hit = first_nonfinite(reports)
        if hit is not None:
            raise NumericalAbort(*hit)

    def alm_results_global(self):
        """(rho, u, blade force) of every point, each from the rank that owns
        it (the others report zeros, so the sum is exact)."""
        rho, u, blade = self._alm_results()
        parts = [None] * self.nranks
        _dist().all_gather_object(parts, (rho, u, blade), group=self._group)
        return tuple(sum(p[k] for p in parts) for k in range(3))

    def gather_interior(self, root=0):
        """Post-stream populations of the whole lattice on `root` (tests)."""
        mine = self.fields[0].interior.view(np.ndarray)
        parts = [None] * self.nranks
        _dist().all_gather_object(parts, mine, group=self._group)
        return np.concatenate(parts, axis=0) if self.rank == root else None

    def gather_force(self, root=0):
        mine = self.fields[0].interior_force.view(np.ndarray)
        parts = [None] * self.nranks
        _dist().all_gather_object(parts, mine, group=self._group)
        return np.concatenate(parts, axis=0) if self.rank == root else None

    def close(self):
        """Free this slab once every rank has finished its work: the
        neighbours' sweeps store into this slab's ghost planes (and read
        nothing after their own completion), so no rank frees memory a
        neighbour may still write."""
        if getattr(self, "_domain", None):
            try:
                _lib.load().lbw_domain_sync(self._domain)
                _dist().barrier(group=self._group)
            except Exception:
                pass
        super().close()

    def __del__(self):
        # no collective from a finaliser: the other ranks may be gone
        try:
            Simulation.close(self)
        except Exception:
            pass

    # ------------------------------------------------------------ output
    def _probe_tick(self):
        """Output tick of the whole lattice (output.py:33-167) written by
        rank 0, files identical to a single-GPU run.  Position probes only
        need the cells of their sampling cubes: each rank sends rank 0 the
        ones it owns (a few kB), not its field.  The VTK dump is the whole
        field by definition: the slabs' macro and force fields are gathered
        to rank 0 only."""
        from . import output
        cfg = self.cfg
        if not (cfg.probes or cfg.vtk):
            return
        dist = _dist()
        if not self._macro_fresh:
            self._recompute_moments()
        macro = self.fields[0].download_macro()
        results = self.alm_results_global() if self.points else None
        cubes = gather_probe_cells(self, macro, int(self.grid.bounds[self.rank]), self.rank,
                                   self.nranks, self._group)
        fields = None
        if cfg.vtk:
            force = self.fields[0].download_force()
            fields = [None] * self.nranks if self.rank == 0 else None
            dist.gather_object((macro, force), fields, dst=0, group=self._group)
        if self.rank == 0:
            gm = gf = None
            if cfg.vtk:
                gm = np.concatenate([f[0] for f in fields], axis=0)
                gf = np.concatenate([f[1] for f in fields], axis=0)
            view = _GlobalView(self, gm, gf, results)
            output.probe_tick(view, gmacro=cubes)
        dist.barrier(group=self._group)

    def _write_report(self, report):
        if self.rank == 0:
            super()._write_report(report)


class _GlobalField:
    def __init__(self, macro, force):
        self._macro, self._force = macro, force

    def download_macro(self):
        return self._macro

    def download_force(self):
        return self._force


class _GlobalPoint:
    """An ActuatorPoint whose per-step outputs come from the gathered
    (owner) results."""

    def __init__(self, point, results):
        self._p, self._r = point, results

    def __getattr__(self, name):
        return getattr(self._p, name)

    blade_force = property(lambda s: s._r[2][s._p.global_id].copy())
    fluid_force = property(lambda s: -s._r[2][s._p.global_id])
    sampled_rho = property(lambda s: float(s._r[0][s._p.global_id]))
    sampled_u = property(lambda s: s._r[1][s._p.global_id].copy())


class _GlobalView:
    """What output.probe_tick needs of a Simulation, for the whole lattice
    on rank 0 (a single-block grid over the global extent)."""

    def __init__(self, sim, macro, force, results):
        cfg = sim.cfg
        self.cfg, self.units, self.boundary = cfg, sim.units, sim.boundary
        self.step_index = sim.step_index
        self.grid = SlabGrid(cfg.cells, cfg.periodicity, 1, 0)
        self.fields = [_GlobalField(macro, force)]
        self._line_groups = sim._line_groups
        self._avg = sim._avg
        self._macro_fresh = True
        self._kin_view = sim._kin_view
        self.points = [_GlobalPoint(p, results) for p in sim.points] if results else []
        self._alm_results = lambda: results


def run_slab_simulation(cfg, group=None, kinematics=None):
    """Simulation.run over all ranks of torch.distributed (one process per
    GPU, device = LOCAL_RANK); rank 0 writes the probes, VTK and report."""
    import os
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = int(os.environ.get("LOCAL_RANK", rank))
    sim = SlabSimulation(cfg, rank, world, device=device, group=group, kinematics=kinematics)
    try:
        return sim.run()
    finally:
        sim.close()


__all__ = ["SlabGrid", "SlabSimulation", "exchange_neighbour_blobs", "first_nonfinite",
           "gather_probe_cells", "run_slab_simulation", "slab_neighbours"]
