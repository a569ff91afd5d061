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
from .errors import ConfigError, NumericalAbort
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


class SlabSimulation(Simulation):
    """Simulation of one x-slab, linked to its neighbours on other GPUs."""

    def __init__(self, cfg, rank, nranks, device=None, group=None, kinematics=None):
        super().__init__(cfg, rank=rank, nranks=nranks, device=device, kinematics=kinematics)
        self.rank, self.nranks, self._group = int(rank), int(nranks), group
        if self._disk_groups and self.nranks > 1:
            self.close()
            raise ConfigError("actuator disks run on a single GPU in this build "
                              "(ring averages are not exchanged between slabs)")
        self._pending_abort = None
        self._link()

    def _link(self):
        dist = _dist()
        lib = _lib.load()
        n = int(lib.lbw_peer_blob_bytes())
        buf = (ctypes.c_char * n)()
        size = ctypes.c_int64(n)
        _lib.check(lib.lbw_domain_export_handle(self._domain, buf, ctypes.byref(size)), "export")
        blobs = [None] * self.nranks
        dist.all_gather_object(blobs, bytes(buf[:size.value]), group=self._group)
        lo, hi = slab_neighbours(self.rank, self.nranks, self.cfg.periodicity[0])
        lo_b = ctypes.create_string_buffer(blobs[lo], len(blobs[lo])) if lo >= 0 else None
        hi_b = ctypes.create_string_buffer(blobs[hi], len(blobs[hi])) if hi >= 0 else None
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


__all__ = ["SlabGrid", "SlabSimulation", "first_nonfinite", "slab_neighbours"]
