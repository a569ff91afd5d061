"""Outer boundary specification (lbwind.halo.BoundarySpec, halo.py:122-141).

The reference refreshes ghost layers through serialised byte buffers and
then overwrites the x-face ghosts with the inflow equilibrium / outflow copy
(halo.py:92-160).  On the device there is no ghost ring in y/z (wrap by
index) and the x faces are folded into the sweep's pull (XSource in
csrc/lbw_internal.h); across GPUs the nine outgoing direction planes travel
over NVLink.  Only the specification object remains on the host.
"""

import numpy as np

from .collision import equilibrium_pdf


class BoundarySpec:
    """kind "periodic" or "velocity_inflow_outflow" (the -x ghost pinned to
    the polynomial equilibrium of (1, u_in), the +x ghost a copy of the last
    interior plane)."""

    KINDS = ("periodic", "velocity_inflow_outflow")

    def __init__(self, kind="periodic", u_in_lat=(0.0, 0.0, 0.0)):
        if kind not in self.KINDS:
            raise ValueError(f"unknown boundary kind {kind!r}")
        self.kind = kind
        self.u_in_lat = np.asarray(u_in_lat, dtype=np.float64)

    def inflow_populations(self):
        """equilibrium_pdf(1, u_in) exactly as apply_outer_boundary builds it."""
        return np.ascontiguousarray(equilibrium_pdf(1.0, self.u_in_lat), dtype=np.float64)

    def __repr__(self):
        return f"BoundarySpec({self.kind!r}, u_in_lat={tuple(self.u_in_lat)})"
