"""D3Q27 velocity set (stencil.py:15-49 of the reference).

Direction index i = (cx+1)*9 + (cy+1)*3 + (cz+1): cx slowest, i = 13 is the
rest direction and opposite(i) = 26 - i.  The device kernels use the same
order (csrc/lbw_cell.cuh); the halo direction subsets follow from it:
cx = -1 is i = 0..8, cx = +1 is i = 18..26.
"""

import numpy as np

Q = 27
CS2 = 1.0 / 3.0
CS4 = CS2 * CS2
REST = 13


def index_of(cx, cy, cz):
    return (cx + 1) * 9 + (cy + 1) * 3 + (cz + 1)


def _velocity_set():
    axis = (-1, 0, 1)
    c = np.array([[a, b, d] for a in axis for b in axis for d in axis], dtype=np.int64)
    by_speed = (8.0 / 27.0, 2.0 / 27.0, 1.0 / 54.0, 1.0 / 216.0)
    w = np.array([by_speed[int((row * row).sum())] for row in c])
    return c, w, (Q - 1) - np.arange(Q, dtype=np.int64)


C, W, OPP = _velocity_set()
CX = C[:, 0].astype(np.float64)
CY = C[:, 1].astype(np.float64)
CZ = C[:, 2].astype(np.float64)
for _arr in (C, W, OPP, CX, CY, CZ):
    _arr.setflags(write=False)
del _arr
