"""The C ABI without the Python package: what a maintainer binding
liblbw.so into the reference (level 2) writes -- plain
ctypes against include/lbw.h.  Runs a small Taylor-Green vortex for a few
steps on the device and checks mass conservation and the analytic decay
of the kinetic energy.

    python examples/abi_minimal.py [path/to/liblbw.so]
"""

import ctypes
import os
import sys

import numpy as np

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "..", "paper_2402_13171_b200", "liblbw.so")


class DomainDesc(ctypes.Structure):   # lbw_domain_desc (include/lbw.h)
    _fields_ = [("cells", ctypes.c_int64 * 3), ("slab_x0", ctypes.c_int64),
                ("slab_nx", ctypes.c_int64), ("periodic", ctypes.c_int32 * 3),
                ("op", ctypes.c_int32), ("mode", ctypes.c_int32), ("boundary", ctypes.c_int32),
                ("device", ctypes.c_int32), ("omega", ctypes.c_double),
                ("rates", ctypes.c_double * 4), ("u_in", ctypes.c_double * 3),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("feq_in_given", ctypes.c_int32), ("feq_in", ctypes.c_double * 27),
                ("precision", ctypes.c_int32), ("walls", ctypes.c_int32 * 4),
                ("reserved32", ctypes.c_int32), ("reserved", ctypes.c_int64 * 5)]


def main():
    L = ctypes.CDLL(LIB)
    L.lbw_last_error.restype = ctypes.c_char_p
    assert L.lbw_abi_version() == 2, "ABI version"
    P = ctypes.c_void_p

    def ck(rc):
        if rc != 0:
            raise RuntimeError(L.lbw_last_error().decode())

    n = 32
    d = DomainDesc()
    d.cells[:] = (n, n, n)
    d.slab_x0, d.slab_nx = 0, n
    d.periodic[:] = (1, 1, 1)
    d.op, d.mode, d.boundary = 1, 0, 0          # cumulant, exact, periodic
    nu = 0.02
    d.omega = 1.0 / (3.0 * nu + 0.5)
    d.rates[:] = (1.0, 1.0, 1.0, 1.0)
    d.nranks = 1
    dom = P()
    ck(L.lbw_domain_create(ctypes.byref(d), ctypes.byref(dom)))

    # Taylor-Green initial state: product equilibrium of u (collision.py:69-100)
    u0, k = 0.02, 2.0 * np.pi / n
    X, Y = np.meshgrid(np.arange(n) + 0.5, np.arange(n) + 0.5, indexing="ij")
    u = np.zeros((n, n, n, 3))
    u[..., 0] = (u0 * np.sin(k * X) * np.cos(k * Y))[:, :, None]
    u[..., 1] = (-u0 * np.cos(k * X) * np.sin(k * Y))[:, :, None]
    c = np.array([(cx, cy, cz) for cx in (-1, 0, 1) for cy in (-1, 0, 1) for cz in (-1, 0, 1)])

    def g(v):
        vv = v * v
        return np.stack([0.5 * (vv - v + 1 / 3), 1.0 - vv - 1 / 3, 0.5 * (vv + v + 1 / 3)], -1)

    gx, gy, gz = g(u[..., 0]), g(u[..., 1]), g(u[..., 2])
    f = np.ascontiguousarray(gx[..., c[:, 0] + 1] * gy[..., c[:, 1] + 1] * gz[..., c[:, 2] + 1])
    ck(L.lbw_domain_upload_pdf(dom, f.ctypes.data_as(P)))
    m0 = f.sum()

    def energy():
        macro = np.empty((n, n, n, 4))
        ck(L.lbw_domain_recompute_moments(dom, macro.ctypes.data_as(P)))
        return float(np.sum(macro[..., 1:4] ** 2))

    e0 = energy()
    steps = 200
    ck(L.lbw_domain_step(dom, ctypes.c_int32(steps)))
    e1 = energy()
    out = np.empty_like(f)
    ck(L.lbw_domain_download_pdf(dom, out.ctypes.data_as(P)))
    step, cell, field = ctypes.c_int64(), (ctypes.c_int64 * 3)(), ctypes.c_int32()
    assert L.lbw_domain_poll_nonfinite(dom, 1, ctypes.byref(step), cell, ctypes.byref(field)) == 0
    L.lbw_domain_destroy(dom)

    rate = np.log(e1 / e0) / steps
    analytic = -4.0 * nu * k * k
    print(f"mass drift {abs(out.sum() - m0) / m0:.2e}, energy decay rate {rate:.4e} "
          f"(analytic {analytic:.4e})")
    assert abs(out.sum() - m0) < 1e-12 * m0
    assert abs(rate / analytic - 1.0) < 0.05


if __name__ == "__main__":
    main()
