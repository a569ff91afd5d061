"""Walls on non-periodic y / z faces (an extension the north star asks for:
the reference leaves those ghosts unwritten).  No-slip = halfway
bounce-back, free-slip = specular reflection, per face (run.walls).
Device vs the C oracle's ghost-fill restatement bit for bit (exact
arithmetic), and physics: the Poiseuille profile between no-slip walls.
Parity unpinned: no reference golden exists for walls.  -m gpu."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2402_13171_b200 import Simulation, parse_config

pytestmark = pytest.mark.gpu


def _cfg(cells, periodic, walls, op="cumulant", boundary="periodic", wind=(8.0, 0.3, -0.2),
         arithmetic="exact", precision="double"):
    return parse_config({"domain": {"cells": list(cells), "periodicity": list(periodic)},
                         "fluid": {"kinematic_viscosity": 0.05, "wind": list(wind)},
                         "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                        "mach": 0.1},
                         "run": {"boundary": boundary, "arithmetic": arithmetic,
                                 "precision": precision, "walls": walls,
                                 "collision": {"operator": op}}})


@pytest.mark.parametrize("case", [
    dict(cells=(10, 9, 11), periodic=(True, False, False), boundary="periodic", op="cumulant",
         walls={"y_lo": "no_slip", "y_hi": "no_slip", "z_lo": "no_slip", "z_hi": "no_slip"}),
    dict(cells=(14, 8, 37), periodic=(False, False, True), boundary="velocity_inflow_outflow",
         op="bgk", walls={"y_lo": "free_slip", "y_hi": "no_slip"}),
    dict(cells=(12, 7, 9), periodic=(False, False, False), boundary="velocity_inflow_outflow",
         op="cumulant", walls={"z_lo": "no_slip", "z_hi": "free_slip", "y_hi": "free_slip"}),
    dict(cells=(9, 10, 8), periodic=(True, True, False), boundary="periodic", op="bgk",
         walls={"z_lo": "free_slip", "z_hi": "free_slip"}),
])
def test_walls_bitwise_vs_oracle(gpu, case):
    cfg = _cfg(case["cells"], case["periodic"], case["walls"], case["op"], case["boundary"])
    sim = Simulation(cfg)
    nx, ny, nz = case["cells"]
    rng = np.random.default_rng(nx * 100 + nz)
    f0 = orc.W * (1.0 + 0.2 * rng.uniform(-1, 1, (nx, ny, nz, 27)))
    F = rng.uniform(-1e-4, 1e-4, (nx, ny, nz, 3))
    sim.fields[0].interior = f0
    sim.fields[0].interior_force = F
    ref = orc.OracleSim(case["cells"], periodic=case["periodic"], op=case["op"],
                        omega=sim.units.omega, boundary=case["boundary"],
                        u_in=sim.boundary.u_in_lat, walls=cfg.wall_codes())
    ref.interior[...] = f0
    ref.force[1:-1, 1:-1, 1:-1] = F
    for _ in range(10):
        sim.step()
        ref.step()
    got = sim.fields[0].interior
    sim._recompute_moments()
    macro = sim.fields[0].interior_macro
    sim.close()
    assert np.array_equal(got, ref.interior)
    assert np.array_equal(macro, ref.recompute_moments())


@pytest.mark.parametrize("op", ["bgk", "cumulant"])
def test_poiseuille_between_no_slip_walls(gpu, op):
    """Body-force channel between halfway bounce-back walls at y = -1/2 and
    ny - 1/2: u(y) = F/(2 nu) s (H - s), s = y + 1/2, H = ny."""
    H = 24
    cfg = parse_config({"domain": {"cells": [4, H, 4], "periodicity": [True, False, True]},
                        "fluid": {"kinematic_viscosity": 0.3249, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.05},
                        "run": {"arithmetic": "fast", "walls": {"y_lo": "no_slip",
                                                                "y_hi": "no_slip"},
                                "collision": {"operator": op}}})
    sim = Simulation(cfg)
    nu = sim.units.nu_lat
    F0 = 0.02 * 8.0 * nu / H ** 2
    sim.fields[0].interior_force = np.broadcast_to([F0, 0.0, 0.0], (4, H, 4, 3))
    sim.advance(int(15 * H * H / (np.pi ** 2 * nu)))
    sim._recompute_moments()
    ux = sim.fields[0].interior_macro[..., 1].mean(axis=(0, 2))
    sim.close()
    s = np.arange(H) + 0.5
    analytic = F0 / (2.0 * nu) * s * (H - s)
    err = np.linalg.norm(ux - analytic) / np.linalg.norm(analytic)
    assert err < 0.01, err


def test_free_slip_box_keeps_uniform_flow_and_single_precision(gpu):
    """Uniform flow along x between free-slip walls is a fixed point, and
    fp32-storage wall runs match the float32 oracle bit for bit."""
    cells = (8, 6, 5)
    walls = {f: "free_slip" for f in ("y_lo", "y_hi", "z_lo", "z_hi")}
    sim = Simulation(_cfg(cells, (True, False, False), walls, wind=(8.0, 0.0, 0.0)))
    f0 = sim.fields[0].interior
    sim.advance(20)
    np.testing.assert_allclose(sim.fields[0].interior, f0, rtol=0, atol=1e-15)
    sim.close()
    cfg = _cfg(cells, (True, False, False), walls, wind=(8.0, 0.0, 0.0), precision="single")
    sim = Simulation(cfg)
    rng = np.random.default_rng(3)
    f1 = (orc.W * (1.0 + 0.2 * rng.uniform(-1, 1, cells + (27,)))).astype(np.float32)
    sim.fields[0].interior = f1
    ref = orc.OracleSim(cells, periodic=(True, False, False), op="cumulant",
                        omega=sim.units.omega, walls=cfg.wall_codes(), dtype=np.float32)
    ref.interior[...] = f1
    for _ in range(6):
        sim.step()
        ref.step()
    got = sim.fields[0].interior
    sim.close()
    assert np.array_equal(got, ref.interior)
