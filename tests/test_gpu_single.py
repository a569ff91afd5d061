"""``precision: single`` on the device (config.py:30,
_kernels.py:5-7): populations and forces stored fp32, all arithmetic fp64,
values rounded to nearest on every store as the reference's float32 fields
do.  Against the reference's own single-precision runs (golden single.npz)
and the float32 oracle.  -m gpu.

Tolerances: exact arithmetic bit-identical; fast (FMA) arithmetic within
two float32 ulps (the fp64 results differ in the last double bits, which
occasionally moves a float32 rounding).
"""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2402_13171_b200 import NumericalAbort, Simulation, parse_config
from tests.scenarios import rotor_config

pytestmark = pytest.mark.gpu

F32_ULP = 2.0 ** -23


def _close_f32(got, want, ulps=2):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    tol = ulps * F32_ULP * np.maximum(np.abs(want), 1e-30)
    bad = np.abs(got - want) > tol
    assert not bad.any(), (int(bad.sum()), float(np.abs(got - want).max()))


def _tgv_sim(arithmetic):
    cfg = parse_config({"domain": {"cells": [12, 10, 8]},
                        "fluid": {"kinematic_viscosity": 0.1353, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.2},
                        "run": {"precision": "single", "arithmetic": arithmetic,
                                "collision": {"operator": "cumulant",
                                              "higher_order_rates": [1.0, 1.2, 1.0, 0.9]}}})
    return Simulation(cfg)


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_tgv_single_vs_reference(gpu, golden, arithmetic):
    g = golden("single.npz")
    sim = _tgv_sim(arithmetic)
    assert sim.units.omega == float(g["tgv_omega"])
    sim.fields[0].initialize_equilibrium(1.0, g["tgv_vel"], product=True)
    f0 = sim.fields[0].interior
    assert f0.dtype == np.float32
    assert np.array_equal(f0, g["tgv_f0"])
    for _ in range(6):
        sim.step()
    f6 = sim.fields[0].interior
    sim._recompute_moments()
    macro = sim.fields[0].interior_macro
    sim.close()
    assert macro.dtype == np.float32
    if arithmetic == "exact":
        assert np.array_equal(f6, g["tgv_f6"])
        assert np.array_equal(macro, g["tgv_macro6"])
    else:
        _close_f32(f6, g["tgv_f6"])
        _close_f32(macro, g["tgv_macro6"])


def test_inflow_outflow_single_vs_reference(gpu, golden):
    g = golden("single.npz")
    cfg = parse_config({"domain": {"cells": [14, 8, 6], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
                        "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                       "mach": 0.1},
                        "run": {"precision": "single", "boundary": "velocity_inflow_outflow",
                                "collision": {"operator": "bgk"}}})
    sim = Simulation(cfg)
    sim.fields[0].interior = g["inflow_f0"]
    for _ in range(5):
        sim.step()
    got = sim.fields[0].interior
    sim.close()
    assert np.array_equal(got, g["inflow_f5"])


@pytest.mark.parametrize("kinematics", ["host", "device"])
def test_rotor_single_vs_reference(gpu, golden, kinematics):
    g = golden("single.npz")
    cfg, tmp = rotor_config((16, 12, 12), (False, True, True), "velocity_inflow_outflow",
                            (0.9, 0.75, 0.0), precision="single")
    sim = Simulation(cfg, kinematics=kinematics)
    for n in range(g["rotor_samples"].shape[0]):
        sim.step()
        rho, u, blade = sim._alm_results()
        np.testing.assert_allclose(rho, g["rotor_samples"][n, :, 0], rtol=1e-12)
        np.testing.assert_allclose(u, g["rotor_samples"][n, :, 1:], rtol=1e-11, atol=1e-16)
        np.testing.assert_allclose(blade, g["rotor_blade"][n], rtol=1e-10, atol=1e-13)
    f = sim.fields[0].interior
    F = sim.fields[0].interior_force
    sim.close()
    tmp.cleanup()
    assert f.dtype == np.float32 and F.dtype == np.float32
    _close_f32(f, g["rotor_f_final"], ulps=1)
    _close_f32(F, g["rotor_force_final"], ulps=1)


@pytest.mark.parametrize("case", [
    dict(cells=(40, 24, 20), periodic=(True, True, True), boundary="periodic", op="cumulant"),
    dict(cells=(33, 17, 45), periodic=(False, True, True), boundary="velocity_inflow_outflow",
         op="cumulant"),
    dict(cells=(18, 16, 7), periodic=(False, True, False), boundary="velocity_inflow_outflow",
         op="bgk"),
])
def test_random_state_single_vs_oracle(gpu, case):
    """Ragged sizes (z pitch 32 floats), non-periodic y/z, body force:
    exact arithmetic bit-identical to the float32 oracle over 12 steps."""
    nx, ny, nz = case["cells"]
    cfg = parse_config({"domain": {"cells": list(case["cells"]),
                                   "periodicity": list(case["periodic"])},
                        "fluid": {"kinematic_viscosity": 0.05, "wind": [8.0, 0.3, -0.2]},
                        "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                       "mach": 0.1},
                        "run": {"precision": "single", "boundary": case["boundary"],
                                "collision": {"operator": case["op"]}}})
    sim = Simulation(cfg)
    rng = np.random.default_rng(nx * 1000 + nz)
    f0 = (orc.W * (1.0 + 0.2 * rng.uniform(-1, 1, (nx, ny, nz, 27)))).astype(np.float32)
    F = rng.uniform(-1e-4, 1e-4, (nx, ny, nz, 3)).astype(np.float32)
    sim.fields[0].interior = f0
    sim.fields[0].interior_force = F
    ref = orc.OracleSim(case["cells"], periodic=case["periodic"], op=case["op"],
                        omega=sim.units.omega, boundary=case["boundary"],
                        u_in=sim.boundary.u_in_lat, dtype=np.float32)
    ref.interior[...] = f0
    ref.force[1:-1, 1:-1, 1:-1] = F
    for _ in range(12):
        sim.step()
        ref.step()
    got = sim.fields[0].interior
    sim._recompute_moments()
    macro = sim.fields[0].interior_macro
    sim.close()
    assert np.array_equal(got, ref.interior)
    assert np.array_equal(macro, ref.recompute_moments())


def test_single_precision_run(gpu, tmp_path):
    """test_sim.py:284-291 on the device."""
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 5, "precision": "single"},
           "output": {"directory": str(tmp_path / "out")}}
    sim = Simulation(parse_config(raw))
    for _ in range(5):
        sim.step()
    assert sim.fields[0].f.dtype == np.float32
    assert np.all(np.isfinite(sim.fields[0].interior))
    assert sim.report()["kernel"]["bytes_per_update"] == 228
    sim.close()


def test_single_nan_abort(gpu):
    cfg = parse_config({"domain": {"cells": [8, 8, 8]},
                        "fluid": {"kinematic_viscosity": 0.1, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.1},
                        "run": {"precision": "single"}})
    sim = Simulation(cfg)
    f = sim.fields[0].interior
    f[3, 4, 5, 7] = np.nan
    with pytest.raises(NumericalAbort) as e:
        sim.step()
        sim.synchronize()
    assert e.value.step == 0 and tuple(e.value.cell) == (3, 4, 5)
    sim.close()


def test_large_single_uniform_fixed_point(gpu):
    """96x64x80 uniform wind, inflow/outflow, fast arithmetic: stays a fixed
    point to float32 rounding over 50 steps (storage-only change)."""
    cfg = parse_config({"domain": {"cells": [96, 64, 80], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.1, "wind": [8.0, 0.0, 0.0]},
                        "resolution": {"cells_per_diameter": 16, "reference_diameter": 1.0,
                                       "mach": 0.05},
                        "run": {"precision": "single", "arithmetic": "fast",
                                "boundary": "velocity_inflow_outflow"}})
    sim = Simulation(cfg)
    f0 = sim.fields[0].interior
    for _ in range(50):
        sim.step()
    _close_f32(sim.fields[0].interior, f0, ulps=4)
    sim.close()
