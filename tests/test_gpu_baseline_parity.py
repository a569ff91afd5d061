"""Parity at the BASELINE.json configurations' own sizes, against the C
oracle (pinned to the reference's golden vectors, tests/test_oracle.py).

  C1  64^3 periodic Taylor-Green vortex, 600 steps: exact arithmetic is
      bit-identical; fast arithmetic within 1e-10.
  C2  the benchmark itself (bench.py's config: 256x128x128, inflow /
      outflow, the 18-point rotor):
        exact, host kinematics, 20 steps -- the oracle spreads the device's
        blade forces, so every one of the 4.2 M cells' populations and the
        force field are compared BIT FOR BIT every run; the oracle's own
        blade forces (same state) are compared to 1e-10 and the samples
        to 1e-12 each step;
        fast, device kinematics (exactly the benchmarked path), 50 steps:
        samples, blade forces and populations within 1e-10 relative.
  C5' the C5 setup at a quarter of its resolution: an aligned row of three
      rotors at 4D / 11D / 18D with 50 points per blade (450 points: the
      pooled-force K5 path, many points per cell), a turbulent-like
      init_modes start, 10 steps; exact (host kinematics, injected
      forces: populations bit-identical) and fast (device kinematics,
      1e-10).

Tolerances: the actuator path's trilinear sums, dot products and atan2
are not bit-reproducible between numpy/libm and the device (SURVEY.md
§8c), hence 1e-12 (samples) / 1e-10 (blade forces) there; everything the
LBM does is compared bitwise in exact arithmetic.
"""

import os
import tempfile

import numpy as np
import pytest

import bench
from oracle import oracle as orc
from paper_2402_13171_b200 import Simulation, parse_config
from paper_2402_13171_b200.fields import fourier_modes
from paper_2402_13171_b200.sim import HostKinematics
from tests.scenarios import oracle_for

pytestmark = pytest.mark.gpu

RTOL_SAMPLE = 1e-12
RTOL_BLADE = 1e-10
RTOL_FAST = 1e-10


def _rel(a, b):
    scale = max(float(np.abs(b).max()), 1e-300)
    return float(np.abs(a - b).max()) / scale


def _bench_cfg(name, arithmetic):
    tmp = tempfile.TemporaryDirectory()
    cfg, _ = bench.make_config(name, 1, arithmetic, tmp.name)
    return cfg, tmp


# ------------------------------------------------------------------- C1

def _tgv_field(n, u0):
    k = 2.0 * np.pi / n
    c = (np.arange(n) + 0.5) * k
    X, Y, Z = np.meshgrid(c, c, c, indexing="ij")
    u = np.zeros((n, n, n, 3))
    u[..., 0] = u0 * np.sin(X) * np.cos(Y) * np.cos(Z)
    u[..., 1] = -u0 * np.cos(X) * np.sin(Y) * np.cos(Z)
    return orc.product_equilibrium(np.ones((n, n, n)), u)


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_c1_tgv64_600_steps_vs_oracle(gpu, arithmetic):
    raw = {"domain": {"cells": [64, 64, 64]},
           "fluid": {"kinematic_viscosity": 0.02, "wind": [0.0, 0.0, 0.0],
                     "reference_velocity": 1.0},
           "resolution": {"mach": 0.1, "cells_per_diameter": 32},
           "run": {"arithmetic": arithmetic,
                   "collision": {"operator": "cumulant",
                                 "higher_order_rates": [1.0, 1.0, 1.0, 1.0]}}}
    sim = Simulation(parse_config(raw))
    ref = oracle_for(sim)
    f0 = _tgv_field(64, 0.05)
    sim.fields[0].interior = f0
    ref.interior[...] = f0
    sim.advance(600)
    for _ in range(600):
        ref.step()
    got = sim.fields[0].interior
    sim.close()
    if arithmetic == "exact":
        assert np.array_equal(got, ref.interior)
    else:
        assert _rel(got, ref.interior) <= RTOL_FAST
    # the vortex decayed but is still there (not a trivial fixed point)
    assert np.abs(ref.interior - f0).max() > 1e-4


# ------------------------------------------------------------------- C2

def test_c2_bench_config_exact_bitwise_vs_oracle(gpu):
    cfg, tmp = _bench_cfg("c2", "exact")
    cfg2, tmp2 = _bench_cfg("c2", "exact")
    sim = Simulation(cfg, kinematics="host")
    host = HostKinematics(cfg2)
    ref = oracle_for(host)
    for n in range(20):
        kin = host.refresh()
        host.advance()
        sim.step()
        rho, u, blade = sim._alm_results()
        assert np.array_equal(sim._kin_view(), kin), n
        ref.step(kin, blade=blade)
        np.testing.assert_allclose(rho, ref.samples[:, 0], rtol=RTOL_SAMPLE)
        np.testing.assert_allclose(u, ref.samples[:, 1:], rtol=1e-11, atol=1e-16)
        np.testing.assert_allclose(blade, ref.blade_own, rtol=RTOL_BLADE, atol=1e-13)
    assert np.abs(blade).max() > 0.0
    assert np.array_equal(sim.fields[0].interior, ref.interior)
    assert np.array_equal(sim.fields[0].interior_force, ref.force[1:-1, 1:-1, 1:-1])
    sim.close()
    tmp.cleanup()
    tmp2.cleanup()


def test_c2_bench_config_fast_vs_oracle(gpu):
    cfg, tmp = _bench_cfg("c2", "fast")
    cfg2, tmp2 = _bench_cfg("c2", "fast")
    sim = Simulation(cfg)            # device kinematics: the benchmarked path
    assert sim.kinematics == "device"
    host = HostKinematics(cfg2)
    ref = oracle_for(host)
    worst = {"rho": 0.0, "u": 0.0, "blade": 0.0}
    for n in range(50):
        kin = host.refresh()
        host.advance()
        sim.step()
        rho, u, blade = sim._alm_results()
        ref.step(kin)
        worst["rho"] = max(worst["rho"], _rel(rho, ref.samples[:, 0]))
        worst["u"] = max(worst["u"], _rel(u, ref.samples[:, 1:]))
        worst["blade"] = max(worst["blade"], _rel(blade, ref.blade))
    f = sim.fields[0].interior
    sim.close()
    print("C2 fast vs oracle after 50 steps:", worst, "f:", _rel(f, ref.interior))
    assert all(v <= RTOL_FAST for v in worst.values()), worst
    assert _rel(f, ref.interior) <= RTOL_FAST
    tmp.cleanup()
    tmp2.cleanup()


# ------------------------------------------------------------------- C5'

def _c5_reduced_cfg(arithmetic, cpd=16):
    """configs[4] at cpd 16 (quarter resolution): 384x128x128, the three
    rotors of bench.py's c5 at x = 4.05 / 11.05 / 18.05 m, 50 points per
    blade."""
    tmp = tempfile.TemporaryDirectory()
    with open(os.path.join(tmp.name, "rotor.yaml"), "w") as fh:
        fh.write(bench.ROTOR.replace("points: 6", "points: 50"))
    with open(os.path.join(tmp.name, "sym.csv"), "w") as fh:
        fh.write(bench.polar_csv())
    raw = {"domain": {"cells": [24 * cpd, 8 * cpd, 8 * cpd], "periodicity": [False, True, True]},
           "fluid": {"kinematic_viscosity": 0.0866, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": cpd, "reference_diameter": 1.0, "mach": 0.05},
           "run": {"boundary": "velocity_inflow_outflow", "arithmetic": arithmetic,
                   "collision": {"operator": "cumulant"}},
           "turbines": [{"file": "rotor.yaml", "position": [x, 4.0, 3.2]}
                        for x in (4.05, 11.05, 18.05)],
           "polars": [{"id": "sym", "file": "sym.csv"}]}
    return parse_config(raw, base_dir=tmp.name), tmp


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_c5_reduced_three_rotors_450_points_vs_oracle(gpu, arithmetic):
    cfg, tmp = _c5_reduced_cfg(arithmetic)
    cfg2, tmp2 = _c5_reduced_cfg(arithmetic)
    exact = arithmetic == "exact"
    sim = Simulation(cfg, kinematics="host" if exact else "device")
    host = HostKinematics(cfg2)
    assert len(sim.points) == 450 and len(cfg.topologies) == 3
    ref = oracle_for(host)
    u0 = sim.boundary.u_in_lat
    sim.fields[0].initialize_modes(1.0, u0, fourier_modes(cfg.cells, u0), product=True)
    # the device-generated turbulent-like start is the common input
    ref.interior[...] = sim.fields[0].interior
    ref.macro[1:-1, 1:-1, 1:-1] = sim.fields[0].interior_macro
    worst = {"rho": 0.0, "u": 0.0, "blade": 0.0}
    for n in range(10):
        kin = host.refresh()
        host.advance()
        sim.step()
        rho, u, blade = sim._alm_results()
        ref.step(kin, blade=blade if exact else None)
        own = ref.blade_own
        worst["rho"] = max(worst["rho"], _rel(rho, ref.samples[:, 0]))
        worst["u"] = max(worst["u"], _rel(u, ref.samples[:, 1:]))
        worst["blade"] = max(worst["blade"], _rel(blade, own))
    f = sim.fields[0].interior
    F = sim.fields[0].interior_force
    sim.close()
    print(f"C5' {arithmetic} vs oracle after 10 steps:", worst, "f:", _rel(f, ref.interior))
    assert np.abs(blade).max() > 0.0
    if exact:
        assert worst["rho"] <= RTOL_SAMPLE and worst["u"] <= 1e-11, worst
        assert worst["blade"] <= RTOL_BLADE, worst
        assert np.array_equal(f, ref.interior)
        assert np.array_equal(F, ref.force[1:-1, 1:-1, 1:-1])
    else:
        assert all(v <= RTOL_FAST for v in worst.values()), worst
        assert _rel(f, ref.interior) <= RTOL_FAST
    tmp.cleanup()
    tmp2.cleanup()
