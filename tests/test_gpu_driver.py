"""Driver-level behaviour on the GPU: the reference's own driver and
acceptance contracts (test_sim.py, test_acceptance.py) re-run through this
package's Simulation / run_simulation — fixed points, probes and reports,
momentum budgets, actuator disks, the Taylor-Green decay rate and the
Poiseuille profile.  -m gpu.
"""

import json
import os
import warnings

import numpy as np
import pytest

from paper_2402_13171_b200 import C, Simulation, parse_config, run_simulation
from paper_2402_13171_b200.output import gather_global_fields
from tests.scenarios import disk_config

pytestmark = pytest.mark.gpu

FLAT_POLAR = "alpha_deg,cl,cd\n-10,1.0,0.0\n10,1.0,0.0\n"
DISK_YAML = """
name: d
components:
  - name: mast
    position: [2.0, 2.0, 2.0]
  - name: rotor
    parent: mast
    discretization:
      type: disk
      radius: 1.0
      rings: 2
      sectors: 6
      thrust_coefficient: 0.5
"""


def base(tmp_path, **over):
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 5},
           "output": {"directory": str(tmp_path / "out")}}
    for k, v in over.items():
        raw[k] = dict(raw[k], **v) if isinstance(v, dict) and isinstance(raw.get(k), dict) else v
    return raw


def with_disk(tmp_path, raw):
    (tmp_path / "d.yaml").write_text(DISK_YAML)
    raw["turbines"] = [{"file": "d.yaml"}]
    return raw


@pytest.mark.parametrize("kinematics", ["host", "device"])
def test_actuator_disk_vs_reference(gpu, golden, kinematics):
    g = golden("disk.npz")
    cfg, tmp = disk_config(str(g["disk_yaml"]))
    sim = Simulation(cfg, kinematics=kinematics)
    for n in range(g["pos"].shape[0]):
        sim.step()
        pos = sim._kin_view()[:, 0:3]
        if kinematics == "host":
            assert np.array_equal(pos, g["pos"][n])
        else:
            np.testing.assert_allclose(pos, g["pos"][n], rtol=0, atol=1e-12)
        rho, u, blade = sim._alm_results()
        np.testing.assert_allclose(rho, g["samples"][n, :, 0], rtol=1e-12)
        np.testing.assert_allclose(blade, g["blade"][n], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(sim.fields[0].interior, g["f_final"], rtol=0, atol=1e-14)
    sim.close()
    tmp.cleanup()


def test_quiescent_box_is_a_fixed_point(gpu, tmp_path):
    raw = base(tmp_path, fluid={"wind": [0.0, 0.0, 0.0], "kinematic_viscosity": 0.5,
                                "reference_velocity": 1.0})
    sim = Simulation(parse_config(raw))
    before = sim.fields[0].interior
    for _ in range(5):
        sim.step()
    np.testing.assert_allclose(sim.fields[0].interior, before, rtol=0.0, atol=1e-12)
    sim.close()


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_uniform_wind_is_a_fixed_point(gpu, tmp_path, arithmetic):
    raw = base(tmp_path, run={"arithmetic": arithmetic})
    cfg = parse_config(raw)
    sim = Simulation(cfg)
    before = sim.fields[0].interior
    for _ in range(5):
        sim.step()
    np.testing.assert_allclose(sim.fields[0].interior, before, rtol=0.0, atol=1e-12)
    wind_lat = cfg.units.velocity_to_lattice(np.array([8.0, 0.0, 0.0]))
    macro = sim.fields[0].interior_macro
    np.testing.assert_allclose(macro[..., 1:4], np.broadcast_to(wind_lat, macro[..., 1:4].shape),
                               atol=1e-13)
    sim.close()


def test_zero_steps_is_a_valid_run(gpu, tmp_path):
    raw = base(tmp_path, run={"steps": 0},
               output={"probes": [{"kind": "axial_line", "samples": 4, "name": "ax"}]})
    report = run_simulation(parse_config(raw))
    assert report["performance"]["steps"] == 0
    assert "mlups" not in report["performance"]
    assert os.path.exists(tmp_path / "out" / "report.json")
    rows = np.loadtxt(tmp_path / "out" / "ax_00000000.csv", delimiter=",", skiprows=1)
    np.testing.assert_allclose(rows[:, 1], 8.0, atol=1e-12)


def test_blade_loads_probe_matches_blade_element_theory(gpu, tmp_path):
    (tmp_path / "blade.yaml").write_text("""
name: b
components:
  - name: root
    position: [2.0, 2.0, 1.5]
  - name: blade
    parent: root
    discretization: {type: line, points: 3, r_end: 0.8, chord: 0.1, polar: flat}
""")
    (tmp_path / "flat.csv").write_text(FLAT_POLAR)
    raw = base(tmp_path, run={"steps": 1},
               output={"cadence": 1, "probes": [{"kind": "blade_loads", "name": "loads",
                                                 "turbine": 0, "component": "blade"}]})
    raw["turbines"] = [{"file": "blade.yaml"}]
    raw["polars"] = [{"id": "flat", "file": "flat.csv"}]
    run_simulation(parse_config(raw, base_dir=str(tmp_path)))
    rows = np.loadtxt(tmp_path / "out" / "loads_00000001.csv", delimiter=",", skiprows=1)
    np.testing.assert_allclose(rows[:, 0], [0.0, 0.5, 1.0], atol=1e-15)
    np.testing.assert_allclose(rows[:, 1], 0.0, atol=1e-12)
    np.testing.assert_allclose(rows[:, 2], -0.5 * 1.225 * 8.0 ** 2 * 0.1, rtol=1e-9)


def test_driver_momentum_budget_with_disk(gpu, tmp_path):
    cfg = parse_config(with_disk(tmp_path, base(tmp_path, run={"steps": 1})),
                       base_dir=str(tmp_path))
    sim = Simulation(cfg)

    def momentum():
        return np.einsum("xyzi,ic->c", sim.fields[0].interior, C.astype(np.float64))

    before = momentum()
    sim.step()
    deposited = sim.fields[0].interior_force.sum(axis=(0, 1, 2))
    np.testing.assert_allclose(momentum() - before, deposited, rtol=1e-10, atol=5e-12)
    total_newton = sum(p.fluid_force for p in sim.points)
    np.testing.assert_allclose(deposited, cfg.units.force_to_lattice(total_newton), rtol=1e-12,
                               atol=1e-16)
    sim.close()


def test_probe_running_average(gpu, tmp_path):
    raw = with_disk(tmp_path, base(tmp_path, run={"steps": 4},
                                   output={"cadence": 2, "probes": [
                                       {"kind": "radial_profile", "name": "rp", "x_m": 3.0,
                                        "samples": 6, "average_from_step": 0}]}))
    run_simulation(parse_config(raw, base_dir=str(tmp_path)))
    out = tmp_path / "out"
    inst2 = np.loadtxt(out / "rp_00000002.csv", delimiter=",", skiprows=1)
    inst4 = np.loadtxt(out / "rp_00000004.csv", delimiter=",", skiprows=1)
    avg2 = np.loadtxt(out / "rp_avg_00000002.csv", delimiter=",", skiprows=1)
    avg4 = np.loadtxt(out / "rp_avg_00000004.csv", delimiter=",", skiprows=1)
    np.testing.assert_array_equal(avg2, inst2)
    np.testing.assert_allclose(avg4[:, 1], 0.5 * (inst2[:, 1] + inst4[:, 1]), rtol=1e-14)


def test_inflow_outflow_preserves_uniform_wind(gpu, tmp_path):
    raw = base(tmp_path, domain={"cells": [32, 16, 16], "periodicity": [False, True, True]},
               run={"steps": 10, "boundary": "velocity_inflow_outflow"})
    cfg = parse_config(raw)
    sim = Simulation(cfg)
    for _ in range(10):
        sim.step()
    _, vel, _ = gather_global_fields(sim)
    np.testing.assert_allclose(vel, 8.0 * np.broadcast_to([1.0, 0.0, 0.0], vel.shape),
                               atol=1e-9)
    sim.close()


def test_report_contents(gpu, tmp_path):
    raw = base(tmp_path, run={"steps": 3})
    raw["machine"] = {"name": "desk", "stream_bandwidth_GB_s": 10.0, "peak_tflops": 1.0}
    report = run_simulation(parse_config(raw))
    perf = report["performance"]
    assert perf["steps"] == 3 and perf["mlups"] > 0 and perf["percent_of_peak"] > 0
    assert sum(perf["phase_seconds"].values()) <= perf["wall_seconds"] + 1e-6
    assert report["machine"]["lightspeed"] <= 1.0
    with open(tmp_path / "out" / "report.json") as fh:
        assert json.load(fh)["performance"]["steps"] == 3


def test_repeat_runs_bitwise(gpu, tmp_path):
    outs = []
    for k in range(2):
        raw = with_disk(tmp_path, base(tmp_path, run={"steps": 8}))
        sim = Simulation(parse_config(raw, base_dir=str(tmp_path)))
        for _ in range(8):
            sim.step()
        outs.append(sim.fields[0].interior)
        sim.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_taylor_green_decay_rate(gpu, arithmetic):
    """test_acceptance.py:216-255: kinetic energy of a z-invariant TGV at
    64^3, Mach 0.02, decays at 4 nu k^2 within 2 % (601 steps)."""
    cfg = parse_config({"domain": {"cells": [64, 64, 64]},
                        "fluid": {"kinematic_viscosity": 0.1353, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.02},
                        "run": {"arithmetic": arithmetic, "collision": {"operator": "cumulant"}}})
    sim = Simulation(cfg)
    k = 2.0 * np.pi / 64.0
    u0 = cfg.units.u_lat
    X, Y = np.meshgrid(np.arange(64) + 0.5, np.arange(64) + 0.5, indexing="ij")
    vel = np.zeros((64, 64, 64, 3))
    vel[..., 0] = (u0 * np.sin(k * X) * np.cos(k * Y))[:, :, None]
    vel[..., 1] = (-u0 * np.cos(k * X) * np.sin(k * Y))[:, :, None]
    sim.fields[0].initialize_equilibrium(1.0, vel, product=True)
    ts, es = [], []
    for n in range(601):
        if n >= 100 and n % 50 == 0:
            sim._recompute_moments()
            ts.append(float(n))
            es.append(float(np.sum(sim.fields[0].interior_macro[..., 1:4] ** 2)))
        sim.step()
    sim.close()
    fit = np.polyfit(ts, np.log(es), 1)[0]
    analytic = -4.0 * cfg.units.nu_lat * k * k
    assert abs(fit / analytic - 1.0) < 0.02, (fit, analytic)


def _channel_error(H):
    """test_acceptance.py:258-300: mirrored body-force channel, BGK."""
    cfg = parse_config({"domain": {"cells": [4, 2 * H, 4]},
                        "fluid": {"kinematic_viscosity": 0.3249, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.05},
                        "run": {"collision": {"operator": "bgk"}}})
    u = cfg.units
    sim = Simulation(cfg)
    F0 = 0.02 * 8.0 * u.nu_lat / H ** 2
    F = np.zeros((4, 2 * H, 4, 3))
    F[:, :H, :, 0] = F0
    F[:, H:, :, 0] = -F0
    sim.fields[0].interior_force = F
    steps = int(12 * H * H / (np.pi ** 2 * u.nu_lat))
    lib_steps = 0
    while lib_steps < steps:
        n = min(1000, steps - lib_steps)
        for _ in range(n):
            sim.step()
        lib_steps += n
    sim._recompute_moments()
    ux = sim.fields[0].interior_macro[..., 1].mean(axis=(0, 2))
    sim.close()
    j = np.arange(2 * H)
    y = np.where(j < H, j + 0.5, 2 * H - (j + 0.5))
    analytic = np.where(j < H, 1.0, -1.0) * F0 / (2.0 * u.nu_lat) * y * (H - y)
    return float(np.linalg.norm(ux - analytic) / np.linalg.norm(analytic))


def test_poiseuille_profile_and_convergence(gpu):
    e32, e64 = _channel_error(32), _channel_error(64)
    assert e32 < 0.01, e32
    assert e32 / e64 >= 3.5, (e32, e64)


def test_polar_clamp_warns_once(gpu, tmp_path):
    (tmp_path / "blade.yaml").write_text("""
name: b
components:
  - name: hub
    position: [2.0, 2.0, 2.0]
    rotation: {axis: [1.0, 0.0, 0.0], rate_rad_per_s: 50.0}
  - name: blade
    parent: hub
    discretization: {type: line, points: 3, r_end: 1.0, chord: 0.1, polar: flat}
""")
    (tmp_path / "flat.csv").write_text(FLAT_POLAR)
    raw = base(tmp_path, run={"steps": 3})
    raw["turbines"] = [{"file": "blade.yaml"}]
    raw["polars"] = [{"id": "flat", "file": "flat.csv"}]
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        run_simulation(parse_config(raw, base_dir=str(tmp_path)))
    assert sum("clamping" in str(x.message) for x in w) == 1
