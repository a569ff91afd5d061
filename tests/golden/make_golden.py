"""Generate the golden vectors in tests/golden/ by running the REFERENCE
implementation (/root/reference/pkg/src/lbwind, read-only) in this
container.  The reference does not exist on the GPU box; the fixtures it
produces are committed and travel instead.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_golden \
        python tests/golden/make_golden.py

Fixtures (numpy .npz, fp64):
  collide.npz    batch collide, both operators, several rate sets, with and
                 without force (collision.collide -> _kernels.*_batch)
  block.npz      collide_field / moments_block / stream_pull_block on a
                 ghosted 4x3x5 block
  tgv.npz        12x10x8 periodic cumulant run (Simulation.step x 6)
  inflow.npz     14x8x6 velocity_inflow_outflow BGK + cumulant runs with a
                 perturbed start (x 5)
  rotor_*.npz    rotating 3-blade actuator line on 12^3 periodic and 16x12x12
                 inflow/outflow domains (x 8): per-step kinematics, sampled
                 rho/u, blade forces, final populations and force field
  disk.npz       2-ring actuator disk on 16^3 (x 6)
  single.npz     precision: single TGV, inflow/outflow BGK and rotor runs
  disk_wake.npz  (--wake) test_05's reduced wake case at 8 and 12 cells per
                 diameter: deficit, axis / plane-mean u_x, ring forces
  output.npz     (--output) the files Simulation.run() writes (output.py:44-167):
                 probe CSVs (axial_line, radial_profile, running averages) and
                 the VTK dump of a perturbed inflow/outflow run, and the
                 blade_loads CSVs of a rotor run, verbatim (text)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("LBWIND_SRC", "/root/reference/pkg/src"))

import lbwind  # noqa: E402
from lbwind import _kernels  # noqa: E402
from lbwind.collision import CollisionConfig, collide  # noqa: E402
from lbwind.config import parse_config  # noqa: E402
from lbwind.fields import PdfField, collide_field  # noqa: E402
from lbwind.sim import Simulation  # noqa: E402
from lbwind.stencil import W  # noqa: E402

# test-local fixtures in the style of the reference's own tests
# (test_acceptance.py:48-98)
ROTOR_YAML = """
name: alm
components:
  - name: tower
    position: [0.0, 0.0, 0.0]
  - name: nacelle
    parent: tower
    position: [0.0, 0.0, 0.8]
  - name: hub
    parent: nacelle
    position: [-0.05, 0.0, 0.0]
    rotation: {axis: [1.0, 0.0, 0.0], rate_rad_per_s: 96.0}
  - name: blade1
    parent: hub
    discretization: {type: line, points: 6, r_start: 0.06, r_end: 0.48,
                     chord: 0.08, twist_deg: 8.0, polar: sym}
  - name: blade2
    parent: hub
    orientation: {axis: [1.0, 0.0, 0.0], angle_deg: 120.0}
    discretization: {type: line, points: 6, r_start: 0.06, r_end: 0.48,
                     chord: 0.08, twist_deg: 8.0, polar: sym}
  - name: blade3
    parent: hub
    orientation: {axis: [1.0, 0.0, 0.0], angle_deg: 240.0}
    discretization: {type: line, points: 6, r_start: 0.06, r_end: 0.48,
                     chord: 0.08, twist_deg: 8.0, polar: sym}
"""


def sym_polar_csv():
    a = np.arange(-180.0, 181.0, 15.0)
    r = np.deg2rad(a)
    rows = ["alpha_deg,cl,cd"]
    rows += [f"{x},{0.9 * np.sin(2 * t):.6f},{0.08 + 0.3 * (1 - np.cos(2 * t)):.6f}"
             for x, t in zip(a, r)]
    return "\n".join(rows) + "\n"


def random_states(n, seed, amp=0.3):
    rng = np.random.default_rng(seed)
    return np.tile(W, (n, 1)) * (1.0 + amp * rng.uniform(-1, 1, (n, 27)))


def gen_collide():
    out = {}
    cases = [("bgk", 1.3, (1.0, 1.0, 1.0, 1.0)), ("bgk", 1.0, (1.0, 1.0, 1.0, 1.0)),
             ("cumulant", 1.3, (1.0, 1.0, 1.0, 1.0)),
             ("cumulant", 1.7857, (1.1, 1.2, 0.9, 1.4)),
             ("cumulant", 1.0, (1.0, 1.0, 1.0, 1.0))]
    for k, (op, omega, rates) in enumerate(cases):
        f = random_states(96, seed=5 + k)
        F = np.random.default_rng(100 + k).uniform(-1e-3, 1e-3, (96, 3))
        F[::3] = 0.0            # force-free rows exercise the no-Guo path
        cfg = CollisionConfig(operator=op, omega=omega, higher_order_rates=rates)
        out[f"c{k}_op"] = np.array(op)
        out[f"c{k}_omega"] = np.array(omega)
        out[f"c{k}_rates"] = np.array(rates)
        out[f"c{k}_f"] = f
        out[f"c{k}_F"] = F
        out[f"c{k}_out"] = collide(f, F, cfg)
    out["ncases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "collide.npz"), **out)


def gen_block():
    rng = np.random.default_rng(17)
    blk = PdfField((4, 3, 5))
    f0 = random_states(4 * 3 * 5, seed=17).reshape(4, 3, 5, 27)
    F0 = rng.uniform(-1e-3, 1e-3, (4, 3, 5, 3))
    blk.f[...] = random_states(blk.f[..., 0].size, seed=18).reshape(blk.f.shape)
    blk.interior[...] = f0
    blk.interior_force[...] = F0
    out = {"f_in": blk.f.copy(), "force": blk.force.copy(), "macro_in": blk.macro.copy()}
    _kernels.moments_block(blk.f, blk.force, blk.macro, 1.0)
    out["moments"] = blk.macro.copy()
    fdst = np.zeros_like(blk.f)
    _kernels.stream_pull_block(blk.f, fdst)
    out["stream"] = fdst
    for op in ("bgk", "cumulant"):
        b2 = PdfField((4, 3, 5))
        b2.f[...] = out["f_in"]
        b2.force[...] = out["force"]
        collide_field(b2, CollisionConfig(operator=op, omega=1.45,
                                          higher_order_rates=(1.0, 1.3, 0.8, 1.0)))
        out[f"collide_{op}_f"] = b2.f.copy()
        out[f"collide_{op}_macro"] = b2.macro.copy()
    np.savez_compressed(os.path.join(HERE, "block.npz"), **out)


def _gather(sim):
    nx, ny, nz = sim.cfg.cells
    out = np.zeros((nx, ny, nz, 27))
    for d in sim.grid.blocks:
        sl = tuple(slice(o, o + s) for o, s in zip(d.origin, d.size))
        out[sl] = sim.fields[d.id].interior
    return out


def gen_tgv():
    raw = {"domain": {"cells": [12, 10, 8]},
           "fluid": {"kinematic_viscosity": 0.1353, "wind": [0.0, 0.0, 0.0],
                     "reference_velocity": 1.0},
           "resolution": {"mach": 0.2},
           "run": {"steps": 0, "collision": {"operator": "cumulant",
                                              "higher_order_rates": [1.0, 1.2, 1.0, 0.9]}}}
    cfg = parse_config(raw)
    sim = Simulation(cfg)
    nx, ny, nz = cfg.cells
    X, Y = np.meshgrid(np.arange(nx) + 0.5, np.arange(ny) + 0.5, indexing="ij")
    u0 = cfg.units.u_lat
    vel = np.zeros((nx, ny, nz, 3))
    vel[..., 0] = (u0 * np.sin(2 * np.pi * X / nx) * np.cos(2 * np.pi * Y / ny))[:, :, None]
    vel[..., 1] = (-u0 * np.cos(2 * np.pi * X / nx) * np.sin(2 * np.pi * Y / ny))[:, :, None]
    vel[..., 2] = 0.3 * u0 * np.sin(2 * np.pi * (np.arange(nz) + 0.5) / nz)[None, None, :]
    sim.fields[0].initialize_equilibrium(1.0, vel, product=True)
    out = {"omega": np.array(cfg.units.omega), "rates": np.array(cfg.higher_order_rates),
           "f0": _gather(sim)}
    for n in range(6):
        sim.step()
        if n in (0, 5):
            out[f"f{n + 1}"] = _gather(sim)
    sim._recompute_moments()
    out["macro6"] = sim.fields[0].interior_macro.copy()
    sim.close()
    np.savez_compressed(os.path.join(HERE, "tgv.npz"), **out)


def gen_inflow():
    out = {}
    for op in ("bgk", "cumulant"):
        raw = {"domain": {"cells": [14, 8, 6], "periodicity": [False, True, True]},
               "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
               "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                              "mach": 0.1},
               "run": {"steps": 0, "boundary": "velocity_inflow_outflow",
                       "collision": {"operator": op}}}
        cfg = parse_config(raw)
        sim = Simulation(cfg)
        rng = np.random.default_rng(23)
        fld = sim.fields[0]
        fld.interior[...] *= 1.0 + 0.01 * rng.uniform(-1, 1, fld.interior.shape)
        out[f"{op}_f0"] = _gather(sim)
        out[f"{op}_omega"] = np.array(cfg.units.omega)
        out[f"{op}_u_in"] = np.asarray(sim.boundary.u_in_lat)
        for _ in range(5):
            sim.step()
        out[f"{op}_f5"] = _gather(sim)
        sim.close()
    np.savez_compressed(os.path.join(HERE, "inflow.npz"), **out)


def gen_rotor(tag, cells, periodicity, boundary, position, tmp):
    with open(os.path.join(tmp, "rotor.yaml"), "w") as fh:
        fh.write(ROTOR_YAML)
    with open(os.path.join(tmp, "sym.csv"), "w") as fh:
        fh.write(sym_polar_csv())
    raw = {"domain": {"cells": list(cells), "periodicity": list(periodicity)},
           "fluid": {"kinematic_viscosity": 0.866, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
           "run": {"steps": 0, "boundary": boundary,
                   "collision": {"operator": "cumulant"}},
           "turbines": [{"file": "rotor.yaml", "position": list(position)}],
           "polars": [{"id": "sym", "file": "sym.csv"}]}
    cfg = parse_config(raw, base_dir=tmp)
    sim = Simulation(cfg)
    P = len(sim.points)
    nsteps = 8
    kin = np.zeros((nsteps, P, 15))
    samples = np.zeros((nsteps, P, 4))
    blade = np.zeros((nsteps, P, 3))
    for n in range(nsteps):
        sim.step()
        for p in sim.points:
            kin[n, p.global_id] = np.concatenate([p.position_lat, p.velocity, p.e_chord,
                                                  p.e_normal, p.e_span])
            samples[n, p.global_id, 0] = p.sampled_rho
            samples[n, p.global_id, 1:] = p.sampled_u
            blade[n, p.global_id] = p.blade_force
    u = cfg.units
    out = {"cells": np.array(cells), "periodicity": np.array(periodicity),
           "boundary": np.array(boundary), "position": np.array(position),
           "kin": kin, "samples": samples, "blade": blade, "f_final": _gather(sim),
           "force_final": sim.fields[0].interior_force.copy(),
           "omega": np.array(u.omega), "dx": np.array(u.dx), "dt": np.array(u.dt),
           "rho_ref": np.array(u.rho_ref), "u_in": np.asarray(sim.boundary.u_in_lat),
           "chord": np.array([p.chord for p in sim.points]),
           "element_length": np.array([p.element_length for p in sim.points]),
           "twist": np.array([p.twist for p in sim.points]),
           "polar_alpha": cfg.polars["sym"].alpha, "polar_cl": cfg.polars["sym"].cl,
           "polar_cd": cfg.polars["sym"].cd, "rotor_yaml": np.array(ROTOR_YAML),
           "polar_csv": np.array(sym_polar_csv())}
    sim.close()
    np.savez_compressed(os.path.join(HERE, f"rotor_{tag}.npz"), **out)


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
      thrust_coefficient: [0.5, 0.3]
"""


def gen_disk(tmp):
    """Actuator disk in the style of test_sim.py:18-31 (16^3, 2 rings x 6)."""
    with open(os.path.join(tmp, "d.yaml"), "w") as fh:
        fh.write(DISK_YAML)
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 0, "collision": {"operator": "cumulant"}},
           "turbines": [{"file": "d.yaml"}]}
    cfg = parse_config(raw, base_dir=tmp)
    sim = Simulation(cfg)
    P = len(sim.points)
    nsteps = 6
    pos = np.zeros((nsteps, P, 3))
    samples = np.zeros((nsteps, P, 4))
    blade = np.zeros((nsteps, P, 3))
    for n in range(nsteps):
        sim.step()
        for p in sim.points:
            pos[n, p.global_id] = p.position_lat
            samples[n, p.global_id, 0] = p.sampled_rho
            samples[n, p.global_id, 1:] = p.sampled_u
            blade[n, p.global_id] = p.blade_force
    out = {"pos": pos, "samples": samples, "blade": blade, "f_final": _gather(sim),
           "force_final": sim.fields[0].interior_force.copy(),
           "area": np.array([p.area for p in sim.points]), "disk_yaml": np.array(DISK_YAML)}
    sim.close()
    np.savez_compressed(os.path.join(HERE, "disk.npz"), **out)


def gen_single(tmp):
    """precision: single (fp32 storage, fp64 arithmetic; config.py:30,
    _kernels.py:5-7): a TGV, an inflow/outflow BGK run and the rotor on the
    inflow domain, as float32 fixtures."""
    out = {}
    # TGV (as gen_tgv)
    cfg = parse_config({"domain": {"cells": [12, 10, 8]},
                        "fluid": {"kinematic_viscosity": 0.1353, "wind": [0.0, 0.0, 0.0],
                                  "reference_velocity": 1.0},
                        "resolution": {"mach": 0.2},
                        "run": {"steps": 0, "precision": "single",
                                "collision": {"operator": "cumulant",
                                              "higher_order_rates": [1.0, 1.2, 1.0, 0.9]}}})
    sim = Simulation(cfg)
    nx, ny, nz = cfg.cells
    X, Y = np.meshgrid(np.arange(nx) + 0.5, np.arange(ny) + 0.5, indexing="ij")
    u0 = cfg.units.u_lat
    vel = np.zeros((nx, ny, nz, 3))
    vel[..., 0] = (u0 * np.sin(2 * np.pi * X / nx) * np.cos(2 * np.pi * Y / ny))[:, :, None]
    vel[..., 1] = (-u0 * np.cos(2 * np.pi * X / nx) * np.sin(2 * np.pi * Y / ny))[:, :, None]
    vel[..., 2] = 0.3 * u0 * np.sin(2 * np.pi * (np.arange(nz) + 0.5) / nz)[None, None, :]
    out["tgv_vel"] = vel
    sim.fields[0].initialize_equilibrium(1.0, vel, product=True)
    out["tgv_f0"] = sim.fields[0].interior.copy()
    out["tgv_omega"] = np.array(cfg.units.omega)
    for _ in range(6):
        sim.step()
    out["tgv_f6"] = sim.fields[0].interior.copy()
    sim._recompute_moments()
    out["tgv_macro6"] = sim.fields[0].interior_macro.copy()
    sim.close()
    # inflow/outflow BGK (as gen_inflow)
    cfg = parse_config({"domain": {"cells": [14, 8, 6], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
                        "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                       "mach": 0.1},
                        "run": {"steps": 0, "precision": "single",
                                "boundary": "velocity_inflow_outflow",
                                "collision": {"operator": "bgk"}}})
    sim = Simulation(cfg)
    rng = np.random.default_rng(29)
    fld = sim.fields[0]
    fld.interior[...] *= 1.0 + 0.01 * rng.uniform(-1, 1, fld.interior.shape)
    out["inflow_f0"] = fld.interior.copy()
    for _ in range(5):
        sim.step()
    out["inflow_f5"] = fld.interior.copy()
    sim.close()
    # rotor, inflow/outflow (as gen_rotor "inflow")
    with open(os.path.join(tmp, "rotor.yaml"), "w") as fh:
        fh.write(ROTOR_YAML)
    with open(os.path.join(tmp, "sym.csv"), "w") as fh:
        fh.write(sym_polar_csv())
    cfg = parse_config({"domain": {"cells": [16, 12, 12], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.866, "wind": [8.0, 0.0, 0.0]},
                        "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                       "mach": 0.1},
                        "run": {"steps": 0, "precision": "single",
                                "boundary": "velocity_inflow_outflow",
                                "collision": {"operator": "cumulant"}},
                        "turbines": [{"file": "rotor.yaml", "position": [0.9, 0.75, 0.0]}],
                        "polars": [{"id": "sym", "file": "sym.csv"}]}, base_dir=tmp)
    sim = Simulation(cfg)
    P, nsteps = len(sim.points), 8
    samples = np.zeros((nsteps, P, 4))
    blade = np.zeros((nsteps, P, 3))
    for n in range(nsteps):
        sim.step()
        for p in sim.points:
            samples[n, p.global_id, 0] = p.sampled_rho
            samples[n, p.global_id, 1:] = p.sampled_u
            blade[n, p.global_id] = p.blade_force
    out["rotor_samples"] = samples
    out["rotor_blade"] = blade
    out["rotor_f_final"] = sim.fields[0].interior.copy()
    out["rotor_force_final"] = sim.fields[0].interior_force.copy()
    sim.close()
    for k in ("tgv_f0", "tgv_f6", "tgv_macro6", "inflow_f0", "inflow_f5", "rotor_f_final",
              "rotor_force_final"):
        assert out[k].dtype == np.float32, k
    np.savez_compressed(os.path.join(HERE, "single.npz"), **out)


WAKE_DISK_YAML = """
name: disk
components:
  - name: hub
    discretization: {type: disk, radius: 0.5, rings: 8, sectors: 16,
                     thrust_coefficient: 0.5}
"""


def wake_observables(sim, sample_velocity):
    """Disk-averaged deficit (test_acceptance.py:381-400) plus the recomputed
    axial velocity on the domain axis and its per-plane mean."""
    edges = np.linspace(0.0, 0.5, 7)
    mids = 0.5 * (edges[:-1] + edges[1:])
    theta = (np.arange(12) + 0.5) * 2.0 * np.pi / 12

    def disk_avg_ux(x_plane):
        tot_a = tot_u = 0.0
        for j in range(6):
            a = (edges[j + 1] ** 2 - edges[j] ** 2) / 12
            for t in theta:
                pos = (x_plane, 2.5 + mids[j] * np.cos(t), 2.5 + mids[j] * np.sin(t))
                tot_u += a * sample_velocity(pos)[0]
                tot_a += a
        return tot_u / tot_a

    return 1.0 - disk_avg_ux(3.0) / disk_avg_ux(1.0)


def gen_disk_wake(tmp):
    """test_05's reduced-resolution wake case (test_acceptance.py:355-441)
    at 8 and 12 cells/diameter: ~12 min of reference CPU time, so only with
    --wake."""
    from lbwind.output import _sample_velocity
    with open(os.path.join(tmp, "wdisk.yaml"), "w") as fh:
        fh.write(WAKE_DISK_YAML)
    out = {"disk_yaml": np.array(WAKE_DISK_YAML)}
    for cpd, steps in ((8, 1200), (12, 1800)):
        cfg = parse_config({
            "domain": {"diameters": [10, 5, 5]},
            "fluid": {"kinematic_viscosity": 0.09237, "wind": [8.0, 0.0, 0.0]},
            "resolution": {"cells_per_diameter": cpd, "reference_diameter": 1.0,
                           "mach": 0.05},
            "run": {"steps": 0, "collision": {"operator": "bgk"}},
            "turbines": [{"file": "wdisk.yaml", "position": [3.0, 2.5, 2.5]}]}, base_dir=tmp)
        sim = Simulation(cfg)
        for _ in range(steps):
            sim.step()
        sim._recompute_moments()
        macro = sim.fields[0].interior_macro
        ny, nz = macro.shape[1:3]
        out[f"cpd{cpd}_steps"] = steps
        out[f"cpd{cpd}_deficit"] = wake_observables(sim, lambda p: _sample_velocity(sim, p))
        out[f"cpd{cpd}_ux_axis"] = macro[:, ny // 2, nz // 2, 1].copy()
        out[f"cpd{cpd}_ux_plane_mean"] = macro[..., 1].mean(axis=(1, 2))
        out[f"cpd{cpd}_blade"] = np.array([p.blade_force for p in sim.points])
        sim.close()
    np.savez_compressed(os.path.join(HERE, "disk_wake.npz"), **out)


OUTPUT_FLOW = {
    "name": "outcase",
    "domain": {"cells": [12, 10, 8], "periodicity": [False, True, True]},
    "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
    "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
    "run": {"steps": 6, "boundary": "velocity_inflow_outflow",
            "collision": {"operator": "cumulant"}},
    "output": {"cadence": 3, "vtk": True,
               "probes": [{"kind": "axial_line", "name": "axial", "samples": 12,
                           "average_from_step": 3},
                          {"kind": "radial_profile", "name": "radial", "samples": 10,
                           "x_m": 0.8, "z_m": 0.4},
                          {"kind": "axial_line", "name": "offaxis", "samples": 7,
                           "y_m": 0.3, "z_m": 0.9}]}}

OUTPUT_ROTOR = {
    "name": "outrotor",
    "domain": {"cells": [16, 12, 12], "periodicity": [False, True, True]},
    "fluid": {"kinematic_viscosity": 0.866, "wind": [8.0, 0.0, 0.0]},
    "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
    "run": {"steps": 8, "boundary": "velocity_inflow_outflow",
            "collision": {"operator": "cumulant"}},
    "turbines": [{"file": "rotor.yaml", "position": [0.9, 0.75, 0.0]}],
    "polars": [{"id": "sym", "file": "sym.csv"}],
    "output": {"cadence": 4,
               "probes": [{"kind": "blade_loads", "name": "loads", "turbine": 0,
                           "component": "blade2", "average_from_step": 4},
                          {"kind": "axial_line", "name": "wake", "samples": 16,
                           "y_m": 0.75, "z_m": 0.0}]}}


def gen_output(tmp):
    """Simulation.run() of the reference with probes and VTK output; every
    file it writes (except report.json, which holds timings) is stored as
    text under '<case>/<file name>'."""
    import copy
    import json
    out = {"rotor_yaml": np.array(ROTOR_YAML), "polar_csv": np.array(sym_polar_csv())}
    for case, raw0 in (("flow", OUTPUT_FLOW), ("rotor", OUTPUT_ROTOR)):
        out[f"{case}_raw"] = np.array(json.dumps(raw0))
        raw = copy.deepcopy(raw0)
        odir = os.path.join(tmp, "out_" + case)
        raw["output"]["directory"] = odir
        if case == "rotor":
            with open(os.path.join(tmp, "rotor.yaml"), "w") as fh:
                fh.write(ROTOR_YAML)
            with open(os.path.join(tmp, "sym.csv"), "w") as fh:
                fh.write(sym_polar_csv())
        cfg = parse_config(raw, base_dir=tmp)
        sim = Simulation(cfg)
        if case == "flow":
            rng = np.random.default_rng(29)
            fld = sim.fields[0]
            fld.interior[...] *= 1.0 + 0.02 * rng.uniform(-1, 1, fld.interior.shape)
            out["flow_f0"] = _gather(sim)
        sim.run()
        sim.close()
        for fn in sorted(os.listdir(odir)):
            if fn == "report.json":
                continue
            with open(os.path.join(odir, fn)) as fh:
                out[f"{case}/{fn}"] = np.array(fh.read())
    np.savez_compressed(os.path.join(HERE, "output.npz"), **out)


def main():
    import tempfile
    if "--output" in sys.argv:
        _kernels.warm_up()
        with tempfile.TemporaryDirectory() as tmp:
            gen_output(tmp)
        return
    if "--single" in sys.argv:
        with tempfile.TemporaryDirectory() as tmp:
            gen_single(tmp)
        return
    if "--wake" in sys.argv:
        with tempfile.TemporaryDirectory() as tmp:
            gen_disk_wake(tmp)
        return
    _kernels.warm_up()
    gen_collide()
    gen_block()
    gen_tgv()
    gen_inflow()
    with tempfile.TemporaryDirectory() as tmp:
        gen_rotor("periodic", (12, 12, 12), (True, True, True), "periodic",
                  (0.9, 0.3, 0.0), tmp)
        gen_rotor("inflow", (16, 12, 12), (False, True, True), "velocity_inflow_outflow",
                  (0.9, 0.75, 0.0), tmp)
        gen_disk(tmp)
        gen_single(tmp)
    print("golden vectors written to", HERE, "with lbwind", lbwind.__version__)


if __name__ == "__main__":
    main()
