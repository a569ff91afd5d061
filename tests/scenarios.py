"""Shared test scenarios: configs for the product and matching oracles."""

import os
import tempfile

import numpy as np

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


def write_rotor_files(d, points_per_blade=6):
    with open(os.path.join(d, "rotor.yaml"), "w") as fh:
        fh.write(ROTOR_YAML.replace("points: 6", f"points: {points_per_blade}"))
    with open(os.path.join(d, "sym.csv"), "w") as fh:
        fh.write(sym_polar_csv())


def rotor_raw(cells, periodic, boundary="periodic", position=(0.9, 0.3, 0.0), steps=0,
              arithmetic="exact", nu=0.866, cpd=8, mach=0.1, operator="cumulant",
              precision="double"):
    res = {"mach": mach} if cpd is None else {"cells_per_diameter": cpd,
                                                "reference_diameter": 1.0, "mach": mach}
    return {"domain": {"cells": list(cells), "periodicity": list(periodic)},
            "fluid": {"kinematic_viscosity": nu, "wind": [8.0, 0.0, 0.0]},
            "resolution": res,
            "run": {"steps": steps, "boundary": boundary, "arithmetic": arithmetic,
                    "precision": precision, "collision": {"operator": operator}},
            "turbines": [{"file": "rotor.yaml", "position": list(position)}],
            "polars": [{"id": "sym", "file": "sym.csv"}]}


def rotor_config(cells=(12, 12, 12), periodic=(True, True, True), boundary="periodic",
                 position=(0.9, 0.3, 0.0), steps=0, arithmetic="exact", points_per_blade=6,
                 **kw):
    """(RunConfig, TemporaryDirectory) for the golden-style rotor."""
    from paper_2402_13171_b200 import parse_config
    tmp = tempfile.TemporaryDirectory()
    write_rotor_files(tmp.name, points_per_blade)
    cfg = parse_config(rotor_raw(cells, periodic, boundary, position, steps, arithmetic, **kw),
                       base_dir=tmp.name)
    return cfg, tmp


def oracle_for(sim):
    """OracleSim with the parameters and initial state of a product
    Simulation (uniform wind product equilibrium)."""
    from oracle import oracle as orc
    cfg, u = sim.cfg, sim.units
    points = None
    if sim.points:
        points = {"chord": np.array([p.chord for p in sim.points]),
                  "element_length": np.array([p.element_length for p in sim.points]),
                  "twist": np.array([p.twist for p in sim.points]),
                  "polar": [None if p.polar is None else (p.polar.alpha, p.polar.cl, p.polar.cd)
                            for p in sim.points],
                  "vscale": u.velocity_scale, "rho_ref": u.rho_ref, "dt2": u.dt ** 2,
                  "den": u.rho_ref * u.dx ** 4,
                  "area": np.array([p.area for p in sim.points]),
                  "disks": [(sl.start, spec.rings, spec.sectors, spec.thrust_coefficient)
                            for comp, spec, offs, areas, sl in sim._disk_groups],
                  "spreading": (cfg.spread_kernel, cfg.spread_epsilon)}
    ref = orc.OracleSim(cfg.cells, periodic=cfg.periodicity, op=cfg.operator, omega=u.omega,
                        rates=cfg.higher_order_rates, boundary=cfg.boundary_kind,
                        u_in=sim.boundary.u_in_lat, points=points, dtype=cfg.dtype,
                        walls=cfg.wall_codes())
    ref.initialize_equilibrium(1.0, sim.boundary.u_in_lat, product=(cfg.operator == "cumulant"))
    return ref


def disk_config(disk_yaml):
    """(RunConfig, TemporaryDirectory) of the golden actuator-disk run
    (tests/golden/make_golden.py gen_disk)."""
    from paper_2402_13171_b200 import parse_config
    tmp = tempfile.TemporaryDirectory()
    with open(os.path.join(tmp.name, "d.yaml"), "w") as fh:
        fh.write(disk_yaml)
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 0, "collision": {"operator": "cumulant"}},
           "turbines": [{"file": "d.yaml"}]}
    return parse_config(raw, base_dir=tmp.name), tmp
