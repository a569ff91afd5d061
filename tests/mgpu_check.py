"""Multi-GPU transparency check, run under torchrun (one process per GPU):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mgpu_check.py

Every case runs the same configuration on N x-slabs (N GPUs, peer halo
stores + GPU-side ordering) and on one GPU, and requires the gathered
populations, force fields and actuator loads to be bit-identical (the
reference's decomposition-transparency contract, test_acceptance.py:316-348).
Exit code 0 = all identical.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_13171_b200 import Simulation, parse_config  # noqa: E402
from paper_2402_13171_b200.parallel import SlabSimulation  # noqa: E402
from tests.scenarios import rotor_config  # noqa: E402


def lbm_raw(cells, periodic, boundary, op, arithmetic):
    return {"domain": {"cells": list(cells), "periodicity": list(periodic)},
            "fluid": {"kinematic_viscosity": 0.05, "wind": [0.02, 0.005, -0.003],
                      "reference_velocity": 1.0},
            "resolution": {"mach": 0.1, "cells_per_diameter": 32},
            "run": {"boundary": boundary, "arithmetic": arithmetic,
                    "collision": {"operator": op, "higher_order_rates": [1.1, 0.9, 1.3, 1.0]}}}


DISK = """
name: d
components:
  - name: mast
    position: [2.9, 2.0, 2.0]
    orientation: {axis: [0.0, 0.0, 1.0], angle_deg: YAW}
  - name: rotor
    parent: mast
    discretization: {type: disk, radius: 1.0, rings: 2, sectors: 6,
                     thrust_coefficient: [0.5, 0.3]}
"""


def disk_cfg(nx, yaw):
    import tempfile
    d = tempfile.mkdtemp()
    with open(os.path.join(d, "d.yaml"), "w") as fh:
        fh.write(DISK.replace("YAW", repr(yaw)))
    return parse_config({"domain": {"cells": [nx, 16, 16], "periodicity": [False, True, True]},
                         "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
                         "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0,
                                        "mach": 0.1},
                         "run": {"boundary": "velocity_inflow_outflow", "arithmetic": "fast",
                                 "collision": {"operator": "cumulant"}},
                         "turbines": [{"file": "d.yaml"}]}, base_dir=d)


def run_case(name, make_cfg, steps, perturb, kinematics=None):
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = make_cfg()
    sim = SlabSimulation(cfg, rank, world, device=rank, kinematics=kinematics)
    nx = cfg.cells[0]
    f0 = None
    if perturb:
        rng = np.random.default_rng(11)
        x0 = sim.grid.blocks[0].origin[0]
        full = rng.uniform(-1, 1, (nx,) + tuple(cfg.cells[1:]) + (27,))
        mine = sim.fields[0].interior.view(np.ndarray)
        f0 = mine * (1.0 + 0.02 * full[x0:x0 + mine.shape[0]])
        sim.fields[0].interior = f0
    for _ in range(steps):
        sim.step()
    sim.synchronize()
    got_f = sim.gather_interior()
    got_F = sim.gather_force()
    loads = sim.alm_results_global() if sim.points else None
    sim.close()
    ok = True
    if rank == 0:
        ref = Simulation(make_cfg(), device=0, kinematics=kinematics)
        if perturb:
            rng = np.random.default_rng(11)
            full = rng.uniform(-1, 1, (nx,) + tuple(cfg.cells[1:]) + (27,))
            ref.fields[0].interior = ref.fields[0].interior * (1.0 + 0.02 * full)
        for _ in range(steps):
            ref.step()
        ref.synchronize()
        want_f = ref.fields[0].interior.view(np.ndarray)
        want_F = ref.fields[0].interior_force.view(np.ndarray)
        ok = np.array_equal(got_f, want_f) and np.array_equal(got_F, want_F)
        detail = f"max|df|={np.abs(got_f - want_f).max():.3e}"
        if loads is not None:
            rho, u, blade = ref._alm_results()
            ok = ok and np.array_equal(loads[2], blade) and np.array_equal(loads[0], rho)
            detail += f" max|dF_blade|={np.abs(loads[2] - blade).max():.3e}"
        ref.close()
        print(f"[{name}] world={world} {'OK' if ok else 'MISMATCH'} {detail}", flush=True)
    flag = torch.tensor([0 if ok else 1])
    dist.broadcast(flag, 0)
    return flag.item() == 0


def output_case(world, nx):
    """Probes (axial line, radial profile with running average, blade loads)
    and VTK dumps of a run over N slabs are the same files as one GPU's."""
    import filecmp
    import tempfile
    rank = dist.get_rank()
    base = tempfile.mkdtemp() if rank == 0 else None
    holder = [base]
    dist.broadcast_object_list(holder, 0)
    base = holder[0]
    from tests.scenarios import rotor_raw, write_rotor_files
    files = os.path.join(base, "files")
    if rank == 0:   # one writer, the others read after the barrier
        os.makedirs(files, exist_ok=True)
        write_rotor_files(files)
    dist.barrier()

    def cfg_for(out):
        raw = rotor_raw((nx, 12, 12), (True, True, True), position=(1.5, 0.3, 0.0), steps=6,
                        arithmetic="fast")
        raw["output"] = {"directory": out, "cadence": 3, "vtk": True,
                         "probes": [{"kind": "axial_line", "name": "ax", "samples": 7},
                                    {"kind": "radial_profile", "name": "rp", "x_m": 1.4,
                                     "samples": 5, "average_from_step": 3},
                                    {"kind": "blade_loads", "name": "bl", "turbine": 0,
                                     "component": "blade1"}]}
        return parse_config(raw, base_dir=files)

    from paper_2402_13171_b200.parallel import run_slab_simulation
    multi = os.path.join(base, "multi")
    run_slab_simulation(cfg_for(multi), kinematics="device")
    ok = True
    if rank == 0:
        from paper_2402_13171_b200 import run_simulation
        single = os.path.join(base, "single")
        run_simulation(cfg_for(single))
        names = sorted(f for f in os.listdir(single) if f != "report.json")
        same = [filecmp.cmp(os.path.join(single, f), os.path.join(multi, f), shallow=False)
                for f in names]
        ok = len(names) > 6 and all(same) and os.path.exists(os.path.join(multi, "report.json"))
        print(f"[output-files] world={world} {'OK' if ok else 'MISMATCH'} "
              f"{sum(same)}/{len(names)} identical"
              + ("" if ok else f" differ: {[n for n, e in zip(names, same) if not e]}"),
              flush=True)
    flag = torch.tensor([0 if ok else 1])
    dist.broadcast(flag, 0)
    return flag.item() == 0


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(rank)
    world = dist.get_world_size()
    nx = 12 * world
    ok = True
    ok &= run_case("periodic-cumulant-exact",
                   lambda: parse_config(lbm_raw((nx, 16, 13), (True, True, True), "periodic",
                                                "cumulant", "exact")), 8, True)
    ok &= run_case("inflow-bgk-fast",
                   lambda: parse_config(lbm_raw((nx + 3, 10, 16), (False, True, True),
                                                "velocity_inflow_outflow", "bgk", "fast")), 8, True)
    ok &= run_case("nonperiodic-yz-cumulant",
                   lambda: parse_config(lbm_raw((nx, 9, 7), (True, False, False), "periodic",
                                                "cumulant", "fast")), 6, True)
    # walls on every y / z face (extension): bounce-back / specular sources
    # next to the slab faces
    def walls_cfg():
        raw = lbm_raw((nx + 1, 9, 8), (False, False, False), "velocity_inflow_outflow",
                      "cumulant", "exact")
        raw["run"]["walls"] = {"y_lo": "no_slip", "y_hi": "free_slip", "z_lo": "free_slip",
                               "z_hi": "no_slip"}
        return parse_config(raw)
    ok &= run_case("walls-inflow-cumulant", walls_cfg, 8, True)
    # fp32 storage: float ghost planes across the slab faces
    ok &= run_case("rotor-single",
                   lambda: rotor_config(cells=(nx, 12, 12), position=(1.5, 0.3, 0.0),
                                        arithmetic="exact", precision="single")[0], 8, False)
    # rotor plane at x = 11.6 cells: sampling cubes and Roma supports straddle
    # the face between slabs 0 and 1; blades cross the periodic y face too
    for arith, kin in (("exact", "host"), ("fast", "device")):
        ok &= run_case(f"rotor-{arith}-{kin}",
                       lambda: rotor_config(cells=(nx, 12, 12), position=(1.5, 0.3, 0.0),
                                            arithmetic=arith)[0], 10, False, kinematics=kin)
    # 90 points: the many-point path (K5 fills per-row pools)
    ok &= run_case("rotor-many-points",
                   lambda: rotor_config(cells=(nx, 12, 12), position=(1.5, 0.3, 0.0),
                                        arithmetic="fast", points_per_blade=30)[0], 8, False)
    # Gaussian spreading (support half-width 4 x cells across the slab face)
    def gaussian_cfg():
        import tempfile
        from tests.scenarios import rotor_raw, write_rotor_files
        d = tempfile.mkdtemp()
        write_rotor_files(d)
        raw = rotor_raw((nx, 12, 12), (True, True, True), position=(1.5, 0.3, 0.0),
                        arithmetic="fast")
        raw["run"]["spreading"] = {"kernel": "gaussian", "epsilon": 1.0}
        return parse_config(raw, base_dir=d)
    ok &= run_case("rotor-gaussian", gaussian_cfg, 8, False)
    # actuator disks: an aligned disk on the slab face and a yawed one whose
    # rings spread over neighbouring slabs (ring averages across GPUs)
    for name, yaw in (("disk-aligned", 0.0), ("disk-yawed", 35.0)):
        ok &= run_case(name, lambda yaw=yaw: disk_cfg(nx, yaw), 8, False)
    ok &= output_case(world, nx)
    # the benchmark's weak-scaled C2 configuration itself (256 planes per
    # GPU, rotor, inflow / outflow, fast arithmetic, device kinematics)
    ok &= run_case("bench-c2-weak",
                   lambda: rotor_config(cells=(256 * world, 128, 128), periodic=(False, True, True),
                                        boundary="velocity_inflow_outflow",
                                        position=(2.0, 2.0, 1.2), arithmetic="fast", cpd=32,
                                        nu=0.1732, mach=0.05)[0], 6, False, kinematics="device")
    if os.environ.get("LBW_MGPU_LONG"):
        # test_acceptance.py test_04 at its size: 64^3 periodic, one rotating
        # 3-blade turbine, 200 steps (slabs of 64/world planes)
        ok &= run_case("test04-64cubed-200steps",
                       lambda: rotor_config(cells=(64, 64, 64), position=(1.0, 1.0, 0.2),
                                            nu=0.1732, cpd=None, mach=0.05,
                                            arithmetic="exact")[0], 200, False)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
