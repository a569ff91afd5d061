"""Pin the CPU oracle (oracle/) against the reference's own outputs.

Golden vectors come from tests/golden/make_golden.py, which runs the
reference package.  LBM layers must match bit for bit; the actuator-line
numpy restatement must match to 1e-12 relative (numpy einsum / BLAS dot
summation order is implementation-defined).
"""

import numpy as np
import pytest

from oracle import oracle as orc


def test_batch_collide_bitwise(golden):
    g = golden("collide.npz")
    for k in range(int(g["ncases"])):
        out, _ = orc.collide_batch(str(g[f"c{k}_op"]), g[f"c{k}_f"], g[f"c{k}_F"],
                                   float(g[f"c{k}_omega"]), tuple(g[f"c{k}_rates"]))
        assert np.array_equal(out, g[f"c{k}_out"]), k


def test_block_kernels_bitwise(golden):
    g = golden("block.npz")
    f = g["f_in"].copy()
    force = g["force"].copy()
    macro = g["macro_in"].copy()
    orc.moments_block(f, force, macro)
    assert np.array_equal(macro, g["moments"])
    dst = np.zeros_like(f)
    orc.stream_pull_block(f, dst)
    assert np.array_equal(dst, g["stream"])
    for op in ("bgk", "cumulant"):
        f = g["f_in"].copy()
        macro = g["macro_in"].copy()
        orc.collide_block(op, f, force.copy(), macro, 1.45, (1.0, 1.3, 0.8, 1.0))
        assert np.array_equal(f, g[f"collide_{op}_f"]), op
        inner = (slice(1, -1),) * 3
        assert np.array_equal(macro[inner], g[f"collide_{op}_macro"][inner]), op


def test_tgv_steps_bitwise(golden):
    g = golden("tgv.npz")
    nx, ny, nz = g["f0"].shape[:3]
    sim = orc.OracleSim((nx, ny, nz), op="cumulant", omega=float(g["omega"]),
                        rates=tuple(g["rates"]))
    sim.interior[...] = g["f0"]
    for n in range(6):
        sim.step()
        if n == 0:
            assert np.array_equal(sim.interior, g["f1"])
    assert np.array_equal(sim.interior, g["f6"])
    assert np.array_equal(sim.recompute_moments(), g["macro6"])


@pytest.mark.parametrize("op", ["bgk", "cumulant"])
def test_inflow_outflow_bitwise(golden, op):
    g = golden("inflow.npz")
    f0 = g[f"{op}_f0"]
    sim = orc.OracleSim(f0.shape[:3], periodic=(False, True, True), op=op,
                        omega=float(g[f"{op}_omega"]), boundary="velocity_inflow_outflow",
                        u_in=g[f"{op}_u_in"])
    sim.interior[...] = f0
    for _ in range(5):
        sim.step()
    assert np.array_equal(sim.interior, g[f"{op}_f5"])


@pytest.mark.parametrize("tag", ["periodic", "inflow"])
def test_rotor_alm_matches_reference(golden, tag):
    g = golden(f"rotor_{tag}.npz")
    sim, kin = oracle_rotor(g)
    for n in range(kin.shape[0]):
        sim.step(kin[n])
        np.testing.assert_allclose(sim.samples, g["samples"][n], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(sim.blade, g["blade"][n], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(sim.interior, g["f_final"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(sim.force[1:-1, 1:-1, 1:-1], g["force_final"],
                               rtol=1e-10, atol=1e-16)


def oracle_rotor(g):
    """OracleSim configured like the golden rotor run (the initial state is
    the uniform-wind product equilibrium of Simulation.__init__)."""
    u_in = g["u_in"]
    cells = tuple(int(c) for c in g["cells"])
    dx, dt, rho_ref = float(g["dx"]), float(g["dt"]), float(g["rho_ref"])
    P = g["chord"].shape[0]
    polar = (g["polar_alpha"], g["polar_cl"], g["polar_cd"])
    points = {"chord": g["chord"], "element_length": g["element_length"],
              "twist": g["twist"], "polar": [polar] * P, "vscale": dx / dt,
              "rho_ref": rho_ref, "dt2": dt ** 2, "den": rho_ref * dx ** 4}
    sim = orc.OracleSim(cells, periodic=tuple(bool(p) for p in g["periodicity"]),
                        op="cumulant", omega=float(g["omega"]), boundary=str(g["boundary"]),
                        u_in=u_in, points=points)
    wind = u_in if str(g["boundary"]) != "periodic" else u_in
    sim.initialize_equilibrium(1.0, wind, product=True)
    return sim, g["kin"]


def test_oracle_against_live_reference(reference_lbwind):
    """Beyond the fixtures: random batch states with fresh seeds, run through
    the reference in-process (build container only)."""
    from lbwind.collision import CollisionConfig, collide
    rng = np.random.default_rng(2402)
    for op in ("bgk", "cumulant"):
        f = np.tile(orc.W, (500, 1)) * (1.0 + 0.4 * rng.uniform(-1, 1, (500, 27)))
        F = rng.uniform(-3e-3, 3e-3, (500, 3))
        cfg = CollisionConfig(operator=op, omega=1.61, higher_order_rates=(0.7, 1.5, 1.1, 1.9))
        ref = collide(f, F, cfg)
        out, _ = orc.collide_batch(op, f, F, 1.61, (0.7, 1.5, 1.1, 1.9))
        assert np.array_equal(out, ref), op


def test_disk_oracle_matches_reference(golden):
    """Actuator disk (actuator.py:149-183): host kinematics bit-identical, the
    oracle's samples / ring forces / populations match the reference."""
    from paper_2402_13171_b200.sim import HostKinematics
    from tests.scenarios import disk_config, oracle_for
    g = golden("disk.npz")
    cfg, tmp = disk_config(str(g["disk_yaml"]))
    host = HostKinematics(cfg)
    ref = oracle_for(host)
    for n in range(g["pos"].shape[0]):
        kin = host.refresh()
        assert np.array_equal(kin[:, 0:3], g["pos"][n])
        ref.step(kin)
        host.advance()
        np.testing.assert_allclose(ref.samples, g["samples"][n], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(ref.blade, g["blade"][n], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(ref.interior, g["f_final"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ref.force[1:-1, 1:-1, 1:-1], g["force_final"], rtol=1e-10,
                               atol=1e-18)
    tmp.cleanup()


def test_single_precision_oracle_matches_reference(golden):
    """precision: single (config.py:30; fp32 storage, fp64 arithmetic):
    TGV and inflow/outflow BGK bit-exact; rotor samples / forces to the
    actuator tolerance."""
    from paper_2402_13171_b200 import parse_config
    from paper_2402_13171_b200.sim import HostKinematics
    from tests.scenarios import oracle_for, rotor_config
    g = golden("single.npz")
    # TGV 12x10x8
    ref = orc.OracleSim((12, 10, 8), op="cumulant", omega=float(g["tgv_omega"]),
                        rates=(1.0, 1.2, 1.0, 0.9), dtype=np.float32)
    ref.initialize_equilibrium(1.0, g["tgv_vel"], product=True)
    assert np.array_equal(ref.interior, g["tgv_f0"])
    for _ in range(6):
        ref.step()
    assert np.array_equal(ref.interior, g["tgv_f6"])
    assert np.array_equal(ref.recompute_moments(), g["tgv_macro6"])
    # inflow/outflow BGK
    cfg = parse_config({"domain": {"cells": [14, 8, 6], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
                        "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0,
                                       "mach": 0.1},
                        "run": {"precision": "single", "boundary": "velocity_inflow_outflow",
                                "collision": {"operator": "bgk"}}})
    u_in = cfg.units.velocity_to_lattice(np.array([8.0, 0.5, -0.25]))
    ref = orc.OracleSim((14, 8, 6), periodic=(False, True, True), op="bgk",
                        omega=cfg.units.omega, boundary="velocity_inflow_outflow", u_in=u_in,
                        dtype=np.float32)
    ref.interior[...] = g["inflow_f0"]
    for _ in range(5):
        ref.step()
    assert np.array_equal(ref.interior, g["inflow_f5"])
    # rotor on the inflow domain
    cfg, tmp = rotor_config((16, 12, 12), (False, True, True), "velocity_inflow_outflow",
                            (0.9, 0.75, 0.0), precision="single")
    host = HostKinematics(cfg)
    ref = oracle_for(host)
    for n in range(g["rotor_samples"].shape[0]):
        kin = host.refresh()
        ref.step(kin)
        host.advance()
        np.testing.assert_allclose(ref.samples, g["rotor_samples"][n], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(ref.blade, g["rotor_blade"][n], rtol=1e-10, atol=1e-13)
    # the float32 rounding absorbs the einsum-order noise of the actuator path
    assert np.array_equal(ref.interior, g["rotor_f_final"])
    assert np.array_equal(ref.force[1:-1, 1:-1, 1:-1], g["rotor_force_final"])
    tmp.cleanup()


def test_wall_oracle_free_slip_fixed_point_and_closed_box_mass():
    """Walls (an extension; the reference has none): uniform flow along x
    between free-slip y / z walls is a fixed point, and a closed box
    (periodic x, no-slip y / z) conserves mass exactly."""
    u = np.array([0.03, 0.0, 0.0])
    sim = orc.OracleSim((6, 5, 7), periodic=(True, False, False), op="cumulant", omega=1.3,
                        walls=(2, 2, 2, 2))
    sim.initialize_equilibrium(1.0, u, product=True)
    f0 = sim.interior.copy()
    for _ in range(5):
        sim.step()
    np.testing.assert_allclose(sim.interior, f0, rtol=0, atol=1e-15)
    rng = np.random.default_rng(5)
    box = orc.OracleSim((6, 5, 7), periodic=(True, False, False), op="bgk", omega=1.1,
                        walls=(1, 1, 1, 1))
    box.interior[...] = orc.W * (1.0 + 0.1 * rng.uniform(-1, 1, box.interior.shape))
    m0 = box.interior.sum()
    for _ in range(10):
        box.step()
    assert abs(box.interior.sum() - m0) < 1e-12 * m0
