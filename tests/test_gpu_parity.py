"""GPU parity: liblbw kernels vs the reference (golden vectors) and vs the
bit-exact C oracle, through the C ABI.  Run on a B200: pytest -m gpu.

Tolerances (stated per north star):
  * LBM populations, exact arithmetic: bit-identical (np.array_equal).
  * LBM populations, fast (FMA) arithmetic: |f - f_ref| <= 1e-13 per step
    horizon tested, <= 1e-10 after 200 steps.
  * Actuator samples (rho, u): 1e-12 relative; blade forces 1e-10 relative
    (numpy einsum/BLAS/libm summation and atan2 are not reproducible
    bit-for-bit).
"""

import warnings

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2402_13171_b200 import (CollisionConfig, NumericalAbort, Simulation, collide,
                                   kernels, parse_config)
from paper_2402_13171_b200 import _lib
from tests.scenarios import oracle_for, rotor_config

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ K0

def test_batch_collide_exact_bitwise(gpu, golden):
    g = golden("collide.npz")
    for k in range(int(g["ncases"])):
        cfg = CollisionConfig(str(g[f"c{k}_op"]), float(g[f"c{k}_omega"]),
                              tuple(g[f"c{k}_rates"]))
        out = collide(g[f"c{k}_f"], g[f"c{k}_F"], cfg)
        assert np.array_equal(out, g[f"c{k}_out"]), k


def test_batch_collide_fast_close(gpu, golden):
    g = golden("collide.npz")
    for k in range(int(g["ncases"])):
        cfg = CollisionConfig(str(g[f"c{k}_op"]), float(g[f"c{k}_omega"]),
                              tuple(g[f"c{k}_rates"]))
        out = collide(g[f"c{k}_f"], g[f"c{k}_F"], cfg, mode="fast")
        np.testing.assert_allclose(out, g[f"c{k}_out"], rtol=0, atol=2e-15)


def test_batch_collide_large_random_vs_oracle(gpu):
    rng = np.random.default_rng(99)
    n = 200_000
    f = np.tile(orc.W, (n, 1)) * (1.0 + 0.4 * rng.uniform(-1, 1, (n, 27)))
    F = rng.uniform(-2e-3, 2e-3, (n, 3))
    F[rng.random(n) < 0.5] = 0.0
    for op in ("bgk", "cumulant"):
        cfg = CollisionConfig(op, 1.37, (0.8, 1.2, 1.6, 0.4))
        want, _ = orc.collide_batch(op, f, F, 1.37, (0.8, 1.2, 1.6, 0.4))
        assert np.array_equal(collide(f, F, cfg), want), op


def test_empty_batch(gpu):
    out = collide(np.zeros((0, 27)), None, CollisionConfig("cumulant", 1.2))
    assert out.shape == (0, 27)


# ---------------------------------------------------- block entry points

def test_block_kernels_bitwise(gpu, golden):
    g = golden("block.npz")
    macro = g["macro_in"].copy()
    kernels.moments_block(g["f_in"].copy(), g["force"].copy(), macro, 1.0)
    assert np.array_equal(macro, g["moments"])
    dst = np.zeros_like(g["f_in"])
    kernels.stream_pull_block(g["f_in"].copy(), dst)
    assert np.array_equal(dst, g["stream"])
    inner = (slice(1, -1),) * 3
    for op in ("bgk", "cumulant"):
        f, macro = g["f_in"].copy(), g["macro_in"].copy()
        if op == "bgk":
            kernels.collide_bgk_block(f, g["force"].copy(), macro, 1.45, 1.0)
        else:
            kernels.collide_cumulant_block(f, g["force"].copy(), macro, 1.45, 1.0, 1.3, 0.8,
                                           1.0, 1.0)
        assert np.array_equal(f, g[f"collide_{op}_f"]), op
        assert np.array_equal(macro[inner], g[f"collide_{op}_macro"][inner]), op


# ----------------------------------------------------- device time step

def _lbm_sim(cells, periodic=(True, True, True), boundary="periodic", op="cumulant",
             arithmetic="exact", nu=0.1353, wind=(0.0, 0.0, 0.0), mach=0.2, cpd=32,
             rates=(1.0, 1.0, 1.0, 1.0)):
    raw = {"domain": {"cells": list(cells), "periodicity": list(periodic)},
           "fluid": {"kinematic_viscosity": nu, "wind": list(wind), "reference_velocity": 1.0},
           "resolution": {"mach": mach, "cells_per_diameter": cpd},
           "run": {"boundary": boundary, "arithmetic": arithmetic,
                   "collision": {"operator": op, "higher_order_rates": list(rates)}}}
    return Simulation(parse_config(raw))


@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
def test_tgv_vs_reference(gpu, golden, arithmetic):
    g = golden("tgv.npz")
    sim = _lbm_sim(g["f0"].shape[:3], rates=tuple(g["rates"]), mach=0.2, arithmetic=arithmetic)
    assert sim.units.omega == float(g["omega"])
    sim.fields[0].interior = g["f0"]
    sim.step()
    got1 = sim.fields[0].interior
    for _ in range(5):
        sim.step()
    got6 = sim.fields[0].interior
    sim._recompute_moments()
    macro = sim.fields[0].interior_macro
    sim.close()
    if arithmetic == "exact":
        assert np.array_equal(got1, g["f1"])
        assert np.array_equal(got6, g["f6"])
        assert np.array_equal(macro, g["macro6"])
    else:
        np.testing.assert_allclose(got6, g["f6"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(macro, g["macro6"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("op", ["bgk", "cumulant"])
def test_inflow_outflow_vs_reference(gpu, golden, op):
    g = golden("inflow.npz")
    raw = {"domain": {"cells": [14, 8, 6], "periodicity": [False, True, True]},
           "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
           "run": {"boundary": "velocity_inflow_outflow", "collision": {"operator": op}}}
    sim = Simulation(parse_config(raw))
    assert np.array_equal(sim.boundary.u_in_lat, g[f"{op}_u_in"])
    sim.fields[0].interior = g[f"{op}_f0"]
    for _ in range(5):
        sim.step()
    got = sim.fields[0].interior
    sim.close()
    assert np.array_equal(got, g[f"{op}_f5"])


@pytest.mark.parametrize("case", [
    dict(cells=(40, 24, 20), periodic=(True, True, True), boundary="periodic", op="cumulant"),
    dict(cells=(33, 17, 13), periodic=(False, True, True), boundary="velocity_inflow_outflow",
         op="cumulant"),
    dict(cells=(20, 9, 35), periodic=(True, False, True), boundary="periodic", op="bgk"),
    dict(cells=(18, 16, 7), periodic=(False, True, False), boundary="velocity_inflow_outflow",
         op="bgk"),
    dict(cells=(12, 10, 40), periodic=(False, False, False), boundary="periodic",
         op="cumulant"),
])
def test_random_state_many_steps_vs_oracle(gpu, case):
    """Ragged sizes (z not a multiple of 16, odd y), non-periodic y/z (zero
    ghosts), inflow/outflow and both operators: bit-identical after 12
    steps of a perturbed state."""
    sim = _lbm_sim(case["cells"], case["periodic"], case["boundary"], case["op"],
                   nu=0.05, wind=(0.02, 0.005, -0.003), mach=0.1, rates=(1.1, 0.9, 1.3, 1.0))
    ref = oracle_for(sim)
    rng = np.random.default_rng(7)
    f0 = ref.interior * (1.0 + 0.02 * rng.uniform(-1, 1, ref.interior.shape))
    ref.interior[...] = f0
    sim.fields[0].interior = f0
    for _ in range(12):
        sim.step()
        ref.step()
    got = sim.fields[0].interior
    sim.close()
    assert np.array_equal(got, ref.interior)


def test_body_force_field_bitwise(gpu):
    """A user force field persists across steps when no actuator points exist
    (Poiseuille-style forcing, test_acceptance.py:258-300)."""
    sim = _lbm_sim((16, 24, 8), op="bgk", nu=0.3249, mach=0.05)
    ref = oracle_for(sim)
    F = np.zeros((16, 24, 8, 3))
    F[:, :12, :, 0] = 1e-5
    F[:, 12:, :, 0] = -1e-5
    F[3, 5, :, 1] = 2e-6
    sim.fields[0].interior_force[...] = F
    ref.force[1:-1, 1:-1, 1:-1] = F
    for _ in range(20):
        sim.step()
        ref.step()
    assert np.array_equal(sim.fields[0].interior, ref.interior)
    assert np.array_equal(sim.fields[0].interior_force, F)
    sim.close()


def test_fast_mode_drift_200_steps(gpu):
    sims = [_lbm_sim((32, 32, 32), arithmetic=a, nu=0.02, wind=(0.03, 0.0, 0.0), mach=0.1)
            for a in ("exact", "fast")]
    rng = np.random.default_rng(3)
    f0 = sims[0].fields[0].interior * (1.0 + 0.01 * rng.uniform(-1, 1, (32, 32, 32, 27)))
    for s in sims:
        s.fields[0].interior = f0
        for _ in range(200):
            s.step()
    a, b = (s.fields[0].interior for s in sims)
    for s in sims:
        s.close()
    assert np.abs(a - b).max() <= 1e-10


def test_large_domain_properties(gpu):
    """Size-independent properties at a bench-sized domain: mass is conserved
    and a uniform product-equilibrium flow is a fixed point."""
    sim = _lbm_sim((256, 128, 128), nu=0.02, wind=(0.03, 0.01, 0.0), mach=0.1,
                   arithmetic="fast")
    f0 = sim.fields[0].interior
    for _ in range(10):
        sim.step()
    f1 = sim.fields[0].interior
    sim.close()
    assert np.abs(f1 - f0).max() < 1e-15
    assert abs(f1.sum() / f0.sum() - 1.0) < 1e-13


def test_bench_size_rotor_momentum_budget(gpu):
    """test_sim.py:207-231's momentum budget at the benchmark's size (C2,
    256x128x128, periodic so nothing leaves): each step's change of the
    lattice momentum equals the force that step's collide applied, summed
    over the 4.2 M cells -- a size-independent check of sampling, blade
    forces, spreading and Guo forcing together.  The change is summed from
    per-population differences, so the sum is accurate to ~1e-12."""
    cfg, tmp = rotor_config(cells=(256, 128, 128), periodic=(True, True, True),
                            position=(2.0, 2.0, 1.2), arithmetic="fast", cpd=32, nu=0.1732,
                            mach=0.05)
    sim = Simulation(cfg)
    c = orc.C.astype(np.float64)            # (27, 3)
    for _ in range(3):
        sim.step()
    prev = sim.fields[0].interior
    for _ in range(3):
        sim.step()
        cur = sim.fields[0].interior
        dP = np.einsum("xyzi,ic->c", cur - prev, c)
        F = sim.fields[0].interior_force.sum(axis=(0, 1, 2))
        assert np.abs(F).max() > 0.0
        np.testing.assert_allclose(dP, F, rtol=1e-9, atol=1e-15)
        prev = cur
    sim.close()
    tmp.cleanup()


def test_bench_config_deterministic_and_round_trip(gpu):
    """The benchmark configuration itself (C2: 256x128x128, inflow /
    outflow, rotor, fast arithmetic): two runs are bit-identical (no
    float atomics anywhere in the step), and the state round-trips through
    upload / download unchanged."""
    cfg, tmp = rotor_config(cells=(256, 128, 128), periodic=(False, True, True),
                            boundary="velocity_inflow_outflow", position=(2.0, 2.0, 1.2),
                            arithmetic="fast", cpd=32, nu=0.1732, mach=0.05)
    runs = []
    for _ in range(2):
        sim = Simulation(cfg)
        sim.advance(6)
        runs.append((sim.fields[0].interior, sim.fields[0].interior_force,
                     sim._alm_results()[2]))
        sim.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b)
    sim = Simulation(cfg)
    sim.fields[0].interior = runs[0][0]
    assert np.array_equal(sim.fields[0].interior, runs[0][0])
    sim.close()
    tmp.cleanup()


# ----------------------------------------------------------- actuator line

@pytest.mark.parametrize("arithmetic", ["exact", "fast"])
@pytest.mark.parametrize("kinematics", ["host", "device"])
@pytest.mark.parametrize("tag", ["periodic", "inflow"])
def test_rotor_vs_reference(gpu, golden, tag, kinematics, arithmetic):
    """The reference's own rotor runs (golden): exact arithmetic to the
    actuator tolerances (samples 1e-12, blade forces 1e-10, populations
    1e-14); the benchmark's fast arithmetic within 1e-10 relative."""
    g = golden(f"rotor_{tag}.npz")
    cfg, tmp = rotor_config(cells=tuple(int(c) for c in g["cells"]),
                            periodic=tuple(bool(p) for p in g["periodicity"]),
                            boundary=str(g["boundary"]), position=tuple(g["position"]),
                            arithmetic=arithmetic)
    fast = arithmetic == "fast"
    sim = Simulation(cfg, kinematics=kinematics)
    for n in range(g["kin"].shape[0]):
        sim.step()
        kin = sim._kin_view()[:, :15]
        if kinematics == "host":
            assert np.array_equal(kin, g["kin"][n])
        else:
            np.testing.assert_allclose(kin, g["kin"][n], rtol=1e-13, atol=1e-14)
        rho, u, blade = sim._alm_results()
        np.testing.assert_allclose(rho, g["samples"][n, :, 0], rtol=1e-10 if fast else 1e-12)
        np.testing.assert_allclose(u, g["samples"][n, :, 1:], rtol=1e-10 if fast else 1e-11,
                                   atol=1e-15 if fast else 1e-16)
        np.testing.assert_allclose(blade, g["blade"][n], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(sim.fields[0].interior, g["f_final"], rtol=0,
                               atol=1e-13 if fast else 1e-14)
    np.testing.assert_allclose(sim.fields[0].interior_force, g["force_final"], rtol=1e-10,
                               atol=1e-18)
    sim.close()
    tmp.cleanup()


@pytest.mark.parametrize("ppb", [6, 30])
def test_rotor_vs_oracle_point_counts(gpu, ppb):
    """18 points (forces summed inside the sweep) and 90 points (per-row
    pools filled by K5) against the oracle over 6 steps."""
    from paper_2402_13171_b200.sim import HostKinematics
    cfg, tmp = rotor_config(cells=(16, 12, 12), periodic=(False, True, True),
                            boundary="velocity_inflow_outflow", position=(0.9, 0.75, 0.0),
                            points_per_blade=ppb)
    sim = Simulation(cfg, kinematics="host")
    cfg2, tmp2 = rotor_config(cells=(16, 12, 12), periodic=(False, True, True),
                              boundary="velocity_inflow_outflow", position=(0.9, 0.75, 0.0),
                              points_per_blade=ppb)
    host = HostKinematics(cfg2)
    ref = oracle_for(host)
    for _ in range(6):
        sim.step()
        ref.step(host.refresh())
        host.advance()
        rho, u, blade = sim._alm_results()
        np.testing.assert_allclose(rho, ref.samples[:, 0], rtol=1e-12)
        np.testing.assert_allclose(blade, ref.blade, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(sim.fields[0].interior, ref.interior, rtol=0, atol=1e-14)
    np.testing.assert_allclose(sim.fields[0].interior_force, ref.force[1:-1, 1:-1, 1:-1],
                               rtol=1e-9, atol=1e-17)
    sim.close()
    tmp.cleanup()
    tmp2.cleanup()


def test_initialize_modes_matches_host_equilibrium(gpu):
    """The device-side initial field (lbw_domain_init_modes) equals the host
    initialize_equilibrium of the same u(x) to libm rounding."""
    from paper_2402_13171_b200.collision import equilibrium_pdf, product_equilibrium
    from paper_2402_13171_b200.fields import fourier_modes
    for op in ("cumulant", "bgk"):
        sim = _lbm_sim((12, 10, 8), op=op)
        u0 = np.array([0.03, 0.0, 0.0])
        modes = fourier_modes((12, 10, 8), u0, intensity=0.1, n_modes=8, seed=3)
        sim.fields[0].initialize_modes(1.0, u0, modes, product=(op == "cumulant"))
        X, Y, Z = np.meshgrid(np.arange(12) + 0.5, np.arange(10) + 0.5, np.arange(8) + 0.5,
                              indexing="ij")
        u = np.broadcast_to(u0, (12, 10, 8, 3)).copy()
        for m in modes:
            sn = np.sin(m[0] * X + m[1] * Y + m[2] * Z + m[6])
            u += m[3:6] * sn[..., None]
        want = (product_equilibrium if op == "cumulant" else equilibrium_pdf)(1.0, u)
        np.testing.assert_allclose(sim.fields[0].interior, want, rtol=0, atol=1e-15)
        np.testing.assert_allclose(sim.fields[0].interior_macro[..., 1:], u, rtol=0, atol=1e-16)
        assert np.sqrt(np.mean(np.sum((u - u0) ** 2, axis=-1))) > 0.05 * 0.03
        sim.close()


@pytest.mark.parametrize("kinematics", ["host", "device"])
def test_rotor_loads_time_series_vs_reference(gpu, golden, kinematics):
    """Thrust / torque / power series (output.rotor_loads) against the same
    sums over the reference's own blade forces (golden rotor run) at the
    reference's point positions (HostKinematics, bit-identical)."""
    from paper_2402_13171_b200 import rotor_loads
    from paper_2402_13171_b200.sim import HostKinematics
    g = golden("rotor_inflow.npz")
    args = dict(cells=tuple(int(c) for c in g["cells"]),
                periodic=tuple(bool(p) for p in g["periodicity"]),
                boundary=str(g["boundary"]), position=tuple(g["position"]))
    cfg, tmp = rotor_config(**args)
    cfg2, tmp2 = rotor_config(**args)
    host = HostKinematics(cfg2)
    sim = Simulation(cfg, kinematics=kinematics)
    hub = next(c for c in cfg2.topologies[0].components if c.rate != 0.0)
    for n in range(g["blade"].shape[0]):
        sim.step()
        sim.synchronize()
        host.refresh()
        pos_m = host._pos_m.copy()
        hub_p, rate = hub.world.p.copy(), hub.rate
        axis = np.array([1.0, 0.0, 0.0])
        host.advance()
        F = g["blade"][n]
        thrust = np.sum(F @ axis)
        torque = np.sum(np.cross(pos_m - hub_p, F) @ axis)
        got = rotor_loads(sim)
        np.testing.assert_allclose(got, (thrust, torque, torque * rate), rtol=1e-9, atol=1e-12)
    assert abs(got[0]) > 0 and abs(got[2]) > 0
    sim.close()
    tmp.cleanup()
    tmp2.cleanup()


def test_device_kinematics_long_run(gpu):
    """600 steps of device kinematics stay on the host (reference-identical)
    kinematics to 1e-12 m, and sync_topologies restores the host objects."""
    cfgs = [rotor_config(cells=(12, 12, 12))[0] for _ in range(2)]
    host_topo = cfgs[0].topologies[0]
    sim = Simulation(cfgs[1], kinematics="device")
    for n in range(600):
        sim.step()
        if n < 599:
            host_topo.advance(cfgs[0].units.dt)
    sim.synchronize()
    # host topology advanced 599 times = state used by step 599; device's
    # last kinematics are those of step 599
    pos_host = host_topo.point_positions()
    np.testing.assert_allclose(sim._kin_view()[:, 15:18], pos_host, rtol=0, atol=1e-12)
    host_topo.advance(cfgs[0].units.dt)
    np.testing.assert_allclose(cfgs[1].topologies[0].point_positions(),
                               host_topo.point_positions(), rtol=0, atol=1e-12)
    sim.close()


def test_prelaunched_actuator_chain_survives_state_changes(gpu):
    """Device kinematics queue step n+1's actuator chain during sweep n.
    Mutating the state between steps (moments recompute, new populations)
    must invalidate it: the run must track a run without prelaunch."""
    sims = []
    for kin in ("host", "device"):
        cfg, tmp = rotor_config(cells=(16, 12, 12))
        sims.append((Simulation(cfg, kinematics=kin), tmp))
    rng = np.random.default_rng(5)
    bump = 1.0 + 1e-3 * rng.uniform(-1, 1, (16, 12, 12, 27))
    for sim, _ in sims:
        for _ in range(3):
            sim.step()
        sim._recompute_moments()
        for _ in range(2):
            sim.step()
        sim.fields[0].interior = sim.fields[0].interior * bump
        for _ in range(3):
            sim.step()
    (a, ta), (b, tb) = sims
    np.testing.assert_allclose(b.fields[0].interior, a.fields[0].interior, rtol=0, atol=1e-13)
    np.testing.assert_allclose(b._alm_results()[2], a._alm_results()[2], rtol=1e-10,
                               atol=1e-12)
    for sim, tmp in sims:
        sim.close()
        tmp.cleanup()


def test_rotor_spreading_matches_oracle_bitwise_given_forces(gpu):
    """With identical point forces the deposit is bit-identical: compare the
    device force field against the oracle fed the device's blade forces."""
    cfg, tmp = rotor_config(cells=(12, 12, 12), position=(0.9, 0.3, 0.0))
    sim = Simulation(cfg, kinematics="host")
    sim.step()
    blade = sim._alm_results()[2]
    kin = sim._kin.copy()
    dims = cfg.cells
    recs = [(p, kin[p, 0:3].copy(), -blade[p]) for p in range(len(blade))]
    routed = orc.route_single_block(recs, dims, cfg.periodicity)
    force = np.zeros((dims[0] + 2, dims[1] + 2, dims[2] + 2, 3))
    orc.spread(routed, force, dims, cfg.units.dt ** 2, cfg.units.rho_ref * cfg.units.dx ** 4)
    assert np.array_equal(sim.fields[0].interior_force, force[1:-1, 1:-1, 1:-1])
    sim.close()
    tmp.cleanup()


def test_nan_aborts_with_step_and_cell(gpu, tmp_path):
    (tmp_path / "blow.yaml").write_text("""
name: blow
components:
  - name: hub
    position: [2.0, 2.0, 2.0]
  - name: blade
    parent: hub
    discretization: {type: line, points: 3, r_end: 1.0, chord: 1.0e+308, polar: flat}
""")
    (tmp_path / "flat.csv").write_text("alpha_deg,cl,cd\n-10,1.0,0.0\n10,1.0,0.0\n")
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 10}, "output": {"directory": str(tmp_path / "out")},
           "turbines": [{"file": "blow.yaml"}], "polars": [{"id": "flat", "file": "flat.csv"}]}
    from paper_2402_13171_b200 import run_simulation
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        with pytest.raises(NumericalAbort) as exc:
            run_simulation(parse_config(raw, base_dir=str(tmp_path)))
    assert exc.value.step == 0
    assert len(exc.value.cell) == 3
    assert "global cell" in str(exc.value)


def test_kernels_are_native(gpu):
    before = _lib.kernel_launches()
    sim = _lbm_sim((16, 16, 16))
    sim.step()
    sim.synchronize()
    sim.close()
    assert _lib.kernel_launches() > before



@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pdffield_collide_and_stream(gpu, dtype):
    """The reference's block-level API (fields.py PdfField / collide_field /
    stream) on the GPU block kernels, float64 and float32 storage, against
    the oracle."""
    from paper_2402_13171_b200 import PdfField, collide_field, stream
    rng = np.random.default_rng(7)
    fld = PdfField((6, 5, 7), dtype=dtype)
    f = (orc.W * (1.0 + 0.3 * rng.uniform(-1, 1, fld.f.shape))).astype(dtype)
    F = rng.uniform(-1e-3, 1e-3, fld.force.shape).astype(dtype)
    fld.f[...] = f
    fld.force[...] = F
    cfg = CollisionConfig("cumulant", 1.6, (1.0, 1.2, 0.9, 1.1))
    collide_field(fld, cfg)
    ref_f = f.astype(np.float64)
    ref_m = np.zeros(fld.macro.shape)
    orc.collide_block("cumulant", ref_f, F.astype(np.float64), ref_m, 1.6, (1.0, 1.2, 0.9, 1.1))
    inner = (slice(1, -1),) * 3
    assert fld.f.dtype == dtype
    assert np.array_equal(fld.f[inner], ref_f[inner].astype(dtype))
    assert np.array_equal(fld.macro[inner], ref_m[inner].astype(dtype))
    stream(fld)
    dst = np.zeros_like(ref_f)
    orc.stream_pull_block(fld.f_next.astype(np.float64), dst)
    assert np.array_equal(fld.f[inner], dst[inner].astype(dtype))


def test_immediate_abort_leaves_reference_state(gpu, tmp_path):
    """run.abort: immediate -- the step that produces a non-finite macro
    raises right after its collide (sim.py:254-262, 281): step_index not
    advanced, populations post-collision and not streamed, exactly the
    oracle's state when its collide trips the same check (the reference's
    chord: 1e308 fault, test_sim.py:116-138, here on a fast-growing blade
    so the fault appears after a few healthy steps)."""
    from tests.scenarios import oracle_for
    (tmp_path / "blow.yaml").write_text("""
name: blow
components:
  - name: hub
    position: [1.0, 1.0, 1.0]
    rotation: {axis: [1.0, 0.0, 0.0], rate_rad_per_s: 40.0}
  - name: blade
    parent: hub
    discretization: {type: line, points: 3, r_end: 0.5, chord: 1.0e+308, polar: flat}
""")
    (tmp_path / "flat.csv").write_text("alpha_deg,cl,cd\n-10,1.0,0.0\n10,1.0,0.0\n")
    raw = {"domain": {"cells": [16, 16, 16]},
           "fluid": {"kinematic_viscosity": 5.0, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 2.0, "mach": 0.1},
           "run": {"steps": 10, "abort": "immediate"},
           "output": {"directory": str(tmp_path / "out")},
           "turbines": [{"file": "blow.yaml"}], "polars": [{"id": "flat", "file": "flat.csv"}]}
    cfg = parse_config(raw, base_dir=str(tmp_path))
    sim = Simulation(cfg, kinematics="host")
    ref = oracle_for(sim)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        with pytest.raises(NumericalAbort) as exc:
            for _ in range(10):
                sim.refresh_points()
                kin = sim._kin.copy()
                try:
                    ref.step(kin)
                except FloatingPointError as e:
                    ref_abort = e.args[0]
                sim.step()
    assert exc.value.step == ref_abort[0] == sim.step_index
    assert tuple(exc.value.cell) == tuple(ref_abort[1])
    got = sim.fields[0].interior
    np.testing.assert_array_equal(got, ref.interior)      # NaN where the oracle has NaN
    assert np.isnan(got).any()
    sim.close()
