"""The fused time step (csrc/lbw_fused.cuh): one launch per step carrying
sweep m, the point forces of step m and the kinematics + deposit geometry of
step m+2, used on a single slab with device kinematics and <= 64 points.

It must give exactly what the standalone actuator chain + sweep give
(LBW_FUSED=0 selects those): bit for bit in the exact flavour -- the same
arithmetic, the sampled macro taken from the previous collide's own output
instead of a recomputation of it -- and to the fast flavour's tolerance
otherwise, through priming, steady state, state changes mid-run and the
per-step load series."""

import numpy as np
import pytest

from paper_2402_13171_b200 import Simulation
from tests.scenarios import rotor_config

pytestmark = pytest.mark.gpu

CASES = {
    # cells, periodicity, boundary, rotor position (m)
    "periodic": ((24, 20, 16), (True, True, True), "periodic", (0.9, 0.3, 0.0)),
    "inflow": ((32, 20, 20), (False, True, True), "velocity_inflow_outflow", (1.1, 0.75, 0.6)),
    "wrap_z": ((20, 16, 12), (True, True, True), "periodic", (0.6, 0.5, 0.05)),
}


def _run(monkeypatch, fused, case, arithmetic, steps, poke=None, loads=False, chain=None):
    """fused: LBW_FUSED=1; else the standalone chain, event-ordered
    (chain="events") or flag-ordered (chain="flags", the default mode)."""
    monkeypatch.setenv("LBW_FUSED", "1" if fused else "0")
    monkeypatch.setenv("LBW_CHAIN_FLAGS", "0" if chain == "events" else "1")
    cells, per, bc, pos = CASES[case]
    cfg, tmp = rotor_config(cells=cells, periodic=per, boundary=bc, position=pos,
                            arithmetic=arithmetic)
    sim = Simulation(cfg)               # device kinematics (the default)
    if loads:
        sim.record_loads(steps + 4)
    out = {"samples": [], "blade": []}
    for n in range(steps):
        if poke is not None and n in poke:
            poke[n](sim)
        sim.step()
        rho, u, blade = sim._alm_results()
        out["samples"].append(np.column_stack([rho, u]))
        out["blade"].append(blade.copy())
    out["f"] = sim.fields[0].interior.copy()
    out["force"] = sim.fields[0].interior_force.copy()
    out["kin"] = sim._kin_view().copy()
    if loads:
        out["loads"] = sim.read_loads()[1].copy()
    sim.close()
    tmp.cleanup()
    return out


@pytest.mark.parametrize("case", sorted(CASES))
def test_fused_exact_bitwise_vs_standalone_chain(gpu, monkeypatch, case):
    a = _run(monkeypatch, True, case, "exact", 24)
    b = _run(monkeypatch, False, case, "exact", 24, chain="events")
    for n in range(24):
        assert np.array_equal(a["samples"][n], b["samples"][n]), n
        assert np.array_equal(a["blade"][n], b["blade"][n]), n
    assert np.array_equal(a["kin"], b["kin"])
    assert np.array_equal(a["f"], b["f"])
    assert np.array_equal(a["force"], b["force"])


@pytest.mark.parametrize("case", ["periodic", "inflow"])
def test_fused_fast_vs_standalone_chain(gpu, monkeypatch, case):
    a = _run(monkeypatch, True, case, "fast", 40)
    b = _run(monkeypatch, False, case, "fast", 40, chain="events")
    for n in range(40):
        np.testing.assert_allclose(a["samples"][n], b["samples"][n], rtol=1e-12, atol=1e-16)
        np.testing.assert_allclose(a["blade"][n], b["blade"][n], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(a["f"], b["f"], rtol=0, atol=1e-14)


def test_fused_survives_state_changes(gpu, monkeypatch):
    """Uploads, moment recomputes and downloads between steps re-prime the
    pipeline (the sampled macro then comes from a recomputation); the
    result stays bit-identical to the standalone chain."""
    def upload(sim):
        f = sim.fields[0].interior
        sim.fields[0].interior = f

    def recompute(sim):
        sim._recompute_moments()

    poke = {3: upload, 7: recompute, 8: upload, 15: lambda s: s.fields[0].interior}
    a = _run(monkeypatch, True, "inflow", "exact", 20, poke=poke)
    b = _run(monkeypatch, False, "inflow", "exact", 20, poke=poke, chain="events")
    for n in range(20):
        assert np.array_equal(a["blade"][n], b["blade"][n]), n
    assert np.array_equal(a["f"], b["f"])


def test_fused_load_series(gpu, monkeypatch):
    """The per-step blade loads the fused step writes in-kernel into the
    pinned ring equal the standalone chain's copies."""
    a = _run(monkeypatch, True, "periodic", "exact", 12, loads=True)
    b = _run(monkeypatch, False, "periodic", "exact", 12, loads=True, chain="events")
    assert a["loads"].shape == b["loads"].shape == (12, 18, 3)
    assert np.array_equal(a["loads"], b["loads"])
    assert np.array_equal(a["loads"][-1], a["blade"][-1])


def test_fused_advance_many_steps(gpu, monkeypatch):
    """advance(n) (one native call, PDL-chained fused launches) equals n
    single steps of the standalone chain."""
    monkeypatch.setenv("LBW_FUSED", "1")
    cells, per, bc, pos = CASES["inflow"]
    cfg, tmp = rotor_config(cells=cells, periodic=per, boundary=bc, position=pos)
    sim = Simulation(cfg)
    sim.advance(30)
    fa = sim.fields[0].interior.copy()
    ba = sim._alm_results()[2].copy()
    sim.close()
    b = _run(monkeypatch, False, "inflow", "exact", 30, chain="events")
    assert np.array_equal(ba, b["blade"][-1])
    assert np.array_equal(fa, b["f"])
    tmp.cleanup()
