"""The flag-ordered actuator chain (default for a single slab with device
kinematics and <= 64 points; lbw_alm.cu "chain B"): KK two steps ahead
computes the geometry, the sweep stores the (rho, u) of the next step's
sampling rows and signals when they are stored, K4 waits for that in-kernel
and samples them, the sweep's force tiles wait in-kernel for K4 -- no stream
event on the main stream.  It must equal the event-ordered chain
(LBW_CHAIN_FLAGS=0): bit for bit in the exact flavour (the pooled macro IS
the collide's output, which the event-ordered chain recomputes with the same
arithmetic), within the fast flavour's tolerance otherwise; across priming,
state changes, advance(n) and the load series."""

import numpy as np
import pytest

from tests.test_gpu_fused import CASES, _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", sorted(CASES))
def test_flags_exact_bitwise_vs_events(gpu, monkeypatch, case):
    a = _run(monkeypatch, False, case, "exact", 30, chain="flags")
    b = _run(monkeypatch, False, case, "exact", 30, chain="events")
    for n in range(30):
        assert np.array_equal(a["samples"][n], b["samples"][n]), n
        assert np.array_equal(a["blade"][n], b["blade"][n]), n
    assert np.array_equal(a["kin"], b["kin"])
    assert np.array_equal(a["f"], b["f"])
    assert np.array_equal(a["force"], b["force"])


@pytest.mark.parametrize("case", ["periodic", "inflow"])
def test_flags_fast_vs_events(gpu, monkeypatch, case):
    a = _run(monkeypatch, False, case, "fast", 40, chain="flags")
    b = _run(monkeypatch, False, case, "fast", 40, chain="events")
    for n in range(40):
        np.testing.assert_allclose(a["samples"][n], b["samples"][n], rtol=1e-12, atol=1e-16)
        np.testing.assert_allclose(a["blade"][n], b["blade"][n], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(a["f"], b["f"], rtol=0, atol=1e-14)


def test_flags_state_changes_and_loads(gpu, monkeypatch):
    def upload(sim):
        sim.fields[0].interior = sim.fields[0].interior

    poke = {2: upload, 5: lambda s: s._recompute_moments(), 6: upload,
            11: lambda s: s.fields[0].interior}
    a = _run(monkeypatch, False, "inflow", "exact", 16, poke=poke, loads=True, chain="flags")
    b = _run(monkeypatch, False, "inflow", "exact", 16, poke=poke, loads=True, chain="events")
    for n in range(16):
        assert np.array_equal(a["blade"][n], b["blade"][n]), n
    assert np.array_equal(a["f"], b["f"])
    assert np.array_equal(a["loads"], b["loads"])


def test_flags_advance_many_steps(gpu, monkeypatch):
    from paper_2402_13171_b200 import Simulation
    from tests.scenarios import rotor_config
    monkeypatch.setenv("LBW_FUSED", "0")
    monkeypatch.setenv("LBW_CHAIN_FLAGS", "1")
    cells, per, bc, pos = CASES["periodic"]
    cfg, tmp = rotor_config(cells=cells, periodic=per, boundary=bc, position=pos)
    sim = Simulation(cfg)
    sim.advance(50)
    sim.synchronize()
    fa, ba = sim.fields[0].interior.copy(), sim._alm_results()[2].copy()
    sim.close()
    tmp.cleanup()
    b = _run(monkeypatch, False, "periodic", "exact", 50, chain="events")
    assert np.array_equal(ba, b["blade"][-1])
    assert np.array_equal(fa, b["f"])


def _run_raw(monkeypatch, chain, raw, steps, upload_first=False):
    import os
    import tempfile

    from paper_2402_13171_b200 import Simulation, parse_config
    from tests.scenarios import write_rotor_files
    monkeypatch.setenv("LBW_FUSED", "0")
    monkeypatch.setenv("LBW_CHAIN_FLAGS", "1" if chain == "flags" else "0")
    tmp = tempfile.TemporaryDirectory()
    write_rotor_files(tmp.name)
    sim = Simulation(parse_config(raw, base_dir=tmp.name))
    if upload_first:   # a pre-collision state: the first sweep collides in place
        f = sim.fields[0].interior
        sim.fields[0].interior = f * (1.0 + 1e-3 * np.sin(np.arange(f.size)).reshape(f.shape))
    blades = []
    for _ in range(steps):
        sim.step()
        blades.append(sim._alm_results()[2].copy())
    out = (np.array(blades), sim.fields[0].interior.copy(), sim.fields[0].interior_force.copy())
    sim.close()
    tmp.cleanup()
    return out


VARIANTS = {
    "single": dict(precision="single"),
    "gauss": dict(spreading={"kernel": "gaussian", "epsilon": 1.5}),
    "walls": dict(periodic=(True, False, False),
                  walls={"y_lo": "no_slip", "y_hi": "free_slip", "z_lo": "no_slip"}),
    "bgk": dict(operator="bgk"),
    "pre": dict(upload_first=True),
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_flags_variants_bitwise_vs_events(gpu, monkeypatch, variant):
    """fp32 storage, Gaussian spreading (9 deposit cells per axis), walls,
    BGK and a first in-place collide through the flag-ordered chain: bit
    for bit the event-ordered chain."""
    from tests.scenarios import rotor_raw
    v = dict(VARIANTS[variant])
    upload_first = v.pop("upload_first", False)
    periodic = v.pop("periodic", (True, True, True))
    raw = rotor_raw((24, 20, 16), periodic, "periodic", (0.9, 1.25, 0.2),
                    precision=v.pop("precision", "double"), operator=v.pop("operator", "cumulant"))
    if "spreading" in v:
        raw["run"]["spreading"] = v.pop("spreading")
    if "walls" in v:
        raw["run"]["walls"] = v.pop("walls")
    a = _run_raw(monkeypatch, "flags", raw, 16, upload_first)
    b = _run_raw(monkeypatch, "events", raw, 16, upload_first)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _calls(monkeypatch, loop, case, arithmetic):
    from paper_2402_13171_b200 import Simulation
    from tests.scenarios import rotor_config
    monkeypatch.setenv("LBW_FUSED", "0")
    monkeypatch.setenv("LBW_CHAIN_FLAGS", "1")
    monkeypatch.setenv("LBW_CHAIN_LOOP", "1" if loop else "0")
    cells, per, bc, pos = CASES[case]
    cfg, tmp = rotor_config(cells=cells, periodic=per, boundary=bc, position=pos,
                            arithmetic=arithmetic)
    sim = Simulation(cfg)
    out = []
    # long calls (one resident chain kernel each), short calls (per-step
    # launches) and a state change between them
    for n in (7, 1, 2, 10, 1, 4, 3, 12):
        sim.advance(n)
        out.append(sim._alm_results()[2].copy())
        if n == 2:
            sim.fields[0].interior = sim.fields[0].interior
    out.append(sim.fields[0].interior.copy())
    sim.close()
    tmp.cleanup()
    return out


@pytest.mark.parametrize("case,arithmetic", [("periodic", "exact"), ("inflow", "exact"),
                                             ("periodic", "fast"), ("inflow", "fast")])
def test_resident_loop_bitwise_vs_per_step(gpu, monkeypatch, case, arithmetic):
    """The resident chain kernel (K4 / kinematics / geometry of a call's
    steps in one launch, lbw_alm.cu k_cb_persist; the default with the FMA
    arithmetic): bit for bit the per-step chain launches, across calls of
    every length and a state change."""
    a = _calls(monkeypatch, True, case, arithmetic)
    b = _calls(monkeypatch, False, case, arithmetic)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("variant", ["single", "gauss", "walls", "bgk"])
def test_resident_loop_variants_bitwise(gpu, monkeypatch, variant):
    """The resident chain (FMA arithmetic) against the per-step launches for
    fp32 storage, Gaussian spreading, walls and BGK, through advance(n)."""
    import tempfile

    from paper_2402_13171_b200 import Simulation, parse_config
    from tests.scenarios import rotor_raw, write_rotor_files

    def run(loop):
        monkeypatch.setenv("LBW_FUSED", "0")
        monkeypatch.setenv("LBW_CHAIN_FLAGS", "1")
        monkeypatch.setenv("LBW_CHAIN_LOOP", "1" if loop else "0")
        v = dict(VARIANTS[variant])
        periodic = v.pop("periodic", (True, True, True))
        raw = rotor_raw((24, 20, 16), periodic, "periodic", (0.9, 1.25, 0.2), arithmetic="fast",
                        precision=v.pop("precision", "double"),
                        operator=v.pop("operator", "cumulant"))
        if "spreading" in v:
            raw["run"]["spreading"] = v.pop("spreading")
        if "walls" in v:
            raw["run"]["walls"] = v.pop("walls")
        with tempfile.TemporaryDirectory() as tmp:
            write_rotor_files(tmp)
            sim = Simulation(parse_config(raw, base_dir=tmp))
            out = []
            for n in (6, 2, 5):   # 13 steps: the walls case goes unstable near 17
                sim.advance(n)
                out.append(sim._alm_results()[2].copy())
            out.append(sim.fields[0].interior.copy())
            sim.close()
        return out

    for x, y in zip(run(True), run(False)):
        assert np.array_equal(x, y)
