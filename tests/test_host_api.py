"""Host-side API (no GPU): config grammar, units, polars, turbine kinematics
against the reference's own per-step kinematics, C-ABI exports."""

import ctypes
import os
import re
import warnings

import numpy as np
import pytest

from paper_2402_13171_b200 import (ConfigError, PolarTable, build_topology, parse_config,
                                   rotation_matrix)
from paper_2402_13171_b200 import _lib
from paper_2402_13171_b200.turbine import reorthonormalize
from tests.scenarios import rotor_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ C ABI

def _header_functions():
    text = open(os.path.join(ROOT, "include", "lbw.h")).read()
    return sorted(set(re.findall(r"\b(lbw_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table and header disagree"
    assert lib.lbw_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_calls_fail_loudly_here():
    lib = _lib.load()
    if lib.lbw_device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _lib.require_gpu()
    d = _lib.DomainDesc()
    d.cells[:] = (8, 8, 8)
    d.slab_nx = 8
    d.omega = 1.2
    d.nranks = 1
    h = ctypes.c_void_p()
    assert lib.lbw_domain_create(ctypes.byref(d), ctypes.byref(h)) == _lib.LBW_EINVAL
    assert "no CUDA device" in _lib.last_error()


# ----------------------------------------------------------------- config

def test_minimal_config_defaults():
    cfg = parse_config({"domain": {"cells": [32, 32, 32]}})
    assert cfg.operator == "cumulant" and cfg.boundary_kind == "periodic"
    assert cfg.periodicity == (True, True, True) and cfg.arithmetic == "exact"
    assert cfg.higher_order_rates == (1.0, 1.0, 1.0, 1.0)


@pytest.mark.parametrize("raw,match", [
    ({}, "domain"),
    ({"domain": {"cells": [8, 8, 8]}, "bogus": 1}, "unknown key"),
    ({"domain": {"cells": [8, 8, 2]}}, "below 4"),
    ({"domain": {"cells": [8, 8, 8]}, "run": {"collision": {"operator": "mrt"}}}, "operator"),
    ({"domain": {"cells": [8, 8, 8]}, "run": {"boundary": "velocity_inflow_outflow"}},
     "periodicity"),
    ({"domain": {"cells": [8, 8, 8]}, "run": {"arithmetic": "sloppy"}}, "arithmetic"),
    ({"domain": {"cells": [8, 8, 8]}, "resolution": {"mach": 0.5}}, "lattice speed"),
])
def test_config_errors(raw, match):
    with pytest.raises(ConfigError, match=match):
        parse_config(raw)


def test_units_match_survey_c2():
    """u_lat 0.028868, omega 1.78572, dt 1.1276e-4."""
    cfg = parse_config({"domain": {"cells": [256, 128, 128], "periodicity": [False, True, True]},
                        "fluid": {"kinematic_viscosity": 0.1732, "wind": [8, 0, 0]},
                        "resolution": {"cells_per_diameter": 32, "mach": 0.05},
                        "run": {"boundary": "velocity_inflow_outflow"}})
    u = cfg.units
    assert abs(u.u_lat - 0.028868) < 1e-6
    assert abs(u.omega - 1.78572) < 1e-4
    assert abs(u.dt - 1.1276e-4) < 1e-8


def test_config_matches_reference_units(reference_lbwind):
    from lbwind.config import parse_config as ref_parse
    raw = {"domain": {"cells": [24, 16, 16]},
           "fluid": {"kinematic_viscosity": 0.5, "wind": [7.0, 1.0, 0.5]},
           "resolution": {"cells_per_diameter": 8, "mach": 0.08}}
    a, b = parse_config(raw), ref_parse(raw)
    for k in ("dx", "dt", "u_lat", "nu_lat", "tau", "omega"):
        assert getattr(a.units, k) == getattr(b.units, k), k


# ----------------------------------------------------------------- polars

def test_polar_interp_and_clamp_warns_once():
    t = PolarTable("p", np.deg2rad([-10.0, 0.0, 10.0]), [-1.0, 0.0, 1.0], [0.1, 0.05, 0.1])
    cl, cd = t.lookup(np.deg2rad(5.0))
    assert abs(cl - 0.5) < 1e-15 and abs(cd - 0.075) < 1e-15
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert t.lookup(1.0)[0] == 1.0
        assert t.lookup(-1.0)[0] == -1.0
    assert len(w) == 1


def test_polar_validation():
    with pytest.raises(ConfigError):
        PolarTable("p", [0.0, 0.0], [0, 0], [0, 0])
    with pytest.raises(ConfigError):
        PolarTable("p", [0.0], [0], [0])


# -------------------------------------------------------------- kinematics

def test_rotation_and_gram_schmidt():
    R = rotation_matrix([1.0, 2.0, 3.0], 0.7)
    assert np.abs(R.T @ R - np.eye(3)).max() < 1e-15
    noisy = R + 1e-9
    Q = reorthonormalize(noisy)
    assert np.abs(Q.T @ Q - np.eye(3)).max() < 1e-15


@pytest.mark.parametrize("tag", ["periodic", "inflow"])
def test_kinematics_bitwise_vs_reference(golden, tag):
    """refresh_points + advance reproduce the reference's per-step point
    state bit for bit (stacked matmul == per-point matmul)."""
    from paper_2402_13171_b200.sim import Simulation
    g = golden(f"rotor_{tag}.npz")
    cells = tuple(int(c) for c in g["cells"])
    cfg, tmp = rotor_config(cells=cells, periodic=tuple(bool(p) for p in g["periodicity"]),
                            boundary=str(g["boundary"]), position=tuple(g["position"]))
    sim = Simulation.__new__(Simulation)   # host half only: no device here
    sim.cfg, sim.units = cfg, cfg.units
    from paper_2402_13171_b200.sim import SlabGrid
    sim.grid = SlabGrid(cfg.cells, cfg.periodicity, 1, 0)
    sim._line_groups, sim._disk_groups = [], []
    gid = 0
    for topo in cfg.topologies:
        for comp in topo.components:
            if comp.discretization is not None:
                n = comp.discretization.n_points
                sim._line_groups.append((comp, comp.discretization, slice(gid, gid + n)))
                gid += n
    sim._kin = np.zeros((gid, 18))
    sim._pos_m = np.zeros((gid, 3))
    for n in range(g["kin"].shape[0]):
        sim.refresh_points()
        assert np.array_equal(sim._kin[:, :15], g["kin"][n]), n
        for topo in cfg.topologies:
            topo.advance(cfg.units.dt)
    tmp.cleanup()


def test_flat_and_nested_definitions_agree():
    flat = {"name": "t", "components": [
        {"name": "hub", "rotation": {"axis": [1, 0, 0], "rate_rpm": 60}},
        {"name": "b", "parent": "hub",
         "discretization": {"type": "line", "points": 4, "r_end": 1.0}}]}
    nested = {"name": "t", "root": {
        "name": "hub", "rotation": {"axis": [1, 0, 0], "rate_rpm": 60},
        "children": [{"name": "b", "discretization": {"type": "line", "points": 4,
                                                        "r_end": 1.0}}]}}
    a, b = build_topology(flat), build_topology(nested)
    for _ in range(10):
        a.advance(0.01)
        b.advance(0.01)
    assert np.array_equal(a.point_positions(), b.point_positions())


def test_topology_cycle_and_parent_errors():
    with pytest.raises(ConfigError, match="cycle"):
        build_topology({"components": [{"name": "a"}, {"name": "b", "parent": "c"},
                                       {"name": "c", "parent": "b"}]})
    with pytest.raises(ConfigError, match="unknown parent"):
        build_topology({"components": [{"name": "a"}, {"name": "b", "parent": "zz"}]})


def test_extension_config_keys_validate():
    """run.walls / run.spreading / run.precision (extensions and the
    reference's single precision) parse, echo and reject bad values."""
    from paper_2402_13171_b200 import ConfigError, parse_config
    base = {"domain": {"cells": [8, 8, 8], "periodicity": [True, False, False]},
            "fluid": {"kinematic_viscosity": 0.1, "wind": [0, 0, 0], "reference_velocity": 1.0},
            "resolution": {"mach": 0.1}}
    cfg = parse_config(dict(base, run={"walls": {"y_lo": "no_slip", "z_hi": "free_slip"},
                                       "spreading": {"kernel": "gaussian", "epsilon": 1.5},
                                       "precision": "single"}))
    assert cfg.wall_codes() == (1, 0, 0, 2)
    assert cfg.echo()["run"]["walls"] == {"y_lo": "no_slip", "z_hi": "free_slip"}
    assert cfg.echo()["run"]["spreading"] == {"kernel": "gaussian", "epsilon": 1.5}
    for bad in ({"walls": {"x_lo": "no_slip"}}, {"walls": {"y_lo": "sticky"}},
                {"spreading": {"kernel": "gaussian"}},
                {"spreading": {"kernel": "gaussian", "epsilon": 3.0}},
                {"spreading": {"kernel": "tophat"}}):
        with pytest.raises(ConfigError):
            parse_config(dict(base, run=bad))
    periodic = dict(base, domain={"cells": [8, 8, 8]})
    with pytest.raises(ConfigError):
        parse_config(dict(periodic, run={"walls": {"y_lo": "no_slip"}}))


def test_oracle_gaussian_weights_normalised_and_roma_unchanged():
    from oracle import oracle as orc
    for x in (3.2, 7.5, 10.01):
        cw = orc.axis_weights(x, "gaussian", 1.3)
        assert abs(sum(w for _, w in cw) - 1.0) < 1e-15
        assert all(abs(x - (c + 0.5)) <= 3.9 + 1e-12 for c, _ in cw)
        # centred on the point up to the 3-eps truncation (exp(-9) tails)
        assert abs(sum(w * (c + 0.5) for c, w in cw) - x) < 1e-3
        roma = orc.axis_weights(x, "roma")
        assert [c for c, _ in roma] == [int(np.floor(x)) - 1 + q for q in range(3)]
        assert abs(sum(w for _, w in roma) - 1.0) < 1e-15


@pytest.mark.gpu
def test_standalone_abi_example(gpu):
    """examples/abi_minimal.py: the ABI bound with plain ctypes (no package)."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "abi_minimal.py")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "energy decay rate" in r.stdout


def test_abort_mode_config():
    base = {"domain": {"cells": [8, 8, 8]},
            "fluid": {"kinematic_viscosity": 0.1, "wind": [1.0, 0.0, 0.0]},
            "resolution": {"mach": 0.1}}
    assert parse_config(base).abort == "deferred"
    raw = dict(base, run={"abort": "immediate"})
    cfg = parse_config(raw)
    assert cfg.abort == "immediate"
    assert cfg.echo()["run"]["abort"] == "immediate"
    with pytest.raises(ConfigError, match="run.abort"):
        parse_config(dict(base, run={"abort": "sometimes"}))


def test_bench_clock_summary_uses_timed_region_samples():
    """bench.py's NVML clock sampler: the median and reasons come from the
    samples inside the timed region when there are any (else the whole
    window), throttle reasons are decoded from the NVML bit mask."""
    import types

    import bench
    nv = types.SimpleNamespace(nvmlClocksEventReasonHwSlowdown=8,
                               nvmlClocksEventReasonHwThermalSlowdown=64,
                               nvmlClocksEventReasonSwThermalSlowdown=32,
                               nvmlClocksEventReasonSwPowerCap=4)
    cs = bench.ClockSampler(0)
    cs.nv, cs.smax = nv, 1965.0
    cs.samples = [(0.0, 1965.0, 0), (1.0, 1500.0, 4), (2.0, 1600.0, 4), (3.0, 1965.0, 0)]
    cs.window = [0.5, 2.5]
    s = cs.summary()
    assert s["samples_in_timed_region"] == 2 and s["sm_mhz"] == 1550.0
    assert s["reasons"] == ["sw_power_cap"] and s["window"] == "timed region"
    cs.window = [10.0, 11.0]
    s = cs.summary()
    assert s["samples_in_timed_region"] == 0 and s["samples"] == 4
    assert s["window"] == "warm-up + timed region"
    cs.nv = None
    cs.error = "NVML unavailable: test"
    assert cs.summary()["reasons"] == ["NVML unavailable: test"]
