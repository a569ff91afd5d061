"""The output files of Simulation.run() against the files the REFERENCE
itself wrote for the same configuration (tests/golden/output.npz,
make_golden.py --output; reference output.py:44-167, sim.py:304-333).

flow:  a perturbed inflow/outflow cumulant run with axial_line /
       radial_profile probes, a running average and VTK dumps every 3 steps
       -- exact arithmetic, so every file is byte-identical (repr floats of
       bit-identical states, the same trilinear einsum on the host).
rotor: the rotating 3-blade rotor with a blade_loads probe (+ average) and
       a wake line -- the actuator path is parity-tested to 1e-10 (BLAS /
       atan2 rounding), so values are compared to that
       tolerance and the layout (file names, headers, first columns) exactly.
"""
import json
import os

import numpy as np
import pytest

from paper_2402_13171_b200 import Simulation, parse_config

pytestmark = pytest.mark.gpu


def _files(g, case):
    return {k.split("/", 1)[1]: str(g[k]) for k in g.files if k.startswith(case + "/")}


def _run(g, case, tmp_path, **sim_kw):
    raw = json.loads(str(g[f"{case}_raw"]))
    raw["output"]["directory"] = str(tmp_path / case)
    raw["run"]["arithmetic"] = "exact"
    if case == "rotor":
        (tmp_path / "rotor.yaml").write_text(str(g["rotor_yaml"]))
        (tmp_path / "sym.csv").write_text(str(g["polar_csv"]))
    sim = Simulation(parse_config(raw, base_dir=str(tmp_path)), **sim_kw)
    if case == "flow":
        sim.fields[0].interior = g["flow_f0"]
    sim.run()
    sim.close()
    out = {}
    for fn in sorted(os.listdir(tmp_path / case)):
        if fn != "report.json":
            out[fn] = (tmp_path / case / fn).read_text()
    return out


def test_flow_output_files_byte_identical(gpu, golden, tmp_path):
    g = golden("output.npz")
    want = _files(g, "flow")
    got = _run(g, "flow", tmp_path)
    assert sorted(got) == sorted(want)
    for fn in want:
        assert got[fn] == want[fn], fn


def _csv(text):
    lines = text.strip().split("\n")
    return lines[0], np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])


@pytest.mark.parametrize("kinematics", ["device", "host"])
def test_rotor_output_files_match_reference(gpu, golden, tmp_path, kinematics):
    g = golden("output.npz")
    want = _files(g, "rotor")
    got = _run(g, "rotor", tmp_path, kinematics=kinematics)
    assert sorted(got) == sorted(want)
    for fn in want:
        hw, vw = _csv(want[fn])
        hg, vg = _csv(got[fn])
        assert hg == hw, fn
        assert vg.shape == vw.shape, fn
        assert np.array_equal(vg[:, 0], vw[:, 0]), fn          # stations / positions
        scale = np.abs(vw[:, 1:]).max()
        np.testing.assert_allclose(vg[:, 1:], vw[:, 1:], rtol=1e-9, atol=1e-12 * scale,
                                   err_msg=fn)
