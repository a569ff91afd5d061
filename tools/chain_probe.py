"""Advance a rotor case n^3 for a few hundred steps (for the LBW_K4_PROF /
LBW_KK_PROF builds, which printf their phase clocks every 50 steps)."""
import sys
import tempfile

sys.path.insert(0, ".")
from paper_2402_13171_b200 import Simulation, parse_config
from tests.scenarios import write_rotor_files

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 300
alone = len(sys.argv) > 4 and sys.argv[4] == "alone"   # synchronize after every step
bare = len(sys.argv) > 4 and sys.argv[4] == "bare"     # no turbine
tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
raw = {"domain": {"cells": [n, n, n]},
       "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
       "resolution": {"mach": 0.05},
       "run": {"arithmetic": arith, "collision": {"operator": "cumulant"}},
       "turbines": [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}],
       "polars": [{"id": "sym", "file": "sym.csv"}]}
if bare:
    del raw["turbines"], raw["polars"]
sim = Simulation(parse_config(raw, base_dir=tmp))
if alone:
    for _ in range(steps):
        sim.step()
        sim.synchronize()
else:
    sim.advance(steps)
    sim.synchronize()
sim.close()
