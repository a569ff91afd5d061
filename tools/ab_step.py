"""A/B of the 64^3 rotor step between two builds of the library, alternating
in one process each (LBW_LIB picks the build): median of repeated
domain_step(400) timings.  usage: python tools/ab_step.py n arith reps"""
import os
import statistics
import sys
import tempfile
import time

sys.path.insert(0, ".")
from paper_2402_13171_b200 import Simulation, parse_config
from tests.scenarios import write_rotor_files

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 15
tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
raw = {"domain": {"cells": [n, n, n]},
       "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
       "resolution": {"mach": 0.05},
       "run": {"arithmetic": arith, "collision": {"operator": "cumulant"}},
       "turbines": [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}],
       "polars": [{"id": "sym", "file": "sym.csv"}]}
sim = Simulation(parse_config(raw, base_dir=tmp))
sim.advance(200)
sim.synchronize()
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    sim.advance(400)
    sim.synchronize()
    ts.append((time.perf_counter() - t0) / 400 * 1e6)
print(f"{os.environ.get('LBW_LIB', 'in-tree')} {n}^3 {arith}: median {statistics.median(ts):.2f} "
      f"us/step, min {min(ts):.2f}")
