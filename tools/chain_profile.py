"""64^3 rotor, a few device-kinematics steps: the actuator chain kernels for
ncu (LBW_ALM_CHAIN=0 selects the multi-kernel chain)."""
import sys

sys.path.insert(0, ".")
import tempfile

from paper_2402_13171_b200 import Simulation, parse_config
from tests.scenarios import write_rotor_files

tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
raw = {"domain": {"cells": [n, n, n]},
       "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
       "resolution": {"mach": 0.05},
       "run": {"arithmetic": "fast", "collision": {"operator": "cumulant"}},
       "turbines": [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}],
       "polars": [{"id": "sym", "file": "sym.csv"}]}
sim = Simulation(parse_config(raw, base_dir=tmp))
sim.advance(30)
sim.synchronize()
sim.close()
