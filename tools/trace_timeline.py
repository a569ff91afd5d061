"""Kernel timeline of a few device-kinematics steps (needs the LBW_TRACE
build: make -C paper_2402_13171_b200/csrc EXTRA=-DLBW_TRACE
OUT=/root/repo/build/liblbw_trace.so BUILD=/root/repo/build/lbw_trace, run with
LBW_LIB pointing at it).  Prints per step the start/end (us) of the sweep,
kinematics, K4 and K5 relative to the first sweep start."""
import ctypes
import sys

sys.path.insert(0, ".")
import tempfile

import numpy as np

from paper_2402_13171_b200 import Simulation, _lib, parse_config
from tests.scenarios import write_rotor_files

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
raw = {"domain": {"cells": [n, n, n]},
       "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
       "resolution": {"mach": 0.05},
       "run": {"arithmetic": arith, "collision": {"operator": "cumulant"}},
       "turbines": [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}],
       "polars": [{"id": "sym", "file": "sym.csv"}]}
sim = Simulation(parse_config(raw, base_dir=tmp))
lib = _lib.load()
sim.advance(40)
sim.synchronize()
for tu in ("fast", "alm"):
    getattr(lib, f"lbw_trace_reset_{tu}")()
s0 = sim.step_index
sim.advance(12)
sim.synchronize()
tabs = {}
for tu in ("fast", "alm"):
    buf = np.zeros((8, 64, 2), dtype=np.uint64)
    getattr(lib, f"lbw_trace_dump_{tu}")(buf.ctypes.data_as(ctypes.c_void_p))
    tabs[tu] = buf
t0 = int(tabs["fast"][0, s0 & 63, 0])
names = [("fast", 0, "sweep"), ("alm", 1, "KK"), ("alm", 2, "K4"), ("alm", 4, "K5")]
print("step  " + "  ".join(f"{nm:>17s}" for _, _, nm in names))
for st in range(s0, s0 + 12):
    cols = []
    for tu, kid, nm in names:
        b, e = tabs[tu][kid, st & 63]
        if b == np.uint64(~np.uint64(0)) or e == 0:
            cols.append(f"{'-':>17s}")
        else:
            cols.append(f"{(int(b) - t0) / 1e3:8.1f}-{(int(e) - t0) / 1e3:8.1f}")
    print(f"{st:4d}  " + "  ".join(cols))
