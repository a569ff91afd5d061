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
turbine = not (len(sys.argv) > 3 and sys.argv[3] == "none")
tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
raw = {"domain": {"cells": [n, n, n]},
       "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
       "resolution": {"mach": 0.05},
       "run": {"arithmetic": arith, "collision": {"operator": "cumulant"}},
       "turbines": [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}],
       "polars": [{"id": "sym", "file": "sym.csv"}]}
if not turbine:
    del raw["turbines"], raw["polars"]
sim = Simulation(parse_config(raw, base_dir=tmp))
lib = _lib.load()
sim.advance(40)
sim.synchronize()
SW = "exact" if arith == "exact" else "fast"   # the TU holding the sweep kernels
for tu in (SW, "alm"):
    getattr(lib, f"lbw_trace_reset_{tu}")()
s0 = sim.step_index
sim.advance(40)
sim.synchronize()
tabs = {}
for tu in (SW, "alm"):
    buf = np.zeros((8, 64, 2), dtype=np.uint64)
    getattr(lib, f"lbw_trace_dump_{tu}")(buf.ctypes.data_as(ctypes.c_void_p))
    tabs[tu] = buf
t0 = int(tabs[SW][0, s0 & 63, 0])
names = [(SW, 0, "sweep"), ("alm", 1, "KK"), ("alm", 2, "K4"), ("alm", 4, "K5")]
# chain-B sweep events: first force-tile wait start / last release, samples stored
for st in range(s0 + 30, s0 + 34):
    b = int(tabs[SW][0, st & 63, 0])
    fb, fe = (int(v) for v in tabs[SW][6, st & 63])
    pe = int(tabs[SW][5, st & 63, 1])
    sb, se = (int(v) for v in tabs[SW][7, st & 63])
    if fe and pe:
        print(f"sweep({st}): force tiles wait {(fb - b) / 1e3:.2f} .. {(fe - b) / 1e3:.2f} us, "
              f"sample tiles {(sb - b) / 1e3:.2f} .. {(se - b) / 1e3:.2f}, "
              f"samples stored at {(pe - b) / 1e3:.2f} us (after the sweep start)")
# chain-B KK phase ends (END markers only: kinematics, geometry), as offsets from KK start
for st in range(s0 + 30, s0 + 34):
    b = int(tabs["alm"][1, st & 63, 0])
    e5, e6, e1 = (int(tabs["alm"][i, st & 63, 1]) for i in (5, 6, 1))
    if b != int(np.uint64(~np.uint64(0))) and e5 and e6:
        print(f"KK({st}) phases: kinematics {(e5 - b) / 1e3:.2f} us, geometry "
              f"{(e6 - e5) / 1e3:.2f} us, count+publish {(e1 - e6) / 1e3:.2f} us")
print("step  " + "  ".join(f"{nm:>17s}" for _, _, nm in names))
spans = {nm: [] for _, _, nm in names}
for st in range(s0, s0 + 40):
    for tu, kid, nm in names:
        b, e = tabs[tu][kid, st & 63]
        if not (b == np.uint64(~np.uint64(0)) or e == 0):
            spans[nm].append((int(b), int(e), st))
for nm, sp in spans.items():
    if len(sp) > 2:
        dur = np.mean([e - b for b, e, _ in sp[2:]]) / 1e3
        gap = np.mean([sp[i][0] - sp[i - 1][1] for i in range(2, len(sp))]) / 1e3
        per = (sp[-1][0] - sp[2][0]) / (len(sp) - 3) / 1e3
        print(f"{nm:6s} mean duration {dur:6.2f} us, gap after the previous {gap:6.2f} us, "
              f"period {per:6.2f} us")
for st in range(s0 + 28, s0 + 40):
    cols = []
    for tu, kid, nm in names:
        b, e = tabs[tu][kid, st & 63]
        if b == np.uint64(~np.uint64(0)) or e == 0:
            cols.append(f"{'-':>17s}")
        else:
            cols.append(f"{(int(b) - t0) / 1e3:8.1f}-{(int(e) - t0) / 1e3:8.1f}")
    print(f"{st:4d}  " + "  ".join(cols))
