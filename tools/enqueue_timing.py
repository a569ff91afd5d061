"""Host enqueue time vs device time of lbw_domain_step(N) (is a small
domain launch-bound?)."""
import sys
import time

sys.path.insert(0, ".")
import tempfile

from paper_2402_13171_b200 import Simulation, _lib, parse_config
from tests.scenarios import write_rotor_files

tmp = tempfile.mkdtemp()
write_rotor_files(tmp)
for n in (64, 128):
    for turb in (False, True):
        raw = {"domain": {"cells": [n, n, n]},
               "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
               "resolution": {"mach": 0.05},
               "run": {"arithmetic": "fast", "collision": {"operator": "cumulant"}}}
        if turb:
            raw["turbines"] = [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}]
            raw["polars"] = [{"id": "sym", "file": "sym.csv"}]
        sim = Simulation(parse_config(raw, base_dir=tmp))
        lib = _lib.load()
        sim.advance(50)
        sim.synchronize()
        # short bursts stay below the launch-queue depth, so the enqueue
        # time is the host's own cost, not back-pressure from the device
        for N in (60, 2000):
            t0 = time.perf_counter()
            lib.lbw_domain_step(sim._domain, N)
            t1 = time.perf_counter()
            lib.lbw_domain_sync(sim._domain)
            t2 = time.perf_counter()
            print(f"{n}^3 turbine={turb!s:5s} N={N}: enqueue {(t1 - t0) / N * 1e6:6.1f} "
                  f"us/step, total {(t2 - t0) / N * 1e6:6.1f} us/step", flush=True)
        sim.close()
