"""Per-step wall time on a small domain (64^3, the reference's test_07
case): Python step() loop vs one lbw_domain_step(n) call, with and without
the rotor."""
import os
import sys
import time

sys.path.insert(0, ".")
import tempfile

from paper_2402_13171_b200 import Simulation, _lib, parse_config
from tests.scenarios import write_rotor_files

tmp = tempfile.mkdtemp()
write_rotor_files(tmp)


def make(turbine, arithmetic, n=64):
    raw = {"domain": {"cells": [n, n, n]},
           "fluid": {"kinematic_viscosity": 0.1732, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"mach": 0.05},
           "run": {"arithmetic": arithmetic, "collision": {"operator": "cumulant"}}}
    if turbine:
        raw["turbines"] = [{"file": "rotor.yaml", "position": [1.0, 1.0, 0.2]}]
        raw["polars"] = [{"id": "sym", "file": "sym.csv"}]
    return Simulation(parse_config(raw, base_dir=tmp))


N = 400
for n in ([int(a) for a in sys.argv[1:]] or (64, 128)):
    for arith in ("exact", "fast"):
        for turb, fused in ((False, "1"), (True, "0"), (True, "1")):
            os.environ["LBW_FUSED"] = fused   # read at domain creation
            sim = make(turb, arith, n)
            lib = _lib.load()
            for _ in range(20):
                sim.step()
            sim.synchronize()
            t = time.perf_counter()
            for _ in range(N):
                sim.step()
            sim.synchronize()
            py = (time.perf_counter() - t) / N * 1e6
            t = time.perf_counter()
            lib.lbw_domain_step(sim._domain, N)
            lib.lbw_domain_sync(sim._domain)
            c = (time.perf_counter() - t) / N * 1e6
            l0 = lib.lbw_kernel_launches()
            lib.lbw_domain_step(sim._domain, 10)
            lib.lbw_domain_sync(sim._domain)
            launches = (lib.lbw_kernel_launches() - l0) / 10
            print(f"{n}^3 {arith:5s} turbine={turb!s:5s} fused={fused}: step() {py:7.1f} us/step  "
                  f"domain_step(N) {c:7.1f} us/step  launches/step {launches:.1f}", flush=True)
            sim.close()
