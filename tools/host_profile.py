"""Host-side cost per step of the C2 bench loop (no device sync)."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2402_13171_b200 import Simulation, _lib

tmp = tempfile.TemporaryDirectory()
cfg, desc = bench.make_config("c2", 1, "fast", tmp.name)
sim = Simulation(cfg)
lib = _lib.load()
for _ in range(5):
    sim.step()
sim.synchronize()
acc = {"refresh": 0.0, "setkin": 0.0, "step": 0.0, "poll": 0.0, "advance": 0.0}
N = 50
t0 = time.perf_counter()
for _ in range(N):
    a = time.perf_counter(); sim.refresh_points(); b = time.perf_counter()
    lib.lbw_alm_set_kinematics(sim._domain, _lib.ptr(sim._kin)); c = time.perf_counter()
    lib.lbw_domain_step(sim._domain, 1); d = time.perf_counter()
    sim._poll(False); e = time.perf_counter()
    for topo in cfg.topologies:
        topo.advance(cfg.units.dt)
    f = time.perf_counter()
    acc["refresh"] += b - a; acc["setkin"] += c - b; acc["step"] += d - c
    acc["poll"] += e - d; acc["advance"] += f - e
t_host = time.perf_counter() - t0
sim.synchronize()
t_all = time.perf_counter() - t0
print({k: round(v / N * 1e6, 1) for k, v in acc.items()}, "us/step host;",
      "host loop", round(t_host / N * 1e6, 1), "us/step; incl. drain", round(t_all / N * 1e6, 1))
sim.close()
