import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2402_13171_b200 import Simulation
from paper_2402_13171_b200.sim import HostKinematics
from tests.scenarios import rotor_config
np.set_printoptions(precision=4, suppress=True, linewidth=150)
cfg, tmp = rotor_config(cells=(12, 12, 12))
cfg2, tmp2 = rotor_config(cells=(12, 12, 12))
host = HostKinematics(cfg2)
sim = Simulation(cfg, kinematics="device")
for n in range(2):
    sim.step()
    kin = host.refresh(); host.advance()
    dk = sim._kin_view()
    print(n, np.abs(dk[:, 0:3] - kin[:, 0:3]).max(axis=0), flush=True)
    print(np.c_[dk[:4, 0:3], kin[:4, 0:3], dk[:4,15:18]])
