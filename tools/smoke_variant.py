import sys
sys.path.insert(0, ".")
from paper_2402_13171_b200 import Simulation
from tests.scenarios import rotor_config
kin = sys.argv[1]
cfg, tmp = rotor_config(cells=(16, 12, 12), periodic=(True, True, True), steps=3)
sim = Simulation(cfg, kinematics=kin)
for _ in range(3):
    sim.step()
    sim._alm_results()
sim.close()
print("ok", kin)
