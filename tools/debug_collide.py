import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_13171_b200 import kernels, collide, CollisionConfig
g = np.load("tests/golden/collide.npz")
f = g["c0_f"]; F = g["c0_F"]; n = f.shape[0]
cfg = CollisionConfig("bgk", 1.3, (1.0, 1.0, 1.0, 1.0))
a = collide(f, F, cfg)
f2 = np.ascontiguousarray(f).copy(); m2 = np.zeros((n, 4))
kernels.collide_bgk_batch(f2, np.ascontiguousarray(F), m2, 1.3, 1.0)
print("collide==kernels", np.array_equal(a, f2), "kernels==golden", np.array_equal(f2, g["c0_out"]),
      "collide==golden", np.array_equal(a, g["c0_out"]))
print(f.dtype, f.flags["C_CONTIGUOUS"], F.dtype, F.flags["C_CONTIGUOUS"], g["c0_op"], g["c0_omega"])
