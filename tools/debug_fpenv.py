import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as orc
g = np.load("tests/golden/collide.npz")
f = g["c0_f"]; F = g["c0_F"]
a, _ = orc.collide_batch("bgk", f, F, 1.3)
print("before: oracle==golden", np.array_equal(a, g["c0_out"]))
from paper_2402_13171_b200 import _lib, kernels
lib = _lib.load()
print("devices", lib.lbw_device_count())
b, _ = orc.collide_batch("bgk", f, F, 1.3)
print("after load: oracle==golden", np.array_equal(b, g["c0_out"]))
if lib.lbw_device_count():
    f2 = np.ascontiguousarray(f).copy(); m2 = np.zeros((f.shape[0], 4))
    kernels.collide_bgk_batch(f2, np.ascontiguousarray(F), m2, 1.3, 1.0)
    c, _ = orc.collide_batch("bgk", f, F, 1.3)
    print("after kernel: oracle==golden", np.array_equal(c, g["c0_out"]), "gpu==golden", np.array_equal(f2, g["c0_out"]), "gpu==oracle_now", np.array_equal(f2, c))
