import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_13171_b200 import kernels
from oracle import oracle as orc
g = np.load("tests/golden/collide.npz")
f = np.ascontiguousarray(g["c0_f"]); F = np.ascontiguousarray(g["c0_F"]); n = f.shape[0]
for op in ("bgk", "cumulant"):
    f2 = f.copy(); m2 = np.zeros((n, 4))
    if op == "bgk":
        kernels.collide_bgk_batch(f2, F, m2, 1.3, 1.0)
    else:
        kernels.collide_cumulant_batch(f2, F, m2, 1.3, 1, 1, 1, 1, 1.0)
    fo, mo = orc.collide_batch(op, f, F, 1.3)
    print(op, "rho equal", np.array_equal(m2[:, 0], mo[:, 0]), "u equal", np.array_equal(m2[:, 1:], mo[:, 1:]),
          "f equal", np.array_equal(f2, fo))
    rho = f.sum(axis=1)
    # sequential sums
    rs = np.zeros(n)
    for i in range(27): rs = rs + f[:, i]
    print("  rho gpu==seq", np.array_equal(m2[:, 0], rs), "oracle==seq", np.array_equal(mo[:, 0], rs))
    inv = 1.0 / rs
    print("  inv: gpu ux == (mx)*inv?", )
    bad = np.nonzero(m2[:, 1] != mo[:, 1])[0]
    if len(bad):
        r = bad[0]
        print("  row", r, m2[r].tolist(), mo[r].tolist())
