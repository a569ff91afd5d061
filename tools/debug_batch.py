import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_13171_b200 import CollisionConfig, collide
g = np.load("tests/golden/collide.npz")
for k in range(int(g["ncases"])):
    cfg = CollisionConfig(str(g[f"c{k}_op"]), float(g[f"c{k}_omega"]), tuple(g[f"c{k}_rates"]))
    out = collide(g[f"c{k}_f"], g[f"c{k}_F"], cfg)
    ref = g[f"c{k}_out"]
    bad = np.argwhere(out != ref)
    F = g[f"c{k}_F"]
    rows = np.unique(bad[:, 0]) if len(bad) else []
    print(k, cfg.operator, cfg.omega, "mismatches", len(bad), "rows", len(rows),
          "rows with F=0:", sum(1 for r in rows if not F[r].any()), "maxdiff", np.abs(out-ref).max())
    if len(bad):
        r, i = bad[0]
        print("  first", r, i, repr(out[r, i]), repr(ref[r, i]), "dirs", sorted(set(bad[:, 1].tolist()))[:30])
