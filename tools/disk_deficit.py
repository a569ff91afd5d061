"""Print the test_05 disk-deficit for (cpd, steps, arithmetic) triples."""
import sys
import time

sys.path.insert(0, ".")
import pathlib
import tempfile

from tests.test_gpu_acceptance import DISK_TURBINE, INDUCTION, _disk_deficit

d = pathlib.Path(tempfile.mkdtemp())
(d / "disk.yaml").write_text(DISK_TURBINE)
for arg in sys.argv[1:]:
    cpd, steps, arith = arg.split(":")
    t = time.time()
    dd = _disk_deficit(int(cpd), int(steps), d, arithmetic=arith)
    print(f"cpd={cpd} steps={steps} {arith}: deficit={dd:.6f} a={INDUCTION:.6f} "
          f"ratio={dd / INDUCTION:.4f} ({time.time() - t:.1f}s)", flush=True)
