"""Multi-GPU x-slab decomposition.

CPU part (gloo, world size 2): the host-side logic — slab bounds,
neighbour rings, non-finite consensus over ranks.
GPU part: tests/mgpu_check.py under torchrun on every visible GPU (needs
>= 2): N slabs vs one GPU, bit for bit.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2402_13171_b200.parallel import first_nonfinite, slab_neighbours
from paper_2402_13171_b200.sim import SlabGrid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_slab_bounds_and_owner():
    g = SlabGrid((100, 8, 8), (True, True, True), 3, 1)
    assert g.bounds == [0, 33, 66, 100]
    assert g.blocks[0].origin == (33, 0, 0) and g.blocks[0].size == (33, 8, 8)
    assert g.owner_block_of_position((65.9, 1.0, 1.0)) == 1
    assert g.owner_block_of_position((-0.5, 1.0, 1.0)) == 2     # periodic wrap
    with pytest.raises(Exception):
        SlabGrid((3, 8, 8), (True, True, True), 4, 0)


@pytest.mark.parametrize("n,periodic,expect", [
    (1, True, [(-1, -1)]),
    (2, True, [(1, 1), (0, 0)]),
    (3, False, [(-1, 1), (0, 2), (1, -1)]),
    (4, True, [(3, 1), (0, 2), (1, 3), (2, 0)]),
])
def test_neighbour_rings(n, periodic, expect):
    assert [slab_neighbours(r, n, periodic) for r in range(n)] == expect


def test_first_nonfinite_consensus():
    assert first_nonfinite([None, None]) is None
    reports = [None, (5, (40, 1, 2), "velocity"), (5, (3, 9, 9), "density"),
               (7, (0, 0, 0), "density")]
    assert first_nonfinite(reports) == (5, (3, 9, 9), "density")


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    report = (3, (rank, 0, 0), "velocity") if rank == 1 else None
    reports = [None] * world
    dist.all_gather_object(reports, report)
    # exact-sum reduction of owner-zeroed per-point loads
    blade = np.zeros((4, 3))
    blade[rank::world] = rank + 1.0
    parts = [None] * world
    dist.all_gather_object(parts, blade)
    q.put((rank, first_nonfinite(reports), sum(parts)))
    dist.destroy_process_group()


def test_gloo_two_rank_consensus():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, hit, blade in out:
        assert hit == (3, (1, 0, 0), "velocity")
        np.testing.assert_array_equal(blade[0::2], 1.0)
        np.testing.assert_array_equal(blade[1::2], 2.0)


@pytest.mark.gpu
def test_slabs_bitwise_equal_single_gpu(gpu):
    n = gpu.lbw_device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={min(n, 4)}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.join(ROOT, "tests", "mgpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
