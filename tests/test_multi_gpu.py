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


def _wiring_worker(rank, world, port, q):
    """Handle-blob exchange and neighbour wiring (SlabSimulation._link) and
    the sparse probe-cube gather of an output tick (SlabSimulation.
    _probe_tick), over gloo with fake blobs and a host macro field."""
    import types

    import torch.distributed as dist

    from paper_2402_13171_b200 import output, parse_config
    from paper_2402_13171_b200.halo import BoundarySpec
    from paper_2402_13171_b200.parallel import exchange_neighbour_blobs, gather_probe_cells
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for periodic in (False, True):
        blob = f"handle-of-rank-{rank}".encode() * (rank + 1)
        out[periodic] = exchange_neighbour_blobs(blob, rank, world, periodic)
    raw = {"domain": {"cells": [3 * world + 2, 9, 7], "periodicity": [False, True, True]},
           "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
           "run": {"boundary": "velocity_inflow_outflow"},
           "output": {"probes": [{"kind": "axial_line", "name": "a", "samples": 23},
                                 {"kind": "radial_profile", "name": "r", "samples": 9,
                                  "x_m": 0.31}]}}
    cfg = parse_config(raw)
    grid = SlabGrid(cfg.cells, cfg.periodicity, world, rank)
    sim = types.SimpleNamespace(cfg=cfg, units=cfg.units, grid=grid, step_index=4,
                                boundary=BoundarySpec("velocity_inflow_outflow",
                                                      u_in_lat=(0.03, 0.0, 0.0)))
    macro = np.random.default_rng(11).uniform(0.5, 1.5, tuple(cfg.cells) + (4,))
    x0, x1 = grid.bounds[rank], grid.bounds[rank + 1]
    cubes = gather_probe_cells(sim, macro[x0:x1], x0, rank, world)
    ok = None
    if rank == 0:
        dense = output.ghosted_macro(sim, macro)
        ok = all(np.array_equal(output.probe_rows(sim, p, dense)[1],
                                output.probe_rows(sim, p, cubes)[1]) for p in cfg.probes)
    q.put((rank, out, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_neighbour_wiring_and_probe_gather(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_wiring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, out, ok = q.get(timeout=120)
        res[rank] = (out, ok)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    blob = lambda r: f"handle-of-rank-{r}".encode() * (r + 1)   # noqa: E731
    for rank in range(world):
        for periodic in (False, True):
            lo, hi = slab_neighbours(rank, world, periodic)
            got = res[rank][0][periodic]
            assert got == (blob(lo) if lo >= 0 else None, blob(hi) if hi >= 0 else None)
    assert res[0][1] is True


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


# ------------------------------------------------ multi-GPU output ticks
# SlabSimulation._probe_tick sends rank 0 only the cells of the position
# probes' sampling cubes (output.CubeSource); the samples must equal the
# ones a dense ghosted field gives, bit for bit, for every ghost rule.

@pytest.mark.parametrize("boundary,periodic,step", [
    ("velocity_inflow_outflow", (False, True, True), 3),
    ("velocity_inflow_outflow", (False, True, False), 0),
    ("periodic", (True, True, True), 5),
    ("periodic", (True, False, True), 2),
])
def test_sparse_probe_cubes_equal_dense_ghosted_field(boundary, periodic, step):
    import types

    from paper_2402_13171_b200 import output, parse_config
    from paper_2402_13171_b200.halo import BoundarySpec
    raw = {"domain": {"cells": [13, 9, 7], "periodicity": list(periodic)},
           "fluid": {"kinematic_viscosity": 0.3, "wind": [8.0, 0.5, -0.25]},
           "resolution": {"cells_per_diameter": 8, "reference_diameter": 1.0, "mach": 0.1},
           "run": {"boundary": boundary},
           "output": {"probes": [
               {"kind": "axial_line", "name": "a", "samples": 29},
               {"kind": "axial_line", "name": "b", "samples": 11, "y_m": 0.05, "z_m": 0.83},
               {"kind": "radial_profile", "name": "r", "samples": 17, "x_m": 1.59, "z_m": 0.02},
               {"kind": "radial_profile", "name": "s", "samples": 5, "x_m": 0.01}]}}
    cfg = parse_config(raw)
    sim = types.SimpleNamespace(
        cfg=cfg, units=cfg.units, grid=SlabGrid(cfg.cells, cfg.periodicity, 1, 0),
        boundary=BoundarySpec(boundary, u_in_lat=(0.03, -0.01, 0.002)), step_index=step)
    rng = np.random.default_rng(5)
    macro = rng.uniform(0.5, 1.5, tuple(cfg.cells) + (4,))
    dense = output.ghosted_macro(sim, macro)
    cells = {}
    for key in output.probe_cube_cells(sim):
        kind, src = output.ghost_source(sim, key)
        cells[key] = macro[src] if kind == "cell" else src
        assert np.array_equal(cells[key], dense[key]), key
    sparse = output.CubeSource(cells)
    for probe in cfg.probes:
        h1, r1 = output.probe_rows(sim, probe, dense)
        h2, r2 = output.probe_rows(sim, probe, sparse)
        assert h1 == h2 and np.array_equal(r1, r2)
