#!/usr/bin/env python
"""Benchmark of the lbwind time step on B200 (BASELINE.json metric:
"MLUP/s (D3Q27 cumulant fp64 + ALM) at 1/2/4/8 B200; % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--arithmetic exact|fast] [--config c2|c1|c3|c4]
                    [--precision double|single]

Workload (BASELINE.json configs[1], "C2"): 256x128x128 D3Q27 cumulant fp64,
velocity inflow / zero-gradient outflow in x, periodic y/z, one rotating
three-bladed actuator-line rotor (6 points per blade, r = 0.48 m, 96 rad/s,
symmetric polar) in a uniform 8 m/s inflow, 32 cells per diameter, Mach
0.05, nu 0.1732 -> omega 1.7857.  Synthetic data: the rotor and polar are
generated here (no files), the state starts from the uniform-wind product
equilibrium.  With N > 1 the run is weak-scaled: (256 N)x128x128 on N
GPUs, one x-slab of 256 planes per GPU, the same single rotor.

A step = actuator kinematics + sampling + blade forces + Roma spreading +
fused pull-stream-collide sweep over every cell (sim.py:264-300).  value:
device time (CUDA events on the domain stream, max over ranks) of K steps
with the state resident in HBM.  e2e: the same K steps through the public
Simulation.step() API with each step's kinematics copied host->device and
its blade loads (the thrust/power time series) read back device->host,
wall-clock, synchronised.  The state (2 x 0.9 GB) exceeds the 126 MB L2, so
no flush is needed between steps.

--impl reference times the reference algorithm on the host cores: the
bit-exact C restatement in oracle/ (OpenMP, all host threads) on the same
config; rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ROTOR = """
name: hawt
components:
  - name: tower
    position: [0.0, 0.0, 0.0]
  - name: nacelle
    parent: tower
    position: [0.0, 0.0, 0.8]
  - name: hub
    parent: nacelle
    position: [-0.05, 0.0, 0.0]
    rotation: {axis: [1.0, 0.0, 0.0], rate_rad_per_s: 96.0}
  - name: blade1
    parent: hub
    discretization: {type: line, points: 6, r_end: 0.48, chord: 0.08, twist_deg: 8.0,
                     polar: sym}
  - name: blade2
    parent: hub
    orientation: {axis: [1.0, 0.0, 0.0], angle_deg: 120.0}
    discretization: {type: line, points: 6, r_end: 0.48, chord: 0.08, twist_deg: 8.0,
                     polar: sym}
  - name: blade3
    parent: hub
    orientation: {axis: [1.0, 0.0, 0.0], angle_deg: 240.0}
    discretization: {type: line, points: 6, r_end: 0.48, chord: 0.08, twist_deg: 8.0,
                     polar: sym}
"""

BYTES_PER_LUP = 2 * 27 * 8     # algorithmic bytes of the fused sweep (fp64)
METRIC = "MLUP/s (D3Q27 cumulant fp64 + ALM)"
METRIC_SINGLE = "MLUP/s (D3Q27 cumulant fp64 arithmetic, fp32 storage + ALM)"


def polar_csv():
    a = np.arange(-180.0, 181.0, 15.0)
    t = np.deg2rad(a)
    rows = ["alpha_deg,cl,cd"] + [
        f"{float(x)!r},{float(0.9 * np.sin(2 * s))!r},{float(0.08 + 0.3 * (1 - np.cos(2 * s)))!r}"
        for x, s in zip(a, t)]
    return "\n".join(rows) + "\n"


def workload(name, n_gpus):
    """(raw config dict, description) of the benchmark workload."""
    if name == "c1":
        raw = {"domain": {"cells": [64 * n_gpus, 64, 64]},
               "fluid": {"kinematic_viscosity": 0.1353, "wind": [0.0, 0.0, 0.0],
                         "reference_velocity": 1.0},
               "resolution": {"mach": 0.02}, "run": {"collision": {"operator": "cumulant"}}}
        return raw, f"C1 TGV {64 * n_gpus}x64x64 periodic cumulant fp64, no turbine"
    if name == "c5":     # strong scaling, three aligned rotors, turbulent-like start
        cells, cpd, nu = [2048, 512, 512], 64, 0.0866
        raw = {"domain": {"cells": cells, "periodicity": [False, True, True]},
               "fluid": {"kinematic_viscosity": nu, "wind": [8.0, 0.0, 0.0]},
               "resolution": {"cells_per_diameter": cpd, "reference_diameter": 1.0,
                              "mach": 0.05},
               "run": {"boundary": "velocity_inflow_outflow",
                       "collision": {"operator": "cumulant"}},
               "turbines": [{"file": "rotor.yaml", "position": [x, 4.0, 3.2]}
                            for x in (4.05, 11.05, 18.05)],
               "polars": [{"id": "sym", "file": "sym.csv"}]}
        desc = (f"C5 2048x512x512 cumulant fp64, inflow/outflow x, aligned row of 3 rotors "
                f"at 4D/11D/18D ({9 * POINTS_PER_BLADE} points), turbulent-like initial field "
                f"(32 seeded divergence-free Fourier modes, 5 % intensity)")
        return raw, desc
    if name == "c4":     # strong scaling: the global domain is fixed
        cells, cpd, nu, pos = [1024, 512, 512], 64, 0.0866, [4.05, 4.0, 3.2]
    else:                # weak scaling: one slab of this size per GPU
        side = {"c2": (256, 128, 128), "c3": (256, 256, 256)}[name]
        cells = [side[0] * n_gpus, side[1], side[2]]
        cpd, nu = 32, 0.1732
        pos = [2.0, 2.0, 1.2] if name == "c2" else [2.0, 4.0, 3.2]
    raw = {"domain": {"cells": cells, "periodicity": [False, True, True]},
           "fluid": {"kinematic_viscosity": nu, "wind": [8.0, 0.0, 0.0]},
           "resolution": {"cells_per_diameter": cpd, "reference_diameter": 1.0, "mach": 0.05},
           "run": {"boundary": "velocity_inflow_outflow", "collision": {"operator": "cumulant"}},
           "turbines": [{"file": "rotor.yaml", "position": pos}],
           "polars": [{"id": "sym", "file": "sym.csv"}]}
    desc = (f"{name.upper()} {cells[0]}x{cells[1]}x{cells[2]} cumulant fp64, "
            f"inflow/outflow x, one 3-blade ALM rotor ({3 * POINTS_PER_BLADE} points)")
    return raw, desc


POINTS_PER_BLADE = 6


def make_config(name, n_gpus, arithmetic, tmpdir, precision="double"):
    from paper_2402_13171_b200 import parse_config
    with open(os.path.join(tmpdir, "rotor.yaml"), "w") as fh:
        fh.write(ROTOR.replace("points: 6", f"points: {POINTS_PER_BLADE}"))
    with open(os.path.join(tmpdir, "sym.csv"), "w") as fh:
        fh.write(polar_csv())
    raw, desc = workload(name, n_gpus)
    raw.setdefault("run", {})["arithmetic"] = arithmetic
    raw["run"]["precision"] = precision
    if precision == "single":
        desc = desc.replace("fp64", "fp64 arithmetic / fp32 storage")
    return parse_config(raw, base_dir=tmpdir), desc


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML from a background
    thread every ~1 ms while the sampler is open (warm-up + timed region);
    mark() brackets the timed region so the summary can say how many samples
    fell inside it.  Falls back to an nvidia-smi poll when NVML is absent."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device_index):
        self.device_index = device_index
        self.samples = []          # (t, sm_mhz, reason bits)
        self.window = [None, None]
        self.smax = None
        self.error = None

    def _handle(self, nv):
        try:
            import torch
            p = torch.cuda.get_device_properties(self.device_index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.device_index)

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = self._handle(nv)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        except Exception as e:           # no NVML: summary says so
            self.nv = None
            self.error = f"NVML unavailable: {e}"
            return self

        def poll():
            nv, h = self.nv, self.h
            while not self.stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((time.perf_counter(), float(sm), int(rs)))
                except Exception as e:
                    self.error = str(e)
                    return
                time.sleep(0.001)

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        return self

    def mark(self, which):
        self.window[0 if which == "start" else 1] = time.perf_counter()

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=5)

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0,
                    "reasons": [self.error or "NVML unavailable"]}
        t0, t1 = self.window
        inside = [s for s in self.samples
                  if t0 is not None and t1 is not None and t0 <= s[0] <= t1]
        use = inside if inside else self.samples
        reasons = set()
        for nm, attr in self.REASONS:
            bit = getattr(self.nv, attr, 0)
            if any(s[2] & bit for s in use):
                reasons.add(nm)
        out = {"sm_mhz": statistics.median(s[1] for s in use) if use else None,
               "sm_max_mhz": self.smax, "samples": len(use),
               "samples_in_timed_region": len(inside),
               "window": "timed region" if inside else "warm-up + timed region",
               "sm_mhz_min": min(s[1] for s in use) if use else None,
               "reasons": sorted(reasons), "source": "NVML, ~1 ms poll"}
        return out


# --------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2402_13171_b200 import Simulation, _lib

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    tmp = tempfile.TemporaryDirectory()
    cfg, desc = make_config(args.config, world, args.arithmetic, tmp.name, args.precision)
    bytes_per_lup = BYTES_PER_LUP if args.precision == "double" else 2 * 27 * 4
    from paper_2402_13171_b200 import parallel
    from paper_2402_13171_b200.fields import fourier_modes
    if world > 1:
        sim = parallel.SlabSimulation(cfg, rank=rank, nranks=world, device=local_rank)
    else:
        sim = Simulation(cfg, device=local_rank)
    u0 = sim.boundary.u_in_lat
    if args.config == "c5":
        sim.fields[0].initialize_modes(1.0, u0, fourier_modes(cfg.cells, u0), product=True)
    cells_total = int(np.prod(cfg.cells))
    cells_local = int(np.prod(sim.fields[0].size))
    lib = _lib.load()
    stream_ptr = _lib.ctypes.c_void_p()
    _lib.check(lib.lbw_domain_stream(sim._domain, _lib.ctypes.byref(stream_ptr)))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()

    clocks = ClockSampler(local_rank).__enter__()
    for _ in range(args.warmup):
        sim.step()
    sim.synchronize()

    # ---- the sweep kernel alone (roofline): K steps with CUDA events
    # recorded around every sweep launch on the domain stream
    _lib.check(lib.lbw_domain_sweep_timing(sim._domain, 1))
    sim.advance(args.steps)
    sim.synchronize()
    sweep_ms = _lib.ctypes.c_double()
    sweep_n = _lib.ctypes.c_int64()
    _lib.check(lib.lbw_domain_sweep_time(sim._domain, _lib.ctypes.byref(sweep_ms),
                                         _lib.ctypes.byref(sweep_n)))
    _lib.check(lib.lbw_domain_sweep_timing(sim._domain, 0))
    # ---- device-timed region (value): the next K steps queued by one native
    # call with nothing between the sweeps (the timing events above sit
    # between consecutive sweeps and turn off their programmatic launch)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    clocks.mark("start")
    start.record(stream)
    sim.advance(args.steps)
    stop.record(stream)
    sim.synchronize()
    clocks.mark("stop")
    launches = _lib.kernel_launches() - launches0
    torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(stop)
    clocks.__exit__(None, None, None)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = cells_total * args.steps / (ms / 1e3) / 1e6
    sweep_avg_ms = sweep_ms.value / max(1, sweep_n.value)

    # ---- end to end through the public API: a fresh Simulation driven the
    # reference's way -- the host turbine objects produce every step's
    # kinematics, copied host->device from pinned memory each step -- with
    # every step's blade loads copied device->host (the thrust series),
    # asynchronously, consumed after the loop
    P = len(sim.points)
    sim.close()
    if world > 1:
        sim = parallel.SlabSimulation(cfg, rank=rank, nranks=world, device=local_rank,
                                      kinematics="host" if P else None)
    else:
        sim = Simulation(cfg, device=local_rank, kinematics="host" if P else None)
    if args.config == "c5":
        sim.fields[0].initialize_modes(1.0, u0, fourier_modes(cfg.cells, u0), product=True)
    if P:
        sim.record_loads(args.steps + args.warmup + 8)
    for _ in range(args.warmup):
        sim.step()
    sim.synchronize()
    if P:
        sim.read_loads()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.step()
    sim.synchronize()
    thrust = []
    if P:
        first, forces = sim.read_loads()
        thrust = forces[..., 0].sum(axis=1)
    t_e2e = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e = cells_total * args.steps / t_e2e / 1e6

    peaks = _measured_peaks()
    achieved = bytes_per_lup * cells_local / (sweep_avg_ms / 1e3) / 1e9
    out = None
    if rank == 0:
        out = {
            "metric": METRIC if args.precision == "double" else METRIC_SINGLE,
            "value": round(value, 2), "unit": "MLUP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "strong" if args.config in ("c4", "c5") else "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "cells": list(cfg.cells),
                       "cells_per_gpu": cells_local, "actuator_points": P,
                       "arithmetic": cfg.arithmetic, "storage": cfg.precision,
                       "parallelism": f"x-slab x{world}",
                       "l2": f"state (2 x 27 x {bytes_per_lup // 54} B x cells) far larger "
                             "than the 126 MB L2; no flush needed"},
            "e2e": {"value": round(e2e, 2), "unit": "MLUP/s",
                    "h2d_bytes_per_step": P * 18 * 8,
                    "d2h_bytes_per_step": P * 3 * 8 + 8,
                    "path": "Simulation.step() with host kinematics (per-step H2D from "
                            "pinned memory) and per-step async D2H of the blade loads",
                    "thrust_series_len": int(len(thrust))},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1),
                         "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / peaks["hbm_gbs"], 4),
                         "traffic": _ncu_traffic(args.config, cells_local, args.precision),
                         "kernel": "lbw::k_sweep<cumulant,pull> (fused stream-collide)",
                         "bytes_per_lup": bytes_per_lup,
                         "sweep_ms": round(sweep_avg_ms, 4),
                         "sweep_timing": "CUDA events around each sweep launch on the domain "
                                         "stream, K steps right before the value region",
                         "sweep_share_of_step": round(sweep_avg_ms / (ms / args.steps), 4),
                         "peak_source": peaks["source"],
                         "lup_ceiling_mlups": round(peaks["hbm_gbs"] * 1e3 / bytes_per_lup, 1)},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
    sim.close()
    tmp.cleanup()
    if (rank == 0 and world == 1 and not args.no_cpu_baseline
            and args.config not in ("c4", "c5")):
        out["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_budget)
    if dist is not None:
        dist.destroy_process_group()
    return out


def _measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md 6.65 TB/s)"}


def _ncu_traffic(config, cells_local, precision="double"):
    """dram bytes per sweep launch from the committed ncu capture, scaled to
    this launch's cell count (profiles/ncu_sweep.json), or None."""
    path = os.path.join(ROOT, "profiles",
                        "ncu_sweep.json" if precision == "double" else "ncu_sweep_single.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return round(float(d["dram_bytes_per_lup"]) * cells_local)
    except (OSError, KeyError, ValueError):
        return None


# ------------------------------------------------------------ CPU legs

def _oracle_run(cfg, steps, sim_host):
    """Time `steps` reference-algorithm steps (oracle/) of cfg on the host."""
    from oracle import oracle as orc
    from tests.scenarios import oracle_for
    ref = oracle_for(sim_host)
    kins = []
    for _ in range(steps + 1):
        sim_host.refresh_points()
        kins.append(sim_host._kin.copy())
        for topo in cfg.topologies:
            topo.advance(cfg.units.dt)
    ref.step(kins[0] if ref.points else None)      # untimed warm step
    t0 = time.perf_counter()
    for n in range(steps):
        ref.step(kins[n + 1] if ref.points else None)
    return time.perf_counter() - t0


def _HostOnlySim(cfg):
    """The host half of a Simulation (kinematics, parameters) without a GPU,
    used to drive the oracle with identical actuator kinematics."""
    from paper_2402_13171_b200.sim import HostKinematics
    host = HostKinematics(cfg)
    host.refresh_points = host.refresh
    return host


def cpu_baseline(args, budget_s=20.0):
    """Reference algorithm (C oracle, OpenMP over every host thread) on the
    same workload; steps sized to ~budget_s of CPU time."""
    from oracle import oracle as orc
    orc.build()
    cores = len(os.sched_getaffinity(0))
    # every host thread, whatever OMP_NUM_THREADS a launcher set (torchrun
    # sets 1 for each rank; only rank 0 runs this arm)
    orc.set_threads(cores)
    tmp = tempfile.TemporaryDirectory()
    cfg, desc = make_config(_host_sample_config(args.config), 1, "exact", tmp.name,
                            args.precision)
    host = _HostOnlySim(cfg)
    t1 = _oracle_run(cfg, 1, host)
    steps = int(max(1, min(50, budget_s / max(t1, 1e-3))))
    cfg, desc = make_config(_host_sample_config(args.config), 1, "exact", tmp.name,
                            args.precision)
    host = _HostOnlySim(cfg)
    t = _oracle_run(cfg, steps, host)
    cells = int(np.prod(cfg.cells))
    tmp.cleanup()
    return {"value": round(cells * steps / t / 1e6, 3), "unit": "MLUP/s", "cores": cores,
            "kind": "port",
            "sample": f"{steps} full steps of {desc} (after 1 warm step), C oracle "
                      f"(-O2 -ffp-contract=off, OpenMP {cores} threads), {t:.1f} s"}


def _host_sample_config(name):
    """Host-side sample of a workload: C4 / C5 (116 / 232 GB of state) are
    timed on the C3 slab (256^3 + rotor: the same per-cell work)."""
    return "c3" if name in ("c4", "c5") else name


def _numba_child(argv):
    """Child process of the numba leg: the UNMODIFIED reference package from
    baseline/_ref (PYTHONPATH), driven through its own public API --
    lbwind.config.parse_config + lbwind.sim.Simulation.step() -- on the
    host-sample workload, every host thread as a worker (x-slab blocks).
    Prints one JSON object."""
    name, precision, budget = argv[0], argv[1], float(argv[2])
    import lbwind
    from lbwind import _kernels
    from lbwind.config import parse_config as ref_parse
    from lbwind.sim import Simulation as RefSim
    cores = len(os.sched_getaffinity(0))
    tmp = tempfile.mkdtemp()
    with open(os.path.join(tmp, "rotor.yaml"), "w") as fh:
        fh.write(ROTOR.replace("points: 6", f"points: {POINTS_PER_BLADE}"))
    with open(os.path.join(tmp, "sym.csv"), "w") as fh:
        fh.write(polar_csv())
    raw, desc = workload(name, 1)
    nx = raw["domain"]["cells"][0]
    nb = next(b for b in range(1, nx + 1) if nx % b == 0 and b >= min(cores, nx))
    raw["run"].update({"precision": precision, "workers": cores,
                       "block_dims": [nx // nb] + raw["domain"]["cells"][1:]})
    cfg = ref_parse(raw, base_dir=tmp)
    t0 = time.perf_counter()
    _kernels.warm_up((cfg.dtype,))
    sim = RefSim(cfg)
    sim.step()                                   # untimed (JIT, first touch)
    warm = time.perf_counter() - t0
    t0 = time.perf_counter()
    sim.step()
    t1 = time.perf_counter() - t0
    n = int(max(1, min(50, budget / max(t1, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(n):
        sim.step()
    t = time.perf_counter() - t0
    sim.close()
    cells = int(np.prod(cfg.cells))
    print(json.dumps({"value": round(cells * n / t / 1e6, 3), "unit": "MLUP/s", "cores": cores,
                      "kind": "reference",
                      "sample": f"{n} timed steps (after 2 untimed) of {desc}, the reference "
                                f"package lbwind {getattr(lbwind, '__version__', '0.1.0')} "
                                f"(numba, baseline/_ref) through Simulation.step(), "
                                f"{cores} workers on {nb} x-slab blocks, {t:.1f} s "
                                f"(+{warm:.1f} s JIT / first step)",
                      "cells": list(cfg.cells)}))


def numba_reference(args, budget_s=20.0):
    """Time the genuine reference (lbwind + numba from baseline/_ref) in a
    child process; None when it is not installed or fails."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lbwind")):
        return {"unavailable": "baseline/_ref not installed"}
    env = dict(os.environ)
    env["PYTHONPATH"] = ref
    env.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lbw_numba_cache"))
    env["NUMBA_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    env.pop("OMP_NUM_THREADS", None)
    try:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--numba-child",
                            _host_sample_config(args.config), args.precision, str(budget_s),
                            str(POINTS_PER_BLADE)],
                           env=env, capture_output=True, text=True, timeout=600,
                           cwd=tempfile.gettempdir())
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # report, never fail the arm
        return {"unavailable": f"numba reference failed: {type(e).__name__}: {e}"[:300]}


def run_reference(args, rank, budget_s=150.0):
    if rank != 0:
        return None
    cb = cpu_baseline(args, budget_s=args.cpu_budget)
    # time K steps (bounded so the arm ends within a few minutes: fewer
    # steps of the same workload when K would take longer than budget_s)
    from oracle import oracle as orc  # noqa: F401
    tmp = tempfile.TemporaryDirectory()
    sample_name = _host_sample_config(args.config)
    cfg, desc = make_config(sample_name, 1, "exact", tmp.name, args.precision)
    cells = int(np.prod(cfg.cells))
    est = cells / (cb["value"] * 1e6) if cb["value"] > 0 else 1.0
    n = int(max(1, min(args.steps, budget_s / max(est, 1e-6))))
    host = _HostOnlySim(cfg)
    t = _oracle_run(cfg, n, host)
    P = len(host.points) if hasattr(host, "points") else None
    tmp.cleanup()
    value = cells * n / t / 1e6
    cb["value"] = round(value, 3)
    # the line names the workload of this launch (weak-scaled with --gpus, as
    # the GPU arm's) with the GPU arm's config keys; what was actually timed
    # (one GPU's share; C4 / C5 through the C3 slab as a proxy) is measured_*
    raw_full, desc_full = workload(args.config, max(1, args.gpus))
    full_cells = list(raw_full["domain"]["cells"])
    proxy = " (C3 proxy: same per-cell work)" if sample_name != args.config else ""
    cb["sample"] = (f"{n} of {args.steps} requested steps of {desc}{proxy}, C oracle "
                    f"(bit-exact restatement of the reference kernels), {cb['cores']} threads")
    cb["sample_cells"] = list(cfg.cells)
    strong = args.config in ("c4", "c5")
    per_gpu = int(np.prod(full_cells)) // (max(1, args.gpus))
    out = {"metric": METRIC if args.precision == "double" else METRIC_SINGLE,
           "value": round(value, 3), "unit": "MLUP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(1e3 * t / n, 3), "higher_is_better": True,
           "scaling": "strong" if strong else "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": desc_full, "cells": full_cells,
                      "cells_per_gpu": per_gpu, "actuator_points": P,
                      "arithmetic": "exact (reference)", "storage": args.precision,
                      "parallelism": f"host threads x{cb['cores']} (no GPU)",
                      "l2": "n/a (host)"},
           "measured_cells": list(cfg.cells),
           "impl": "reference", "cpu_baseline": cb,
           "e2e": {"value": round(value, 3), "unit": "MLUP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    if not args.no_numba_reference:
        out["reference_numba"] = numba_reference(args, budget_s=args.cpu_budget)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c1", "c2", "c3", "c4", "c5"), default="c2")
    ap.add_argument("--points-per-blade", type=int, default=None,
                    help="default 6 (demo rotor); 50 for c5 (paper-like blades)")
    ap.add_argument("--arithmetic", choices=("exact", "fast"), default="fast")
    ap.add_argument("--precision", choices=("double", "single"), default="double")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-numba-reference", action="store_true",
                    help="reference arm: skip timing the numba reference package")
    if len(sys.argv) > 1 and sys.argv[1] == "--numba-child":
        global POINTS_PER_BLADE
        POINTS_PER_BLADE = int(sys.argv[5])
        _numba_child(sys.argv[2:5])
        return
    args = ap.parse_args()
    POINTS_PER_BLADE = args.points_per_blade or (50 if args.config == "c5" else 6)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)
    if args.impl == "reference":
        out = run_reference(args, rank)
    else:
        out = run_ours(args, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
