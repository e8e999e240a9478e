#!/usr/bin/env python
"""Benchmark of the B200 (I - Lambda Sigma) matvec -- the hot path of rtkrylov.

Workload (BASELINE.json configs[1], "cfg2"): 1D slab, N_z = 2000 log-spaced
optical depths 1e-6..1e6 with a seeded log-normal perturbation (sigma 0.3),
32+32 Gauss-Legendre mu, N_nu = 512 over +-8 Doppler widths, dipole x PRD
(dense 512 x 512 R), eps = 1e-6, implicit-Euler formal solver, FP64:
N = 65,536,000 DOF, 524 MB per vector.  A step is one matvec y = A x.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1: launched under torchrun (one rank per GPU; `--gpus N` without torchrun
re-launches itself through torch.distributed.run).  Default `--mode sharded`:
ONE cfg2 matvec per step, its 64 directions split over the ranks, one NCCL
all-reduce of the 16 MB moment array per matvec (strong scaling, DESIGN.md
section 10); `--mode replicas`: an independent cfg2 matvec per GPU (weak).
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  The vector (524 MB) exceeds the 126 MB L2, so no
explicit flush is needed between steps.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "(I-Lambda Sigma) matvecs/s"
UNIT = "matvec/s"
CFG = 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--formal-solver", default="ie", choices=["ie", "exp_linear", "exp_parabolic"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--no-lattice", action="store_true")
    ap.add_argument("--cfg5-gmres", action="store_true",
                    help="also run cfg5 GMRES(20) to 1e-8 (about 1,550 iterations, ~9 minutes)")
    ap.add_argument("--mode", choices=["replicas", "sharded"], default="sharded",
                    help="N > 1: ONE cfg2 matvec sharded by direction with an NCCL all-reduce of the moments "
                         "(strong scaling, default) or independent cfg2 matvecs per GPU (weak scaling)")
    ap.add_argument("--no-reference-as-shipped", action="store_true",
                    help="skip timing the installed reference package (baseline/_ref) on cfg2 shapes")
    return ap.parse_args()


def dist_setup(backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return world, rank, local


def profile_path(name):
    """profiles/r02_<name> when this round captured it, else round 1's file."""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", f"{rnd}_{name}")
        if os.path.exists(path):
            return path
    return os.path.join(ROOT, "profiles", f"r02_{name}")


def ncu_raw(path, kernel=None):
    """The `raw:` metrics line of a committed ncu summary (profiles/) -- the first one, or the
    one labelled with `kernel` -- as a dict, or {}."""
    try:
        with open(path) as fh:
            for line in fh:
                if "raw:" in line and (kernel is None or kernel in line):
                    out = {}
                    for part in line.split("raw:")[1].split("]", 1)[-1].split(","):
                        if "=" in part:
                            k, v = part.strip().split("=", 1)
                            out[k] = v
                    return out
    except OSError:
        pass
    return {}


def ncu_dmma_pipes(path=None):
    """{kernel: DMMA sub-pipe active fraction} from the committed ncu capture
    (profiles/r02_ncu_dmma_pipes.txt by tools/ncu_dmma_pipes.sh, else round 1's), or {}."""
    path = path or profile_path("ncu_dmma_pipes.txt")
    out, name = {}, None
    try:
        with open(path) as fh:
            for line in fh:
                if line.startswith("=="):
                    name = "sigma_fused_kernel" if "sigma_fused" in line else (
                        "redistribute_dmma_kernel" if "redistribute_dmma" in line else None)
                elif name and "dmma_cycles_active" in line:
                    for part in line.split("raw:")[1].split(","):
                        k, v = part.strip().split("=")
                        if "dmma_cycles_active" in k:
                            out[name] = float(v.rstrip("%")) / 100
    except OSError:
        pass
    return out


def sweep_traffic_source():
    """(path, kernel label) of the committed `ncu --set full` capture of the IE sweep."""
    r02 = os.path.join(ROOT, "profiles", "r02_ncu_cfg2_kernels.txt")
    if os.path.exists(r02) and ncu_raw(r02, "sweep1d_tma"):
        return r02, "sweep1d_tma"
    return os.path.join(ROOT, "profiles", "r01_ncu_sweep_tma_v3.txt"), None


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of the sweep kernel from the committed
    `ncu --set full` capture (profiles/), bytes per launch, or None."""
    path, kernel = sweep_traffic_source()
    vals = ncu_raw(path, kernel)

    def to_bytes(v):
        for unit, mul in (("Gbyte", 1e9), ("Mbyte", 1e6), ("Kbyte", 1e3), ("byte", 1.0)):
            if v.endswith(unit):
                return float(v[: -len(unit)]) * mul
        return float(v)

    try:
        return to_bytes(vals["dram__bytes_read.sum"]) + to_bytes(vals["dram__bytes_write.sum"])
    except (KeyError, ValueError):
        return None


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def workload_config(extra=None):
    from paper_2602_21958_b200 import configs

    c = configs.SLAB_CONFIGS[CFG]
    cfg = {"workload": "cfg2: 1D slab 2000 z x 64 mu x 512 nu, dipole x PRD (dense 512x512 R), eps 1e-6",
           "n_dof": c["n_space"] * c["n_angles"] * c["n_freq"], "n_space": c["n_space"], "n_angles": c["n_angles"],
           "n_freq": c["n_freq"], "l2_policy": "inputs larger than L2 (524 MB vector vs 126 MB L2); no flush"}
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def aggregate(ms_local: float, steps: int, world: int, device: str):
    """Max of the timed region over ranks; whole-job throughput = world * steps / max time
    (weak scaling: every rank runs the full per-GPU workload)."""
    import torch

    t = torch.tensor([ms_local], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    return ms_max, world * steps / (ms_max / 1e3)


def cpu_port_timing(problem, target_s=12.0, max_steps=30):
    """The oracle's C/OpenMP restatement (oracle/librto.so) on this host's cores."""
    from oracle import cport
    from oracle.rt_oracle import desc_from_problem

    port = cport.SlabPort(desc_from_problem(problem))
    rng = np.random.default_rng(7)
    x = rng.standard_normal(problem.n_total)
    y = np.empty_like(x)
    threads = cport.max_threads()
    port.apply_A(x, y)  # warm-up (page faults, thread pool)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_steps and (time.perf_counter() - t_start) < target_s:
        t0 = time.perf_counter()
        port.apply_A(x, y)
        times.append(time.perf_counter() - t0)
    return {"value": 1.0 / statistics.mean(times), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(times)} full cfg2 matvecs (N=65.5M) by oracle/rt_oracle_c.c, OpenMP over {threads} "
                      f"threads, mean {statistics.mean(times) * 1e3:.1f} ms"}


REF_PKG = os.path.join(ROOT, "baseline", "_ref")


def _ref_shipped_child():
    """(child process) The installed, unmodified reference package (baseline/_ref, rtkrylov
    0.1.0) on cfg2 shapes, timed through its own public API: apply_A with its own dipole
    kernel LegendreKernel((1, 0, 1/2)) -- the reference's Sigma is frequency-flat; the PRD
    contraction is not expressible in it -- and apply_transfer alone (its numba
    sweeps, R/transfer.py:134-141, R/_kernels.py:70-88).  Best of k, the reference's own
    benchmark pattern (benchmarks/bench_kernels.py:19-25).  Prints one JSON object."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtk_numba_cache")
    sys.path.insert(0, REF_PKG)
    import numpy as np_

    from rtkrylov import _kernels
    from rtkrylov.grid import Grid
    from rtkrylov.operator import RTProblem, apply_A
    from rtkrylov.quadrature import gauss_legendre, trapezoid
    from rtkrylov.scattering import LegendreKernel, build_scattering
    from rtkrylov.transfer import apply_transfer, build_transfer

    from paper_2602_21958_b200 import configs

    c = configs.SLAB_CONFIGS[CFG]
    t = configs.slab_t_nodes(c["n_space"], c["t_range"], c["sigma"], configs.SEED_BASE + CFG)
    dn = gauss_legendre(c["n_angles"] // 2, -1.0, 0.0)
    up = gauss_legendre(c["n_angles"] // 2, 0.0, 1.0)
    fr = trapezoid(c["n_freq"], -c["x_max"], c["x_max"])

    def gauss(nu):
        nu = np_.asarray(nu, dtype=float)
        return np_.exp(-nu * nu) / np_.sqrt(np_.pi)

    grid = Grid(t, np_.concatenate([dn.nodes, up.nodes]), np_.concatenate([dn.weights, up.weights]), fr.nodes,
                fr.weights, gauss)
    eps = c["eps"]
    wsum = float(fr.weights.sum())
    scat = build_scattering(grid, LegendreKernel((1.0, 0.0, 0.5)),
                            lambda tt, mu, nu: (1.0 - eps) / (2.0 * wsum) * np_.ones_like(tt + mu + nu))
    tr = build_transfer(grid, 0.0, 0.0)
    prob = RTProblem(grid, tr, scat, thermal=np_.full(grid.n_total, eps))
    v = np_.random.default_rng(7).standard_normal(grid.n_total)

    def best_of(fn, k):
        best = float("inf")
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
        return best

    apply_transfer(tr, v)   # numba compile / page-in
    t_lam = best_of(lambda: apply_transfer(tr, v), 2)
    apply_A(prob, v)
    t_a = best_of(lambda: apply_A(prob, v), 2)
    print(json.dumps({"apply_A_s": t_a, "apply_transfer_s": t_lam, "backend": _kernels.backend(),
                      "n_dof": int(grid.n_total)}), flush=True)


def reference_as_shipped(timeout_s=900):
    """The installed reference (baseline/_ref) timed as shipped (numba sweeps on one core, numpy
    BLAS on all cores) and with OPENBLAS_NUM_THREADS=1, each in a fresh process; plus the host's
    CPU model and core count.  {} entries say why a leg is missing."""
    import platform

    cpu_model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    cpu_model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    out = {"cpu_model": cpu_model, "nproc": os.cpu_count(), "package": "rtkrylov 0.1.0 (baseline/_ref, unmodified)",
           "workload": "cfg2 shapes (2000 x 64 x 512 = 65.5 M DOF), the reference's own frequency-flat dipole "
                       "kernel LegendreKernel((1, 0, 1/2)); best of 2 after a warm-up call"}
    if not os.path.isdir(os.path.join(REF_PKG, "rtkrylov")):
        out["unavailable"] = "baseline/_ref not installed (pip install --target baseline/_ref /root/reference)"
        return out
    for name, extra in (("as_shipped", {}), ("openblas_1_thread", {"OPENBLAS_NUM_THREADS": "1",
                                                                   "OMP_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"})):
        env = dict(os.environ, **extra)
        try:
            res = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-shipped-child"], env=env,
                                 capture_output=True, text=True, timeout=timeout_s)
            rec = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
            rec["matvecs_per_s"] = 1.0 / rec["apply_A_s"]
            out[name] = rec
        except Exception as exc:  # pragma: no cover - reported, not fatal
            out[name] = {"unavailable": f"{type(exc).__name__}: {str(exc)[:200]}"}
    return out


def run_reference(args):
    """--impl reference: the oracle port of the reference CPU path on the host cores (rank 0 only)."""
    world, rank, _ = dist_setup("gloo")
    if rank != 0:
        return
    from oracle import cport
    from oracle.rt_oracle import desc_from_problem
    from paper_2602_21958_b200 import configs

    problem = configs.slab_problem(CFG, formal_solver=args.formal_solver)
    port = cport.SlabPort(desc_from_problem(problem))
    x = np.random.default_rng(7).standard_normal(problem.n_total)
    y = np.empty_like(x)
    for _ in range(max(args.warmup, 0)):
        port.apply_A(x, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        port.apply_A(x, y)
    elapsed = time.perf_counter() - t0
    value = args.steps / elapsed
    threads = cport.max_threads()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config({"formal_solver": args.formal_solver}),
            "gdof_per_s": value * problem.n_total / 1e9,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"each step one full cfg2 matvec by oracle/rt_oracle_c.c (C restatement of "
                                       f"R/operator.py:48-53 + R/_kernels.py:70-88), OpenMP {threads} threads",
                             "reference_as_shipped": None if args.no_reference_as_shipped
                             else reference_as_shipped()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class _PlumbingShardOps:
    """BENCH_PLUMBING=1 only (tests/test_bench_multirank.py, CPU ranks): stand-ins with the
    shapes of the two device halves and NO radiative-transfer arithmetic, so the multi-rank
    bench path (torchrun relaunch, all-reduce, barriers, max over ranks, the JSON line) runs
    end to end without a GPU.  Its line says so in "data"; it is never a measurement."""

    def __init__(self, local):
        import torch

        from paper_2602_21958_b200.scattering import separable_form

        g = local.grid
        self.torch = torch
        self.n_m = g.n_space * separable_form(local.scattering.kernel, g)[0].shape[0] * g.n_freq

    def partial_moments(self, x):
        return self.torch.zeros(self.n_m, dtype=self.torch.float64)

    def apply_with_moments(self, x, m):
        return x.clone()


def run_sharded(args):
    """--mode sharded (default for N > 1): ONE cfg2 matvec per step, the 64 directions split
    over the ranks (paper_2602_21958_b200.sharding), one NCCL all-reduce of the 16 MB moment
    array per matvec.  `value` = whole-job matvecs/s (strong scaling); e2e adds each rank's
    H2D of its x slice and D2H of its y slice (pinned host buffers) inside the timed region."""
    import torch

    plumbing = os.environ.get("BENCH_PLUMBING") == "1"
    world, rank, local = dist_setup("gloo" if plumbing else "nccl")
    from paper_2602_21958_b200 import _native, configs
    from paper_2602_21958_b200.sharding import NativeShardOps, ShardedOperator

    if plumbing:
        problem = configs.slab_problem(CFG, n_space=40, n_angles=8, n_freq=16)
        op = ShardedOperator(problem, rank=rank, world=world, ops_factory=_PlumbingShardOps)
        dev = "cpu"
    else:
        torch.cuda.set_device(local)
        problem = configs.slab_problem(CFG, formal_solver=args.formal_solver)
        op = ShardedOperator(problem, rank=rank, world=world, ops_factory=NativeShardOps)
        dev = "cuda"
    gen = torch.Generator(device=dev).manual_seed(1234)
    x = torch.randn(problem.n_total, dtype=torch.float64, device=dev, generator=gen)
    x_local = op.local_slice(x).contiguous()
    del x

    def sync():
        if not plumbing:
            torch.cuda.synchronize()

    def timed(fn, steps):
        """ms of `steps` calls: CUDA events on the launching stream (wall clock on CPU ranks)."""
        sync()
        torch.distributed.barrier()
        if plumbing:
            t0 = time.perf_counter()
            for _ in range(steps):
                fn()
            ms = (time.perf_counter() - t0) * 1e3
        else:
            stream = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        torch.distributed.barrier()
        return ms

    for _ in range(max(args.warmup, 3)):
        op(x_local)
    clocks = None if plumbing else ClockSampler(local)
    if clocks:
        clocks.start()
    launches0 = 0 if plumbing else _native.launch_count()
    ms = timed(lambda: op(x_local), args.steps)
    launches = 0 if plumbing else _native.launch_count() - launches0
    clk = clocks.stop() if clocks else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["cpu plumbing run"]}
    ms_max, _ = aggregate(ms, args.steps, world, dev)
    value = args.steps / (ms_max / 1e3)   # whole-job matvecs/s: every step is ONE global matvec

    # e2e: host slices in, host slices out (pinned), one sharded matvec per step
    hx = torch.empty(x_local.numel(), dtype=torch.float64, pin_memory=not plumbing)
    hx.copy_(x_local.cpu())
    hy = torch.empty_like(hx)

    def e2e_step():
        xd = hx.to(dev, non_blocking=True)
        yd = op(xd)
        hy.copy_(yd, non_blocking=True)
        sync()

    ms_e = timed(e2e_step, max(3, min(args.steps, 10)))
    ms_e_max, _ = aggregate(ms_e, max(3, min(args.steps, 10)), world, dev)
    e2e = {"value": max(3, min(args.steps, 10)) / (ms_e_max / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": 8 * problem.n_total, "d2h_bytes_per_step": 8 * problem.n_total,
           "path": "ShardedOperator (rtk_partial_moments + all-reduce + rtk_apply_A_with_moments) with each "
                   "rank's x slice copied H2D and its y slice D2H every step (bytes summed over ranks)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": ("PLUMBING TEST: CPU gloo ranks, stand-in halves with no transfer arithmetic, reduced cfg2 "
                         "shapes -- not a measurement") if plumbing else "synthetic (seeded; BASELINE cfg2 shapes)",
                "config": workload_config({"formal_solver": args.formal_solver}),
                "parallelism": f"direction-sharded x{world} (NCCL all-reduce of moments)",
                "gdof_per_s": value * problem.n_total / 1e9, "gpu_launches": launches, "clocks": clk,
                "e2e": e2e, "mode": "sharded", "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def run_b200(args):
    import torch

    world, rank, local = dist_setup("nccl")
    torch.cuda.set_device(local)
    import paper_2602_21958_b200 as P
    from paper_2602_21958_b200 import _device, _native, configs

    lib = _native.lib()
    problem = configs.slab_problem(CFG, formal_solver=args.formal_solver)
    n = problem.n_total
    h = problem.device()
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)

    def step():
        _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _native.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    # K matvecs last only K x 0.3 ms, shorter than nvidia-smi's 200 ms sampling period: keep the
    # same matvec loop running (untimed) for 1.2 s so the clock / throttle samples are taken
    # under the timed region's own load
    t_hold = time.perf_counter() + 1.2
    while time.perf_counter() < t_hold:
        for _ in range(50):
            step()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    clk["window"] = "timed region + 1.2 s of the same matvec loop (untimed)"
    ms_max, value = aggregate(ms, args.steps, world, "cuda")
    ms_per_step = ms_max / args.steps

    # per-kernel durations inside the same matvec (events on the launching stream)
    kms = np.zeros(3)
    buf = (ctypes.c_float * 3)()
    kreps = max(5, min(args.steps, 20))
    for _ in range(kreps):
        _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr, buf))
        kms += np.array(list(buf), dtype=float)
    kms /= kreps
    g = problem.grid
    n_mom = P.separable_form(problem.scattering.kernel, g)[0].shape[0]
    mom_elems = n_mom * g.n_freq * g.n_space
    peaks, peak_src = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    sweep_bytes = 16 * n + 8 * mom_elems + 8 * g.n_space
    moments_bytes = 8 * n + 8 * mom_elems
    r_flops = 2.0 * g.n_freq * mom_elems   # 2 N_nu^2 n_mom N_s
    fp64_peak = 37.1  # DMMA TF/s measured by tools/peaks_fp64.cu (profiles/r01_peaks_fp64.json)
    kernels = {
        "sweep": {"ms": kms[2], "bytes": sweep_bytes, "achieved_gbs": sweep_bytes / kms[2] / 1e6,
                  "frac_hbm": sweep_bytes / kms[2] / 1e6 / hbm},
    }
    if kms[1] < 0:
        # the unfused pair (K2a moments, K2b DMMA GEMM) on the same input, for the per-kernel roofline
        h.set_tuning("sigma_unfused", 1)
        kun = np.zeros(3)
        for _ in range(kreps):
            _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr, buf))
            kun += np.array(list(buf), dtype=float)
        kun /= kreps
        h.set_tuning("sigma_unfused", 0)
        kernels["unfused_pair"] = {
            "moments": {"ms": kun[0], "bytes": moments_bytes, "achieved_gbs": moments_bytes / kun[0] / 1e6,
                        "frac_hbm": moments_bytes / kun[0] / 1e6 / hbm},
            "redistribute": {"ms": kun[1], "flops": r_flops, "achieved_tflops": r_flops / kun[1] / 1e9,
                             "frac_fp64": r_flops / kun[1] / 1e9 / fp64_peak}}
        # FP64 tensor (DMMA) pipe utilisation from the committed ncu capture (north star: "FP64
        # tensor-pipe utilisation (redistribution) taken from ncu")
        dm = ncu_dmma_pipes()
        if "redistribute_dmma_kernel" in dm:
            kernels["unfused_pair"]["redistribute"]["ncu_dmma_pipe_active"] = dm["redistribute_dmma_kernel"]
        if "sigma_fused_kernel" in dm:
            kernels.setdefault("sigma_fused_ncu", {})["dmma_pipe_active"] = dm["sigma_fused_kernel"]
        # K2a + K2b ran as ONE kernel (sigma_fused_kernel): x streamed once while the DMMA
        # contraction runs; it is bound by both HBM (x) and the FP64 pipe (R contraction + the
        # 2 n_mom flops per x element of the moment reduction), so both fractions are given
        fl = r_flops + 2.0 * n_mom * n
        kernels["sigma_fused"] = {"ms": kms[0], "bytes": moments_bytes, "achieved_gbs": moments_bytes / kms[0] / 1e6,
                                  "frac_hbm": moments_bytes / kms[0] / 1e6 / hbm, "flops": fl,
                                  "achieved_tflops": fl / kms[0] / 1e9, "frac_fp64": fl / kms[0] / 1e9 / fp64_peak}
    else:
        kernels["moments"] = {"ms": kms[0], "bytes": moments_bytes, "achieved_gbs": moments_bytes / kms[0] / 1e6,
                              "frac_hbm": moments_bytes / kms[0] / 1e6 / hbm}
        kernels["redistribute"] = {"ms": kms[1], "flops": r_flops, "achieved_tflops": r_flops / kms[1] / 1e9,
                                   "frac_fp64": r_flops / kms[1] / 1e9 / fp64_peak}
    matvec_bytes = 24 * n + 16 * mom_elems + 8 * g.n_freq ** 2 + 8 * g.n_space
    roofline = {"bound": "hbm", "kernel": "sweep1d_tma_kernel (K1: fused source expansion + IE sweep + y = x - acc)",
                "achieved": sweep_bytes / kms[2] / 1e6, "peak": hbm, "unit": "GB/s",
                "frac": sweep_bytes / kms[2] / 1e6 / hbm, "traffic": ncu_traffic(), "peak_source": peak_src,
                "traffic_source": os.path.relpath(sweep_traffic_source()[0], ROOT) +
                                  " (ncu --set full, dram read+write per launch)",
                "algorithmic_bytes_per_launch": sweep_bytes,
                "matvec_algorithmic_bytes": matvec_bytes,
                "matvec_frac_hbm": matvec_bytes / (ms_per_step / 1e3) / 1e9 / hbm}

    # e2e: reference-facing calls with host buffers (pinned), H2D + matvec + D2H per step
    e2e = None
    if rank == 0 or world > 1:
        nbuf = 4
        hx = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(nbuf)]
        hy = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(nbuf)]
        for t_ in hx:
            t_.copy_(x.cpu())
        k_e2e = max(4, min(args.steps, 12))
        # (a) one call per step: rtk_apply_A_host (H2D, matvec, D2H, synchronise)
        hxp, hyp = ctypes.c_void_p(hx[0].data_ptr()), ctypes.c_void_p(hy[0].data_ptr())
        for _ in range(2):
            _native.check(lib.rtk_apply_A_host(h.h, hxp, hyp, n, sptr))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            _native.check(lib.rtk_apply_A_host(h.h, hxp, hyp, n, sptr))
        el_seq = time.perf_counter() - t0
        # (b) batched public API: apply_A_batch overlaps the H2D of step k+1 with the D2H of step k
        xs = [hx[k % nbuf].numpy() for k in range(k_e2e)]
        ys = [hy[k % nbuf].numpy() for k in range(k_e2e)]
        P.apply_A_batch(problem, xs[:2], ys[:2])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.apply_A_batch(problem, xs, ys)
        el_b = time.perf_counter() - t0
        # ceiling: the same bytes moved H2D and D2H at once with no compute (pinned buffers)
        d_tmp = torch.empty_like(x)
        s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()

        def copies():
            with torch.cuda.stream(s_a):
                d_tmp.copy_(hx[0], non_blocking=True)
            with torch.cuda.stream(s_b):
                hy[0].copy_(y, non_blocking=True)

        copies()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(4):
            copies()
        torch.cuda.synchronize()
        ceiling = 4 / (time.perf_counter() - t0)
        del d_tmp
        e2e = {"value": world * k_e2e / el_b, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "copy_ceiling": world * ceiling,
               "copy_ceiling_note": "H2D + D2H of the same bytes at once, no compute: the PCIe bound of this metric",
               "path": "paper_2602_21958_b200.apply_A_batch -> rtk_apply_A_host_batch (pinned host buffers; "
                       "H2D of step k+1 overlaps D2H of step k)",
               "value_one_call_per_step": world * k_e2e / el_seq,
               "one_call_path": "rtk_apply_A_host (H2D + matvec + D2H, synchronous)"}
        # the drop-in call a reference user makes: apply_A(problem, numpy array), pageable
        # buffers staged through pinned chunks inside the library
        import time as _time
        xv = np.random.default_rng(1).standard_normal(n)
        P.apply_A(problem, xv)
        t0 = _time.perf_counter()
        for _ in range(3):
            P.apply_A(problem, xv)
        e2e["drop_in_numpy_apply_A_per_s"] = 3.0 / (_time.perf_counter() - t0)
        del xv
        del hx, hy, xs, ys

    extra = {}
    if rank == 0 and not args.no_gmres:
        extra["gmres"] = gmres_timings(torch)
        extra["gmres_cfg2_moment_layout"] = gmres_cfg2_moments(torch)
        extra["krylov_cfg2"] = krylov_cfg2(torch, problem, ms_per_step, hbm)
    if rank == 0 and not args.no_gmres:
        extra["formal_solvers_cfg2"] = formal_solver_timings(torch, lib, hbm)
    if rank == 0 and not args.no_lattice:
        extra["lattice"] = lattice_timings(torch)
        if not args.no_gmres:
            extra["gmres_lattice"] = lattice_gmres_timings(torch, cfg5=args.cfg5_gmres)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_port_timing(problem)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
        if not args.no_reference_as_shipped:
            cpu["reference_as_shipped"] = reference_as_shipped()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE cfg2 shapes)",
                "config": workload_config({"formal_solver": args.formal_solver}),
                "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                "gdof_per_s": value * n / 1e9, "gpu_launches": launches, "clocks": clk, "roofline": roofline,
                "kernels": kernels, "e2e": e2e, "cpu_baseline": cpu}
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_gmres_cfg1(p, b_host):
    """The reference GMRES algorithm (oracle restatement of R/krylov.py:56-158, numpy MGS) with the
    numpy oracle matvec on one host core: CPU time-to-1e-8 on cfg1 (the OpenMP C port is slower at
    this tiny size: thread start-up dominates a 50k-DOF matvec)."""
    from oracle import rt_oracle as ro

    d = ro.desc_from_problem(p)
    out = {}
    for name, restart in (("cfg1_gmres30", 30), ("cfg1_gmres_full", None)):
        t0 = time.perf_counter()
        rep = ro.gmres(lambda v: ro.apply_A(d, v), b_host, rel_tol=1e-8, max_iter=6000, restart=restart)
        out[name] = {"iterations": rep.iterations, "converged": rep.converged, "time_s": time.perf_counter() - t0,
                     "cores": 1, "kind": "port"}
    return out


def gmres_timings(torch):
    """Time-to-1e-8 of the device GMRES on cfg1 (restart 30 and unrestarted)."""
    import paper_2602_21958_b200 as P
    from paper_2602_21958_b200 import configs

    p = configs.slab_problem(1)
    b = P.build_rhs(p, device=True)
    out = {"cpu": cpu_gmres_cfg1(p, b.cpu().numpy())}
    # the fused CGS2 Arnoldi (north star) and the reference's own MGS (SolveConfig default)
    for orth in ("cgs2", None):
        tag = "" if orth == "cgs2" else "_mgs"
        for name, restart in (("cfg1_gmres30", 30), ("cfg1_gmres_full", None)):
            cfg = P.SolveConfig(rel_tol=1e-8, max_iter=6000, restart=restart, orthogonalization=orth)
            P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=5, restart=restart, orthogonalization=orth))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = P.gmres(p, b, cfg)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            out[name + tag] = {"iterations": rep.iterations, "converged": rep.converged, "time_s": el,
                               "true_residual": rep.true_residual, "matvecs": rep.matvecs,
                               "orthogonalization": orth or "mgs (reference default)"}
    return out


def gmres_cfg2_moments(torch):
    """cfg2 time-to-1e-8 in the moment layout (unknown u = R_w M I, 16 MB): unrestarted GMRES
    (basis of up to ~1500 x 16 MB in HBM), and the residual GMRES(30) reaches in 3000 iterations.
    The CPU reference cannot run this solve (about 3 s per matvec and an N-sized MGS basis)."""
    import paper_2602_21958_b200 as P
    from paper_2602_21958_b200 import configs

    p = configs.slab_problem(2, layout="moments")
    b = P.build_rhs(p, device=True)
    out = {}
    for name, restart, its in (("gmres30_3000", 30, 3000), ("gmres_unrestarted", None, 4000)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=its, restart=restart, orthogonalization="cgs2"))
        torch.cuda.synchronize()
        out[name] = {"iterations": rep.iterations, "converged": rep.converged, "time_s": time.perf_counter() - t0,
                     "true_residual": rep.true_residual, "matvecs": rep.matvecs, "unknowns": p.n_total,
                     "orthogonalization": "cgs2"}
    return out


def krylov_cfg2(torch, problem, matvec_ms, hbm):
    """30 GMRES(30) iterations on cfg2: per-iteration time and the CGS2 passes' achieved bandwidth."""
    import paper_2602_21958_b200 as P

    n = problem.n_total
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    cfg = P.SolveConfig(rel_tol=1e-30, max_iter=30, restart=30, orthogonalization="cgs2")
    P.gmres(problem, b, cfg)   # warm the memory pool
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(problem, b, cfg)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    its = rep.iterations
    orth_s = el - rep.matvecs * matvec_ms / 1e3
    # CGS2 + normalisation traffic per step j: 3(j+1) basis reads + 7 vector reads/writes
    orth_bytes = sum((3 * (j + 1) + 7) * 8 * n for j in range(its))
    return {"iterations": its, "matvecs": rep.matvecs, "time_s": el, "ms_per_iteration": el / its * 1e3,
            "orth_s": orth_s, "orth_algorithmic_bytes": orth_bytes,
            "orth_achieved_gbs": orth_bytes / orth_s / 1e9 if orth_s > 0 else None,
            "orth_frac_hbm": orth_bytes / orth_s / 1e9 / hbm if orth_s > 0 else None}


def formal_solver_timings(torch, lib, hbm):
    """cfg2 matvec with the exponential integrators (the north star's formal solver; the
    headline uses the reference's implicit Euler): matvec rate and the sweep's HBM fraction."""
    from paper_2602_21958_b200 import _device, _native, configs

    out = {}
    for fs in ("exp_linear", "exp_parabolic"):
        p = configs.slab_problem(2, formal_solver=fs)
        n = p.n_total
        h = p.device()
        x = torch.randn(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        sptr = _device.stream_ptr()
        for _ in range(3):
            _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        buf = (ctypes.c_float * 3)()
        sweep_ms = 0.0
        for _ in range(5):
            _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sptr, buf))
            sweep_ms += buf[2] / 5
        g = p.grid
        sweep_bytes = 16 * n + 8 * 2 * g.n_freq * g.n_space + 8 * g.n_space
        out[fs] = {"matvecs_per_s": 1e3 / ms, "ms_per_matvec": ms, "sweep_ms": sweep_ms,
                   "sweep_gbs": sweep_bytes / sweep_ms / 1e6, "sweep_frac_hbm": sweep_bytes / sweep_ms / 1e6 / hbm,
                   "kernel": "sweep1d_tma_kernel<EXP_*> (branch-free range-reduced weights in the chain warps)"}
        del p, x, y
        torch.cuda.empty_cache()
    return out


def lattice_gmres_timings(torch, cfg5=False):
    """GMRES time-to-1e-8 on the multi-D configurations that reach it within a bench run:
    cfg4 (moment layout) unrestarted; cfg3 in BOTH layouts -- intensity (2.75 GB vectors)
    GMRES(40), moment layout (129 MB vectors) unrestarted.  cfg5 GMRES(20) (BASELINE's
    restart) with --cfg5-gmres.  Arnoldi: the fused CGS2."""
    import paper_2602_21958_b200 as P
    from paper_2602_21958_b200 import configs

    runs = [(4, "moments", None, 600), (3, "intensity", 40, 1200), (3, "moments", None, 1500)]
    if cfg5:
        runs.append((5, "moments", 20, 2500))
    out = {}
    for cfg, layout, restart, its in runs:
        p = configs.lattice_config_problem(cfg, layout=layout)
        b = P.build_rhs(p, device=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=its, restart=restart, orthogonalization="cgs2"))
        torch.cuda.synchronize()
        key = f"cfg{cfg}" if layout == configs.LATTICE_CONFIGS[cfg]["layout"] else f"cfg{cfg}_{layout}"
        out[key] = {"restart": restart, "iterations": rep.iterations, "converged": bool(rep.converged),
                    "time_s": time.perf_counter() - t0, "true_residual": float(rep.true_residual),
                    "unknowns": p.n_total, "layout": layout, "orthogonalization": "cgs2"}
        del p, b, rep
        torch.cuda.empty_cache()
    return out


def lattice_timings(torch):
    """Matvec time of the multi-D configurations (cfg3 intensity layout, cfg4/5 moment layout)."""
    import paper_2602_21958_b200 as P
    from paper_2602_21958_b200 import lattice as L

    from paper_2602_21958_b200 import configs

    cfgs = {cfg: dict(configs.LATTICE_CONFIGS[cfg]) for cfg in (3, 4, 5)}
    out = {}

    def time_matvec(p):
        x = torch.randn(p.n_total, dtype=torch.float64, device="cuda")
        P.apply_A(p, x)
        torch.cuda.synchronize()
        reps = 2 if p.nz >= 128 else 4
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            P.apply_A(p, x)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for cfg, kw in cfgs.items():
        p = L.lattice_problem(seed=21958 + cfg, **kw)
        ms = time_matvec(p)
        if cfg == 3:   # cfg3 also in the moment layout (u = 129 MB instead of I = 2.75 GB)
            pm = L.lattice_problem(seed=21958 + cfg, **dict(kw, layout="moments"))
            ms_m = time_matvec(pm)
            del pm
            torch.cuda.empty_cache()
        dof = p.n_space * p.n_dirs * p.n_freq
        n_total = p.n_total
        del p
        torch.cuda.empty_cache()
        # hybrid characteristics (short for steep, long for grazing directions; TRIP)
        ph = L.lattice_problem(seed=21958 + cfg, characteristics="hybrid", **kw)
        ms_h = time_matvec(ph)
        del ph
        torch.cuda.empty_cache()
        out[f"cfg{cfg}"] = {"layout": kw["layout"], "unknowns": n_total, "dof": dof, "ms_per_matvec": ms,
                            "matvecs_per_s": 1e3 / ms, "gdof_per_s": dof / ms / 1e6,
                            "hybrid_characteristics": {"ms_per_matvec": ms_h, "gdof_per_s": dof / ms_h / 1e6}}
        if cfg == 3:
            out["cfg3"]["moment_layout"] = {"ms_per_matvec": ms_m, "gdof_per_s": dof / ms_m / 1e6}
        if cfg in (3, 4):   # the exponential integrators (cfg5 skipped to keep the default run short)
            fsd = {}
            for fs in ("exp_linear", "exp_parabolic"):
                pf = L.lattice_problem(seed=21958 + cfg, formal_solver=fs, **kw)
                ms_f = time_matvec(pf)
                del pf
                torch.cuda.empty_cache()
                fsd[fs] = {"ms_per_matvec": ms_f, "gdof_per_s": dof / ms_f / 1e6}
            out[f"cfg{cfg}"]["formal_solvers"] = fsd
        # the multi-D sweeps are bound by the FP64 pipe / latency, not HBM -- report the
        # transfer kernel's FP64-pipe utilisation from the committed ncu capture of this config
        src = profile_path(f"ncu_lattice_cfg{cfg}.txt")
        raw = ncu_raw(src)
        key = "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
        if key in raw:
            out[f"cfg{cfg}"]["transfer_kernel_fp64_pipe_frac"] = float(raw[key].rstrip("%")) / 100
            out[f"cfg{cfg}"]["fp64_source"] = f"{os.path.relpath(src, ROOT)} (ncu --set full, one launch)"
    return out


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: run this same command line under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous) and return its
    exit code.  BENCH_BACKEND=gloo lets the CPU tests drive the multi-rank path."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    if "--ref-shipped-child" in sys.argv:
        _ref_shipped_child()
        return
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "sharded" and world > 1:
        run_sharded(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
