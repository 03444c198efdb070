"""Benchmark: time-to-solution of the pseudo-hermitian ChASE solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c1] [--impl ours|reference]

A "step" is one complete solve (Lanczos bounds -> filtered subspace iteration
until nev pairs lock) of the BASELINE.json configuration the metric is quoted
on: n = 40k (m = 20,000) complex128, nev = 1000, nex = 200, deg = 20,
tol = 1e-10 relative (SolverConfig(rel_res=True); the reference's absolute
1e-10 is below the FP64 residual floor at this n).
Synthetic input built on the GPU with the reference construction
(generate.py:60-83).  The inputs (A|B = 12.8 GB) exceed L2 (126 MB), so no
L2 flush is needed between steps.

value            device-resident time-to-solution (s), max over ranks
e2e              same solve through the public drop-in API with HOST numpy blocks:
                 H2D of A, B and the start block and D2H of the nev vectors inside the timed region
roofline         the filter kernel (fused H-operator DMMA GEMM) vs the measured FP64 DMMA peak
cpu_baseline     the CPU oracle (numpy/OpenBLAS restatement of the reference) on a bounded sample
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (m, nev, nex, deg, tol, rel_res)
    "c1": (500, 50, 20, 20, 1e-10, False),
    "c2": (10000, 500, 100, 20, 1e-10, True),
    "c3": (20000, 1000, 200, 20, 1e-10, True),
    "c3b0": (20000, 1000, 200, 20, 1e-10, True),  # configs[4]: C3 with B = 0 (coupling_ratio 0)
    "c4": (50000, 3000, 500, 20, 1e-10, True),    # configs[3]: n = 100k (8 GPUs in BASELINE.json)
    "c3c64": (20000, 1000, 200, 20, 1e-5, True),  # configs[4]: C3 with the complex64 (tcgen05) filter,
                                                  # c64 policy rel tol 1e-5
    "c3mixed": (20000, 1000, 200, 20, 1e-10, True),  # C3, mixed-precision filter policy (early iterations
}                                                    # c64 on tcgen05, FP64 from 1e-4 |mu_1| residuals on)
MIXED = {"c3mixed"}
PRECISION = {"c3c64": "c64"}
COUPLING = {"c3b0": 0.0}
METRIC = "time-to-solution, nev eigenpairs @ n=40k; filter FP64 TFLOP/s as % of peak"
FP64_PEAK_FILE = ROOT / "profiles" / "fp64_peak.json"
TRAFFIC_FILE = ROOT / "profiles" / "r02" / "ncu_traffic.json"


def ncu_traffic(algo: str):
    """DRAM bytes per launch of the filter kernel at k = 1200 from the committed ncu capture."""
    try:
        d = json.loads(TRAFFIC_FILE.read_text())
        key = "c64" if algo.startswith("c64") else algo
        if key not in d:
            return None, None
        return d[key]["bytes"], f"ncu --set full, {d[key]['kernel']} at k={d[key]['k']} ({TRAFFIC_FILE.name})"
    except Exception:
        return None, None
# expected modeled flops of one C3 solve (from our own trace, profiles/); used by the CPU arm
TRACE_FILE = ROOT / "profiles" / "solve_trace_{cfg}.json"


def pinned_fortran(x: np.ndarray) -> np.ndarray:
    """F-ordered copy of x in page-locked host memory (the e2e contract's pinned inputs)."""
    import torch

    t = torch.empty((x.shape[1], x.shape[0]), dtype=torch.complex128, pin_memory=True)
    out = t.numpy().T
    out[...] = x
    return out


def fp64_peak() -> tuple[float, str]:
    try:
        d = json.loads(FP64_PEAK_FILE.read_text())
        return float(d["dmma_tflops"]), "measured DMMA.8x8x4 peak (profiles/fp64_peak.json)"
    except Exception:
        return 37.2, "nominal 148 SM x 64 FP64 FMA/clk x 1.965 GHz"


class ClockSampler:
    """SM clocks and throttle reasons sampled in-process through NVML during the timed region
    (an nvidia-smi subprocess per sample stalls the solver's synchronous CUDA calls)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int, period: float = 0.5):
        self.index, self.period = index, period
        self.sm, self.mx, self.reasons, self.power = [], [], set(), []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.h = None
        try:
            import pynvml as nv
            import torch

            nv.nvmlInit()
            self.nv = nv
            try:
                props = torch.cuda.get_device_properties(index)
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.h = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mx.append(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons |= {name for bit, name in self.REASONS.items() if bits & bit}
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.h is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t.is_alive():
            self._t.join(timeout=15)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "power_w_max": max(self.power) if self.power else None,
                "source": "NVML (in-process)"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL communicator init lines (rank count, transports): NCCL_DEBUG=INFO / SUBSYS=INIT into
        # per-process files, which rank 0 echoes to stderr (nccl_init_lines) so stdout carries only the
        # JSON line; an image default of NCCL_DEBUG=VERSION is raised
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", str(NCCL_LOG_DIR / "nccl_init.%h.%p.log"))
        NCCL_LOG_DIR.mkdir(parents=True, exist_ok=True)
        if os.environ.get("BSE200_DIST_BACKEND", "nccl") == "gloo":
            # test only: more ranks than GPUs (the 2 x 4 grid of an 8-GPU box on 4 GPUs); not a bench number
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU arms
CACHE = ROOT / ".bench_cache"
NCCL_LOG_DIR = ROOT / ".bench_cache" / "nccl" / (os.environ.get("TORCHELASTIC_RUN_ID", "")
                                                  + "-" + os.environ.get("MASTER_PORT", ""))


def nccl_init_lines(world: int) -> dict | None:
    """The NCCL communicator init lines of this run's ranks (NCCL_DEBUG_FILE), echoed to stderr."""
    if world == 1:
        return None
    lines = []
    for p in sorted(NCCL_LOG_DIR.glob("nccl_init.*.log")):
        lines += [ln.rstrip() for ln in p.read_text(errors="replace").splitlines()
                  if "Init COMPLETE" in ln or " nRanks " in ln]
    for ln in lines:
        print(ln, file=sys.stderr)
    ranks = sorted({int(x) for ln in lines for x in __import__("re").findall(r"nranks (\d+)", ln)})
    return {"comm_sizes_seen": ranks, "init_complete_lines": sum("Init COMPLETE" in ln for ln in lines)}


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def solve_trace(cfg_name: str):
    from oracle import cpu_model

    return cpu_model.reference_trace(ROOT / "tests" / "golden" / f"large_{cfg_name}.npz",
                                     Path(str(TRACE_FILE).format(cfg=cfg_name)))


def cpu_reference_time(cfg_name: str, blocks=None, quick: bool = False, samples: int = 0):
    """Reference CPU time-to-solution from timed reference-path phases (oracle/cpu_model.py):
    every phase of the reference code path timed at the full n and the solve's own widths on this
    host's cores (median of 3), the solve's per-iteration (k, l) applied to those timings;
    ``samples`` further per-step samples of the H application rescale the filter rate (median
    reported).  ``quick`` (our arm's cpu_baseline leg): the reference arm's cached calibration on
    this host when present, else the same calibration (~3 min at C3 on 16 cores)."""
    from oracle import cpu_model

    m, nev, nex, deg, tol, rel = CONFIGS[cfg_name]
    nevex = nev + nex
    tr = solve_trace(cfg_name)
    if tr is None:
        return None
    tk, tl, lsteps, tsrc = tr
    host = f"{cores()}c"
    cache = CACHE / f"cpu_calibration_{cfg_name}_{host}.json"
    cal = None
    if quick and cache.exists():
        cal = json.loads(cache.read_text())
    t0 = time.perf_counter()
    if blocks is None:
        blocks = cpu_model.timing_instance(m)
    a, b = blocks
    if cal is None:
        # the same calibration as the reference arm (the solve's own widths, medians of 3)
        cal = cpu_model.calibrate(a, b, nevex, max(min(tk), 32), nev)
        cal["sample_k"] = 64
        cal["sample_s"] = cpu_model.sample_step(a, b, 64)
        cal["quick"] = quick
        if not quick:
            CACHE.mkdir(exist_ok=True)
            cache.write_text(json.dumps(cal, indent=1) + "\n")
        cal["source"] = "timed here"
    else:
        cal["source"] = f"timed by this host's --impl reference run ({cache.name})"
    vals = []
    for _ in range(samples):
        sc = cpu_model.sample_step(a, b, cal["sample_k"]) / cal["sample_s"]
        vals.append(cpu_model.model(cal, tk, tl, deg, lsteps, step_scale=sc, nevex=nevex))
    base = cpu_model.model(cal, tk, tl, deg, lsteps, nevex=nevex)
    tot = [v["total"] for v in vals] or [base["total"]]
    return {"value": statistics.median(tot), "phases": {k: round(v, 2) for k, v in base.items()},
            "per_step": [round(x, 2) for x in tot], "calibration": cal, "trace_source": tsrc,
            "wall_s": time.perf_counter() - t0,
            "sample": (f"reference code path (oracle restatement: numpy temporaries + OpenBLAS/LAPACK, "
                       f"{cores()} threads) timed phase by phase at n={2 * m}: filter step at k={cal['k_lo']} "
                       f"and {cal['k_hi']}, Householder QR of S Y_locked at l={cal['l_hi']}, CholQR2 and "
                       f"hermitian RR at both k, residuals, Lanczos step ({cal['source']}); evaluated over "
                       f"the {len(tk)} iterations of the {tsrc}")}


def run_reference(args, world, rank):
    if rank != 0:
        return
    r = cpu_reference_time(args.config, samples=args.warmup + args.steps)
    val = statistics.median(r["per_step"][args.warmup:]) if r is not None else None
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": val * 1e3 if val else None, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": config_dict(args.config),
        "cpu_baseline": {"value": val, "unit": "s", "cores": cores(), "kind": "port",
                         "sample": r["sample"] if r else "no solve trace"},
        "cpu_phases_s": r["phases"] if r else None,
        "cpu_calibration": r["calibration"] if r else None,
        "cpu_model_check": model_check_summary(),
        "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def model_check_summary():
    """The CPU model against measured full solves (profiles/r02/cpu_model_check_*.json)."""
    out = {}
    for p in sorted((ROOT / "profiles" / "r02").glob("cpu_model_check_*.json")):
        try:
            d = json.loads(p.read_text())
            out[p.stem] = {k: d.get(k) for k in ("measured_s", "model_s", "ratio", "cores", "where")}
        except Exception:
            pass
    return out or None


def config_dict(name):
    m, nev, nex, deg, tol, rel = CONFIGS[name]
    cpl = COUPLING.get(name, 0.5)
    return {"workload": f"{name}: synthetic definite BSE H, n={2 * m} complex128, nev={nev}, nex={nex}, deg={deg}, "
                        f"tol={tol:g} {'relative' if rel else 'absolute'}, coupling_ratio={cpl}",
            "n": 2 * m, "nev": nev, "nex": nex, "deg": deg, "tol": tol, "rel_res": rel,
            "l2_flush": "inputs (A|B 32m^2 B) larger than L2", "parallelism": "1 GPU"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    import torch

    import paper_2601_10557_b200 as bse
    from paper_2601_10557_b200 import _lib
    from paper_2601_10557_b200.hamiltonian import BseHamiltonian, Definiteness

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    bse.set_filter_precision(PRECISION.get(args.config, "c128"))
    bse.set_mixed_precision(args.config in MIXED)
    m, nev, nex, deg, tol, rel = CONFIGS[args.config]
    n = 2 * m
    t0 = time.perf_counter()
    spec = bse.GeneratorSpec(m=m, seed=0, coupling_ratio=COUPLING.get(args.config, 0.5))
    if world == 1 or os.environ.get("BSE200_DIST_BACKEND", "nccl") == "gloo":
        ham = bse.generate(spec, device=dev)
    else:
        # rank 0 builds the instance (host rng, device GEMM / eigensolvers) and broadcasts [A|B] over
        # NVLink: the other ranks neither redraw 2 m^2 host normals nor rerun the eigensolvers
        import torch.distributed as tdist

        from paper_2601_10557_b200.hamiltonian import colmajor_empty

        if rank == 0:
            ham = bse.generate(spec, device=dev)
            ab = ham.device_blocks(dev)
        else:
            ab = colmajor_empty(m, 2 * m, dev)
        tdist.broadcast(torch.view_as_real(ab.T), src=0)  # (2m, m) storage: contiguous
        if rank != 0:
            ham = BseHamiltonian.from_device(ab, Definiteness.DEFINITE)  # rank 0 ran the certificate
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    cfg = bse.SolverConfig(nev=nev, nex=nex, deg=deg, tol=tol, seed=0, rel_res=rel)
    ctx = _lib.Context.get(local)

    filt = {"ms": 0.0, "flops": 0.0}
    if world == 1:
        # filter-kernel timing: CUDA events around every filter call (same stream as the kernels)
        import paper_2601_10557_b200.solver as solver_mod

        events = []
        orig = solver_mod.filter_inplace

        def timed_filter(ham_, v, fcfg, work=None, ledger=None):
            prec = _lib.filter_precision()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = orig(ham_, v, fcfg, work, ledger)
            e1.record()
            events.append((e0, e1, fcfg.degree * 8.0 * n * n * v.shape[1], prec))
            return out

        solver_mod.filter_inplace = timed_filter

        def one_solve():
            return bse.solve(ham, cfg, device=dev, keep_on_device=True)

        def filter_stats():
            # the roofline is the dominant kernel's: FP64 filter launches only, unless the run is all c64
            sel = [e for e in events if e[3] == "c128"] or events
            return sum(a.elapsed_time(b) for a, b, _, _ in sel), sum(f for _, _, f, _ in sel)
    else:
        from paper_2601_10557_b200.dist import DistributedSolver, tile_blocks_host

        ds = DistributedSolver(ham, device=dev)
        pieces = None if args.no_e2e else tile_blocks_host(ds.grid, ham)  # this rank's tile, for the e2e leg
        ham.release_device()
        ham._dev.clear()
        torch.cuda.empty_cache()
        events = []

        def one_solve():
            r = ds.solve(cfg)
            events.append((r.ledger.seconds["filter"] * 1e3, r.ledger.flops["filter"] / world))
            return r

        def filter_stats():
            return sum(e[0] for e in events), sum(e[1] for e in events)

    for _ in range(args.warmup):
        one_solve()
    events.clear()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    profile_range = os.environ.get("BSE200_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if profile_range:
            torch.cuda.profiler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        results = [one_solve() for _ in range(args.steps)]
        e1.record()
        torch.cuda.synchronize()
        if profile_range:
            torch.cuda.profiler.stop()
        barrier(world)
    launches = ctx.launches - launches0
    step_s = e0.elapsed_time(e1) / 1e3 / args.steps
    step_s = max_over_ranks(step_s, world)
    # device memory: this rank's operator storage and the peak allocation of the timed solves
    op_bytes = ds.operator_bytes() if world > 1 else None
    peak_gb = max_over_ranks(torch.cuda.max_memory_allocated(dev) / 1e9, world)
    fms, ffl = filter_stats()
    res = results[-1]
    if world == 1:
        solver_mod.filter_inplace = orig

    # end to end through the public API with HOST buffers: upload inside the timed region
    if args.no_e2e:
        r_e2e, e2e_s, h2d, d2h = res, None, 0, 0
    elif world == 1:
        a_h, b_h = (pinned_fortran(x) for x in ham.host_blocks())  # user inputs staged in pinned host memory
        host_ham = BseHamiltonian(a_h, b_h, Definiteness.DEFINITE)  # definiteness certified by the generator
        h2d = 2 * m * m * 16 + n * cfg.nevex * 16 + 8 * n * 16
    else:
        pieces["fwd"] = tuple(pinned_fortran(x) for x in pieces["fwd"])  # user inputs staged in pinned memory
        # every rank uploads its own tile of A and B (bytes summed over ranks) and its start-block rows
        h2d = world * sum(x.nbytes for x in pieces["fwd"]) + world * 2 * ds.grid.nc * cfg.nevex * 16
    if not args.no_e2e:
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            r_e2e = bse.solve(host_ham, cfg, device=dev)  # returns numpy v
            v_host = r_e2e.v
        else:
            ds.load(pieces)
            r_e2e = ds.solve(cfg)
            v_host = r_e2e.v.T.contiguous().cpu().numpy().T if rank == 0 else None
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world)
        d2h = n * nev * 16 + 8 * (cfg.nevex + 64)
        if world == 1:
            host_ham.release_device()

    peak, peak_src = fp64_peak()
    model_rate = ffl / (fms / 1e3) / 1e12 if fms > 0 else None  # reference model flops (8 n^2 k per step)
    algo = _lib.filter_algorithm() if _lib.filter_precision() == "c128" else "c64-3xtf32-tcgen05"
    if algo.startswith("rs") and (ham.flags & 1 or (world > 1 and not ds.planes)):
        algo = "3m"  # B = 0 (or tiles without room for the planes) runs the 3M kernel
    exec_ratio = 0.75 if algo.startswith("3m") else 1.0  # 3M: 6 real DMMA per complex block pair instead of 8
    if algo.startswith("rs"):
        exec_ratio = 0.5  # real split: 4 n^2 k DMMA flops per step (csrc/hop_rs.cuh)
    if algo.startswith("c64"):
        peak, peak_src = 1177.7, ("dense tf32 tcgen05 peak as ncu reports it at 1965 MHz (sm__ops_path_tensor_op_utchmma_"
                                  "src_tf32 peak); measured probe GEMMs: 433 TF/s (1 CTA), 663 TF/s (CTA pair)")
        exec_ratio = 3.0  # 3 TF32 MMAs per real product
    if ham.flags & 1 and model_rate:  # B = 0: the B half is skipped, count 4 n^2 k
        model_rate *= 0.5
    achieved = model_rate * exec_ratio if model_rate else None  # flops the tensor pipe executes
    total_model = res.ledger.total_flops()
    if rank == 0 and args.config != "c1" and world == 1:
        TRACE_FILE.parent.mkdir(exist_ok=True)
        Path(str(TRACE_FILE).format(cfg=args.config)).write_text(json.dumps({
            "total_model_flops": total_model, "iterations": res.iterations_used, "converged": res.converged,
            "lanczos_steps": res.bounds.steps,
            "trace": [[t.it, t.locked, t.k, t.max_res, t.mu_nevex, t.flops] for t in res.trace],
            "ledger_seconds": res.ledger.seconds, "ledger_flops": res.ledger.flops}, indent=1) + "\n")

    parity = parity_vs_reference(args.config, res) if rank == 0 else None
    defin = None
    if rank == 0 and world == 1 and not args.no_e2e and m <= 20000:
        defin = time_is_definite(ham, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_reference_time(args.config, blocks=ham.host_blocks(), quick=True)
        if r is not None:
            cpu = {"value": r["value"], "unit": "s", "cores": cores(), "kind": "port", "sample": r["sample"],
                   "phases_s": r["phases"]}
    if rank == 0:
        cfgd = config_dict(args.config)
        if world > 1:
            from paper_2601_10557_b200.dist import grid_shape

            p, q = grid_shape(world)
            backend = os.environ.get("BSE200_DIST_BACKEND", "nccl")
            cfgd["parallelism"] = (f"2D block grid {p}x{q} (one tile of real-split planes per GPU), "
                                   f"{'NCCL' if backend == 'nccl' else backend + ' (functional test mode)'} "
                                   f"row/col allreduce")
        line = {
            "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (GPU generator, reference construction)",
            "config": cfgd,
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches // args.steps,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic(algo)[0],
                         "traffic_source": ncu_traffic(algo)[1],
                         "kernel": ("bse::c64::step_kernel (tcgen05 3xTF32 complex64 filter step)" if algo.startswith("c64")
                                    else "bse::hop3m_tma_kernel (fused H-operator 3M DMMA GEMM, TMA-fed by a producer warp, mbarrier rings, Chebyshev epilogue)"
                                    if algo == "3m" else
                                    "bse::hop_rs_tma_kernel (real-split H operator: folded block, four real planes, 4 n^2 k DMMA flops per step, TMA-fed by a producer warp, Chebyshev epilogue)"
                                    if algo.startswith("rs") else "bse::hop_kernel (fused H-operator DMMA GEMM + Chebyshev epilogue)"),
                         "peak_source": peak_src,
                         "algorithmic": ("EXECUTED tensor-pipe flops per filter step: 4 n^2 k with the real-split "
                                         "kernel (6 n^2 k 3M, 8 n^2 k 4M; DESIGN.md §Roofline), summed over the "
                                         "solve's filter calls / their CUDA-event time on the launching stream "
                                         "(1 GPU) or synchronised time (N GPUs)")},
            "filter_tflops_model": model_rate,
            "filter_model_note": "reference model 8 n^2 k flops per step (metrics.py:11-39) / filter time; exceeds "
                                 "the FP64 peak because the real-split kernel executes half of it",
            "filter_algorithm": algo,
            "solve": {"iterations": res.iterations_used, "converged": res.converged,
                      "ledger_seconds": {k: round(v, 4) for k, v in res.ledger.seconds.items()},
                      "model_tflop": total_model / 1e12, "generator_s": round(gen_s, 2),
                      "lambda_1": float(res.lambdas[0]), "lambda_nev": float(res.lambdas[-1]),
                      "max_residual": float(res.residual_norms.max()),
                      "locked_per_iter": [t.locked for t in res.trace],
                      "filter_precision_per_iter": getattr(res, "filter_precisions", None),
                      "phase_events_s": [[ph, round(dt, 4)] for ph, dt in res.ledger.events],
                      "e2e_iterations": r_e2e.iterations_used,
                      "e2e_max_dlambda_rel": float(np.max(np.abs(r_e2e.lambdas - res.lambdas) / np.abs(res.lambdas)))},
            "parity_vs_reference": parity,
            "is_definite": defin,
            "nccl": nccl_init_lines(world),
            "memory": {"operator_gb_per_gpu": round(op_bytes / 1e9, 3) if op_bytes else None,
                       "peak_allocated_gb_max_over_ranks": round(peak_gb, 2),
                       "note": "operator = one tile's real-split planes, 32 m^2/(p q) bytes (N > 1); "
                               "peak includes the generator's full instance on each rank"},
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def parity_vs_reference(cfg_name, res):
    """The solve against the REFERENCE's own result at this config (tests/golden/large_<cfg>.npz,
    made by oracle/make_golden_large.py from bsesolve.solve on the reference instance)."""
    p = ROOT / "tests" / "golden" / f"large_{cfg_name}.npz"
    if cfg_name not in ("c2", "c3") or not p.exists():
        return None
    g = np.load(p, allow_pickle=False)
    ref = g["lambdas"]
    same_it = res.iterations_used == int(g["iterations_used"])
    v = res.v if isinstance(res.v, np.ndarray) else None
    out = {"golden": p.name, "max_dlambda_rel": float(np.max(np.abs(res.lambdas - ref) / np.abs(ref))),
           "iterations": res.iterations_used, "iterations_ref": int(g["iterations_used"]),
           "trace_locked_equal": same_it and [t.locked for t in res.trace] == [int(x) for x in g["trace_locked"]],
           "trace_k_equal": same_it and [t.k for t in res.trace] == [int(x) for x in g["trace_k"]],
           "max_residual_over_tol": float(res.residual_norms.max() / (float(g["tol"]) * abs(res.bounds.mu_1))),
           "mu_1_rel": float(abs(res.bounds.mu_1 - float(g["mu_1"])) / abs(float(g["mu_1"]))),
           "reference_solve_s": float(g["solve_seconds"]),
           "reference_host": json.loads(str(g["host_json"]))}
    if v is None:
        v = res.v[:, :4].T.contiguous().cpu().numpy().T
        v2 = res.v[:, -4:].T.contiguous().cpu().numpy().T
    else:
        v, v2 = v[:, :4], v[:, -4:]
    ov = np.concatenate([np.abs(np.einsum("ij,ij->j", g["v_first4"].conj(), v)),
                         np.abs(np.einsum("ij,ij->j", g["v_last4"].conj(), v2))])
    out["ritz_vector_overlap_min"] = float(ov.min())
    out["pass"] = bool(out["max_dlambda_rel"] <= 1e-10 and abs(out["iterations"] - out["iterations_ref"]) <= 1
                       and out["max_residual_over_tol"] <= 1.0 and out["ritz_vector_overlap_min"] >= 1 - 1e-8)
    return out


def time_is_definite(ham, dev):
    """The definiteness check a host-supplied input pays (solver.py:128 -> hamiltonian.py:208-218):
    upload of A, B plus the device Cholesky of the n x n S H, timed on its own (the generated input
    skips it as the reference's generate() does, generate.py:77)."""
    import torch

    import paper_2601_10557_b200 as bse
    from paper_2601_10557_b200.hamiltonian import BseHamiltonian

    a_h, b_h = (pinned_fortran(x) for x in ham.host_blocks())
    h = BseHamiltonian(a_h, b_h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.device(dev):
        out = bse.is_definite(h)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h.release_device()
    return {"seconds": round(dt, 3), "outcome": out.name,
            "what": "H2D of A, B + device Cholesky of S H (16 n^2 bytes) -- not in value/e2e, like the "
                    "reference's generate()-cached check"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end solve (long demo runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        # CPU arm: rank 0 alone works; the other ranks exit at once (no process group needed)
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
