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
TRAFFIC_FILE = ROOT / "profiles" / "r01" / "ncu_traffic.json"


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
_BLOCKS = {}


def cpu_sample(m: int, k_sample: int, ham=None) -> dict:
    """Time the oracle's H-application (the reference's 86 %-of-wall kernel, 4 zgemm) on
    k_sample columns at the full m, on the host cores (OpenBLAS threads = all)."""
    from oracle import bse_oracle as o

    if ham is not None:
        a, b = ham.host_blocks()
    else:  # reference arm without a GPU-built input: same-shaped blocks (zgemm time is data independent)
        if m not in _BLOCKS:
            z = o.gauss_c(12345, m * m)
            a = np.asfortranarray(z.reshape(m, m))
            _BLOCKS[m] = (a, a)
        a, b = _BLOCKS[m]
    x = o.gauss_c_matrix(o.child_seed(0, 3), 2 * m, k_sample)
    o.h_times(a[:64, :64], b[:64, :64], x[:128, :2])  # warm BLAS
    t0 = time.perf_counter()
    o.h_times(a, b, x)
    dt = time.perf_counter() - t0
    flops = 8.0 * (2 * m) ** 2 * k_sample
    return {"seconds": dt, "flops": flops, "gflops": flops / dt / 1e9}


def expected_solve_flops(cfg_name: str, nevex: int, m: int, deg: int) -> tuple[float, str]:
    p = Path(str(TRACE_FILE).format(cfg=cfg_name))
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["total_model_flops"]), f"modeled flops of our {cfg_name} solve trace ({p.name})"
    n = 2 * m
    sum_k = 6.9 * nevex  # measured Sigma k / nevex at the C2 shape
    return (deg + 2) * 8.0 * n * n * sum_k, "model (deg+2) 8 n^2 Sigma k, Sigma k = 6.9 nevex (SURVEY 6.4)"


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    if rank != 0:
        return
    m, nev, nex, deg, tol, rel = CONFIGS[args.config]
    nevex = nev + nex
    k_sample = 16 if m >= 10000 else 64
    total, how = expected_solve_flops(args.config, nevex, m, deg)
    times = []
    for i in range(args.warmup + args.steps):
        s = cpu_sample(m, k_sample)
        if i >= args.warmup:
            times.append(total / (s["flops"] / s["seconds"]))
    val = statistics.median(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": config_dict(args.config),
        "cpu_baseline": {"value": val, "unit": "s", "cores": cores(), "kind": "port",
                         "sample": f"oracle H-application (4 OpenBLAS zgemm) at m={m} on {k_sample} columns per step, "
                                   f"extrapolated to the solve's total modeled flops ({how})"},
        "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    ham = bse.generate(bse.GeneratorSpec(m=m, seed=0, coupling_ratio=COUPLING.get(args.config, 0.5)), device=dev)
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
        from paper_2601_10557_b200.dist import DistributedSolver

        ds = DistributedSolver(ham, device=dev)
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
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        results = [one_solve() for _ in range(args.steps)]
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    launches = ctx.launches - launches0
    step_s = e0.elapsed_time(e1) / 1e3 / args.steps
    step_s = max_over_ranks(step_s, world)
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
        pieces = ds.tile_pieces_host()
        for name in ("fwd", "trn"):  # user inputs staged in pinned host memory
            pieces[name] = tuple(pinned_fortran(x) for x in pieces[name])
        h2d = world * sum(x.nbytes for name in ("fwd", "trn") for x in pieces[name]) + world * (n // world) * cfg.nevex * 16
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
    achieved = ffl / (fms / 1e3) / 1e12 if fms > 0 else None
    algo = _lib.filter_algorithm() if _lib.filter_precision() == "c128" else "c64-3xtf32-tcgen05"
    if algo.startswith("rs") and (ham.flags & 1 or (world > 1 and ds.fwd.g is None)):
        algo = "3m"  # B = 0 (or tiles without room for the planes) runs the 3M kernel
    exec_ratio = 0.75 if algo.startswith("3m") else 1.0  # 3M: 6 real DMMA per complex block pair instead of 8
    if algo.startswith("rs"):
        exec_ratio = 0.5  # real split: 4 n^2 k DMMA flops per step (csrc/hop_rs.cuh)
    if algo.startswith("c64"):
        peak, peak_src = 1177.7, ("dense tf32 tcgen05 peak as ncu reports it at 1965 MHz (sm__ops_path_tensor_op_utchmma_"
                                  "src_tf32 peak); measured probe GEMMs: 433 TF/s (1 CTA), 663 TF/s (CTA pair)")
        exec_ratio = 3.0  # 3 TF32 MMAs per real product
    if ham.flags & 1 and achieved:  # B = 0: the B half is skipped, count 4 n^2 k
        achieved *= 0.5
    total_model = res.ledger.total_flops()
    if rank == 0 and args.config != "c1" and world == 1:
        TRACE_FILE.parent.mkdir(exist_ok=True)
        Path(str(TRACE_FILE).format(cfg=args.config)).write_text(json.dumps({
            "total_model_flops": total_model, "iterations": res.iterations_used, "converged": res.converged,
            "trace": [[t.it, t.locked, t.k, t.max_res, t.mu_nevex, t.flops] for t in res.trace],
            "ledger_seconds": res.ledger.seconds, "ledger_flops": res.ledger.flops}, indent=1) + "\n")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        k_sample = 16 if m >= 10000 else 64
        s = cpu_sample(m, k_sample, ham)
        cpu = {"value": total_model / (s["flops"] / s["seconds"]), "unit": "s", "cores": cores(), "kind": "port",
               "sample": f"oracle H-application (4 OpenBLAS zgemm, {s['gflops']:.0f} GF/s) at m={m} on {k_sample} "
                         f"columns, extrapolated to this solve's {total_model:.3e} modeled flops"}
    if rank == 0:
        cfgd = config_dict(args.config)
        if world > 1:
            from paper_2601_10557_b200.dist import grid_shape

            p, q = grid_shape(world)
            cfgd["parallelism"] = f"2D block grid {p}x{q} (A/B tiles + block transposes per GPU), NCCL row/col allreduce"
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
                         "algorithmic": "8 n^2 k flops per filter step (bsesolve metrics model, BASELINE.md §3.5) "
                                        "per GPU, summed over the solve's filter calls / CUDA-event (1 GPU) or "
                                        "synchronised (N GPUs) time of those calls; with the 3M filter the DMMA pipe "
                                        "executes 6 n^2 k, with the real-split filter 4 n^2 k (filter_executed_*)"},
            "filter_tflops_per_gpu": achieved, "filter_frac_of_fp64_peak": (achieved / peak) if achieved else None,
            "filter_algorithm": algo,
            "filter_executed_tflops_per_gpu": achieved * exec_ratio if achieved else None,
            "filter_executed_frac_of_fp64_peak": achieved * exec_ratio / peak if achieved else None,
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
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


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
