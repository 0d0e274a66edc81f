"""Benchmark: GMRES-IR time-to-1e-10 on north_star's config C4 (Laplace3D
200^3, 8M rows, restart 50, fp32 inner / fp64 outer) by default, with the
fp64 GMRES time (the paper's IR speedup), per-kernel HBM roofline and the
reference CPU path (oracle port) beside it.  --config C2 gives the BentPipe2D
1500^2 headline of BASELINE.json's single-GPU config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4|C1|C2|C3|C5] [--no-fp64] [--no-cpu]

A step = one full solve (b = ones, x0 = 0, m = 50, rtol 1e-10) with inputs
resident in HBM (value), timed with per-kernel profiling OFF; a separate
profiled solve gives the per-kernel CUDA-event times for the roofline.  e2e
repeats the solve through the public API with host (pinned) b/x0 and the
solution copied back.  Working set (Krylov basis 1.6 GB fp32 at C4, 459 MB at
C2) exceeds the 126 MB L2, so no explicit flush.
N > 1 (torchrun): the same system row-partitioned across the ranks
(paper_2105_07544_b200.distributed: P2P halo stores and in-kernel cross-GPU
reductions inside each rank's persistent cycle kernel), strong scaling, max
over ranks.  MPK_SHARE_GPU=1 puts every rank on GPU 0 (gloo host
collectives) to exercise the multi-process IPC path on a one-GPU box.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": ("Laplace3D", 40, "Laplace3D 7-point 40^3 (64k rows)"),
    "C2": ("BentPipe2D", 1500, "BentPipe2D convection-diffusion 1500^2 (2.25M rows)"),
    "C3": ("UniFlow2D", 2500, "UniFlow2D convection-diffusion 2500^2 (6.25M rows)"),
    "C4": ("Laplace3D", 200, "Laplace3D 7-point 200^3 (8M rows)"),
    "C5": ("synthetic", 4000000, "synthetic irregular nonsymmetric CSR, 4M rows, ~49 nnz/row, + Jacobi(1)"),
}
# C5 family calibrated so that fp64 GMRES(50)+J1 needs hundreds of
# iterations (SURVEY 8(d) warning: the default family converges in 18)
C5_PARAMS = dict(signs="negative", dominance=1.001, shift=1e-3, far_frac=0.01, band=2000)
# reference (mpkrylov) iteration counts on these configs (tests/golden/runs.json)
# C4 IR runs under breakdown rule "u"; its count is the paper's
# Trilinos count, equal to this solver's and the oracle's
REF_ITERS = {"C1": {"ir": 200, "fp64": 206}, "C2": {"ir": 10650, "fp64": 10833},
             "C3": {"ir": None, "fp64": None}, "C4": {"ir": 4100, "fp64": 4053},
             "C5": {"ir": None, "fp64": None}}


def breakdown_rule(cfg_name):
    """the reference's beta <= n*u*||w|| test (n*u32 = 0.24 at 4M,
    0.37 at 6.25M, 0.48 at 8M rows) declares false breakdowns on C3-C5; they
    run with "u" (in both arms)."""
    return "u" if cfg_name in ("C3", "C4", "C5") else "n_u"


def shared_config(args):
    """The workload description both arms print verbatim (same_config)."""
    preset, nx, desc = CONFIGS[args.config]
    basis = 51 * (nx if args.config == "C5" else nx ** (3 if preset == "Laplace3D" else 2)) * 4
    cfg = {"workload": "%s, GMRES-IR restart 50, rtol 1e-10, b = ones, x0 = 0" % desc,
           "config": args.config, "solver": "gmres-ir", "m": 50, "rtol": 1e-10,
           "breakdown_rule": breakdown_rule(args.config),
           "precond": ("jacobi:1" if args.config == "C5" else "poly:%d" % args.poly if args.poly else "none"),
           "l2": ("no flush: working set > 126 MB L2 (Krylov basis alone %.2f GB fp32)" % (basis / 1e9)
                  if basis > 126e6 else "working set fits in L2 (not flushed; latency-bound config)"),
           "parallelism": "row-partitioned x%d" % args.gpus if args.gpus > 1 else "single",
           "iteration_budget": args.max_iters or (5000 if args.config == "C3" else 100000)}
    return cfg


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def note(msg):
    """Progress to stderr (the JSON line stays alone on stdout)."""
    if os.environ.get("MPK_BENCH_VERBOSE"):
        print("[bench %.1fs] %s" % (time.perf_counter() - T0, msg), file=sys.stderr, flush=True)


T0 = time.perf_counter()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


_CPU_SYS = {}


def cpu_sample(cfg_name, solver, steps_budget=50):
    """Oracle port (CPU restatement of the reference) on a bounded sample:
    `steps_budget` inner iterations of the same workload; returns s/iteration.
    The matrix is assembled once (setup, untimed as in cli.py:166-168)."""
    from oracle import mpk_oracle as O

    preset, nx, _ = CONFIGS[cfg_name]
    if cfg_name not in _CPU_SYS:
        rp, ci, v = O.stencil_csr(preset, nx)
        _CPU_SYS[cfg_name] = (rp, ci, v, v.astype(np.float32))
    rp, ci, v, v32 = _CPU_SYS[cfg_name]
    n = rp.size - 1
    b = np.ones(n)
    rule = breakdown_rule(cfg_name)
    t0 = time.perf_counter()
    if solver == "ir":
        out = O.refine((rp, ci, v), b, np.zeros(n), 50, 1e-10, steps_budget,
                       A32=(rp, ci, v32), rule=rule)
    else:
        out = O.restarted((rp, ci, v), None, b, np.zeros(n), 50, 1e-10, steps_budget, rule=rule)
    dt = time.perf_counter() - t0
    return dt / max(out.iters, 1), out.iters, dt


def cycle_steps(history):
    """Inner steps of each refinement, from an IR report's history rows."""
    out, cur = [], 0
    for e in history:
        if e.phase == "inner":
            cur += 1
        elif e.phase == "outer" and e.iteration > 0:
            out.append(cur)
            cur = 0
    return out


def run_reference_arm(args):
    """Reference CPU path (the oracle port, pinned to the unmodified
    reference's goldens) on the box's host cores: each step is a bounded
    sample of the same solve (one refinement = 50 inner iterations plus the
    outer fp64 residual pass).  value = median s/iteration x the reference's
    iteration count for the config (an extrapolation, stated in `note`;
    profiles/r02_cpu_full_runs.json holds full runs to convergence that
    validate it).  ms_per_step is the sample's own wall time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.config not in ("C1", "C2", "C4"):
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for C1/C2/C4 only"}))
        return
    iters_full = REF_ITERS[args.config]["ir"]
    cpu_sample(args.config, "ir", 5)   # assembly (setup) + page-in, untimed
    for _ in range(args.warmup):
        cpu_sample(args.config, "ir", 5)
    per_it, walls = [], []
    for _ in range(args.steps):
        s, it, dt = cpu_sample(args.config, "ir", 50)
        per_it.append(s)
        walls.append(dt)
    value = float(np.median(per_it)) * iters_full
    line = {
        "impl": "reference", "metric": "GMRES-IR time-to-1e-10 residual (s)", "value": value,
        "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(walls)) * 1e3, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32-inner/f64-outer", "data": "synthetic (generated stencil, b = ones, x0 = 0)",
        "config": shared_config(args),
        "cpu_baseline": {"value": value, "unit": "s", "cores": cpu_cores(), "kind": "port",
                         "sample": "50 inner iterations (one refinement) of the same solve per step, "
                                   "median s/iteration x reference iteration count %d" % iters_full},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "value extrapolated: median s/iteration over the samples x the reference's iteration "
                "count; ms_per_step = measured wall time of one 50-iteration sample",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--poly", type=int, default=0, help="GMRES-polynomial preconditioner degree (0: none)")
    ap.add_argument("--fd", type=int, default=0, help="also time GMRES-FD switching precision at this iteration")
    ap.add_argument("--max-iters", type=int, default=None,
                    help="iteration budget (default 100000; C3 5000: UniFlow2D does not reach 1e-10, DESIGN.md 8)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    rank, world, local = dist_env()
    share = os.environ.get("MPK_SHARE_GPU") == "1"   # test mode: N ranks on one GPU (gloo host collectives)
    dev = 0 if share else local
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    import paper_2105_07544_b200 as mk
    from paper_2105_07544_b200 import _lib
    from paper_2105_07544_b200 import distributed as dd

    lib = _lib.load()
    P = mk.Precision
    preset, nx, desc = CONFIGS[args.config]
    rule = breakdown_rule(args.config)
    if args.config == "C5":
        A = mk.synthetic_irregular(nx, **C5_PARAMS)
    else:
        A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
    A_low = mk.convert_matrix(A, P.binary32)
    M32 = M64 = None
    if args.config == "C5":
        if world > 1:
            raise SystemExit("C5 (Jacobi) runs on one GPU")
        M32 = mk.build_block_jacobi(A_low, 1)   # setup, outside the timed region (cli.py:166-168)
        M64 = mk.build_block_jacobi(A, 1)
    if args.poly:
        if world > 1:
            raise SystemExit("the polynomial preconditioner runs on one GPU")
        # setup outside the timed region (cli.py:166-168): fp32 polynomial for
        # the IR inner cycles, fp64 polynomial for the fp64 GMRES comparison.
        # NB on UniFlow2D the reference's poly (seed = ones) stalls GMRES
        # (DESIGN.md 5), so C3's time-to-solution is quoted unpreconditioned
        M32 = mk.build_gmres_poly(A_low, args.poly, np.ones(A.n, np.float32), rule=rule)
        M64 = mk.build_gmres_poly(A, args.poly, np.ones(A.n))
    n = A.n
    budget = args.max_iters or (5000 if args.config == "C3" else 100000)
    inner = mk.SolverConfig(m=50, rtol=1e-4, precision=P.binary32, max_iters=budget, breakdown_rule=rule)
    icfg = mk.IrConfig(inner=inner, rtol=1e-10)
    cfg64 = mk.SolverConfig(m=50, rtol=1e-10, max_iters=budget)
    if world > 1:
        comm = dd.TorchComm()
        if share:
            comm.ctas = max(1, int(lib.mpk_sm_count()) // world)
        sysm = dd.LocalSystem(comm, A, A_low)
        n_loc = sysm.n
        b_dev = torch.ones(n_loc, dtype=torch.float64, device="cuda")
        x0_dev = torch.zeros(n_loc, dtype=torch.float64, device="cuda")
        solve_ir = lambda b, x0: dd.dist_gmres_ir(sysm, b, x0, icfg)  # noqa: E731
        solve_64 = lambda b, x0: dd.dist_gmres_restarted(sysm, b, x0, cfg64)  # noqa: E731
        wsi = sysm.workspace(50, P.binary32)
    else:
        from paper_2105_07544_b200.engine import CycleWorkspace

        n_loc = n
        b_dev = torch.ones(n, dtype=torch.float64, device="cuda")
        x0_dev = torch.zeros(n, dtype=torch.float64, device="cuda")
        solve_ir = lambda b, x0: mk.gmres_ir(A, b, x0, icfg, M=M32, A_low=A_low)  # noqa: E731
        solve_64 = lambda b, x0: mk.gmres_restarted(A, M64, b, x0, cfg64)  # noqa: E731
        wsi = CycleWorkspace.get(n, 50, P.binary32)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            got = [None] * world
            torch.distributed.all_gather_object(got, float(v))
            return max(got)
        return v

    def timed(fn, steps):
        """CUDA-event time of `steps` back-to-back calls, max over ranks (ms)."""
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        reps = [fn() for _ in range(steps)]
        ev1.record()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1)), reps

    note("setup done (n=%d)" % n)
    for _ in range(args.warmup):
        rep = solve_ir(b_dev, x0_dev)
        note("warmup solve: %d iters" % rep.total_iters)
    # timed region: K solves, per-kernel profiling off
    launches0 = lib.mpk_launch_count()
    wsi.flags = 0
    with ClockSampler(dev) as clk:
        ms_ir, reps = timed(lambda: solve_ir(b_dev, x0_dev), args.steps)
    launches = lib.mpk_launch_count() - launches0
    # separate profiled solve: per-kernel CUDA events on the launching stream
    lib.mpk_prof_reset()
    wsi.flags = 1
    ms_prof, reps_prof = timed(lambda: solve_ir(b_dev, x0_dev), 1)
    wsi.flags = 0
    NC = 8
    import ctypes
    pm = (ctypes.c_double * NC)()
    pc = (ctypes.c_int64 * NC)()
    pb = (ctypes.c_double * NC)()
    lib.mpk_prof_read(pm, pc, pb, NC)
    rep = reps[-1]
    ms_step = ms_ir / args.steps
    # algorithmic bytes of the inner cycles on this rank's rows:
    # per Arnoldi step at basis size j: SpMV + CGS2 sv*n*(4j+10); per cycle
    # the correction sv*n*(k+2)
    sv = 4
    # matrix-free stencil: x read + y write; CSR: sv*(nnz+2n) + 4*(nnz+n+1)
    spmv_b = 2.0 * sv * n_loc if A.stencil is not None else sv * (A.nnz + 2.0 * n) + 4.0 * (A.nnz + n + 1)
    steps_per_cycle = cycle_steps(reps_prof[-1].history)
    alg = sum(sum(spmv_b + sv * n_loc * (4 * (k + 1) + 10) for k in range(st)) + sv * n_loc * (st + 2)
              for st in cycle_steps(reps_prof[-1].history))
    names = ["spmv+norm+dot1", "update1+dot2", "update2+norm+givens", "normalise", "precond",
             "correction", "residual", "persistent Arnoldi cycle (k_cycle_reg)"]
    kern = {}
    for i in range(NC):
        if pc[i]:
            b_i = alg if i == 7 else pb[i]
            kern[names[i]] = {"ms_total": pm[i], "launches": int(pc[i]),
                              "alg_GBs": b_i / (pm[i] * 1e-3) / 1e9 if pm[i] > 0 else None}
    top = max(range(NC), key=lambda i: pm[i])
    peak, peak_kind = peaks()
    achieved = (alg if top == 7 else pb[top]) / (pm[top] * 1e-3) / 1e9
    # ncu DRAM bytes per launch of the cycle kernel (one 50-step cycle), from
    # profiles/traffic_<config>.json (ncu --set full of the same kernel)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.config)
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("bytes_per_launch")
        except Exception:
            traffic = None
    traffic_gbs = None
    if traffic and top == 7 and pc[7]:
        full = [st for st in steps_per_cycle if st == 50]
        if len(full) == len(steps_per_cycle):   # every launch is a full cycle
            traffic_gbs = traffic / (pm[7] * 1e-3 / pc[7]) / 1e9

    out = {
        "metric": "GMRES-IR time-to-1e-10 residual (s)",
        "value": ms_step / 1e3,
        "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32-inner/f64-outer",
        "data": "synthetic (generated %s, b = ones, x0 = 0)" % preset,
        "config": shared_config(args),
        "details": {"n": n, "nnz": A.nnz, "operator": "matrix-free stencil (bit-identical to CSR)",
                    "parallelism": ("row-partitioned x%d (P2P halo + in-kernel cross-GPU reductions)" % world
                                    if world > 1 else "single"),
                    "rows_per_rank": n_loc, "profiled_solve_s": ms_prof / 1e3},
        "iters": rep.total_iters, "refinements": rep.restarts, "final_relres": rep.final_explicit_relres,
        "converged": bool(rep.converged),
        "ref_iters": REF_ITERS[args.config]["ir"],
        "us_per_iter": ms_step * 1e3 / max(rep.total_iters, 1),
        "gpu_launches": int(launches),
        "kernels": kern,
        "roofline": {"bound": "hbm", "kernel": names[top], "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_GBs": traffic_gbs,
                     "traffic_frac": (traffic_gbs / peak) if traffic_gbs else None,
                     "note": "achieved = SURVEY 8(d) algorithmic bytes (two CGS2 GEMV pairs = 4 passes over V); "
                             "the kernel reads V 3 times per step, so traffic_GBs (ncu DRAM bytes per launch / "
                             "mean launch time) is the physical HBM rate",
                     "algorithmic_bytes": "per step: stencil SpMV 2*4*n + CGS2 4*n*(4j+10); "
                                          "per cycle: correction 4*n*(k+2) (SURVEY 8(d))"},
    }
    note("timed IR done")
    if not args.no_fp64:
        solve64 = lambda: solve_64(b_dev, x0_dev)  # noqa: E731
        solve64()
        ms64, reps64 = timed(solve64, 1)
        out["fp64_gmres_s"] = ms64 / 1e3
        out["fp64_iters"] = reps64[-1].total_iters
        out["ir_speedup_vs_fp64"] = (ms64 / 1e3) / (ms_step / 1e3)
        if world == 1 and (M64 is None or args.config == "C5"):
            # the lagged one-reduction CGS2 (opt-in, SolverConfig.orthogonalization
            # = "dcgs2"): 2 basis passes and 2 grid barriers per step instead of
            # 3 and 3; reported beside the reference-order headline
            cfg64d = dataclasses.replace(cfg64, orthogonalization="dcgs2")
            solve64d = lambda: mk.gmres_restarted(A, M64, b_dev, x0_dev, cfg64d)  # noqa: E731
            solve64d()
            ms64d, reps64d = timed(solve64d, 1)
            icfgd = dataclasses.replace(icfg, inner=dataclasses.replace(inner, orthogonalization="dcgs2"))
            solve_ird = lambda: mk.gmres_ir(A, b_dev, x0_dev, icfgd, M=M32, A_low=A_low)  # noqa: E731
            solve_ird()
            msird, repsird = timed(solve_ird, 1)
            out["dcgs2"] = {"ir_s": msird / 1e3, "ir_iters": repsird[-1].total_iters,
                            "ir_converged": bool(repsird[-1].converged),
                            "fp64_s": ms64d / 1e3, "fp64_iters": reps64d[-1].total_iters,
                            "ir_speedup_vs_fp64": ms64d / msird}
        if world == 1 and (M32 is None or args.config == "C5"):
            # third precision: the fp32 inner
            # cycles keep the Krylov basis in binary16 (scaled by a power of
            # two); arithmetic stays fp32 / fp64.  Reported beside the headline.
            icfgh = dataclasses.replace(icfg, inner=dataclasses.replace(inner, basis_precision="binary16"))
            solve_irh = lambda: mk.gmres_ir(A, b_dev, x0_dev, icfgh, M=M32, A_low=A_low)  # noqa: E731
            solve_irh()
            msirh, repsirh = timed(solve_irh, args.steps)
            out["binary16_basis"] = {"ir_s": msirh / args.steps / 1e3, "ir_iters": repsirh[-1].total_iters,
                                     "refinements": repsirh[-1].restarts,
                                     "ir_converged": bool(repsirh[-1].converged),
                                     "final_relres": repsirh[-1].final_explicit_relres,
                                     "speedup_vs_fp32_basis_ir": (ms_ir / args.steps) / (msirh / args.steps),
                                     "ir_speedup_vs_fp64": ms64 / (msirh / args.steps)}
            icfgb = dataclasses.replace(icfg, inner=dataclasses.replace(inner, basis_precision="bfloat16"))
            solve_irb = lambda: mk.gmres_ir(A, b_dev, x0_dev, icfgb, M=M32, A_low=A_low)  # noqa: E731
            solve_irb()
            msirb, repsirb = timed(solve_irb, 1)
            out["bfloat16_basis"] = {"ir_s": msirb / 1e3, "ir_iters": repsirb[-1].total_iters,
                                     "ir_converged": bool(repsirb[-1].converged),
                                     "ir_speedup_vs_fp64": ms64 / msirb}
            # both opt-ins at once: the lagged one-reduction CGS2 (2 basis
            # passes per step) over the binary16 basis (half the bytes per pass)
            icfghd = dataclasses.replace(icfg, inner=dataclasses.replace(inner, basis_precision="binary16",
                                                                         orthogonalization="dcgs2"))
            solve_irhd = lambda: mk.gmres_ir(A, b_dev, x0_dev, icfghd, M=M32, A_low=A_low)  # noqa: E731
            solve_irhd()
            msirhd, repsirhd = timed(solve_irhd, args.steps)
            out["dcgs2_binary16_basis"] = {"ir_s": msirhd / args.steps / 1e3, "ir_iters": repsirhd[-1].total_iters,
                                           "refinements": repsirhd[-1].restarts,
                                           "ir_converged": bool(repsirhd[-1].converged),
                                           "final_relres": repsirhd[-1].final_explicit_relres,
                                           "speedup_vs_headline_ir": (ms_ir / args.steps) / (msirhd / args.steps),
                                           "ir_speedup_vs_fp64": ms64 / (msirhd / args.steps)}
    note("fp64 done")
    if not args.no_e2e:
        # public API with host (pinned) inputs; every step copies b and x0 in
        # and the solution out (each rank its own rows when partitioned)
        bh = torch.ones(n_loc, dtype=torch.float64).pin_memory()
        xh = torch.zeros(n_loc, dtype=torch.float64).pin_memory()
        if world > 1:
            solve_e2e = lambda: dd.dist_gmres_ir(sysm, bh, xh, icfg).x.cpu()  # noqa: E731
        else:
            solve_e2e = lambda: mk.gmres_ir(A, bh, xh, icfg, M=M32, A_low=A_low).x  # noqa: E731
        solve_e2e()
        ms_e2e, xs_e = timed(solve_e2e, args.steps)
        assert not xs_e[-1].is_cuda
        out["e2e"] = {"value": ms_e2e / args.steps / 1e3, "unit": "s", "h2d_bytes_per_step": 2 * 8 * n,
                      "d2h_bytes_per_step": 8 * n, "note": "whole job: b and x0 in, x out (all ranks)"}
    if world == 1 and A.stencil is not None:
        # SpMV GB/s (the metric's second half): standalone mpk_spmv on this
        # matrix, stencil and CSR forms, fp64 and fp32, algorithmic bytes of
        # SURVEY 8(d) (CSR) / x read + y write (stencil), CUDA events
        from paper_2105_07544_b200.sparse import spmv_into

        spmv_rates = {}
        for prec, M in ((P.binary64, A), (P.binary32, A_low)):
            svb = 8 if prec is P.binary64 else 4
            # enough x/y pairs that consecutive launches never find their
            # vectors in the 126 MB L2 (>= 384 MB of pairs, cycled)
            npair = max(1, min(20, -(-384 * 2**20 // (2 * svb * n))))
            pairs = [(torch.randn(n, dtype=prec.torch_dtype, device="cuda"),
                      torch.empty(n, dtype=prec.torch_dtype, device="cuda")) for _ in range(npair)]
            xs, ys = pairs[0]
            for form in ("stencil", "csr"):
                M.use_stencil = form == "stencil"
                spmv_into(M, xs, ys)
                torch.cuda.synchronize()
                # 20 launches captured in a CUDA graph and replayed: a
                # Python-issued loop measures the host's launch rate
                # (~12 us per call) once a kernel is shorter than that
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    spmv_into(M, xs, ys)
                torch.cuda.current_stream().wait_stream(side)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    for i in range(20):
                        spmv_into(M, *pairs[i % npair])
                graph.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 20
                del graph
                byt = 2.0 * svb * n if form == "stencil" else svb * (M.nnz + 2.0 * n) + 4.0 * (M.nnz + n + 1)
                spmv_rates["%s_%s" % (form, prec.value)] = {"ms": ms, "GBs": byt / ms / 1e6,
                                                            "frac": byt / ms / 1e6 / peak}
            M.use_stencil = True
            del pairs
        spmv_rates["timing"] = ("CUDA graph of 20 back-to-back launches cycling through x/y pairs of >= 384 MB "
                                "(no vector is L2-resident when its launch starts), CUDA events around one replay")
        out["spmv"] = spmv_rates
    out["clocks"] = clk.summary()
    if args.fd and world == 1:
        # GMRES-FD (multiprecision.py:236-288): fp32 restarted GMRES for
        # switch_iter iterations, then fp64 against the original baseline
        fcfg = mk.FdConfig(switch_iter=args.fd, low=mk.SolverConfig(m=50, rtol=1e-10, precision=P.binary32,
                                                                    breakdown_rule=rule, max_iters=100000),
                           high=cfg64)
        solve_fd = lambda: mk.gmres_fd(A, b_dev, x0_dev, fcfg, M_low=M32, M_high=M64, A_low=A_low)  # noqa: E731
        solve_fd()
        msfd, repfd = timed(solve_fd, 1)
        out["fd"] = {"switch_iter": args.fd, "s": msfd / 1e3, "iters": repfd[-1].total_iters,
                     "converged": bool(repfd[-1].converged)}
    if args.poly and world == 1:
        # the same IR solve with the polynomial on the multi-kernel cycle
        # (desc flag 4: one launch per SpMV / update) -- what fusing the
        # polynomial into the persistent kernel bought
        wsi.flags = 4
        try:
            solve_ir(b_dev, x0_dev)
            msmk, repsmk = timed(lambda: solve_ir(b_dev, x0_dev), 1)
        finally:
            wsi.flags = 0
        out["poly_multikernel"] = {"ir_s": msmk / 1e3, "iters": repsmk[-1].total_iters,
                                   "us_per_iter": msmk * 1e3 / max(repsmk[-1].total_iters, 1),
                                   "fused_speedup": msmk / ms_step}
    if args.config == "C5":
        out["details"]["precond"] = {"kind": "block-jacobi", "block": 1, "fused": "diagonal scaling in k_cycle_reg"}
        out["details"]["operator"] = "CSR, warp-cooperative bit-exact rows"
        out["details"]["generator"] = dict(C5_PARAMS, seed=20240817)
    elif M32 is not None:
        out["details"]["precond"] = {"kind": "gmres-poly", "degree_ir": M32.data.degree,
                                     "degree_fp64": M64.data.degree, "seed": "ones"}
        out["details"]["operator"] = "matrix-free stencil; poly apply = degree SpMVs per step"
    if rank == 0 and world == 1 and not args.no_cpu and not args.poly and args.config != "C5":
        s_it, it, dt = cpu_sample(args.config, "ir", 50)
        full = REF_ITERS[args.config]["ir"] or rep.total_iters
        out["cpu_baseline"] = {"value": s_it * full, "unit": "s", "cores": cpu_cores(), "kind": "port",
                               "sample": "%d inner iterations (one refinement, %.1f s) of the same "
                                         "GMRES-IR solve; s/iteration x reference count %d" % (it, dt, full)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        sysm.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
