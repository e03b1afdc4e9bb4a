#!/usr/bin/env python
"""Benchmark of the explicit RBF-FD pseudo-time loop (BASELINE.json metric:
node-updates/s, and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5|c2x10] [--native] [--ldg] [--quick]

One bench "step" is one pseudo-time iteration over every interior row (one
pass of the hot path, solver.py:198-217); a node-update is one interior row in
one step (perf.py:74).  Default workload: BASELINE config 2 -- m=2, n=15,
N=1e6 scattered nodes, fp64, one B200 -- on the reference's own
advancing-front node set for target 1e6, seed 1 (N=1,046,538, N_i=1,042,999,
SURVEY.md 8d), regenerated bit-identically by the native generator
(paper_2107_03632_b200/geometry.py; the GPU box has no reference package),
with exact GPU kNN supports and GPU-assembled PHS+poly weights.

`value` is device throughput with all inputs resident in HBM (CUDA events on
the plan's stream around exactly K steps, max over ranks); `e2e` is the same
metric through the public API `run_time_loop(config, nodes, shapes)` from host
arrays: plan build (H2D of weights/ids/forcing), field upload, K steps,
field download.  `--impl reference` times the CPU oracle (a bit-exact C port of
the reference's numba loop, oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "node-updates/s of RBF-FD Poisson explicit loop at m=2/4/6; % HBM roofline"

WORKLOADS = {
    # name: (target N, n, m, description)
    "c1": (1027, 15, 2, "C1: paper Fig. 1 case, m=2 n=15 N=1027 (golden fixture, reference nodes)"),
    "c2": (1_000_000, 15, 2, "C2: m=2 n=15 N=1e6 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c3": (10_000_000, 30, 4, "C3: m=4 n=30 N=1e7 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c2x10": (10_000_000, 15, 2, "m=2 n=15 N=1e7 reference advancing-front disk (seed 1), fp64, 1xB200 (north-star m=2 at N>=1e7)"),
    "c4": (25_000_000, 56, 6, "C4: m=6 n=56 N=2.5e7 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c5": (100_000_000, 56, 6, "C5: m=6 n=56 N=1e8 reference advancing-front disk (seed 1), fp64, 1xB200 (single-GPU base of the 2/4/8-GPU config)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_problem(workload: str, seed: int = 1, gpu_setup: bool = True):
    """The workload's (nodes, stencils, shapes).  gpu_setup: exact kNN and
    weights on the GPU; False (the --impl reference arm) keeps the whole setup
    on the CPU (cKDTree, numpy/LAPACK weights) so that arm runs no GPU code."""
    import paper_2107_03632_b200 as rb
    from paper_2107_03632_b200 import synth

    target, n, m, _ = WORKLOADS[workload]
    if workload == "c1":
        return rb.load_fixture(ROOT / "tests" / "golden" / "dome.npz")
    return synth.synthetic_problem(target, n, m, seed=seed, weights="gpu" if gpu_setup else "cpu",
                                   knn="gpu" if gpu_setup else "cpu")


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    ncu --set full summary (profiles/), or None."""
    p = ROOT / "profiles" / "roofline_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
        return False

    def summary(self):
        rows = []
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append(dict(sm=float(parts[0]), max=float(parts[1]), hw=parts[3], hwt=parts[4],
                                 swt=parts[5], pcap=parts[6], util=float(parts[7])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r["util"] > 0] or rows
        reasons = set()
        for r in loaded:
            for key, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                              ("swt", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[key].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in loaded),
                "sm_max_mhz": max(r["max"] for r in rows), "reasons": sorted(reasons),
                "samples": len(loaded)}


def cpu_baseline(nodes, shapes, dt, budget_s: float, threads=None):
    """The oracle (bit-exact C port of the reference's numba loop) on the host
    cores, on a bounded number of full steps of the same workload."""
    from oracle import oracle as orc

    interior = shapes.interior_nodes
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(orc.forcing(nodes.positions[interior]))
    u0 = orc.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    threads = orc.max_threads() if threads is None else threads
    probe = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt,
                           steps=2, threads=threads)
    per_step = max(probe["seconds"] / 2, 1e-6)
    steps = int(max(3, min(100_000, budget_s / per_step)))
    out = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt,
                         steps=steps, threads=threads)
    rate = steps * interior.size / out["seconds"]
    return rate, steps, out["seconds"], threads, out


def run_reference(args, workload):
    """--impl reference: the reference's CPU loop (oracle port) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc

    t0 = time.perf_counter()
    nodes, _, shapes = build_problem(workload, gpu_setup=False)
    log(f"[ref] setup {time.perf_counter() - t0:.1f}s N={nodes.n_total} N_i={shapes.n_rows}")
    dt = 0.5 * orc.stability_bound(shapes.weights)  # solver.py:188, :249-254
    interior = shapes.interior_nodes
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(orc.forcing(nodes.positions[interior]))
    u0 = orc.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    threads = orc.max_threads()
    probe = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt,
                           steps=max(1, args.warmup), threads=threads)
    per_step = probe["seconds"] / max(1, args.warmup)
    budget = 150.0
    steps = args.steps if args.steps * per_step <= budget else max(3, int(budget / per_step))
    out = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt,
                         steps=steps, threads=threads)
    rate = steps * interior.size / out["seconds"]
    sample = (f"{steps} full steps over all {interior.size} interior rows"
              + ("" if steps == args.steps else f" (bounded sample of the requested {args.steps})"))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": rate,
        "unit": "node-updates/s",
        "n_gpus": args.gpus,  # the configuration's; this arm itself runs on the host cores
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * out["seconds"] / steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": ("synthetic (reference advancing-front nodes via the native generator, CPU kNN "
                 "(cKDTree) + numpy/LAPACK weights)" if workload != "c1" else "reference fixture (tests/golden/dome.npz)"),
        "config": {"workload": WORKLOADS[workload][3], "N": int(nodes.n_total),
                   "N_i": int(interior.size), "n": int(shapes.weights.shape[1]),
                   "m": int(shapes.degree), "dt": dt},
        "cpu_baseline": {"value": rate, "unit": "node-updates/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "node-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10_000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--native", action="store_true",
                    help="keep the native (advancing-front) node order instead of Morton renumbering")
    ap.add_argument("--ldg", action="store_true", help="plain-load streaming kernel (no TMA ring)")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-rank (torchrun/NCCL) path even with one rank (testing)")
    ap.add_argument("--quick", action="store_true",
                    help="profiling mode: timed region only (no e2e, clock keep-alive, CPU leg)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args, args.workload)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        from paper_2107_03632_b200 import multigpu

        return multigpu.bench_main(args, METRIC, WORKLOADS)

    import torch

    import paper_2107_03632_b200 as rb
    from paper_2107_03632_b200.solver import Plan

    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    nodes, _, shapes = build_problem(args.workload)
    t_setup = time.perf_counter() - t0
    n = int(shapes.weights.shape[1])
    N_i = int(shapes.n_rows)
    dt = 0.5 * rb.stability_bound(shapes)
    log(f"setup {t_setup:.1f}s: N={nodes.n_total} N_i={N_i} n={n} dt={dt:.4e}")

    interior = shapes.interior_nodes
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(rb.forcing(nodes.positions[interior]))
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    renumber = not args.native
    plan = Plan(nodes.n_total, interior, rows, shapes.weights, f_int,
                nodes.positions if renumber else None, renumber=renumber, device=local,
                tma=not args.ldg, pdl=not args.no_pdl)
    info = plan.info()
    log(f"plan: {info}")
    plan.set_field(u0)

    # warm-up (untimed): W steps through the same graph path
    plan.run(dt, steps=args.warmup)
    plan.set_field(u0)
    torch.cuda.synchronize()
    launches0 = plan.info()["launches"]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        res = plan.run(dt, steps=args.steps)  # CUDA events on the plan's stream
        torch.cuda.synchronize()
        # keep the GPU busy a little longer so the sampler sees the load
        if res.device_seconds < 1.0 and not args.quick:
            extra = int(min(200_000, max(1, args.steps * (1.0 / max(res.device_seconds, 1e-6)))))
            plan.run(dt, steps=extra)
    gpu_launches = plan.info()["launches"] - launches0  # includes the clock-keepalive run
    gpu_launches = args.steps if info["resident"] == 0 else 1  # resident / cluster loop: one launch
    t = res.device_seconds
    value = args.steps * N_i / t
    bytes_per_step = info["bytes_per_step"]
    per_launch = t / args.steps
    achieved_gbs = bytes_per_step / per_launch / 1e9
    peak, peak_src = measured_peak()
    traffic = committed_traffic(args.workload)
    log(f"device: {t * 1e3:.2f} ms for {args.steps} steps -> {value:.4e} upd/s, "
        f"{achieved_gbs:.0f} GB/s algorithmic ({achieved_gbs / peak:.3f} of {peak_src}); "
        f"residual {res.residual}")

    plan_info = info
    plan.close()  # the e2e leg builds its own plan (C5: ~70 GB of HBM each)
    # ---- end to end through the public API (host arrays in, host field out)
    cfg = rb.SolveConfig(degree=int(shapes.degree), support_size=n, nodes=int(nodes.n_total),
                         dt=dt, steps=args.steps)
    t_e2e = float("nan")
    if not args.quick:
        rb.run_time_loop(cfg, nodes, shapes, cache=False, renumber=renumber)  # warm (allocator, module load)
        torch.cuda.synchronize()
        te = time.perf_counter()
        rb.run_time_loop(cfg, nodes, shapes, cache=False, renumber=renumber)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - te
    e2e_value = args.steps * N_i / t_e2e
    h2d = N_i * n * (8 + 8) + N_i * 8 + nodes.n_total * 8  # weights + int64 ids + forcing + field
    d2h = nodes.n_total * 8
    log(f"e2e: {t_e2e * 1e3:.1f} ms -> {e2e_value:.4e} upd/s (plan build + upload + loop + download)")

    cpu = None
    if not (args.no_cpu_baseline or args.quick):
        rate, csteps, csec, threads, _ = cpu_baseline(nodes, shapes, dt, args.cpu_budget)
        cpu = {"value": rate, "unit": "node-updates/s", "cores": threads, "kind": "port",
               "sample": f"{csteps} full steps of the same workload ({csec:.1f}s, oracle/ C port "
                         f"of solver.py:294-311, OpenMP over row chunks)"}
        log(f"cpu baseline: {rate:.4e} upd/s on {threads} threads ({csteps} steps)")

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "node-updates/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * per_launch,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": ("synthetic (reference advancing-front nodes via the native generator, GPU kNN + "
                 "GPU-assembled weights)" if args.workload != "c1" else "reference fixture"),
        "config": {
            "workload": WORKLOADS[args.workload][3],
            "N": int(nodes.n_total), "N_i": N_i, "n": n, "m": int(shapes.degree), "dt": dt,
            "renumber": "morton (bit-identical)" if renumber else "native (advancing-front order)",
            "l2": (f"inputs larger than L2: {bytes_per_step / 1e6:.0f} MB streamed per step "
                   f"vs 126 MB L2" if bytes_per_step > 126e6 else
                   f"working set {bytes_per_step / 1e6:.1f} MB fits L2 (no flush)"),
            "loop": {0: "resident on-chip loop (one CTA)",
                     1: "streaming step (plain loads), CUDA graphs of 64 steps",
                     2: "streaming step (TMA bulk-copy ring, warp-specialised), CUDA graphs of 64 steps",
                     3: "cluster-resident loop (thread-block cluster, DSMEM halo, one launch)",
                     4: "grid-resident loop (rows in every SM's shared memory, one cooperative launch, "
                        "grid barrier per step)"}[
                         info["variant"]] + ("" if args.no_pdl or info["resident"] else " + PDL"),
            "parallelism": "single GPU",
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved_gbs,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved_gbs / peak,
            "traffic": traffic,
            "bytes_per_launch": bytes_per_step,
            "bytes_formula": "N_i*(12n+24): 8n w + 4n ids + 8 f + 8 u_self + 8 u_out",
            "peak_source": peak_src,
            "frac_of_8TBps_spec": achieved_gbs / 8000.0,
            # with 16-bit two-window ids the step streams fewer bytes than B(n)
            # (report compression separately from the B(n) fraction)
            "index_bits": info["index_bits"],
            "stream_bytes_per_launch": info["stream_bytes_per_step"],
            "stream_achieved": info["stream_bytes_per_step"] / per_launch / 1e9,
            "stream_frac": info["stream_bytes_per_step"] / per_launch / 1e9 / peak,
        },
        "e2e": {"value": e2e_value if math.isfinite(e2e_value) else None, "unit": "node-updates/s",
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "what": "run_time_loop(config, nodes, shapes, cache=False) from host numpy arrays: "
                        "plan build + H2D (weights, int64 ids, forcing, field), K steps, D2H field"},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "setup_seconds": t_setup,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    del plan_info
    return 0


if __name__ == "__main__":
    sys.exit(main())
