#!/usr/bin/env python
"""Benchmark of the explicit RBF-FD pseudo-time loop (BASELINE.json metric:
node-updates/s, and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c2x10|c3|c4|c5] [--no-per-config] [--quick]

One bench "step" is one pseudo-time iteration over every interior row (one
pass of the hot path, solver.py:198-217); a node-update is one interior row in
one step (perf.py:74).

Workload of the headline line (N=1): BASELINE config 2 -- m=2, n=15, N=1e6,
fp64, one B200 -- built by the reference pipeline on the host: the
reference's advancing-front node set for (target 1e6, seed 1) (N=1,046,538,
N_i=1,042,999), exact kNN supports (cKDTree, the reference's
tie rules) and PHS+poly weights (numpy/LAPACK, the reference's solve).  Both
arms build byte-identical arrays: this arm through the package's CPU setup
(synth.py), the reference arm through oracle/problem.py, which never maps the
product library; `config.arrays_sha256` is the digest of (positions,
interior, stencil rows, weights) and is the same in both lines.

Keys of the line:
* `value`: K steps x N_i / CUDA-event time of exactly K device steps
  (rbf_run on the plan's stream), inputs resident in HBM, after W warm-up
  steps.  Inputs (182-213 MB per step at C2) exceed the 126 MB L2.
* `e2e`: the same metric through the public API run_time_loop(config,
  nodes, shapes) from host numpy arrays: plan build (H2D of weights, ids,
  forcing, positions), field upload, K steps, field download, error norms.
* `roofline`: the dominant kernel (the TMA-ring step), achieved = bytes it
  actually streams per launch (16-bit ids: 10n+24 per row + window bases)
  / per-launch event time; `frac` against the measured copy peak.  The B(n) =
  12n+24 algorithmic equivalent (int32 ids) is reported separately.
* `cpu_baseline`: the reference's loop (oracle/ C port of the numba kernel,
  bitwise equal to it) on the host cores, threads=1 and all threads, min of
  3 repeats, each run >= 1 s (perf.py:139-143).
* `parity`: the GPU run for the same step count as the all-thread CPU leg,
  sha256 of both final fields (perf.py:75).
* `per_config`: the north-star N>=1e7 configs (m=2 N=1e7, C3 m=4 N=1e7,
  C4 m=6 N=2.5e7) timed in the same run, each with its streamed-bytes
  roofline and a GPU-vs-oracle digest (device setup: GPU kNN + weights).

`--impl reference` times the reference's CPU loop (the oracle port) on all
host threads on the same arrays and prints the same line with
"impl": "reference".
"""

from __future__ import annotations

import argparse
import hashlib
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
SEED = 1

WORKLOADS = {
    # name: (target N, n, m, description)
    "c1": (1027, 15, 2, "C1: paper Fig. 1 case, m=2 n=15 N=1027 (golden fixture, reference nodes)"),
    "c2": (1_000_000, 15, 2, "C2: m=2 n=15 N=1e6 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c2x10": (10_000_000, 15, 2, "m=2 n=15 N=1e7 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c3": (10_000_000, 30, 4, "C3: m=4 n=30 N=1e7 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c4": (25_000_000, 56, 6, "C4: m=6 n=56 N=2.5e7 reference advancing-front disk (seed 1), fp64, 1xB200"),
    "c5": (100_000_000, 56, 6, "C5: m=6 n=56 N=1e8 reference advancing-front disk (seed 1), fp64"),
}
# per_config block of the default line: (workload, timed steps, parity steps)
PER_CONFIG = (("c2x10", 64, 10), ("c3", 40, 6), ("c4", 24, 4))

DATA = ("synthetic: the reference's advancing-front node set for (target, seed 1), exact kNN "
        "supports, PHS r^3 + monomial weights (reference solve)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def setup_text(gpu: bool) -> str:
    if gpu:
        return ("device setup: native advancing-front nodes (bit-identical to the reference), "
                "exact GPU kNN, GPU-assembled weights")
    return "host setup: advancing-front nodes, cKDTree kNN (reference tie rules), numpy/LAPACK weights"


def arrays_digest(nodes, shapes) -> str:
    """sha256 over (positions, interior, neighbors[interior], weights): the
    exact arrays the timed loop consumes."""
    h = hashlib.sha256()
    interior = np.ascontiguousarray(shapes.interior_nodes, dtype=np.int64)
    h.update(np.ascontiguousarray(nodes.positions, dtype=np.float64).tobytes())
    h.update(interior.tobytes())
    nb = shapes.stencils.neighbors
    for lo in range(0, interior.size, 1 << 20):
        h.update(np.ascontiguousarray(nb[interior[lo:lo + (1 << 20)]], dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(shapes.weights, dtype=np.float64).tobytes())
    return h.hexdigest()[:24]


def field_digest(u: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()  # perf.py:75


def l2_note(n_rows: int, n: int) -> str:
    b = n_rows * (12 * n + 24)
    return (f"inputs larger than L2: {b / 1e6:.0f} MB (B(n)) streamed per step vs 126 MB L2" if b > 126e6
            else f"working set {b / 1e6:.1f} MB fits L2 (no flush; latency-bound config)")


def common_config(workload: str, nodes, shapes, dt: float, digest: str) -> dict:
    """The config dict both arms print (identical keys and values)."""
    n = int(shapes.weights.shape[1])
    return {"workload": WORKLOADS[workload][3], "N": int(nodes.n_total), "N_i": int(shapes.n_rows), "n": n,
            "m": int(shapes.degree), "seed": SEED, "dt": dt, "arrays_sha256": digest,
            "l2": l2_note(int(shapes.n_rows), n)}


def cpu_info() -> dict:
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    physical = None
    try:
        import psutil

        physical = psutil.cpu_count(logical=False)
    except Exception:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "physical_cores": physical}


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
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the step
    kernel from the committed ncu --set full summary (profiles/), or None."""
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
        self.lines = []

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
        for l in self.lines:
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


# ---------------------------------------------------------------------------
# CPU legs (oracle/: the reference's loop, bitwise equal to its numba kernel)

def _oracle_arrays(nodes, shapes):
    from oracle import oracle as orc

    interior = np.ascontiguousarray(shapes.interior_nodes, dtype=np.int64)
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(orc.forcing(nodes.positions[interior]))
    u0 = orc.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    return interior, rows, f_int, u0


def cpu_legs(nodes, shapes, dt, min_seconds: float = 1.0, repeats: int = 3):
    """BASELINE.md 3 / perf.py:108-157: threads=1 and threads=all, min of
    `repeats`, steps chosen so each run takes >= min_seconds; the field
    digest of each leg (they must agree: thread count never changes bits)."""
    from oracle import oracle as orc

    interior, rows, f_int, u0 = _oracle_arrays(nodes, shapes)
    N = nodes.n_total
    legs = {}
    for threads in sorted({1, orc.max_threads()}):
        orc.run_arrays(N, interior, rows, shapes.weights, f_int, u0, dt, steps=1, threads=threads)  # warm
        probe = orc.run_arrays(N, interior, rows, shapes.weights, f_int, u0, dt, steps=4, threads=threads)
        per_step = max(probe["seconds"] / 4, 1e-7)
        steps = int(max(3, min(200_000, math.ceil(1.25 * min_seconds / per_step))))
        best, out = None, None
        while True:
            for _ in range(repeats):
                out = orc.run_arrays(N, interior, rows, shapes.weights, f_int, u0, dt, steps=steps,
                                     threads=threads)
                best = out["seconds"] if best is None else min(best, out["seconds"])
            if best >= min_seconds or steps >= 200_000:
                break
            # the probe over-estimated the step time: rescale, time again
            steps = int(min(200_000, math.ceil(1.25 * steps * min_seconds / max(best, 1e-9))))
            best = None
        legs[threads] = {"threads": threads, "steps": steps, "seconds_min": best,
                         "value": steps * interior.size / best, "digest": field_digest(out["field"]),
                         "residual": out["residual"]}
        log(f"cpu leg threads={threads}: {steps} steps, min {best:.3f}s -> {legs[threads]['value']:.4e} upd/s")
    # thread count never changes bits (test_perf.py:111-114): the all-thread
    # loop over the 1-thread leg's step count must give the 1-thread digest
    if len(legs) > 1:
        top = max(legs)
        same = orc.run_arrays(N, interior, rows, shapes.weights, f_int, u0, dt, steps=legs[1]["steps"],
                              threads=top)
        legs[top]["digest_at_1thread_steps"] = field_digest(same["field"])
    return legs


def oracle_steps(nodes, shapes, dt, steps):
    from oracle import oracle as orc

    interior, rows, f_int, u0 = _oracle_arrays(nodes, shapes)
    out = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt, steps=steps)
    return out


# ---------------------------------------------------------------------------
# reference arm

def build_reference_problem(workload: str):
    from oracle import problem as op

    target, n, m, _ = WORKLOADS[workload]
    if workload == "c1":
        z = np.load(ROOT / "tests" / "golden" / "dome.npz")
        nodes = op.Nodes(positions=z["positions"], is_boundary=z["is_boundary"], h=float(z["h"]))
        st = op.Stencils(n=int(z["neighbors"].shape[1]), neighbors=z["neighbors"].astype(np.int64))
        shapes = op.Shapes(degree=int(z["degree"]), interior_nodes=z["interior"].astype(np.int64),
                           weights=z["weights"], stencils=st)
        return nodes, st, shapes
    return op.reference_problem(target, n, m, seed=SEED)


def check_reference_nodes(nodes):
    """The C2 node set must be the reference's own (tests/golden/nodes.json)."""
    try:
        cases = json.loads((ROOT / "tests" / "golden" / "nodes.json").read_text())["cases"]
    except OSError:
        return None
    for c in cases:
        if c["n_total"] == nodes.n_total and abs(c["h"] - nodes.h) == 0.0 and str(c["seed"]) == str(SEED):
            return hashlib.sha256(nodes.positions.tobytes()).hexdigest() == c["sha256"]
    return None


def run_reference(args, workload):
    """--impl reference: the reference's CPU loop (oracle port, all host
    threads) on the same arrays as the GPU arm; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc

    t0 = time.perf_counter()
    nodes, _, shapes = build_reference_problem(workload)
    pinned = check_reference_nodes(nodes)
    if pinned is False:
        raise SystemExit("reference arm: node set differs from the reference's digest")
    dt = 0.5 * orc.stability_bound(shapes.weights)  # solver.py:188, :249-254
    digest = arrays_digest(nodes, shapes)
    log(f"[ref] setup {time.perf_counter() - t0:.1f}s N={nodes.n_total} N_i={shapes.n_rows} "
        f"arrays {digest} nodes pinned={pinned}")
    interior, rows, f_int, u0 = _oracle_arrays(nodes, shapes)
    threads = orc.max_threads()
    orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt, steps=args.warmup,
                   threads=threads)
    probe = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt, steps=2,
                           threads=threads)
    per_step = probe["seconds"] / 2
    budget = 150.0
    steps = args.steps if args.steps * per_step <= budget else max(3, int(budget / per_step))
    out = orc.run_arrays(nodes.n_total, interior, rows, shapes.weights, f_int, u0, dt, steps=steps,
                         threads=threads)
    rate = steps * interior.size / out["seconds"]
    sample = (f"{steps} full steps over all {interior.size} interior rows, {threads} threads"
              + ("" if steps == args.steps else f" (bounded sample of the requested {args.steps})"))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": rate,
        "unit": "node-updates/s",
        "n_gpus": args.gpus,  # the configuration's; this arm runs on the host cores
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * out["seconds"] / steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": DATA,
        "config": common_config(workload, nodes, shapes, dt, digest),
        "cpu_baseline": {"value": rate, "unit": "node-updates/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu": cpu_info(),
                         "what": "oracle/rbffd_oracle.c: C port of solver.py:294-311 + :190-225, bitwise "
                                 "equal to the reference's numba kernel (OpenMP over 1024-row chunks)"},
        "e2e": {"value": rate, "unit": "node-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup": setup_text(False) + " (oracle/problem.py; no product library mapped)",
        "field_sha256": field_digest(out["field"]),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def build_problem(workload: str, gpu_setup: bool):
    import paper_2107_03632_b200 as rb
    from paper_2107_03632_b200 import synth

    target, n, m, _ = WORKLOADS[workload]
    if workload == "c1":
        return rb.load_fixture(ROOT / "tests" / "golden" / "dome.npz")
    if gpu_setup:
        return synth.synthetic_problem(target, n, m, seed=SEED, weights="gpu", knn="gpu")
    return synth.synthetic_problem(target, n, m, seed=SEED, weights="cpu", knn="cpu")


LOOPS = {0: "resident on-chip loop (one CTA)",
         1: "streaming step (plain loads), CUDA graphs of 64 steps",
         2: "streaming step (TMA bulk-copy ring, warp-specialised), CUDA graphs of 64 steps",
         5: "persistent streaming loop (TMA bulk-copy ring, warp-specialised; one cooperative launch per run, "
            "grid barrier per step, the ring streams the next step while the consumers finish)",
         3: "cluster-resident loop (thread-block cluster, DSMEM halo, one launch)",
         4: "grid-resident loop (rows in every SM's shared memory, one cooperative launch, grid barrier per step)"}


def roofline(info: dict, per_launch: float, peak: float, peak_src: str, traffic) -> dict:
    stream = info["stream_bytes_per_step"]
    bn = info["bytes_per_step"]
    return {
        "bound": "hbm",
        "kernel": ("stream_loop_kernel" if info.get("persist") else
                   "step_tma_kernel" if info["variant"] == 2 else LOOPS[info["variant"]]),
        "achieved": stream / per_launch / 1e9,
        "peak": peak,
        "unit": "GB/s",
        "frac": stream / per_launch / 1e9 / peak,
        "traffic": traffic,
        "bytes_per_launch": stream,
        "bytes_formula": ("N_i*(10n+24) + 16*slices (+ int32 ids of overflow slices): 8n w + 2n ids (16-bit "
                          "two-window) + 8 f + 8 u_self + 8 u_out, the bytes the kernel streams"
                          if info["index_bits"] == 16 else
                          "N_i*(12n+24): 8n w + 4n ids + 8 f + 8 u_self + 8 u_out"),
        "peak_source": peak_src,
        "per": ("step: the persistent loop runs all K steps in one launch; achieved = K x bytes_per_launch "
                "/ that launch's event time, traffic = ncu DRAM bytes of one launch / its steps"
                if info.get("persist") else "launch (one step)"),
        "index_bits": info["index_bits"],
        "Bn_bytes_per_launch": bn,
        "Bn_equivalent_GBps": bn / per_launch / 1e9,
        "Bn_frac_of_8TBps_spec": bn / per_launch / 1e9 / 8000.0,
        "Bn_note": "SURVEY.md 8d algorithmic B(n)=12n+24 (int32 ids); with 16-bit ids this rate exceeds "
                   "the bytes moved, so it is not the fraction",
    }


def time_plan(plan, dt, steps, warmup, u0):
    plan.set_field(u0)
    plan.run(dt, steps=warmup)
    plan.set_field(u0)
    l0 = plan.info()["launches"]
    res = plan.run(dt, steps=steps)
    return res, plan.info()["launches"] - l0


def run_per_config(workloads, peak, peak_src):
    """North-star configs in the same run (device setup), each with its
    roofline and a GPU-vs-oracle digest on the same arrays."""
    import torch

    import paper_2107_03632_b200 as rb
    from paper_2107_03632_b200.solver import Plan

    out = {}
    for name, steps, psteps in workloads:
        t0 = time.perf_counter()
        try:
            nodes, _, shapes = build_problem(name, gpu_setup=True)
        except Exception as exc:  # keep the headline line even if a config cannot be set up
            out[name] = {"error": f"setup: {exc}"}
            continue
        t_setup = time.perf_counter() - t0
        n = int(shapes.weights.shape[1])
        N_i = int(shapes.n_rows)
        dt = 0.5 * rb.stability_bound(shapes)
        interior = shapes.interior_nodes
        plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                    rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
        info = plan.info()
        u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
        res, launches = time_plan(plan, dt, steps, 3, u0)
        torch.cuda.synchronize()
        per_launch = res.device_seconds / steps
        plan.set_field(u0)
        pres = plan.run(dt, steps=psteps)
        gfield = plan.get_field()
        plan.close()
        want = oracle_steps(nodes, shapes, dt, psteps)
        g, o = field_digest(gfield), field_digest(want["field"])
        out[name] = {
            "workload": WORKLOADS[name][3], "N": int(nodes.n_total), "N_i": N_i, "n": n,
            "m": int(shapes.degree), "dt": dt, "steps": steps, "warmup": 3,
            "value": steps * N_i / res.device_seconds, "ms_per_step": 1e3 * per_launch,
            "gpu_launches": launches, "loop": LOOPS[5] if info["persist"] else LOOPS[info["variant"]],
            "roofline": roofline(info, per_launch, peak, peak_src, committed_traffic(name)),
            "parity": {"steps": psteps, "sha256_gpu": g, "sha256_oracle": o, "equal": g == o,
                       "residual_equal": pres.residual == want["residual"]},
            "cpu_port_value": psteps * N_i / want["seconds"],
            "setup": setup_text(True), "setup_seconds": t_setup,
        }
        log(f"[{name}] {out[name]['value']:.4e} upd/s, {1e3 * per_launch:.3f} ms/step, stream frac "
            f"{out[name]['roofline']['frac']:.3f}, parity {g == o} (setup {t_setup:.1f}s)")
        del nodes, shapes, want, gfield
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--gpu-setup", action="store_true",
                    help="headline workload set up on the device (GPU kNN + weights) instead of the host")
    ap.add_argument("--native", action="store_true",
                    help="keep the native (advancing-front) node order instead of Morton renumbering")
    ap.add_argument("--ldg", action="store_true", help="plain-load streaming kernel (no TMA ring)")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=1.0, help="minimum seconds per CPU run")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-rank (torchrun/NCCL) path even with one rank (testing)")
    ap.add_argument("--quick", action="store_true",
                    help="profiling mode: timed region only (no e2e, clock keep-alive, CPU legs, per_config)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args, args.workload)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        from paper_2107_03632_b200 import multigpu

        return multigpu.bench_main(args, METRIC, WORKLOADS)

    import torch

    import paper_2107_03632_b200 as rb
    from paper_2107_03632_b200.solver import Plan

    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    nodes, _, shapes = build_problem(args.workload, gpu_setup=args.gpu_setup)
    t_setup = time.perf_counter() - t0
    n = int(shapes.weights.shape[1])
    N_i = int(shapes.n_rows)
    dt = 0.5 * rb.stability_bound(shapes)
    digest = arrays_digest(nodes, shapes)
    log(f"setup {t_setup:.1f}s: N={nodes.n_total} N_i={N_i} n={n} dt={dt!r} arrays {digest}")

    # ---- CPU legs first (host arrays only): threads=1 / all, min of 3
    legs = None
    if not (args.no_cpu_baseline or args.quick):
        legs = cpu_legs(nodes, shapes, dt, min_seconds=args.cpu_seconds)

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

    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        res, launches = time_plan(plan, dt, args.steps, args.warmup, u0)  # CUDA events, plan stream
        torch.cuda.synchronize()
        # median and min of 5 more timed runs of the same K steps
        # (reported beside `value`, which is the single run above)
        reps = []
        for _ in range(5):
            plan.set_field(u0)
            reps.append(plan.run(dt, steps=args.steps).device_seconds / args.steps)
        torch.cuda.synchronize()
        # keep the GPU busy a little longer so the sampler sees the load (not counted)
        if res.device_seconds < 1.0 and not args.quick:
            extra = int(min(200_000, max(1, args.steps * (1.0 / max(res.device_seconds, 1e-6)))))
            plan.run(dt, steps=extra)
    t = res.device_seconds
    value = args.steps * N_i / t
    per_launch = t / args.steps
    peak, peak_src = measured_peak()
    roof = roofline(info, per_launch, peak, peak_src, committed_traffic(args.workload))
    log(f"device: {t * 1e3:.3f} ms for {args.steps} steps -> {value:.4e} upd/s, streamed "
        f"{roof['achieved']:.0f} GB/s ({roof['frac']:.3f} of {peak_src}); residual {res.residual!r}")

    # ---- parity: the GPU run for the all-thread CPU leg's step count, same arrays
    parity = None
    if legs is not None:
        ref_leg = legs[max(legs)]
        plan.set_field(u0)
        pres = plan.run(dt, steps=ref_leg["steps"])
        g = field_digest(plan.get_field())
        parity = {"steps": ref_leg["steps"], "sha256_gpu": g, "sha256_oracle": ref_leg["digest"],
                  "equal": g == ref_leg["digest"], "residual_equal": pres.residual == ref_leg["residual"],
                  "threads_agree": legs[max(legs)].get("digest_at_1thread_steps", legs[1]["digest"])
                  == legs[1]["digest"]}
        log(f"parity over {ref_leg['steps']} steps: {parity['equal']}")
    plan.close()  # the e2e leg builds its own plan

    # ---- end to end through the public API (host arrays in, host field out)
    cfg = rb.SolveConfig(degree=int(shapes.degree), support_size=n, nodes=int(nodes.n_total),
                         dt=dt, steps=args.steps)
    t_e2e = t_plan = float("nan")
    if not args.quick:
        rb.run_time_loop(cfg, nodes, shapes, renumber=renumber)  # warm (module load, pools)
        torch.cuda.synchronize()
        te = time.perf_counter()
        rep = rb.run_time_loop(cfg, nodes, shapes, renumber=renumber)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - te
        log(f"e2e: {t_e2e * 1e3:.1f} ms (device loop {rep.device_seconds * 1e3:.2f} ms)")
        # the plan upload alone (reported separately): host arrays -> packed device plan
        torch.cuda.synchronize()
        tp = time.perf_counter()
        Plan(nodes.n_total, interior, rows, shapes.weights, f_int,
             nodes.positions if renumber else None, renumber=renumber, device=local).close()
        torch.cuda.synchronize()
        t_plan = time.perf_counter() - tp
    e2e_value = args.steps * N_i / t_e2e
    N = nodes.n_total
    # bytes copied per call: weights, int32 ids (converted in the staging
    # copy), forcing, interior ids, the interior mask, positions (renumbering),
    # the start field; back: the field
    h2d = N_i * (8 * n + 4 * n + 8 + 8) + N + (16 * N if renumber else 0) + 8 * N
    d2h = 8 * N

    cpu = None
    if legs is not None:
        best = legs[max(legs)]
        cpu = {"value": best["value"], "unit": "node-updates/s", "cores": best["threads"], "kind": "port",
               "sample": (f"{best['steps']} full steps of the same workload per run, min of 3 runs "
                          f"({best['seconds_min']:.2f} s); oracle/ C port of solver.py:294-311, bitwise equal "
                          f"to the numba kernel, OpenMP over 1024-row chunks"),
               "threads_1": {"value": legs[1]["value"], "steps": legs[1]["steps"],
                             "seconds_min": legs[1]["seconds_min"]},
               "threads_all": {"value": best["value"], "threads": best["threads"], "steps": best["steps"],
                               "seconds_min": best["seconds_min"]},
               "repeats": 3, "cpu": cpu_info()}

    per_config = None
    if args.workload == "c2" and not (args.quick or args.no_per_config):
        per_config = run_per_config(PER_CONFIG, peak, peak_src)

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
        "data": DATA,
        "config": common_config(args.workload, nodes, shapes, dt, digest),
        "impl_config": {
            "setup": setup_text(args.gpu_setup),
            "renumber": "morton (bit-identical)" if renumber else "native (advancing-front order)",
            "loop": (LOOPS[5] if info["persist"] else
                     LOOPS[info["variant"]] + ("" if args.no_pdl or info["resident"] else " + PDL")),
            "index_bits": info["index_bits"],
            "parallelism": "single GPU",
        },
        "roofline": roof,
        "e2e": {"value": e2e_value if math.isfinite(e2e_value) else None, "unit": "node-updates/s",
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "what": "run_time_loop(config, nodes, shapes) from host numpy arrays: plan build + H2D "
                        "(weights, ids, forcing, positions, field), K steps, D2H field, error norms",
                "plan_upload_ms": 1e3 * t_plan if math.isfinite(t_plan) else None},
        "timing_repeats": {"runs": len(reps), "steps_each": args.steps,
                           "median_ms_per_step": 1e3 * statistics.median(reps),
                           "min_ms_per_step": 1e3 * min(reps)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "setup_seconds": t_setup,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if parity is not None:
        line["parity"] = parity
    if per_config is not None:
        line["per_config"] = per_config
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
