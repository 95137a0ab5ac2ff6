"""bench.py -- RTCUR on B200 (BASELINE.json metric: RTCUR iters/sec & sec-to-tol).

Default workload (N=1): BASELINE config 1 -- RTCUR-R, 400^3 float64, ranks
(5,5,5), Bernoulli(0.3) outliers c=10, eps=1e-5, max_iters=100, BASELINE
sample sizes |I|=90, |J|=2693 (seeded synthetic instance, paper_2108_10448_b200.synth).

A *step* is one complete solve to tolerance (``rtcur(x, cfg)``) with X
resident in HBM; ``value`` = iterations/sec over the K timed solves (sum of
iterations / device time), ``ms_per_step`` = seconds-to-tolerance.  X is
512 MB > the 126 MB L2, so no explicit flush is needed between steps.

``e2e``: the same metric through the public API with HOST buffers: each step
copies X from pinned host memory to HBM, solves, and materialises the full
SolveResult on the host (sparse blocks, FiberCur pieces).

``--impl reference`` times the CPU port of the reference loop (oracle/, the
reference itself is Python and cannot be installed as a GPU-box baseline) on
the host cores: one step = one steady-state RTCUR-R iteration of the same
config.

Multi-GPU (torchrun, N>1): config 1 does not shard (BASELINE runs it on one
GPU), so N ranks run N independent replicas ("scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RTCUR iters/sec & sec-to-tol (eps=1e-5) per config; achieved HBM GB/s vs B200 peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _make_problem(config: int):
    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config

    xf, low, _, bc = make_config(config)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    return xf, low, bc, rows, cols


def _algorithmic_bytes(bc, rows, cols):
    """Per-launch algorithmic bytes of each HBM-bound phase."""
    E = 8 if bc.dtype == "f64" else 4
    n_core = int(np.prod(rows))
    n_fib = sum(d * c for d, c in zip(bc.shape, cols))
    n_blk = n_core + n_fib
    inter = sum(r * c for r, c in zip(rows, cols))
    return {
        "gather": 2 * E * n_blk + E * inter,  # read the sampled X entries, write the blocks + X(I_k, J_k) copies
        "threshold": (E + 8) * inter,         # read the X(I_k, J_k) copies, write the fp64 intersections M_k
        "error": E * n_blk,                   # read blocks
        "apass": E * n_fib,                   # read fiber blocks
        "gpass": E * n_core,                  # read core block
    }, n_blk


FP64_PEAK_TFMA = 18.5   # measured fp64 FMA-pipe rate (DFMA and DMMA share it): profiles/r01_fp64_pipes.txt


def _fp64_fmas(bc, rows, cols):
    """Per-launch fp64 FMAs of the fiber-pass phases (the reconstruction L = A_k(I,:) W_k(:, j)
    is r_k FMAs per entry and state): error = 2 r_k + 2 per block entry (previous and new
    iterate, two sums; the core rides with mode 1), A pass = 2 r_k per fiber entry (previous
    iterate + the C V accumulation), threshold = r_k per intersection entry."""
    n_core = int(np.prod(rows))
    fib = [d * c for d, c in zip(bc.shape, cols)]
    inter = [r * c for r, c in zip(rows, cols)]
    rk = list(bc.ranks)
    return {
        "error": n_core * (2 * rk[0] + 2) + sum(f * (2 * r + 2) for f, r in zip(fib, rk)),
        "apass": sum(f * 2 * r for f, r in zip(fib, rk)),
        "threshold": sum(i * r for i, r in zip(inter, rk)),
    }


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle import rtcur_oracle as orc

    orc.build_oracle_lib()
    xf, _, bc, rows, cols = _make_problem(args.config)
    x64 = xf.astype(np.float64)
    n_iters = args.warmup + args.steps
    t0 = time.perf_counter()
    res = orc.solve(x64, bc.shape, bc.ranks, eps=bc.eps, variant=bc.variant, max_iters=n_iters, seed=bc.seed_solver,
                    row_sample_sizes=rows, col_sample_sizes=cols)
    wall = time.perf_counter() - t0
    its = res.iter_times
    timed = its[args.warmup:args.warmup + args.steps]
    if len(timed) < args.steps:   # converged early: time the trailing iterations available
        timed = its[-args.steps:]
    value = len(timed) / sum(timed)
    cores = os.cpu_count()
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "impl": "reference", "n_gpus": world,
        "steps": len(timed), "warmup": args.warmup, "ms_per_step": 1e3 * sum(timed) / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": bc.dtype,
        "data": "synthetic (seeded, paper_2108_10448_b200.synth)",
        "config": _config_dict(bc, rows, cols, world),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": f"RTCUR-{bc.variant} iterations {args.warmup + 1}..{args.warmup + len(timed)} of "
                                   f"config {bc.index} on the host (numpy/OpenBLAS all cores; einsum and SVD "
                                   f"single-threaded as in the reference)"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(bc, rows, cols, world, shard=False):
    return {"workload": f"config{bc.index}: RTCUR-{bc.variant} {'x'.join(map(str, bc.shape))} {bc.dtype} ranks "
                        f"{tuple(bc.ranks)} alpha={bc.alpha} c={bc.c} eps={bc.eps} max_iters=100",
            "shape": list(bc.shape), "ranks": list(bc.ranks), "variant": bc.variant, "row_samples": list(rows),
            "col_samples": list(cols), "l2": "inputs larger than L2 (X = %.0f MB > 126 MB)" % (
                np.prod(bc.shape) * (8 if bc.dtype == "f64" else 4) / 1e6),
            "parallelism": (f"mode-1 slabs x{world} (NCCL all-reduce of the sampled blocks)" if shard else
                            f"replicas x{world}" if world > 1 else "single GPU")}


def _cpu_baseline(bc, rows, cols, xf, budget_iters=2):
    from oracle import rtcur_oracle as orc

    orc.build_oracle_lib()
    res = orc.solve(xf.astype(np.float64), bc.shape, bc.ranks, eps=bc.eps, variant=bc.variant,
                    max_iters=budget_iters, seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
    t = res.iter_times[-1]
    return {"value": 1.0 / t, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"iteration {len(res.iter_times)} (steady state, both _eval_blocks) of a config-{bc.index} "
                      f"RTCUR-{bc.variant} solve by the oracle port on the host; setup (sample+gather) "
                      f"{res.timings['gather'] + res.timings['sample']:.2f}s excluded"}


def _ncu_traffic(config: int, phase: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None when that capture does not exist."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    return d.get(f"config{config}", {}).get(phase)


def _full_tensor_rooflines(res, x_dev, bc, phases, peak, steps):
    """K3 (k_full: full L, S = HT(X - L, zeta_final) and the residual sums,
    cli.py:237-243) and K0 (k_absmax, solver.py:184-192) against the HBM peak.
    K3 runs `steps` times on the solved iterate with CUDA events on the engine's
    stream around the kernel (the Tf contraction it needs is a separate ~us
    launch); algorithmic bytes 3*E*N_local (read X, write L and S), K0 E*N_local."""
    import torch
    from paper_2108_10448_b200.full import full_output

    eng = res.cur._engine
    E = 8 if bc.dtype == "f64" else 4
    n_loc = int(x_dev.flat.numel())
    full_output(res, x_dev)   # warm (allocator, Tf scratch)
    torch.cuda.synchronize()
    eng.profile(True, ["full"])
    eng.profile_read(reset=True)
    rel = None
    for _ in range(max(1, steps)):
        _, _, rel = full_output(res, x_dev)
    ph = eng.profile_read(reset=True)
    eng.profile(False)
    ms, n = ph["full"]
    k3_us = 1e3 * ms / max(n, 1)
    k3_bytes = 3 * E * n_loc
    out = {"k3_full": {"bound": "hbm", "kernel": "k_full", "alg_bytes_per_launch": k3_bytes,
                       "launch_us": k3_us, "launches_timed": int(n),
                       "achieved": k3_bytes / (k3_us * 1e-6) / 1e9, "peak": peak, "unit": "GB/s",
                       "frac": k3_bytes / (k3_us * 1e-6) / 1e9 / peak, "full_relative_residual": rel}}
    if "absmax" in phases:
        k0_us = 1e3 * phases["absmax"]["ms_per_step"] / max(phases["absmax"]["launches_per_step"], 1)
        out["k0_absmax"] = {"bound": "hbm", "kernel": "k_absmax", "alg_bytes_per_launch": E * n_loc,
                            "launch_us": k0_us, "achieved": E * n_loc / (k0_us * 1e-6) / 1e9, "peak": peak,
                            "unit": "GB/s", "frac": E * n_loc / (k0_us * 1e-6) / 1e9 / peak}
    return out


def _sharded(config: int) -> bool:
    """BASELINE shards configs 2 and 4 in mode-1 slabs; the others run replicas."""
    return config in (2, 4)


def run_b200(args):
    import torch

    world, rank, local = _dist()
    group = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    torch.cuda.set_device(local)
    from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
    from paper_2108_10448_b200 import _native
    from paper_2108_10448_b200 import solver as solver_mod
    from paper_2108_10448_b200.dist import rtcur_sharded
    from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes, make_config_device, slab_bounds

    bc = CONFIGS[args.config]
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    dt = torch.float64 if bc.dtype == "f64" else torch.float32
    shard = _sharded(args.config) and world > 1
    slab = slab_bounds(bc.shape[0], world, rank) if shard else None
    xf = None
    if args.config <= 1:
        xf, _, bc, rows, cols = _make_problem(args.config)
        host = torch.from_numpy(xf).to(dt)
        x_dev = DeviceTensor(host.cuda(), bc.shape)
    else:
        x_dev, _ = make_config_device(args.config, slab=slab, group=group if shard else None)
        host = None
    cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=100,
                       seed=bc.seed_solver + (0 if shard else 1000 * rank), row_sample_sizes=rows,
                       col_sample_sizes=cols)

    def solve(x):
        if shard:
            return rtcur_sharded(x, bc.shape, slab, cfg, group=group)
        return rtcur(x, cfg)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        solve(x_dev)
    torch.cuda.synchronize()

    # ---------------- per-phase breakdown: one profiled pass (every phase timed), outside the timed region
    peak, peak_src = _peaks()
    alg, n_blk = _algorithmic_bytes(bc, rows, cols)
    if shard:   # the slab gather reads only this rank's entries; the other passes work on the full blocks
        alg["gather"] = alg["gather"] // 2 + alg["gather"] // 2 // world
    solver_mod.PROFILE, solver_mod.PROFILE_PHASES = True, None
    bd_steps = max(1, min(args.steps, 2))
    phase_ms, phase_n = {}, {}
    res = None
    for _ in range(bd_steps):
        res = None   # one engine throughout: the previous result returns it to the pool
        res = solve(x_dev)
        for k, v in res.timings["device_ms"].items():
            phase_ms[k] = phase_ms.get(k, 0.0) + v
            phase_n[k] = phase_n.get(k, 0) + res.timings["device_launches"][k]
    torch.cuda.synchronize()
    total_dev = sum(phase_ms.values())
    hbm_phases = {k: v for k, v in phase_ms.items() if k in alg and phase_n.get(k)}
    dom = max(hbm_phases, key=hbm_phases.get)
    phases = {k: {"ms_per_step": v / bd_steps, "launches_per_step": phase_n[k] / bd_steps,
                  "share": v / total_dev if total_dev else None}
              for k, v in sorted(phase_ms.items(), key=lambda kv: -kv[1]) if phase_n.get(k)}

    # ---------------- device-resident timed region (only the dominant HBM phase carries CUDA events)
    solver_mod.PROFILE_PHASES = (dom,)
    res = None
    solve(x_dev)   # untimed: the engine's per-iteration CUDA graphs for this profiling setting exist now
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    iters, conv, dom_ms, dom_n = 0, True, 0.0, 0
    for _ in range(args.steps):
        res = None
        res = solve(x_dev)
        iters += res.iterations
        conv &= res.converged
        dom_ms += res.timings["device_ms"][dom]
        dom_n += res.timings["device_launches"][dom]
    ev1.record()
    res_dev = res
    torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - l0
    clk = clocks.stop()
    solver_mod.PROFILE, solver_mod.PROFILE_PHASES = False, None
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    it = torch.tensor([iters], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        if not shard:   # replicas: every rank's iterations count; sharded: one solve spans all ranks
            torch.distributed.all_reduce(it, op=torch.distributed.ReduceOp.SUM)
    ms_max = float(t.item())
    value = float(it.item()) / (ms_max / 1e3)

    # K3 / K0 rooflines on the timed solve's iterate (before the e2e loop, so that loop
    # recycles the warmed-up engines instead of building a new one)
    full_roof = _full_tensor_rooflines(res_dev, x_dev, bc, phases, peak, args.steps)
    del res_dev, res

    # ---------------- e2e through the public API with host buffers
    if host is None:
        host = x_dev.flat.cpu()
    pinned = host.pin_memory()
    x_buf = torch.empty_like(x_dev.flat)
    e2e_iters, d2h = 0, 0
    e2e_steps = max(1, args.steps if args.config <= 1 else min(args.steps, 2))
    # untimed warm-up of the host-buffer path: the exports' pinned staging buffer and
    # the result arrays' first touch are one-time costs (~0.2 s at config 1)
    res = None
    x_buf.copy_(pinned, non_blocking=True)
    res = solve(DeviceTensor(x_buf, x_dev.shape))
    _ = (res.sparse.core, res.sparse.fibers, res.cur.core, res.cur.fibers, res.cur.intersections, res.cur.factors)
    del _
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        x_buf.copy_(pinned, non_blocking=True)
        res = None   # the previous result returns its engine to the pool
        res = solve(DeviceTensor(x_buf, x_dev.shape))
        e2e_iters += res.iterations
        sc = res.sparse.core
        sf = res.sparse.fibers
        core = res.cur.core
        fib = res.cur.fibers
        inters = res.cur.intersections
        facs = res.cur.factors
        d2h = (sc.nbytes + sum(f.nbytes for f in sf) + core.data.nbytes + sum(f.nbytes for f in fib)
               + sum(i.u.nbytes + i.v.nbytes + i.singular_values.nbytes for i in inters)
               + sum(f.nbytes for f in facs) + 8 * res.iterations)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    ie = torch.tensor([e2e_iters], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        if not shard:
            torch.distributed.all_reduce(ie, op=torch.distributed.ReduceOp.SUM)
    e2e_value = float(ie.item()) / float(te.item())

    # ---------------- roofline of the dominant HBM-bound kernel (events from the timed region)
    per_launch_ms = dom_ms / max(dom_n, 1)
    achieved = alg[dom] / (per_launch_ms / 1e3) / 1e9
    kname = {"threshold": "k_fiber_pass (threshold over X(I_k, J_k))", "error": "k_fiber_pass (error: core + fibers)",
             "gather": "k_gather_fibers + k_gather", "apass": "k_fiber_pass (A pass) + k_fiber_areduce",
             "gpass": "k_block_pass (G pass)"}[dom]
    traffic = _ncu_traffic(args.config, dom)
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "traffic_source": traffic.get("source") if traffic else None,
            "alg_bytes_per_launch": alg[dom], "launch_us": 1e3 * per_launch_ms, "launches_timed": dom_n,
            "peak_source": peak_src,
            "share_of_device_time": phases[dom]["share"] if dom in phases else None}
    fmas = _fp64_fmas(bc, rows, cols)
    if dom in fmas:   # the same launch against the fp64 pipe (the fiber passes sit near the ridge)
        tf = fmas[dom] / (per_launch_ms / 1e3) / 1e12
        roof["fp64"] = {"achieved": tf, "peak": FP64_PEAK_TFMA, "unit": "TFMA/s", "frac": tf / FP64_PEAK_TFMA,
                        "fma_per_launch": fmas[dom],
                        "peak_source": "measured: tools/fp64_pipes.cu (profiles/r01_fp64_pipes.txt)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if xf is not None:
            cpu = _cpu_baseline(bc, rows, cols, xf)
        else:
            cpu = {"value": None, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"not run for config {bc.index}: one CPU iteration of the port takes minutes "
                             "(SURVEY §6: ~12 min/iter config 2, ~91 s config 3, ~6.5 s config 4)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": bc.dtype,
            "data": "synthetic (seeded, paper_2108_10448_b200.synth)",
            "config": _config_dict(bc, rows, cols, world, shard),
            "sec_to_tol": ms_max / args.steps / 1e3, "iterations_per_solve": iters / args.steps,
            "converged": bool(conv), "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": int(host.numel() * host.element_size()),
                    "d2h_bytes_per_step": int(d2h), "sec_per_solve": e2e_s / e2e_steps},
            "roofline": roof, "full_tensor_rooflines": full_roof, "phases": phases,
            "phases_note": f"per-phase CUDA-event times from a separate profiled pass of {bd_steps} solve(s); "
                           "the timed region carries events on the dominant phase only",
            "clocks": clk, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
