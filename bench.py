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

``parity``: the timed solve against the real reference's solve of the same
instance (tests/golden/cfg1_summary.npz).  ``per_config``: configs 0, 2, 3, 4
measured the same way (3 solves each) with their phase HBM fractions.

``--impl reference`` times the REAL reference package (oracle/_ref, built by
oracle/build_ref.sh from /root/reference/pkg with its Cython backend) through
its public rtcur() API on the host cores: one step = one RTCUR iteration
(steady-state iterations W+1..W+K of the same config's solve); it falls back to
the oracle port only when oracle/_ref is missing.

Multi-GPU (torchrun, N>1): config 4 by default, sharded in mode-1 slabs
(``"scaling": "strong"``, all-gather of the owned sampled entries); an
explicit ``--config 0|1|3`` runs N independent replicas (``"weak"``).
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
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    The sampler is started well before the timed region (nvidia-smi's own start-up
    attaches to the driver for tens of milliseconds and was seen stalling graph
    launches when it fell inside a short region); ``begin()`` / ``stop()`` bracket
    the region and only the samples that arrived inside it (plus one polling period)
    are reported."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t_begin = None

    def wait_ready(self, timeout: float = 5.0):
        """nvidia-smi is past its start-up once its first sample has arrived."""
        t_wait = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t_wait < timeout:
            time.sleep(0.01)

    def begin(self):
        self.t_begin = time.perf_counter()

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS") == "1":   # diagnostics only: no nvidia-smi polling
            return
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
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t_end = time.perf_counter()
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        t_b = self.t_begin if self.t_begin is not None else 0.0
        inside = [ln for (t, ln) in self.lines if t_b <= t <= t_end + 0.12]
        if not inside:   # a region shorter than the polling period: the samples around it
            inside = [ln for (t, ln) in self.lines if t >= t_b - 0.12]
        for ln in inside:
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
        "factors": sum(f * 2 * r for f, r in zip(fib, rk)) + n_core * 2 * rk[0],
        "threshold": sum(i * r for i, r in zip(inter, rk)),
    }


def _default_config(args, world: int) -> int:
    """config 1 (BASELINE's single-GPU headline) at N=1; config 4 (mode-1 slabs,
    BASELINE's sharded R config) under torchrun."""
    if args.config is not None:
        return int(args.config)
    return 1 if world == 1 else 4


def _host_problem(config: int):
    """(bc, rows, cols, x64 flat F-order) -- configs 0-1 from the host generator,
    2-4 from the device generator copied back (exact fp32 -> fp64)."""
    from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes, make_config

    bc = CONFIGS[config]
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    if config <= 1 or bc.kind == "video":
        xf, _, _, bc = make_config(config)
        return bc, rows, cols, xf.astype(np.float64)
    import torch

    from paper_2108_10448_b200.synth import make_config_device

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    x_dev, bc = make_config_device(config)
    x64 = x_dev.flat.cpu().numpy().astype(np.float64)
    del x_dev
    torch.cuda.empty_cache()
    return bc, rows, cols, x64


def _reference_sample(bc, rows, cols, x64, warmup: int, steps: int):
    """Time the REAL reference (oracle/_ref: rtcur with its compiled Cython backend,
    driven through its public rtcur()/TensorAccessor API) on iterations
    warmup+1 .. warmup+steps of this config's solve.  Falls back to the oracle
    port (kind "port", its einsum evaluation = the reference's cost) when
    oracle/_ref was not built."""
    from oracle import ref_runner

    kw = dict(eps=bc.eps, variant=bc.variant, max_iters=warmup + steps, seed=bc.seed_solver,
              row_sample_sizes=rows, col_sample_sizes=cols)
    if ref_runner.available():
        res, info = ref_runner.run(x64, bc.shape, bc.ranks, **kw)
        its = info["iter_times"]
        kind = "reference"
        what = ("the reference package itself (oracle/_ref, built from /root/reference/pkg by oracle/build_ref.sh; "
                "RTCUR_BACKEND=compiled), rtcur.rtcur() through its TensorAccessor API")
        extra = {"error_history": info["error_history"], "iterations": res.iterations,
                 "s_core_support_sha256": info["s_core_support_sha256"], "backend": info["backend"],
                 "setup_s": info["setup_s"], "wall_s": info["wall_s"]}
    else:
        from oracle import rtcur_oracle as orc

        orc.build_oracle_lib()
        r = orc.solve(x64, bc.shape, bc.ranks, eval_mode="einsum", **kw)
        its = list(r.iter_times)
        kind = "port"
        what = "the oracle port (oracle/rtcur_oracle.py, einsum evaluation as the reference) -- oracle/_ref missing"
        extra = {"error_history": list(r.error_history), "iterations": r.iterations, "wall_s": sum(its)}
    timed = [t for t in its[warmup:warmup + steps] if t is not None]
    if len(timed) < steps:   # converged early / untimed first iteration: the trailing timed iterations
        timed = [t for t in its if t is not None][-steps:]
    value = len(timed) / sum(timed)
    first = len(its) - len(timed) + 1 if len(timed) < steps else warmup + 1
    sample = (f"RTCUR-{bc.variant} iterations {first}..{first + len(timed) - 1} of config {bc.index} "
              f"({'x'.join(map(str, bc.shape))}) on the host: {what}; numpy/OpenBLAS on all host threads, einsum "
              f"and the Cython kernels single-threaded as in the reference")
    return {"value": value, "unit": "iters/s", "cores": os.cpu_count(), "kind": kind, "sample": sample,
            "ms_per_iteration": 1e3 * sum(timed) / len(timed), "iterations_timed": len(timed)}, extra


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:   # the CPU reference runs once per box (rank 0)
        return 0
    config = _default_config(args, world)
    bc, rows, cols, x64 = _host_problem(config)
    t0 = time.perf_counter()
    cpu, extra = _reference_sample(bc, rows, cols, x64, args.warmup, args.steps)
    wall = time.perf_counter() - t0
    line = {
        "metric": METRIC, "value": cpu["value"], "unit": "iters/s", "impl": "reference", "n_gpus": world,
        "steps": cpu["iterations_timed"], "warmup": args.warmup, "ms_per_step": cpu["ms_per_iteration"],
        "higher_is_better": True, "scaling": "strong" if (world > 1 and _sharded(config)) else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, paper_2108_10448_b200.synth)",
        "config": _config_dict(bc, rows, cols, 1),
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_run": extra, "wall_s": wall,
        "step_note": "one step = one RTCUR iteration of the reference's solve (a full GPU-arm step is a whole "
                     "solve; iters/s is the common unit)",
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(bc, rows, cols, world, shard=False):
    return {"workload": f"config{bc.index}: RTCUR-{bc.variant} {'x'.join(map(str, bc.shape))} {bc.dtype} ranks "
                        f"{tuple(bc.ranks)} alpha={bc.alpha} c={bc.c} eps={bc.eps} max_iters=100",
            "shape": list(bc.shape), "ranks": list(bc.ranks), "variant": bc.variant, "row_samples": list(rows),
            "col_samples": list(cols), "l2": "inputs larger than L2 (X = %.0f MB > 126 MB)" % (
                np.prod(bc.shape) * (8 if bc.dtype == "f64" else 4) / 1e6),
            "parallelism": (f"mode-1 slabs x{world} (one all-gather of the owned sampled entries per sample)" if shard else
                            f"replicas x{world}" if world > 1 else "single GPU")}


def _cpu_baseline(bc, rows, cols, x64):
    """Reported CPU baseline for the b200 arm's line: the real reference on
    iterations 2..3 of the same solve (a bounded sample, ~30 s on the box)."""
    cpu, _ = _reference_sample(bc, rows, cols, x64, 1, 2)
    return cpu


def _parity_block(config: int, res):
    """The timed solve against the REAL reference's solve of the same instance
    (tests/golden/cfg1_summary.npz, tests/golden/make_cfg1_golden.py): error
    history (1e-10 abs), iteration count, final S support of the core block
    (bit-exact) and singular values (1e-10 rel).  Config 1 only."""
    p = os.path.join(ROOT, "tests", "golden", f"cfg{config}_summary.npz")
    if not os.path.exists(p):
        return None
    g = np.load(p)
    eh = np.asarray(res.error_history)
    ref_eh = np.asarray(g["error_history"])
    same_len = eh.size == ref_eh.size
    err_diff = float(np.max(np.abs(eh - ref_eh))) if same_len else None
    core = np.asarray(res.sparse.core).reshape(-1, order="F")
    supp = bool(np.array_equal(np.packbits(core != 0), g["s_core_bits"]))
    sv = max(float(np.max(np.abs(res.cur.intersections[m].singular_values - g[f"sv{m}"]) / g[f"sv{m}"][0]))
             for m in range(len(res.cur.indices.rows)))
    ok = bool(same_len and err_diff <= 1e-10 and supp and sv <= 1e-10 and res.converged == bool(g["converged"]))
    return {"vs": "the real reference's solve of this instance (tests/golden/cfg1_summary.npz)", "ok": ok,
            "iterations": [int(res.iterations), int(g["iterations"])], "error_history_max_abs_diff": err_diff,
            "s_core_support_equal": supp, "sigma_max_rel_diff": sv,
            "full_record": "profiles/r02_parity_config*.json (tools/parity_configs.py, per-iteration lockstep)"}


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
        # K0 on its own, events around the scan (inside a solve it shares the GPU with the
        # mode-k copies an RTCUR-R solve builds on the side stream while zeta_0 is scanned)
        eng.profile(True, ["absmax"])
        eng.profile_read(reset=True)
        for _ in range(max(1, min(steps, 5))):
            eng.absmax()
        ph0 = eng.profile_read(reset=True)
        eng.profile(False)
        ms0, n0 = ph0["absmax"]
        k0_us = 1e3 * ms0 / max(n0, 1)
        out["k0_absmax"] = {"bound": "hbm", "kernel": "k_absmax", "alg_bytes_per_launch": E * n_loc,
                            "launch_us": k0_us, "launches_timed": int(n0),
                            "achieved": E * n_loc / (k0_us * 1e-6) / 1e9, "peak": peak,
                            "unit": "GB/s", "frac": E * n_loc / (k0_us * 1e-6) / 1e9 / peak,
                            "in_solve_launch_us": 1e3 * phases["absmax"]["ms_per_step"]
                            / max(phases["absmax"]["launches_per_step"], 1)}
    return out


def _sharded(config: int) -> bool:
    """BASELINE shards configs 2 and 4 in mode-1 slabs; the others run replicas."""
    return config in (2, 4)


def _per_config(configs, local: int, peak: float, steps: int = 3):
    """Compact single-GPU measurements of the other BASELINE configs: iters/s and
    seconds-to-tolerance over `steps` device-resident solves (CUDA events, one
    warm-up solve), the HBM fraction of every sampled-block phase from one
    profiled solve (events around each phase), K3 / K0 fractions, clocks."""
    import torch

    from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
    from paper_2108_10448_b200 import solver as solver_mod
    from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes, make_config_device

    out = {}
    clocks = ClockSampler(local)
    clocks.start()
    for c in configs:
        bc = CONFIGS[c]
        rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
        if c <= 1:
            xf, _, bc, rows, cols = _make_problem(c)
            x_dev = DeviceTensor(torch.from_numpy(xf).cuda(), bc.shape)
        else:
            x_dev, _ = make_config_device(c)
        cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=100,
                           seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
        solver_mod.PROFILE, solver_mod.PROFILE_PHASES = True, None
        res = rtcur(x_dev, cfg)   # warm (engine) + the profiled breakdown pass
        res = None
        res = rtcur(x_dev, cfg)
        solver_mod.PROFILE = False
        dm, dn = res.timings["device_ms"], res.timings["device_launches"]
        total_dev = sum(dm.values())
        alg, _ = _algorithmic_bytes(bc, rows, cols)
        fr = {}
        for ph, b in alg.items():
            if dn.get(ph):
                us = 1e3 * dm[ph] / dn[ph]
                fr[ph] = {"frac": b / (us * 1e-6) / 1e9 / peak, "launch_us": us, "alg_bytes_per_launch": b,
                          "share": dm[ph] / total_dev}
                tr = _ncu_traffic(c, ph)
                if tr:
                    fr[ph]["traffic"] = tr["bytes_per_launch"]
                    fr[ph]["traffic_frac"] = tr["bytes_per_launch"] / (us * 1e-6) / 1e9 / peak
        if "apass" in fr and "gpass" in fr and os.environ.get("RTCUR_AG_FORK", "1") != "0":
            # parallel branches of the iteration's graph: one phase, both passes' bytes over
            # the longer interval (see run_b200)
            a_, g_ = fr.pop("apass"), fr.pop("gpass")
            us = max(a_["launch_us"], g_["launch_us"])
            b = a_["alg_bytes_per_launch"] + g_["alg_bytes_per_launch"]
            fr["factors"] = {"frac": b / (us * 1e-6) / 1e9 / peak, "launch_us": us, "alg_bytes_per_launch": b,
                             "share": max(a_["share"], g_["share"]), "phases": ["apass", "gpass"]}
            if "traffic" in a_ and "traffic" in g_:
                fr["factors"]["traffic"] = a_["traffic"] + g_["traffic"]
                fr["factors"]["traffic_frac"] = fr["factors"]["traffic"] / (us * 1e-6) / 1e9 / peak
        shares = {k: round(v / total_dev, 4) for k, v in sorted(dm.items(), key=lambda kv: -kv[1]) if dn.get(k)}
        phases = {"absmax": {"ms_per_step": dm["absmax"], "launches_per_step": dn["absmax"]}} if dn.get("absmax") \
            else {}
        full = _full_tensor_rooflines(res, x_dev, bc, phases, peak, 1)
        res = None
        res = rtcur(x_dev, cfg)   # untimed: per-iteration graphs without profiling events
        res = None
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters, conv = 0, True
        ev0.record()
        for _ in range(steps):
            res = None
            res = rtcur(x_dev, cfg)
            iters += res.iterations
            conv &= res.converged
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        out[str(c)] = {"workload": _config_dict(bc, rows, cols, 1)["workload"], "iters_per_s": iters / (ms / 1e3),
                       "ms_per_solve": ms / steps, "iterations_per_solve": iters / steps, "converged": bool(conv),
                       "hbm_phases": fr, "device_time_shares": shares,
                       "k3_full_frac": full["k3_full"]["frac"], "k0_absmax_frac": full.get("k0_absmax", {}).get("frac")}
        res = None
        del x_dev
        torch.cuda.empty_cache()
    out["clocks"] = clocks.stop()
    out["note"] = (f"{steps} timed device-resident solves per config after one warm-up; phase fractions from one "
                   "profiled solve; alg bytes per DESIGN.md §3")
    return out


def run_b200(args):
    import torch

    world, rank, local = _dist()
    group = None
    # NCCL over NVLink; RTCUR_BENCH_BACKEND=gloo exercises the N > 1 code path with
    # all ranks on however many devices exist (validation on a one-GPU box)
    backend = os.environ.get("RTCUR_BENCH_BACKEND", "nccl")
    device = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    torch.cuda.set_device(device)
    local = device
    red_dev = "cuda" if backend == "nccl" else "cpu"
    from paper_2108_10448_b200 import DeviceTensor, SolverConfig, rtcur
    from paper_2108_10448_b200 import _native
    from paper_2108_10448_b200 import solver as solver_mod
    from paper_2108_10448_b200.dist import rtcur_sharded
    from paper_2108_10448_b200.synth import CONFIGS, baseline_sample_sizes, make_config_device, slab_bounds

    config = _default_config(args, world)
    bc = CONFIGS[config]
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    dt = torch.float64 if bc.dtype == "f64" else torch.float32
    shard = _sharded(config) and world > 1
    slab = slab_bounds(bc.shape[0], world, rank) if shard else None
    xf = None
    if config <= 1:
        xf, _, bc, rows, cols = _make_problem(config)
        host = torch.from_numpy(xf).to(dt)
        x_dev = DeviceTensor(host.cuda(), bc.shape)
    else:
        x_dev, _ = make_config_device(config, slab=slab, group=group if shard else None)
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
    clocks = ClockSampler(local)   # started early: see ClockSampler
    clocks.start()
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
    # The A pass (+ reduce) and the G pass (+ mode products) are two parallel branches of the
    # iteration's graph: their event intervals start at the same fork and
    # overlap, so they are one phase here -- "factors": both passes' bytes over the longer of
    # the two intervals.
    merged = {}
    if (os.environ.get("RTCUR_AG_FORK", "1") != "0" and os.environ.get("RTCUR_GRAPHS", "1") != "0"
            and "apass" in hbm_phases and "gpass" in hbm_phases):
        merged["factors"] = ("apass", "gpass")
        alg["factors"] = alg["apass"] + alg["gpass"]
        phase_n["factors"] = max(phase_n["apass"], phase_n["gpass"])
        hbm_phases["factors"] = max(hbm_phases.pop("apass"), hbm_phases.pop("gpass"))
    # The roofline goes to the HBM-bound pass with the most device time ON THE ITERATION'S
    # STREAM (its critical path).  An RTCUR-R solve stages its next sample (prep + gather) on a
    # side stream under the eigensolver, so its events time it while it shares the GPU: it is
    # listed in k1_rooflines (concurrent_with_iteration) but does not carry the headline.
    # Likewise the error pass when the engine holds an iteration's tail back and runs it under
    # the next iteration's eigensolver (always for RTCUR-F, for RTCUR-R while
    # the sampled blocks are <= 48 MB; one process per GPU only -- a sharded solve runs its
    # iterations one at a time).
    tail_deferred = (not shard) and os.environ.get("RTCUR_SPECULATE", "1") != "0" and (
        os.environ["RTCUR_TAIL_DEFER"] != "0" if "RTCUR_TAIL_DEFER" in os.environ
        else (bc.variant != "R" or n_blk * (8 if bc.dtype == "f64" else 4) <= (48 << 20)))
    off_path = {"gather"} if bc.variant == "R" else set()
    if tail_deferred:
        off_path.add("error")
    on_path = {k: v for k, v in hbm_phases.items() if k not in off_path} or hbm_phases
    dom = max(on_path, key=on_path.get)
    k1_roof = {k: {"alg_bytes_per_launch": alg[k], "launch_us": 1e3 * v / phase_n[k],
                   "frac": alg[k] / (v / phase_n[k] / 1e3) / 1e9 / peak,
                   "launches_per_step": phase_n[k] / bd_steps,
                   "concurrent_with_iteration": k in off_path}
               for k, v in hbm_phases.items()}
    for k, v in k1_roof.items():   # DRAM bytes ncu counted for the phase's kernels (committed capture)
        tr = _ncu_traffic(config, k)
        if k in merged:
            parts = [_ncu_traffic(config, m) for m in merged[k]]
            tr = {"bytes_per_launch": sum(p_["bytes_per_launch"] for p_ in parts)} if all(parts) else None
            v["phases"] = list(merged[k])
        if tr:
            v["traffic"] = tr["bytes_per_launch"]
            v["traffic_frac"] = tr["bytes_per_launch"] / (v["launch_us"] * 1e-6) / 1e9 / peak
    phases = {k: {"ms_per_step": v / bd_steps, "launches_per_step": phase_n[k] / bd_steps,
                  "share": v / total_dev if total_dev else None}
              for k, v in sorted(phase_ms.items(), key=lambda kv: -kv[1]) if phase_n.get(k)}

    # ---------------- device-resident timed region (only the dominant HBM phase carries CUDA events)
    solver_mod.PROFILE_PHASES = merged.get(dom, (dom,))
    res = None
    clocks.wait_ready()
    solve(x_dev)   # untimed: the engine's per-iteration CUDA graphs for this profiling setting exist now
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks.begin()
    l0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    iters, conv, dom_ms, dom_n = 0, True, 0.0, 0
    # the roofline phase carries its CUDA events on every 4th solve of the timed region: two
    # event-record nodes on the iteration's critical path cost ~8 us each (config 1: 7.5 vs
    # 7.0 ms per solve with them in every iteration), and 1/4 of the launches is plenty
    for step in range(args.steps):
        res = None
        solver_mod.PROFILE = step % 4 == 0
        res = solve(x_dev)
        iters += res.iterations
        conv &= res.converged
        if solver_mod.PROFILE:
            dom_ms += max(res.timings["device_ms"][m] for m in merged.get(dom, (dom,)))
            dom_n += max(res.timings["device_launches"][m] for m in merged.get(dom, (dom,)))
    ev1.record()
    res_dev = res
    torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - l0
    clk = clocks.stop()
    solver_mod.PROFILE, solver_mod.PROFILE_PHASES = False, None
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    it = torch.tensor([iters], dtype=torch.float64, device=red_dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        if not shard:   # replicas: every rank's iterations count; sharded: one solve spans all ranks
            torch.distributed.all_reduce(it, op=torch.distributed.ReduceOp.SUM)
    ms_max = float(t.item())
    value = float(it.item()) / (ms_max / 1e3)

    # K3 / K0 rooflines on the timed solve's iterate (before the e2e loop, so that loop
    # recycles the warmed-up engines instead of building a new one)
    full_roof = _full_tensor_rooflines(res_dev, x_dev, bc, phases, peak, args.steps)
    parity = _parity_block(config, res_dev) if not shard else None
    del res_dev, res

    # ---------------- e2e through the public API with host buffers
    if host is None:
        host = x_dev.flat.cpu()
    pinned = host.pin_memory()
    x_buf = torch.empty_like(x_dev.flat)
    e2e_iters, d2h = 0, 0
    e2e_steps = max(1, args.steps if config <= 1 else min(args.steps, 2))
    # two untimed warm-up steps of the host-buffer path: the result arrays are views of
    # page-locked D2H blocks (engine.to_host) that torch's host allocator recycles once a
    # result is gone; a step's arrays live until the next step replaces them, so two
    # blocks circulate and allocating them (~30 ms each) is a one-time cost
    res = None
    t0 = None
    for step in range(-2, e2e_steps):
        if step == 0:
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_iters = 0
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
    te = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
    ie = torch.tensor([e2e_iters], dtype=torch.float64, device=red_dev)
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
             "factors": "k_fiber_pass (A pass) + k_fiber_areduce || k_block_pass (G pass) + k_modeprod (parallel branches)",
             "gpass": "k_block_pass (G pass)"}[dom]
    traffic = _ncu_traffic(config, dom)
    if dom in merged:
        parts = [_ncu_traffic(config, m) for m in merged[dom]]
        traffic = ({"bytes_per_launch": sum(p_["bytes_per_launch"] for p_ in parts),
                    "source": "; ".join(p_["source"] for p_ in parts)} if all(parts) else None)
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "traffic_source": traffic.get("source") if traffic else None,
            "alg_bytes_per_launch": alg[dom], "launch_us": 1e3 * per_launch_ms, "launches_timed": dom_n,
            "peak_source": peak_src,
            "share_of_device_time": (max(phases[m]["share"] for m in merged[dom] if m in phases) if dom in merged
                                     else phases[dom]["share"] if dom in phases else None)}
    if roof["traffic"]:   # the DRAM bytes ncu counted for this phase, over the same launch time
        roof["traffic_achieved"] = roof["traffic"] / (per_launch_ms / 1e3) / 1e9
        roof["traffic_frac"] = roof["traffic_achieved"] / peak
    fmas = _fp64_fmas(bc, rows, cols)
    if dom in fmas:   # the same launch against the fp64 pipe (the fiber passes sit near the ridge)
        tf = fmas[dom] / (per_launch_ms / 1e3) / 1e12
        roof["fp64"] = {"achieved": tf, "peak": FP64_PEAK_TFMA, "unit": "TFMA/s", "frac": tf / FP64_PEAK_TFMA,
                        "fma_per_launch": fmas[dom],
                        "peak_source": "measured: tools/fp64_pipes.cu (profiles/r01_fp64_pipes.txt)"}

    # the other BASELINE configs (same device, after the headline measurement)
    per_config = None
    if world == 1 and not args.no_per_config:
        del x_buf, pinned
        per_config = _per_config([c for c in (0, 2, 3, 4) if c != config], local, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if xf is not None:
            cpu = _cpu_baseline(bc, rows, cols, xf.astype(np.float64))
        else:
            cpu = {"value": None, "unit": "iters/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"not run for config {bc.index} in the b200 arm (one reference iteration takes "
                             "seconds to minutes here; SURVEY §6); bench.py --impl reference times it"}

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
            "roofline": roof, "k1_rooflines": k1_roof, "full_tensor_rooflines": full_roof, "phases": phases,
            "phases_note": f"phases and k1_rooflines: per-phase CUDA-event times from a separate profiled pass of "
                           f"{bd_steps} solve(s) (every phase bracketed by events, which cuts the iteration's graph "
                           "into segments: ~10 % slower than the timed region); the timed region carries events "
                           "on the roofline's phase only",
            "clocks": clk, "cpu_baseline": cpu, "parity": parity, "per_config": per_config,
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
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 1 at N=1, 4 sharded in mode-1 slabs under torchrun)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
