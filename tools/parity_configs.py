"""Lockstep parity of the GPU solve against the CPU oracle at BASELINE configs.

    python tools/parity_configs.py --config 1                 # full solve
    python tools/parity_configs.py --config 2 --iters 3       # first 3 iterations
    python tools/parity_configs.py --config 4 --json out.json

Both sides solve the SAME X (configs 0-1 generated on the host; configs 2-4
on the device and copied to the host, fp32 -> fp64 upcast is exact) with the
same seed, so the index sets come from the same PCG64 stream.  The oracle
(oracle/rtcur_oracle.py, test infrastructure) runs as a generator one
iteration at a time; the GPU solve calls back after each of its iterations
(``solver._solve(on_iteration=...)``) and the two states are compared there:

* index sets             exact
* zeta                   equal to 1e-15 relative
* sampled error          |e_gpu - e_oracle| <= 1e-10
* S support              bit-exact per block (a flip is logged with its margin
                         (|x - l_prev| - zeta) / zeta from the oracle's values)
* S and L blocks         relative Frobenius error <= 1e-10 (all arithmetic is
                         fp64 on both sides; fp32 X is upcast exactly)
* singular values        |sigma_gpu - sigma_oracle| <= 1e-10 sigma_1
* deficiency flags       equal
* (sigma_r - sigma_{r+1}) / sigma_1 per mode from the oracle's full spectra
  is logged (subspace sensitivity)

After the loop: iteration count and convergence equal, and the full-tensor
low-rank estimate (K3, ``full_output``) against the oracle's
core x_i factors at 4096 random positions (1e-10 relative to max|L|), with
S = HT(X - L, zeta_final) support equal there.

The reference's equivalence pattern this follows:
/root/reference/pkg/tests/test_reference.py:177-214 and
/root/reference/pkg/tests/test_acceptance.py:92-121 over the loop at
/root/reference/pkg/src/rtcur/solver.py:314-375.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TOL_ERR = 1e-10
TOL_REL = 1e-10
TOL_SV = 1e-10


def sha(a) -> np.ndarray:
    """SHA-256 digest as uint8 (as tests/golden/make_cfg1_golden.py stores it)."""
    import hashlib

    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8)


def support_digest(s_flat) -> np.ndarray:
    return sha(np.packbits(np.asarray(s_flat).reshape(-1) != 0.0))


def _rel(a, b):
    den = float(np.linalg.norm(b))
    num = float(np.linalg.norm(a - b))
    return num / den if den > 0 else num


def make_x(config: int):
    """(DeviceTensor, host fp64 flat X, BaselineConfig)."""
    import torch

    from paper_2108_10448_b200 import DeviceTensor
    from paper_2108_10448_b200.synth import CONFIGS, make_config, make_config_device

    bc = CONFIGS[config]
    if config <= 1:
        xf, _, _, bc = make_config(config)
        dt = torch.float64 if bc.dtype == "f64" else torch.float32
        x_dev = DeviceTensor(torch.from_numpy(xf).to(dt).cuda(), bc.shape)
        x64 = xf.astype(np.float64)
    else:
        x_dev, bc = make_config_device(config)
        x64 = x_dev.flat.cpu().numpy().astype(np.float64)
    return x_dev, x64, bc


def lowrank_at(cur, shape, pos, chunk=256):
    """Oracle low-rank estimate core x_i factors[i] at flat F-order positions."""
    n = len(shape)
    midx = []
    rem = np.asarray(pos, dtype=np.int64)
    for d in shape:
        midx.append(rem % d)
        rem = rem // d
    out = np.empty(len(pos))
    for j0 in range(0, len(pos), chunk):
        j1 = min(len(pos), j0 + chunk)
        t = np.tensordot(cur.factors[0][midx[0][j0:j1], :], cur.core, axes=([1], [0]))   # (jc, I2, .., In)
        for m in range(1, n):
            rows = cur.factors[m][midx[m][j0:j1], :]                                      # (jc, I_m)
            lead = t.shape
            t = np.matmul(np.moveaxis(t, 1, -1).reshape(lead[0], -1, lead[1]), rows[:, :, None]).reshape(
                (lead[0],) + lead[2:])
        out[j0:j1] = t.reshape(-1)
    return out


def run(config: int, iters: int | None = None, log=print, full_check: bool = True, ref_summary=None):
    """Run GPU and oracle in lockstep; returns the record dict (``ok`` flag)."""
    import torch

    from oracle import rtcur_oracle as orc
    from paper_2108_10448_b200 import SolverConfig, full_output
    from paper_2108_10448_b200.solver import _solve, _Source
    from paper_2108_10448_b200.synth import baseline_sample_sizes

    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    x_dev, x64, bc = make_x(config)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    max_iters = int(iters) if iters else 100
    n = len(bc.shape)
    t_gen = time.perf_counter() - t0
    orc.build_oracle_lib()
    stats: dict = {}
    it = orc.iter_solve(x64, bc.shape, bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=max_iters,
                        seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols, stats=stats)
    rec = {"config": config, "workload": f"config{config}: RTCUR-{bc.variant} {'x'.join(map(str, bc.shape))} "
                                         f"{bc.dtype} ranks {tuple(bc.ranks)}",
           "max_iters": max_iters, "iterations": [], "failures": [], "gen_s": t_gen,
           "tolerances": {"error_abs": TOL_ERR, "blocks_rel_fro": TOL_REL, "sigma_rel_sigma1": TOL_SV,
                          "support": "bit-exact", "indices": "exact"}}
    last = {}

    def fail(msg):
        rec["failures"].append(msg)
        log("FAIL " + msg)

    def on_iter(k, eng, idx, zeta, err, flags):
        t1 = time.perf_counter()
        o = next(it)
        t_orc = time.perf_counter() - t1
        last["o"] = o
        row = {"k": k, "oracle_s": t_orc}
        if o["iteration"] != k:
            fail(f"iteration numbering {o['iteration']} != {k}")
        same_idx = all(np.array_equal(a, b) for a, b in zip(idx.rows, o["indices"].rows)) and \
            all(np.array_equal(a, b) for a, b in zip(idx.cols, o["indices"].cols))
        row["indices_equal"] = bool(same_idx)
        if not same_idx:
            fail(f"k={k}: index sets differ")
        row["zeta_rel"] = abs(zeta - o["zeta"]) / max(abs(o["zeta"]), 1e-300)
        if row["zeta_rel"] > 1e-15:
            fail(f"k={k}: zeta {zeta!r} vs {o['zeta']!r}")
        row["err_gpu"], row["err_oracle"] = float(err), float(o["error"])
        row["err_abs_diff"] = abs(float(err) - float(o["error"]))
        if not row["err_abs_diff"] <= TOL_ERR:
            fail(f"k={k}: error {err!r} vs {o['error']!r}")
        row["flags_equal"] = tuple(flags) == tuple(o["flags"])
        if not row["flags_equal"]:
            fail(f"k={k}: deficiency flags {flags} vs {o['flags']}")
        s_dev, _, l_dev = eng.export_blocks(True, False, True)
        s_core, s_fib = eng.split_blocks(s_dev.cpu().numpy())
        l_core, l_fib = eng.split_blocks(l_dev.cpu().numpy())
        gs = [s_core.reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in s_fib]
        gl = [l_core.reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in l_fib]
        os_ = [o["s_core"].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in o["s_fibers"]]
        ol = [o["l_core"].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in o["l_fibers"]]
        ox = [o["x_core"].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in o["x_fibers"]]
        olp = [o["l_prev"][0].reshape(-1, order="F")] + [f.reshape(-1, order="F") for f in o["l_prev"][1]]
        flips, margins, nnz = 0, [], []
        for b in range(n + 1):
            ms = (gs[b] != 0) != (os_[b] != 0)
            nf = int(np.count_nonzero(ms))
            nnz.append(int(np.count_nonzero(os_[b])))
            if nf:
                flips += nf
                mg = (np.abs(ox[b][ms] - olp[b][ms]) - o["zeta"]) / o["zeta"]
                margins += [float(v) for v in mg[:8]]
        row["support_flips"], row["s_nnz"] = flips, nnz
        if flips:
            row["flip_margins"] = margins
            fail(f"k={k}: {flips} support flips (margins {margins[:4]})")
        # closest-to-threshold margin over all blocks (how near a flip this iteration was)
        mmin = min(float(np.min(np.abs(np.abs(ox[b] - olp[b]) - o["zeta"]))) for b in range(n + 1)) / o["zeta"]
        row["min_threshold_margin_rel"] = mmin
        row["s_rel_fro"] = _rel(np.concatenate(gs), np.concatenate(os_))
        row["l_rel_fro"] = _rel(np.concatenate(gl), np.concatenate(ol))
        row["s_max_abs"] = max(float(np.max(np.abs(a - b))) if a.size else 0.0 for a, b in zip(gs, os_))
        row["l_max_abs"] = max(float(np.max(np.abs(a - b))) if a.size else 0.0 for a, b in zip(gl, ol))
        if not row["s_rel_fro"] <= TOL_REL:
            fail(f"k={k}: S rel Frobenius {row['s_rel_fro']:.3e}")
        if not row["l_rel_fro"] <= TOL_REL:
            fail(f"k={k}: L rel Frobenius {row['l_rel_fro']:.3e}")
        _, S, _, _, _ = eng.export_cur()
        sv_err, gaps = [], []
        for m in range(n):
            so = o["cur"].intersections[m].singular_values
            sc = max(float(so[0]), 1e-300)
            sv_err.append(float(np.max(np.abs(S[m] - so))) / sc)
            full = o["cur"].spectra[m]
            r = bc.ranks[m]
            gaps.append(float((full[r - 1] - full[r]) / sc) if full.size > r else None)
        row["sigma_rel_err"] = sv_err
        row["gap_r_r1_rel"] = gaps
        if not max(sv_err) <= TOL_SV:
            fail(f"k={k}: singular values off by {max(sv_err):.3e} sigma_1")
        if ref_summary is not None:
            row["vs_reference"] = _vs_reference(ref_summary, k, idx, err, gs, gl, fail)
        rec["iterations"].append(row)
        log(f"k={k:3d} err {err:.6e} (d {row['err_abs_diff']:.1e})  S {row['s_rel_fro']:.1e}  "
            f"L {row['l_rel_fro']:.1e}  flips {flips}  sv {max(sv_err):.1e}  gap "
            f"{min(g for g in gaps if g is not None) if any(g is not None for g in gaps) else float('nan'):.2e}  "
            f"margin {mmin:.1e}  oracle {t_orc:.1f}s")

    cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=max_iters,
                       seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
    t0 = time.perf_counter()
    res = _solve(_Source(x_dev), cfg, on_iteration=on_iter)
    rec["loop_s"] = time.perf_counter() - t0
    rec["gpu_iterations"], rec["oracle_iterations"] = res.iterations, len(stats["iter_times"])
    rec["gpu_converged"], rec["oracle_converged"] = bool(res.converged), bool(stats["converged"])
    if res.iterations != len(stats["iter_times"]) or res.converged != stats["converged"]:
        fail(f"iterations/converged {res.iterations}/{res.converged} vs "
             f"{len(stats['iter_times'])}/{stats['converged']}")
    rec["zeta_final_rel"] = abs(res.zeta_final - last["o"]["zeta"]) / last["o"]["zeta"]
    if full_check:
        L, S, rel = full_output(res, x_dev)
        rng = np.random.default_rng(2024)
        pos = np.sort(rng.integers(0, x64.size, 4096))
        lo = lowrank_at(last["o"]["cur"], bc.shape, pos)
        lg = L.flat[torch.from_numpy(pos).cuda()].double().cpu().numpy()
        sg = S.flat[torch.from_numpy(pos).cuda()].double().cpu().numpy()
        if bc.dtype == "f32":   # K3 stores L in the dtype of X: compare at fp32 resolution
            lo_cmp = lo.astype(np.float32).astype(np.float64)
            tol = 2.0 ** -23 * 4
        else:
            lo_cmp, tol = lo, TOL_REL
        scale = float(np.max(np.abs(lo))) or 1.0
        rec["full_L_max_rel"] = float(np.max(np.abs(lg - lo_cmp))) / scale
        so = orc.hard_threshold(x64[pos] - lo, last["o"]["zeta"])
        so_cmp = so.astype(np.float32).astype(np.float64) if bc.dtype == "f32" else so
        rec["full_S_support_equal"] = bool(np.array_equal(sg != 0, so_cmp != 0))
        rec["full_S_max_rel"] = float(np.max(np.abs(sg - so_cmp))) / max(float(np.max(np.abs(so))), 1.0)
        rec["full_relative_residual_gpu"] = rel
        rec["full_check_tol_rel"] = tol
        if not rec["full_L_max_rel"] <= tol:
            fail(f"full L at random positions off by {rec['full_L_max_rel']:.3e} (tol {tol:.1e})")
        if not rec["full_S_support_equal"]:
            fail("full S support differs at random positions")
        del L, S
    rec["ok"] = not rec["failures"]
    rec["max"] = {key: max(r[key] for r in rec["iterations"]) for key in
                  ("err_abs_diff", "s_rel_fro", "l_rel_fro", "support_flips")}
    rec["max"]["sigma_rel_err"] = max(max(r["sigma_rel_err"]) for r in rec["iterations"])
    gl = [g for r in rec["iterations"] for g in r["gap_r_r1_rel"] if g is not None]
    rec["min_gap_r_r1_rel"] = min(gl) if gl else None
    rec["min_threshold_margin_rel"] = min(r["min_threshold_margin_rel"] for r in rec["iterations"])
    rec["oracle_s"] = sum(r["oracle_s"] for r in rec["iterations"])
    log(f"config {config}: {'PASS' if rec['ok'] else 'FAIL'}  iterations gpu {res.iterations} oracle "
        f"{rec['oracle_iterations']}  max err diff {rec['max']['err_abs_diff']:.2e}  max S/L rel "
        f"{rec['max']['s_rel_fro']:.2e}/{rec['max']['l_rel_fro']:.2e}  flips {rec['max']['support_flips']}")
    return rec


def _vs_reference(g, k, idx, err, gs, gl, fail):
    """Compare iteration k with the real reference's summary (cfg1_summary.npz)."""
    t = k - 1
    out = {}
    if f"t{t}_zeta" not in g:
        return out
    out["idx_equal"] = bool(np.array_equal(sha(np.concatenate([np.asarray(a, dtype=np.int64) for a in
                                                               list(idx.rows) + list(idx.cols)])),
                                           g[f"t{t}_idx_sha"]))
    out["err_abs_diff"] = abs(float(err) - float(g["error_history"][t]))
    supp = [bool(np.array_equal(support_digest(gs[b]), g[f"t{t}_b{b}_supp_sha"])) for b in range(len(gs))]
    out["support_equal"] = supp
    out["s_max_abs"] = max(float(np.max(np.abs(gs[b][g[f"pos{b}"]] - g[f"t{t}_b{b}_s"]))) for b in range(len(gs)))
    out["l_max_abs"] = max(float(np.max(np.abs(gl[b][g[f"pos{b}"]] - g[f"t{t}_b{b}_l"]))) for b in range(len(gs)))
    if not out["idx_equal"]:
        fail(f"k={k}: index sets differ from the reference's")
    if not out["err_abs_diff"] <= TOL_ERR:
        fail(f"k={k}: error differs from the reference's by {out['err_abs_diff']:.2e}")
    if not all(supp):
        fail(f"k={k}: S support differs from the reference's ({supp})")
    if not (out["s_max_abs"] <= TOL_ERR and out["l_max_abs"] <= TOL_ERR):
        fail(f"k={k}: S/L values differ from the reference's ({out['s_max_abs']:.2e}/{out['l_max_abs']:.2e})")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--iters", type=int, default=0, help="stop after this many iterations (0: full solve)")
    ap.add_argument("--json", default="")
    ap.add_argument("--no-full", action="store_true")
    args = ap.parse_args()
    ref = None
    if args.config == 1:
        p = os.path.join(ROOT, "tests", "golden", "cfg1_summary.npz")
        if os.path.exists(p):
            ref = dict(np.load(p))
    rec = run(args.config, args.iters or None, full_check=not args.no_full, ref_summary=ref)
    if ref is not None:
        rec["reference_summary"] = {"error_history_max_abs_diff": float(np.max(np.abs(
            np.array([r["err_gpu"] for r in rec["iterations"]]) - ref["error_history"][:len(rec["iterations"])]))),
            "reference_iterations": int(ref["iterations"])}
        if not args.iters and rec["gpu_iterations"] != int(ref["iterations"]):
            rec["failures"].append("iteration count differs from the reference's")
            rec["ok"] = False
    if args.json:
        os.makedirs(os.path.dirname(os.path.abspath(args.json)), exist_ok=True)
        with open(args.json, "w") as f:
            json.dump(rec, f, indent=1, default=float)
    return 0 if rec["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
