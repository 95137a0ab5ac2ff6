"""Golden summary of BASELINE config 1 (400^3, RTCUR-R, fp64) solved by the REAL
reference (scratch build of /root/reference/pkg, compiled Cython backend).

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_cfg1_golden.py            # ~8 min on 8 cores

Writes tests/golden/cfg1_summary.npz: for every iteration the sampled error,
zeta, SHA-256 of the index sets and of the packed S support of each block,
S-support counts, and S / L values at fixed random positions of every block;
after the solve the singular values, factor norms, the final core-block
support bits, and the low-rank estimate at 2000 random full-tensor positions.
tests/test_oracle_golden.py::test_oracle_cfg1_matches_reference_summary pins
the oracle to it; tools/parity_configs.py pins the GPU path to it on the box.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

NPOS = 64   # sampled positions per block per iteration


def sha(a) -> np.ndarray:
    """32-byte digest as a uint8 array (npz-friendly)."""
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8)


def support_digest(s_flat) -> np.ndarray:
    return sha(np.packbits(np.asarray(s_flat).reshape(-1) != 0.0))


def positions(seed, sizes):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, s, NPOS) for s in sizes]


def main():
    from make_golden import _import_reference

    rtcur = _import_reference()
    from rtcur import DenseTensor, SolverConfig
    from rtcur.fiber_cur import cur_reconstruct_full

    from paper_2108_10448_b200.synth import baseline_sample_sizes, make_config

    xf, low, _, bc = make_config(1)
    rows, cols = baseline_sample_sizes(bc.shape, bc.ranks)
    cfg = SolverConfig(ranks=bc.ranks, eps=bc.eps, gamma=0.7, variant=bc.variant, max_iters=100,
                       seed=bc.seed_solver, row_sample_sizes=rows, col_sample_sizes=cols)
    x = DenseTensor(xf, bc.shape)
    t0 = time.perf_counter()
    res = rtcur.rtcur(x, cfg, record_trace=True)
    wall = time.perf_counter() - t0
    n = len(bc.shape)
    sizes = [int(np.prod(rows))] + [bc.shape[m] * cols[m] for m in range(n)]
    pos = positions(77, sizes)
    out = {"error_history": np.array(res.error_history), "iterations": np.array(res.iterations),
           "converged": np.array(res.converged), "zeta_final": np.array(res.zeta_final),
           "diagnostics": np.array(res.diagnostics, dtype=bool), "wall_s": np.array(wall),
           "npos": np.array(NPOS)}
    for b in range(n + 1):
        out[f"pos{b}"] = pos[b]
    for t, tr in enumerate(res.trace):
        s_blocks = [np.asarray(tr["s_core"]).reshape(-1, order="F")]
        l_blocks = [np.asarray(tr["l_core"]).reshape(-1, order="F")]
        s_blocks += [np.asarray(f).reshape(-1, order="F") for f in tr["s_fibers"]]
        l_blocks += [np.asarray(f).reshape(-1, order="F") for f in tr["l_fibers"]]
        idx = tr["indices"]
        out[f"t{t}_zeta"] = np.array(tr["zeta"])
        out[f"t{t}_idx_sha"] = sha(np.concatenate([np.asarray(a, dtype=np.int64) for a in
                                                   list(idx.rows) + list(idx.cols)]))
        for b in range(n + 1):
            out[f"t{t}_b{b}_supp_sha"] = support_digest(s_blocks[b])
            out[f"t{t}_b{b}_nnz"] = np.array(int(np.count_nonzero(s_blocks[b])))
            out[f"t{t}_b{b}_s"] = s_blocks[b][pos[b]]
            out[f"t{t}_b{b}_l"] = l_blocks[b][pos[b]]
    s_core = np.asarray(res.sparse.core).reshape(-1, order="F")
    out["s_core_bits"] = np.packbits(s_core != 0.0)
    for m in range(n):
        out[f"sv{m}"] = np.asarray(res.cur.intersections[m].singular_values)
        out[f"factor{m}_norm"] = np.array(np.linalg.norm(res.cur.factors[m]))
    lf = cur_reconstruct_full(res.cur).data
    rng = np.random.default_rng(123)
    p = rng.integers(0, lf.size, 2000)
    out["L_pos"] = p
    out["L_val"] = lf[p]
    out["rel_recovery"] = np.array(np.linalg.norm(lf - low) / np.linalg.norm(low))
    np.savez_compressed(os.path.join(HERE, "cfg1_summary.npz"), **out)
    print(f"cfg1: iters={res.iterations} conv={res.converged} err={res.error_history[-1]:.3e} "
          f"rel={float(out['rel_recovery']):.2e} wall={wall:.1f}s")


if __name__ == "__main__":
    main()
