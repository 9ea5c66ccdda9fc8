"""CPU reference time-to-solve (BASELINE config 5): the oracle on the host cores --
leaf-parallel assembly of every leaf in a fork pool, then GMRES(50, 1e-4) with the
threaded oracle H-matvec.  One JSON line; run on the GPU box so the core count matches the bench.

    python tools/cpu_time_to_solve.py [T65k]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import hmatrix as OH  # noqa: E402
from oracle import solve as OS  # noqa: E402


def main(tag):
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    w, ct, nrm, tab, params, desc = bench.cpu_problem(tag)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oh = OH.assemble(w.kind, params, ct.points_tree, None if w.kind != "T" else nrm[ct.perm], ct.perm, tab, w.eps,
                     self_shift=float(w.n_points), workers=cores)
    t_asm = time.perf_counter() - t0
    d = w.d
    m = (tab[:, 2] - tab[:, 1]).astype(np.float64)
    n = (tab[:, 4] - tab[:, 3]).astype(np.float64)
    cost = np.where(tab[:, 0] == 0, d * d * m * n, oh.rank_after * d * (m + n))
    order = np.argsort(-cost, kind="stable")
    chunks = [[] for _ in range(cores)]
    load = np.zeros(cores)
    for b in order:
        i = int(np.argmin(load))
        chunks[i].append(int(b))
        load[i] += cost[b]
    rng = np.random.default_rng(bench.SEED)
    nd = d * w.n_points
    rhs = rng.standard_normal(nd) + 1j * rng.standard_normal(nd)
    with ThreadPoolExecutor(cores) as pool, threadpool_limits(1):
        mv = lambda v: OH.from_tree(oh, OH.matvec_tree_threads(oh, OH.to_tree(oh, v), pool, chunks))  # noqa: E731
        t0 = time.perf_counter()
        x, it, hist, conv = OS.gmres(mv, rhs, 1e-4, 50, 1000)
        t_gm = time.perf_counter() - t0
        res = float(np.linalg.norm(rhs - mv(x)) / np.linalg.norm(rhs))
    out = {"workload": tag, "kind": "port", "cores": cores, "cpu_model": bench.cpu_model(), "sample": desc,
           "assembly_pooled_s": t_asm, "gmres_s": t_gm, "gmres_iterations": it, "converged": bool(conv),
           "true_rel_residual": res, "time_to_solve_s": t_asm + t_gm,
           "max_rank_after": int(oh.rank_after.max()), "n_fallback": int(oh.fallback.sum()),
           "matvec_bytes": 16.0 * float(cost.sum()) + 32.0 * nd}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "T65k")
