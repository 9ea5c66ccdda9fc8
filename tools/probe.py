"""Assemble every BASELINE config on the GPU and print timings / ranks.

    python tools/probe.py [TAG ...]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402
from tests._problems import spec_for  # noqa: E402


def run(tag):
    w = WORKLOADS[tag]
    t0 = time.perf_counter()
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    t_tree = time.perf_counter() - t0
    spec = spec_for(w)
    t0 = time.perf_counter()
    H, rep = hmx.assemble(spec, cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    t_asm = time.perf_counter() - t0
    st = H.stats()
    n = w.d * w.n_points
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n)).cuda()
    y = torch.empty_like(x)
    H.use_stream(torch.cuda.current_stream().cuda_stream)
    ph = (C := __import__("ctypes")).c_float * 4
    times = []
    phases = []
    for it in range(25):
        p = ph()
        _lib.check(_lib.lib().hmx_matvec_profile(H.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), p))
        if it >= 5:
            phases.append(list(p))
    phases = np.median(np.array(phases), axis=0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        hmx.matvec(H, x, out=y)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(50):
        hmx.matvec(H, x, out=y)
    ev1.record()
    torch.cuda.synchronize()
    mv_ms = ev0.elapsed_time(ev1) / 50
    out = dict(tag=tag, N=w.n_points, t_tree_s=t_tree, t_assemble_wall_s=t_asm,
               max_rank_before=rep.max_rank_before, max_rank_after=rep.max_rank_after, tau=rep.tau,
               matvec_ms=mv_ms, matvec_GBps=st["matvec_bytes"] / mv_ms / 1e6, phases_ms=phases.tolist(),
               **{k: st[k] for k in ("t_aca_ms", "t_recompress_ms", "t_dense_ms", "t_form_ms", "t_total_ms",
                                      "matvec_bytes", "n_regularized", "aca_passes", "n_unconverged",
                                      "pairs_evaluated", "flops_assembly", "n_tiles", "n_jobs", "n_levels")})
    if "gmres" in w.runs:
        b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        t0 = time.perf_counter()
        res = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-4, restart=50))
        out.update(gmres_iters=res.iters, gmres_s=time.perf_counter() - t0, gmres_conv=res.converged)
    print(json.dumps(out), flush=True)
    del H


if __name__ == "__main__":
    tags = sys.argv[1:] or list(WORKLOADS)
    for t in tags:
        run(t)
