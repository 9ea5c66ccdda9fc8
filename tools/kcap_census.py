"""ACA rank vs the capacity model (capi.cu): per admissible leaf, K (rank before
recompression) against 60 + 2 d kappa diam; writes gpurun_out/kcap_<tag>.npz and
prints the leaves closest to / above the model.

    python tools/kcap_census.py U131k U32k T65k
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

for tag in sys.argv[1:] or ["U131k"]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    bi = H.block_info()
    t = np.asarray(bt.leaf_table)
    P = np.asarray(ct.points_tree)
    adm = np.flatnonzero(t[:, 0] == 1)

    def diam(a0, a1):
        q = P[a0:a1]
        return float(np.linalg.norm(q.max(0) - q.min(0)))

    cache = {}
    dm = np.empty(len(adm))
    for i, b in enumerate(adm):
        r = (int(t[b, 1]), int(t[b, 2]))
        c = (int(t[b, 3]), int(t[b, 4]))
        for key in (r, c):
            if key not in cache:
                cache[key] = diam(*key)
        dm[i] = max(cache[r], cache[c])
    kap = abs(w.kappa) if w.d == 1 else max(abs(w.ks), abs(w.kp))
    model = 60.0 + 2.0 * w.d * kap * dm
    K = bi["rank_before"][adm]
    mn = (t[adm, 2] - t[adm, 1]) + (t[adm, 4] - t[adm, 3])
    np.savez(f"gpurun_out/kcap_{tag}.npz", K=K, model=model, diam=dm, mn=mn, m=t[adm, 2] - t[adm, 1],
             n=t[adm, 4] - t[adm, 3], steps=bi["steps"][adm])
    ex = K - model
    o = np.argsort(-ex)[:12]
    print(tag, "passes", H.stats()["aca_passes"], "leaves", len(adm), "max K - model", ex.max(), "count K+d>model",
          int(np.sum(K + w.d > model)))
    for i in o:
        print(f"   K {K[i]:4d} model {model[i]:7.1f} diam {dm[i]:.3f} m+n {mn[i]}")
    del H
