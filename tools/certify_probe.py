"""Wall time of assemble(certify=True) vs the default assembly (second call of each in the process).

    python tools/certify_probe.py U32k T65k U131k
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

for tag in sys.argv[1:] or ["U32k"]:
    w = WORKLOADS[tag]
    cl = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cl, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    out = {}
    for cert in (False, True, False, True):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        H, rep = hmx.assemble(w.spec(), cl, ct, bt, hmx.ACAConfig(eps_aca=w.eps, certify=cert))
        torch.cuda.synchronize()
        out[cert] = (time.perf_counter() - t0, H.certify_report)
        del H
    print(f"{tag}: default {out[False][0]:.3f} s, certified {out[True][0]:.3f} s "
          f"(+{out[True][0] - out[False][0]:.3f} s); {out[True][1]}", flush=True)
