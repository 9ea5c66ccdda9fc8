"""Per-phase H-matvec timings (hmx_matvec_profile: gather, V^H x, row GEMV, finalize) per config.

    python tools/mv_phases.py U8k H4k U32k
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

for tag in sys.argv[1:] or ["U8k"]:
    w = WORKLOADS[tag]
    cl = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cl, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, _ = hmx.assemble(w.spec(), cl, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
    st = H.stats()
    n = w.d * w.n_points
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    ph = (C.c_float * 4)()
    acc = np.zeros(4)
    for it in range(30):
        _lib.check(_lib.lib().hmx_matvec_profile(H.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), ph),
                   "profile")
        if it >= 5:
            acc += np.array(ph[:])
    acc /= 25
    tot = acc.sum()
    print(f"{tag}: bytes {st['matvec_bytes'] / 1e9:.3f} GB (phase1 {st['phase1_bytes'] / 1e9:.3f}, phase2 "
          f"{st['phase2_bytes'] / 1e9:.3f}); ms gather {acc[0]:.4f} vhx {acc[1]:.4f} row {acc[2]:.4f} fin {acc[3]:.4f} "
          f"= {tot:.4f} ms; phase1 {st['phase1_bytes'] / acc[1] / 1e6:.0f} GB/s, phase2 "
          f"{st['phase2_bytes'] / acc[2] / 1e6:.0f} GB/s, whole {st['matvec_bytes'] / tot / 1e6:.0f} GB/s; "
          f"jobs {st['n_jobs']} tiles {st['n_tiles']} levels {st['n_levels']}", flush=True)
    del H
