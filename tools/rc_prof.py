"""Recompression phase profile (experiment build with -DHMX_RC_PROF).

    HMX_NVCC_EXTRA=-DHMX_RC_PROF  -> build into a separate lib, then
    HMX_LIB=build/rcprof/libhmx.so python tools/rc_prof.py U32k
Prints, per kernel MODE, the per-phase share of thread-0 clock64 cycles summed
over CTAs (phases: 0 chol, 1 E = R G_U R^H, 2 tridiagonalise, 3 bisection +
truncation, 4 twisted vectors + CGS2, 5 QL fallback, 6 back-transform L_r,
7 W_U, 8 W_V).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

names = ["chol", "E=RGR^H", "tridiag", "bisect", "twist+cgs2", "QL", "backxf", "W_U", "W_V"]
L = C.CDLL(_lib.LIB_PATH)
buf = (C.c_ulonglong * 48)()
for tag in sys.argv[1:] or ["U32k"]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    for rep in range(2):
        L.hmx_debug_rc_prof(buf)
        if hasattr(L, "hmx_debug_tc_prof"):
            L.hmx_debug_tc_prof((C.c_ulonglong * 16)())
        H, r = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
        st = H.stats()
        del H
    L.hmx_debug_rc_prof(buf)
    if hasattr(L, "hmx_debug_tc_prof"):
        tb = (C.c_ulonglong * 16)()
        L.hmx_debug_tc_prof(tb)  # second assembly only (the first call's counts were reset above? no: read now)
    print(f"{tag}: total {st['t_total_ms']:.1f} ms aca {st['t_aca_ms']:.1f} form {st['t_form_ms']:.1f}")
    for mode in range(3):
        v = list(buf[16 * mode:16 * mode + 16])
        tot = sum(v[:9])
        if v[15] == 0:
            continue
        print(f"  MODE {mode}: {v[15]} CTAs, mean K {v[14] / v[15]:.1f}, {tot / v[15] / 1e3:.1f} kcyc/CTA")
        print("    " + "  ".join(f"{n} {100 * x / tot:.1f}%" for n, x in zip(names, v[:9])))
        if hasattr(L, "hmx_debug_tc_prof"):
            pass
    if hasattr(L, "hmx_debug_tc_prof"):
        v = list(tb)
        tn = ["Urow", "row pass", "finalize V+pivot+Vrow", "col pass", "finalize U+decide", "exit"]
        tot = sum(v[:6])
        print("  TC ACA (thread 0, summed over CTAs): " + "  ".join(f"{n} {100 * x / max(tot, 1):.1f}%" for n, x in zip(tn, v[:6])))
        print(f"  TC warps: streaming {v[8] / 1e9:.2f} Gcyc, epilogue {v[9] / 1e9:.2f} Gcyc; thread-0 total {tot / 1e9:.2f} Gcyc")
        print(f"  TC row-pass epilogue parts (lane 0 of each warp): Green's {v[10] / 1e9:.2f} Gcyc, sigma_3 {v[11] / 1e9:.2f} Gcyc")
