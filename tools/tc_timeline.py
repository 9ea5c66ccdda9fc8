"""Per-CTA timeline of the tensor-core ACA (experiment build with -DHMX_TC_PROF).

    python tools/build_variant.py tcprof -DHMX_TC_PROF
    HMX_LIB=build/ab/tcprof.so python tools/tc_timeline.py U32k
Prints how many SMs are busy over the kernel's lifetime (10 slices), the longest CTAs and the
per-CTA streaming rate, i.e. whether the kernel is tail-dominated by its largest leaves.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_09384_b200 as hmx  # noqa: E402
from paper_1706_09384_b200 import _lib  # noqa: E402
from paper_1706_09384_b200.configs import WORKLOADS  # noqa: E402

L = C.CDLL(_lib.LIB_PATH)
for tag in sys.argv[1:] or ["U32k"]:
    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    for rep in range(2):
        H, r = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps))
        st = H.stats()
        del H
    buf = (C.c_ulonglong * (4 * 8192))()
    L.hmx_debug_tc_cta(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)
    a = a[a[:, 1] > 0]
    t0 = a[:, 0].min()
    s = (a[:, 0] - t0).astype(np.float64) * 1e-6
    e = (a[:, 1] - t0).astype(np.float64) * 1e-6
    mn = (a[:, 3] >> np.uint64(32)).astype(np.int64)
    K = (a[:, 3] & np.uint64(0xffffffff)).astype(np.int64)
    T = e.max()
    print(f"{tag}: {len(a)} CTAs, kernel span {T:.1f} ms, assembly {st['t_total_ms']:.1f} ms; sum CTA time {np.sum(e - s):.0f} ms "
          f"= {np.sum(e - s) / T:.1f} SMs busy on average")
    edges = np.linspace(0, T, 21)
    busy = [np.sum(np.clip(np.minimum(e, hi) - np.maximum(s, lo), 0, None)) / (hi - lo) for lo, hi in zip(edges[:-1], edges[1:])]
    print("  busy SMs per 5% slice: " + " ".join(f"{b:.0f}" for b in busy))
    gb = 16.0 * 3 * mn * K.astype(np.float64) ** 2 / 2 / 3 * 1e-9  # panel bytes streamed: sum over steps of 16 * 3(m+n) * K_s
    order = np.argsort(-(e - s))[:12]
    for i in order:
        print(f"  CTA {i}: m+n {mn[i]} K {K[i]} start {s[i]:.1f} dur {e[i] - s[i]:.1f} ms, ~{gb[i]:.2f} GB -> {gb[i] / (e[i] - s[i]) * 1e3:.0f} GB/s")
    rate = gb / (e - s) * 1e3
    print(f"  per-CTA streaming rate GB/s: median {np.median(rate):.0f}, p10 {np.percentile(rate, 10):.0f}, p90 {np.percentile(rate, 90):.0f}")
    for lo, hi in ((320, 512), (512, 1024), (1024, 2048), (2048, 4096), (4096, 1 << 30)):
        sel = (mn >= lo) & (mn < hi)
        if sel.any():
            print(f"  m+n in [{lo},{hi}): {sel.sum()} CTAs, {np.sum((e - s)[sel]):.0f} CTA-ms, mean K {K[sel].mean():.0f}, rate {np.sum(gb[sel]) / np.sum((e - s)[sel]) * 1e3:.0f} GB/s")
