"""H-matrix container, device assembly and H-matvec -- the reference's
``hmatx.hmatrix`` entry points: ``assemble(spec, cloud, ct,
bt, cfg) -> (HMatrix, StorageReport)``, ``matvec(h, x)``,
``storage_report(h)``.  Everything numeric runs in libhmx.so (``hmx_assemble``,
``hmx_matvec``); an assembled HMatrix is immutable and lives in HBM.
"""

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import sparsity_pattern
from .lowrank import ACAConfig, LowRankFactor

HOST, DEVICE = 0, 1


@dataclass(frozen=True)
class StorageReport:
    """N_s, N^2, tau = N_s / N^2, max ranks, and the
    section-5.1 bound 2 C_sp max(r_max, N_leaf) N (log2 N - log2 N_leaf + 1)."""

    n_stored: int
    n_dense_equiv: int
    tau: float
    max_rank_before: int
    max_rank_after: int
    bound: float | None = None


class HMatrix:
    """Device-resident H-matrix."""

    def __init__(self, handle, d, n_points, block_tree=None, perm=None, spec=None, table=None, device=0):
        self._h = handle
        self.d = d
        self.n_points = n_points
        self.block_tree = block_tree
        self.perm = perm
        self.spec = spec
        self.table = table
        self.device = device
        self.self_shift = None
        self.certify_report = None

    def __del__(self):
        try:
            if self._h:
                _lib.lib().hmx_hmatrix_free(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def shape(self):
        n = self.d * self.n_points
        return (n, n)

    @property
    def handle(self):
        return self._h

    def stats(self):
        st = _lib.HmxStats()
        _lib.check(_lib.lib().hmx_hmatrix_stats(self._h, C.byref(st)), "hmx_hmatrix_stats")
        return st.as_dict()

    def block_info(self):
        nb = len(self.table)
        steps = np.empty(nb, np.int64)
        rb = np.empty(nb, np.int64)
        ra = np.empty(nb, np.int64)
        fl = np.empty(nb, np.int32)
        _lib.check(_lib.lib().hmx_hmatrix_block_info(self._h, _lib.ptr(steps), _lib.ptr(rb), _lib.ptr(ra),
                                                     _lib.ptr(fl)), "block_info")
        return dict(steps=steps, rank_before=rb, rank_after=ra, flags=fl)

    def block(self, b):
        """Leaf payload: dense ndarray or LowRankFactor (tree-order index ranges)."""
        k, r0, r1, c0, c1 = (int(t) for t in self.table[b][:5])
        dm, dn = self.d * (r1 - r0), self.d * (c1 - c0)
        if k == 0:
            a = np.empty((dm, dn), np.complex128)
            _lib.check(_lib.lib().hmx_hmatrix_get_block(self._h, b, _lib.ptr(a), None), "get_block")
            return a
        if getattr(self, "_ranks", None) is None:  # immutable H: cache the rank table
            self._ranks = self.block_info()["rank_after"]
        r = int(self._ranks[b])
        u = np.empty((dm, r), np.complex128)
        v = np.empty((dn, r), np.complex128)
        if r:
            _lib.check(_lib.lib().hmx_hmatrix_get_block(self._h, b, _lib.ptr(u), _lib.ptr(v)), "get_block")
        return LowRankFactor(u, v)

    def use_stream(self, stream_ptr):
        """Default launch stream of this H's matvecs (a cudaStream_t such as
        torch.cuda.current_stream().cuda_stream); a per-H setting, not process state.
        ``matvec(h, x, stream=...)`` overrides it per call."""
        self._stream = None if stream_ptr is None else int(stream_ptr)

    @classmethod
    def from_factors(cls, d, n_points, perm, table, payload, device=0):
        """Import leaf payloads (dense arrays / (U, V) pairs, tree-order ranges).
        Used to run the device matvec on oracle-assembled factors."""
        table = np.ascontiguousarray(np.asarray(table)[:, :5], dtype=np.int64)
        nb = len(table)
        keep = []
        A = (C.c_void_p * nb)()
        B = (C.c_void_p * nb)()
        ranks = np.zeros(nb, np.int64)
        for b, p in enumerate(payload):
            if table[b, 0] == 0:
                a = np.ascontiguousarray(p, dtype=np.complex128)
                keep.append(a)
                A[b] = a.ctypes.data
            else:
                u = np.ascontiguousarray(p[0], dtype=np.complex128)
                v = np.ascontiguousarray(p[1], dtype=np.complex128)
                keep += [u, v]
                ranks[b] = u.shape[1]
                A[b] = u.ctypes.data
                B[b] = v.ctypes.data
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(_lib.lib().hmx_hmatrix_load(_lib.context(device), d, n_points, _lib.ptr(perm), _lib.ptr(table),
                                               nb, _lib.ptr(ranks), A, B, C.byref(h)), "hmx_hmatrix_load")
        return cls(h, d, n_points, perm=perm, table=table, device=device)


def _spec_kernel(spec):
    return spec.c_kernel()


def assemble(spec, cloud, ct, bt, cfg=ACAConfig(), self_shift=None, device=0):
    """Device assembly: dense leaves evaluated directly,
    admissible leaves by batched ACA (scalar for d = 1, sigma_3 vector for d = 3)
    + recompression.  ``self_shift`` defaults to zeta = N_c.
    Returns ``(HMatrix, StorageReport)``."""
    if spec.d != cloud.d and cloud.d != 1:
        raise ValueError("kernel dimension does not match the cloud")
    pts = np.ascontiguousarray(ct.points_tree, dtype=np.float64)
    nrm = ct.normals_tree if spec.variant == "elasto_t" else None
    if spec.variant == "elasto_t" and nrm is None:
        raise ValueError("ElastoT requires normals on the cloud")
    perm = np.ascontiguousarray(ct.permutation, dtype=np.int64)
    table = bt.leaf_table
    c = cfg.c_struct()
    kern = _spec_kernel(spec)
    shift = float(cloud.size) if self_shift is None else float(self_shift)
    h = C.c_void_p()
    _lib.check(_lib.lib().hmx_assemble(_lib.context(device), C.byref(kern), _lib.ptr(pts), _lib.ptr(nrm),
                                       pts.shape[0], _lib.ptr(perm), _lib.ptr(table), len(table), C.byref(c),
                                       shift, C.byref(h)), "hmx_assemble")
    H = HMatrix(h, spec.d, pts.shape[0], block_tree=bt, perm=perm, spec=spec, table=bt.table, device=device)
    H.self_shift = shift
    if cfg.certify:
        H = _certify(H, spec, cloud, ct, bt, cfg, shift, device)
    return H, storage_report(H)


def splice(base, sub, idx):
    """New HMatrix = ``base`` with leaf ``idx[j]`` replaced by leaf ``j`` of ``sub`` (hmx_hmatrix_splice,
    a device-side re-layout of the streams)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    if idx.shape != (len(sub.table),):
        raise ValueError("splice: one base leaf index per leaf of sub")
    h = C.c_void_p()
    _lib.check(_lib.lib().hmx_hmatrix_splice(base.handle, sub.handle, _lib.ptr(idx), C.byref(h)), "hmx_hmatrix_splice")
    H = HMatrix(h, base.d, base.n_points, block_tree=base.block_tree, perm=base.perm, spec=base.spec,
                table=base.table, device=base.device)
    H.self_shift = base.self_shift
    return H


def _certify(H, spec, cloud, ct, bt, cfg, shift, device, max_rounds=4):
    """Opt-in per-leaf guarantee ||A_b - U_b V_b^H||_F <= eps ||A_b||_F on every admissible leaf
    (BASELINE north_star; SPEC.md:329 only promises 3 eps): every leaf is regenerated on the device
    (block_errors), the leaves above eps are re-compressed -- ACA stopped at eps / 4^k, truncation at
    eps / (2 4^(k-1)) -- and checked again, at most ``max_rounds`` times, then spliced into H."""
    from dataclasses import replace

    from .shard import LeafSubset

    eps = cfg.eps_aca
    err2, norm2 = block_errors(H, spec, cloud, shift)
    t = np.asarray(H.table)
    rel = np.sqrt(err2 / np.maximum(norm2, np.finfo(float).tiny))
    todo = np.flatnonzero((t[:, 0] == 1) & (rel > eps))
    report = {"leaves_above_eps": int(len(todo)), "worst_before": float(rel[t[:, 0] == 1].max(initial=0.0)),
              "rounds": []}
    f = 4.0
    for _ in range(max_rounds):
        if not len(todo):
            break
        sub_cfg = replace(cfg, eps_aca=eps / f, eps_recompress=eps / (f / 2.0), certify=False)
        Hs, _ = assemble(spec, cloud, ct, LeafSubset(bt, todo), sub_cfg, self_shift=shift, device=device)
        e2, n2 = block_errors(Hs, spec, cloud, shift)
        r = np.sqrt(e2 / np.maximum(n2, np.finfo(float).tiny))
        H = splice(H, Hs, todo)
        report["rounds"].append({"leaves": int(len(todo)), "eps_aca": eps / f, "eps_recompress": eps / (f / 2.0),
                                 "worst_after": float(r.max())})
        todo = todo[r > eps]
        f *= 4.0
    report["leaves_still_above_eps"] = int(len(todo))
    H.certify_report = report
    return H


def block_errors(h, spec, cloud, self_shift=None):
    """Per-leaf ||A_b - U_b V_b^H||_F^2 and ||A_b||_F^2 by regenerating every
    leaf on the device (``hmx_block_errors``; the blockwise accumulation of
    SPEC.md:510).  Dense leaves report error 0.  Returns (err2, norm2), one
    entry per leaf in ``h.table`` order."""
    if h.perm is None:
        raise ValueError("block_errors needs the tree permutation of the H-matrix")
    if spec.d != h.d:
        raise ValueError("kernel dimension does not match the H-matrix")
    pts = np.ascontiguousarray(np.asarray(cloud.points, dtype=np.float64)[h.perm])
    nrm = None
    if spec.variant == "elasto_t":
        if cloud.normals is None:
            raise ValueError("ElastoT requires normals on the cloud")
        nrm = np.ascontiguousarray(np.asarray(cloud.normals, dtype=np.float64)[h.perm])
    if self_shift is None:
        self_shift = h.self_shift if h.self_shift is not None else float(cloud.size)
    nb = len(h.table)
    err2 = np.empty(nb, np.float64)
    norm2 = np.empty(nb, np.float64)
    kern = _spec_kernel(spec)
    _lib.check(_lib.lib().hmx_block_errors(h.handle, C.byref(kern), _lib.ptr(pts), _lib.ptr(nrm), pts.shape[0],
                                           float(self_shift), _lib.ptr(err2), _lib.ptr(norm2)), "hmx_block_errors")
    return err2, norm2


def storage_report(h):
    """SPEC.md:431-439."""
    st = h.stats()
    N = h.d * h.n_points
    bound = None
    if h.block_tree is not None:
        csp = sparsity_pattern(h.block_tree)
        nl = h.d * h.block_tree.rows.n_leaf
        rmax = max(st["max_rank_after"], nl)
        bound = 2.0 * csp * rmax * N * (math.log2(N) - math.log2(nl) + 1.0)
    return StorageReport(n_stored=int(st["n_stored"]), n_dense_equiv=N * N, tau=st["n_stored"] / float(N * N),
                         max_rank_before=int(st["max_rank_before"]), max_rank_after=int(st["max_rank_after"]),
                         bound=bound)


def _is_cuda_tensor(x):
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda", False))


def matvec(h, x, out=None, stream=None):
    """y = A_H x; x in original point order.  numpy in ->
    numpy out (host copies inside); a CUDA complex128 torch tensor in -> a
    CUDA tensor out (no host round trip), launched on ``stream`` (a
    cudaStream_t; default: torch's current stream, so the result is ordered
    with the caller's torch work).  Safe to call concurrently on one H from
    several threads / streams (``hmx_matvec_on``)."""
    n = h.d * h.n_points
    if stream is None:
        stream = getattr(h, "_stream", None)
    if _is_cuda_tensor(x):
        import torch

        if x.dtype != torch.complex128 or x.numel() != n or not x.is_contiguous():
            raise ValueError("dimension mismatch")
        y = torch.empty_like(x) if out is None else out
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        _lib.check(_lib.lib().hmx_matvec_on(h.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), DEVICE,
                                            int(stream)), "hmx_matvec")
        return y
    x = np.ascontiguousarray(x, dtype=np.complex128)
    if x.shape != (n,):
        raise ValueError("dimension mismatch")
    y = np.empty_like(x) if out is None else out
    if stream is None:
        _lib.check(_lib.lib().hmx_matvec(h.handle, _lib.ptr(x), _lib.ptr(y), HOST), "hmx_matvec")
    else:
        _lib.check(_lib.lib().hmx_matvec_on(h.handle, _lib.ptr(x), _lib.ptr(y), HOST, int(stream)), "hmx_matvec")
    return y
