"""Formatted H-arithmetic and the recursive H-LU on the device -- the reference's
``hmatx.hmatrix`` operations ``formatted_addmul``, ``hlu``, ``triangular_solve``
and ``hmatx.solve.solve_direct`` (section 3.2,
"the LU factorization is classically decomposed into 4 steps").  The reference
module is absent from the mount; SURVEY 8(f) row 4.

Layout.  The factorisation works on a device-resident copy of the assembled
H-matrix's leaves, rebuilt into the block tree of ``BlockTree.root``
(``geometry.py:277-295``): ``Dense`` (dm x dn complex128), ``LowRank``
(U dm x k, V dn x k, block = U V^H) and ``Sub`` (grid of children over the
cluster children).  The leaves are taken zero-copy from the assembly's HBM
streams (``hmx_hmatrix_device_layout``) and cloned, so the source H stays
immutable.  All index ranges are dofs in tree order.

Arithmetic (all complex128 on the device, torch's current stream):
* dense diagonal leaves: pivoted LU (cuSOLVER getrf); L = P L~ unit lower,
  U upper, the permutation kept as an index vector;
* triangular solves with dense / low-rank / hierarchical right-hand sides
  (low-rank: only U, resp. V, is transformed);
* ``formatted_addmul`` C <- C + alpha A B over the 27 format cases: a
  low-rank operand multiplies through its thin factors, hierarchical x
  hierarchical recurses over the cluster children (a hierarchical target of
  at most _DENSE_T rows / columns takes the exact product as one GEMM on the
  operands' dense images), dense targets accumulate densely; low-rank targets
  collect addends and are truncated with eps_LU at the truncation points of
  oracle/hlu.py (decision 7).  A product landing on a low-rank target without
  a low-rank operand is formed per child block and agglomerated into one
  factor pair.
* truncations (the recompress rule): batched on the device by
  ``hmx_truncate_batch`` (the assembly's Gram / Cholesky / eigen-solver /
  form kernels), rank-deficient pairs re-submitted as (U V^H, I), problems
  wider than 112 columns reduced first by a seeded Gaussian range sketch.

The LU is in place: ``LUFactors.lower`` / ``.upper`` are the strictly lower /
upper blocks plus the unit-lower / upper factors of the diagonal leaves of the
same tree.
"""

import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import FactorizationError
from .geometry import AdmissibleLeaf, DenseLeaf, Subdivided

_RULES = ("frobenius", "spectral")


_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("hlu: a CUDA device is required (no CPU fallback)")
        _TORCH = torch
    return _TORCH


_EYE = {}


def _eye(n, like):
    """Cached identity (the orthonormal side of the dense-form pairs; read-only)."""
    key = (n, like.device)
    e = _EYE.get(key)
    if e is None:
        e = _EYE[key] = _torch().eye(n, dtype=like.dtype, device=like.device)
    return e


# --------------------------------------------------------------------------------------------
# node types
# --------------------------------------------------------------------------------------------
class Dense:
    __slots__ = ("r0", "r1", "c0", "c1", "a", "L", "U", "pidx", "pinv")

    def __init__(self, r0, r1, c0, c1, a):
        self.r0, self.r1, self.c0, self.c1, self.a = r0, r1, c0, c1, a
        self.L = self.U = self.pidx = self.pinv = None


class LowRank:
    __slots__ = ("r0", "r1", "c0", "c1", "u", "v", "pend", "acc")

    def __init__(self, r0, r1, c0, c1, u, v):
        self.r0, self.r1, self.c0, self.c1, self.u, self.v = r0, r1, c0, c1, u, v
        self.pend = []      # low-rank addends (U_i, V_i) awaiting truncation
        self.acc = None     # dense addend accumulated from small-target products

    @property
    def rank(self):
        return int(self.u.shape[1])


class Sub:
    __slots__ = ("r0", "r1", "c0", "c1", "rs", "cs", "ch", "fin", "dc")

    def __init__(self, r0, r1, c0, c1, rs, cs, ch):
        self.r0, self.r1, self.c0, self.c1, self.rs, self.cs, self.ch = r0, r1, c0, c1, rs, cs, ch
        self.fin = False   # a finished L / U factor block: never modified again
        self.dc = None     # its dense image, built on first use as a product operand


_DC_MAX = 1 << 22      # largest finished block (entries) kept as a dense operand image (64 MB)
_DC_BUDGET = 16 << 30  # HBM bytes all dense operand images of one factorisation may take
_DENSE_T = int(os.environ.get("HMX_HLU_DENSE_T", "512"))  # hierarchical targets up to this size take products densely


def _finalize(x):
    if isinstance(x, Sub):
        x.fin = True
        for row in x.ch:
            for c in row:
                _finalize(c)


def _dense_image(ar, x):
    """Dense image of a finished hierarchical block (one GEMM per product instead of a recursion
    over its leaves), or None (block above _DC_MAX entries, or the images' HBM budget spent)."""
    if not x.fin:
        return None
    if x.dc is None:
        n = (x.r1 - x.r0) * (x.c1 - x.c0)
        if n > _DC_MAX or ar.dc_bytes + 16 * n > _DC_BUDGET:
            return None
        x.dc = _dense(ar, x)
        ar.dc_bytes += 16 * n
    return x.dc


@dataclass
class Arith:
    """Truncation settings + counters of one formatted-arithmetic session."""

    eps: float
    rule: str = "frobenius"
    n_trunc: int = 0
    n_trunc_calls: int = 0
    t_trunc: float = 0.0
    dc_bytes: int = 0
    k_hist: list = field(default_factory=list)
    n_getrf: int = 0
    max_rank: int = 0

    def __post_init__(self):
        if self.rule not in _RULES:
            raise ValueError(f"unknown truncation rule {self.rule!r}")
        if not self.eps >= 0:
            raise ValueError("eps_lu must be >= 0")


def _trank(s, eps, rule):
    """Kept rank for descending singular values (the recompress rule)."""
    if s.size == 0 or s[0] == 0.0:
        return 0
    if rule == "spectral":
        return int(np.count_nonzero(s > eps * s[0]))
    sq = s * s
    tail = np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]])
    return int(np.flatnonzero(tail <= (eps * eps) * tail[0])[0])


_PEND_FLUSH = 400     # pending columns on one low-rank target before it is truncated early
_AGGLO_MAX = 512      # agglomerated product columns before an intermediate truncation
# pairs whose kernel problem would have more columns than this are truncated by cuSOLVER QR + SVD
# instead (the one-CTA eigen-solve of a K x K problem is latency-bound, O(K) dependent phases)
_CUSOLVER_K = 1020   # hmx_truncate_batch accepts K <= 1020 (capi.cu hmx_truncate_batch)
# pairs whose kernel problem would exceed this many columns go through a _SKETCH_L-column range sketch
_SKETCH_K = int(os.environ.get("HMX_HLU_SKETCH_K", "112"))
_SKETCH_L = 112
_SKETCH_S = 56        # narrow sketch (the K <= 60 recompression class) ...
_SKETCH_S_RANK = 24   # ... for targets whose rank before the update was at most this
_TRULES = {"frobenius": 0, "spectral": 1}


def _kernel_batch(ar, items, eps=None):
    """One ``hmx_truncate_batch`` call: list of (U, V) -> list of (U', V') or None for items whose
    V was numerically rank-deficient (regularised Cholesky; not formed)."""
    torch = _torch()
    dev = items[0][0].device
    _lib.bind_torch_stream(dev.index or 0)
    n = len(items)
    dm = np.empty(n, np.int64)
    dn = np.empty(n, np.int64)
    K = np.empty(n, np.int64)
    ptr = np.zeros((4, n), np.uint64)
    keep, outs = [], []
    for i, (u, v) in enumerate(items):
        dm[i], K[i] = u.shape
        dn[i] = v.shape[0]
    # all outputs in one allocation (one torch call instead of 2n); segments start on 256-byte
    # boundaries like the allocator's own blocks
    su = (K * dm + 15) // 16 * 16
    sv = (K * dn + 15) // 16 * 16
    offs = np.concatenate(([0], np.cumsum(su + sv)))
    out = torch.empty(int(offs[-1]), dtype=items[0][0].dtype, device=dev)
    for i, (u, v) in enumerate(items):
        uc = u.mT.contiguous()          # (K, dm) row-major = dm x K column-major
        vc = v.mT.contiguous()
        o = int(offs[i])
        k, m_, n_ = int(K[i]), int(dm[i]), int(dn[i])
        uo = out[o:o + k * m_].view(k, m_)
        vo = out[o + int(su[i]):o + int(su[i]) + k * n_].view(k, n_)
        keep += [uc, vc]
        outs.append((uo, vo))
        ptr[:, i] = (uc.data_ptr(), vc.data_ptr(), uo.data_ptr(), vo.data_ptr())
    ranks = np.zeros(n, np.int64)
    flags = np.zeros(n, np.int32)
    ar.n_trunc_calls += 1
    ar.k_hist.append(int(K.max()))
    t0 = time.perf_counter()
    _lib.check(_lib.lib().hmx_truncate_batch(_lib.context(dev.index or 0), n, _lib.ptr(dm), _lib.ptr(dn),
                                              _lib.ptr(K), _lib.ptr(ptr[0]), _lib.ptr(ptr[1]), _lib.ptr(ptr[2]),
                                              _lib.ptr(ptr[3]), float(ar.eps if eps is None else eps),
                                              _TRULES[ar.rule],
                                              _lib.ptr(ranks), _lib.ptr(flags)), "hmx_truncate_batch")
    ar.t_trunc += time.perf_counter() - t0
    # compact copy of the kept columns (one allocation sized sum r (dm + dn)): the truncated
    # leaves then keep only their final-rank storage alive, not the K-column batch buffer
    kept = [i for i in range(n) if not flags[i] & 1]
    pieces = []
    for i in kept:
        r = int(ranks[i])
        pieces += [outs[i][0][:r].reshape(-1), outs[i][1][:r].reshape(-1)]
    flat = torch.cat(pieces) if pieces else None
    del out, outs[:]
    res = [None] * n
    o = 0
    for i in kept:
        r, m_, n_ = int(ranks[i]), int(dm[i]), int(dn[i])
        u = flat[o:o + r * m_].view(r, m_).mT
        o += r * m_
        v = flat[o:o + r * n_].view(r, n_).mT
        o += r * n_
        res[i] = (u, v)
    return res


def _dense_form(u, v):
    """U V^H as the pair (U V^H, I) -- or, when U has fewer rows, its adjoint (V U^H, I) with the
    result swapped back: the V side is orthonormal, so the kernel's Cholesky is exact.
    Returns (pair, swapped)."""
    torch = _torch()
    if u.shape[0] < v.shape[0]:
        return (v @ u.mH, _eye(u.shape[0], u)), True
    return (u @ v.mH, _eye(v.shape[0], u)), False


def _truncate_batch(ar, items, hints=None):
    """items: list of (U, V) pairs (any strides) -> list of truncated (U', V') pairs, on the device
    through ``hmx_truncate_batch`` (Gram pair, scaled Cholesky, Hermitian eigen-solver, truncation
    rule, U' = U W_U, V' = V W_V -- the assembly's recompression kernels), one call per batch.
    A pair with at least as many columns as V has rows, or whose V turns out numerically
    rank-deficient, is re-submitted as (U V^H, I) (or its adjoint); cuSOLVER QR + SVD only when
    both sides exceed the kernel's 1020-column limit."""
    if not items:
        return []
    torch = _torch()
    res = [None] * len(items)
    sub, idx, swp = [], [], []
    sk_x, sk_meta = [], []
    for i, (u, v) in enumerate(items):
        if u.shape[1] == 0:
            res[i] = (u, v)
            continue
        ar.n_trunc += 1
        if min(u.shape[1], u.shape[0], v.shape[0]) > _CUSOLVER_K:
            res[i] = _trunc_cusolver(ar, u, v)
            ar.max_rank = max(ar.max_rank, res[i][0].shape[1])
            continue
        if min(u.shape[1], u.shape[0], v.shape[0]) > _SKETCH_K and ar.rule == "frobenius":
            sk_x.append((u, v))
            sk_meta.append(i)
            continue
        sub.append(_direct_form(u, v))
        swp.append(sub[-1][1])
        sub[-1] = sub[-1][0]
        idx.append(i)
    if sk_x:
        # U V^H = Q (Q^H U) V^H on a sketched range basis Q, truncated as the (V (U^H Q), Q) pair:
        # its V side is orthonormal and it has at most l columns (the one-CTA eigen-solve stays
        # small); kernel result (P, R) means U V^H ~ R P^H.  The sketch width follows the rank
        # the target had before the update (_SKETCH_S columns when it was small, the fast kernel
        # class), widened to _SKETCH_L where the narrow sketch saturates.
        ls = [_SKETCH_S if hints is not None and hints[i] is not None and hints[i] <= _SKETCH_S_RANK
              else _SKETCH_L for i in sk_meta]
        qs = _sketch_basis(ar, sk_x, ls)
        wide = [j for j, (q, sl) in enumerate(zip(qs, ls)) if q is None and sl < _SKETCH_L]
        if wide:
            for j, q in zip(wide, _sketch_basis(ar, [sk_x[j] for j in wide], [_SKETCH_L] * len(wide))):
                qs[j] = q
        for (u, v), Q, i in zip(sk_x, qs, sk_meta):
            if Q is None:   # sketch saturated: the direct (possibly dense) form
                pair, sw = _direct_form(u, v)
                sub.append(pair)
                swp.append(sw)
            elif Q.shape[1] == 0:
                res[i] = (u[:, :0], v[:, :0])
                continue
            else:
                sub.append((v @ (u.mH @ Q), Q))
                swp.append(True)
            idx.append(i)
    dense_done = [False] * len(idx)
    while idx:
        out = _kernel_batch(ar, sub)
        redo, ridx, rswp, rdone = [], [], [], []
        for i, s_, sw, dd, o in zip(idx, sub, swp, dense_done, out):
            if o is not None:
                res[i] = (o[1], o[0]) if sw else o
                ar.max_rank = max(ar.max_rank, o[0].shape[1])
            elif not dd and min(items[i][0].shape[0], items[i][1].shape[0]) <= 1020:
                pair, sw2 = _dense_form(*items[i])
                redo.append(pair)
                rswp.append(sw2)
                ridx.append(i)
                rdone.append(True)
            else:
                # both sides above the kernel's 1020 limit: Householder QR + SVD (cuSOLVER)
                res[i] = _trunc_cusolver(ar, *items[i])
        sub, idx, swp, dense_done = redo, ridx, rswp, rdone
    return res


def _direct_form(u, v):
    """(pair, swapped) submitted to the kernel without sketching: (U, V) itself, or the dense
    form when U V^H has no more columns than rows on its smaller side."""
    if u.shape[1] >= min(u.shape[0], v.shape[0]):
        return _dense_form(u, v)
    return (u, v), False


def _sketch_basis(ar, pairs_in, ls):
    """Orthonormal bases of the ranges of U V^H (dm x dn) from a seeded Gaussian sketch
    Y = U (V^H Omega) (Omega dn x l, l = ls[i]): the (Y, I) pairs are truncated at max(eps / 10, 1e-8)
    in one kernel call and the orthogonal columns A = Y W_U normalised.  None where the sketch
    saturates (kept rank above l - 8: the range may be larger than the sketch)."""
    torch = _torch()
    pairs = []
    for (u, v), sl in zip(pairs_in, ls):
        g = torch.Generator(device=u.device)
        g.manual_seed(0x5EED + 7 * u.shape[0] + v.shape[0])
        om = torch.randn((v.shape[0], sl), dtype=u.dtype, device=u.device, generator=g)
        pairs.append((u @ (v.mH @ om), _eye(sl, u)))
    out = _kernel_batch(ar, pairs, eps=max(0.1 * ar.eps, 1e-8))
    qs = []
    for o, sl in zip(out, ls):
        if o is None or o[0].shape[1] > sl - 8:
            qs.append(None)
        elif o[0].shape[1] == 0:
            qs.append(o[0])
        else:
            # A = Y W_U has orthogonal columns of norms sqrt(s_i), but the Gram route leaves their
            # trailing directions orthogonal only to ~u s_1 / s_q: one Cholesky-QR pass on the
            # normalised (well-conditioned) columns restores orthonormality
            a = o[0] / o[0].norm(dim=0, keepdim=True)
            r = torch.linalg.cholesky(a.mH @ a).mH
            qs.append(torch.linalg.solve_triangular(r, a, upper=True, left=False))
    return qs


def _trunc_cusolver(ar, u, v):
    torch = _torch()
    qu, ru = torch.linalg.qr(u)
    qv, rv = torch.linalg.qr(v)
    p, s, lh = torch.linalg.svd(ru @ rv.mH, full_matrices=False)
    r = _trank(s.cpu().numpy(), ar.eps, ar.rule)
    root = s[:r].sqrt().to(u.dtype)
    return (qu @ p[:, :r]) * root, (qv @ lh.mH[:, :r]) * root


def _trunc(ar, u, v):
    """(U, V) -> truncated (U', V') with U' V'^H ~ U V^H."""
    return _truncate_batch(ar, [(u, v)])[0]


def _dense_to_lr(ar, m):
    """Truncated SVD of a dense block (operand construction only)."""
    torch = _torch()
    p, s, lh = torch.linalg.svd(m, full_matrices=False)
    r = _trank(s.cpu().numpy(), ar.eps, ar.rule)
    root = s[:r].sqrt().to(m.dtype)
    return p[:, :r] * root, lh.mH[:, :r] * root


def _cat(x):
    torch = _torch()
    us = [x.u] + [p[0] for p in x.pend]
    vs = [x.v] + [p[1] for p in x.pend]
    x.pend = []
    if x.acc is not None:
        # a dense addend is pending: the whole block as the pair (X, I)
        X = x.acc
        x.acc = None
        for u, v in zip(us, vs):
            if u.shape[1]:
                X.addmm_(u, v.mH)
        return X, _eye(X.shape[1], X)
    # stacked as (K, rows) row-major = the column-major panels the truncation kernel reads
    return torch.cat([t.mT for t in us], 0).mT, torch.cat([t.mT for t in vs], 0).mT


def _flush(ar, x):
    if x.pend or x.acc is not None:
        hint = x.u.shape[1]
        x.u, x.v = _truncate_batch(ar, [_cat(x)], [hint])[0]


def _pending(x, out):
    if isinstance(x, LowRank):
        if x.pend or x.acc is not None:
            out.append(x)
    elif isinstance(x, Sub):
        for row in x.ch:
            for c in row:
                _pending(c, out)


def _flush_batch(ar, nodes):
    """Truncate every pending low-rank leaf under ``nodes`` in one batched call."""
    todo = []
    for x in nodes:
        _pending(x, todo)
    if todo:
        hints = [x.u.shape[1] for x in todo]
        for x, (u, v) in zip(todo, _truncate_batch(ar, [_cat(x) for x in todo], hints)):
            x.u, x.v = u, v


# --------------------------------------------------------------------------------------------
# products with dense multivectors, conversion
# --------------------------------------------------------------------------------------------
def _mul(ar, x, X):
    """x @ X for a dense multivector X (rows = x's columns)."""
    if isinstance(x, Dense):
        return x.a @ X
    if isinstance(x, LowRank):
        _flush(ar, x)
        return x.u @ (x.v.mH @ X)
    dc = _dense_image(ar, x)
    if dc is not None:
        return dc @ X
    out = X.new_zeros((x.r1 - x.r0, X.shape[1]))
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            out[a - x.r0:b - x.r0] += _mul(ar, x.ch[i][j], X[c - x.c0:e - x.c0])
    return out


def _mulh(ar, x, X):
    """x^H @ X for a dense multivector X (rows = x's rows)."""
    if isinstance(x, Dense):
        return x.a.mH @ X
    if isinstance(x, LowRank):
        _flush(ar, x)
        return x.v @ (x.u.mH @ X)
    dc = _dense_image(ar, x)
    if dc is not None:
        return dc.mH @ X
    out = X.new_zeros((x.c1 - x.c0, X.shape[1]))
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            out[c - x.c0:e - x.c0] += _mulh(ar, x.ch[i][j], X[a - x.r0:b - x.r0])
    return out


def _dense(ar, x):
    torch = _torch()
    if isinstance(x, Dense):
        return x.a
    if isinstance(x, LowRank):
        _flush(ar, x)
        return x.u @ x.v.mH
    if x.dc is not None:
        return x.dc
    out = torch.empty((x.r1 - x.r0, x.c1 - x.c0), dtype=torch.complex128, device=_dev_of(x))
    _dense_into(ar, x, out)
    return out


def _dense_into(ar, x, out):
    """Dense image of Sub ``x`` written in place into ``out`` (the children tile it): nested
    Subs write straight into their sub-view instead of through a temporary of their own."""
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            ch = x.ch[i][j]
            v = out[a - x.r0:b - x.r0, c - x.c0:e - x.c0]
            if isinstance(ch, Sub) and ch.dc is None:
                _dense_into(ar, ch, v)
            else:
                v.copy_(_dense(ar, ch))


def _dev_of(x):
    while isinstance(x, Sub):
        x = x.ch[0][0]
    if isinstance(x, Dense):
        return (x.a if x.a is not None else x.U).device
    return x.u.device


def _part(ar, x, i, k, r0, r1, c0, c1):
    """Sub-block [r0, r1) x [c0, c1) of operand x: child (i, k) of a Sub, a view of a leaf."""
    if isinstance(x, Sub):
        ch = x.ch[i][k]
        if (ch.r0, ch.r1, ch.c0, ch.c1) != (r0, r1, c0, c1):
            raise ValueError("formatted_addmul: non-conformal block partitions")
        return ch
    if (x.r0, x.r1, x.c0, x.c1) == (r0, r1, c0, c1):
        return x
    if isinstance(x, Dense):
        return Dense(r0, r1, c0, c1, x.a[r0 - x.r0:r1 - x.r0, c0 - x.c0:c1 - x.c0])
    _flush(ar, x)
    return LowRank(r0, r1, c0, c1, x.u[r0 - x.r0:r1 - x.r0], x.v[c0 - x.c0:c1 - x.c0])


def _parts(x, rows):
    if isinstance(x, Sub):
        return x.rs if rows else x.cs
    return [(x.r0, x.r1)] if rows else [(x.c0, x.c1)]


# --------------------------------------------------------------------------------------------
# formatted addition / multiplication
# --------------------------------------------------------------------------------------------
def _pend(ar, C, U, V):
    C.pend.append((U, V))
    if C.u.shape[1] + sum(p[0].shape[1] for p in C.pend) > _PEND_FLUSH:
        _flush(ar, C)


def _add_lr(ar, C, U, V):
    """C += U V^H."""
    if U.shape[1] == 0:
        return
    if isinstance(C, Dense):
        C.a.addmm_(U, V.mH)
    elif isinstance(C, LowRank):
        _pend(ar, C, U, V)
    else:
        for i, (a, b) in enumerate(C.rs):
            for j, (c, e) in enumerate(C.cs):
                _add_lr(ar, C.ch[i][j], U[a - C.r0:b - C.r0], V[c - C.c0:e - C.c0])


def _add_dense(ar, C, M):
    """C += M for a dense M (a low-rank leaf accumulates it densely until its next truncation)."""
    if isinstance(C, Dense):
        C.a.add_(M)
    elif isinstance(C, LowRank):
        if C.acc is None:
            C.acc = M.clone()
        else:
            C.acc.add_(M)
    else:
        for i, (a, b) in enumerate(C.rs):
            for j, (c, e) in enumerate(C.cs):
                _add_dense(ar, C.ch[i][j], M[a - C.r0:b - C.r0, c - C.c0:e - C.c0])


def _dense_op(ar, x):
    """Dense image of an operand (cached for finished hierarchical blocks)."""
    if isinstance(x, Sub):
        img = _dense_image(ar, x)
        if img is not None:
            return img
    return _dense(ar, x)


def _prod_lr(ar, A, B):
    """Low-rank (U, V) with U V^H ~ A B (truncated with eps)."""
    torch = _torch()
    if isinstance(A, LowRank):
        _flush(ar, A)
        return A.u, _mulh(ar, B, A.v)
    if isinstance(B, LowRank):
        _flush(ar, B)
        return _mul(ar, A, B.u), B.v
    if isinstance(A, Dense) and isinstance(B, Dense):
        return A.a, B.a.mH          # untruncated: inner dimension columns
    # at least one hierarchical operand: per child block, then agglomerate with one truncation
    m, n = A.r1 - A.r0, B.c1 - B.c0
    Rp, Cp = _parts(A, True), _parts(B, False)
    Kp = A.cs if isinstance(A, Sub) else B.rs
    us, vs = [], []
    for i, (ra, rb) in enumerate(Rp):
        for j, (ca, cb) in enumerate(Cp):
            for k, (ka, kb) in enumerate(Kp):
                u, v = _prod_lr(ar, _part(ar, A, i, k, ra, rb, ka, kb), _part(ar, B, k, j, ka, kb, ca, cb))
                if u.shape[1] == 0:
                    continue
                up = u.new_zeros((m, u.shape[1]))
                vp = v.new_zeros((n, v.shape[1]))
                up[ra - A.r0:rb - A.r0] = u
                vp[ca - B.c0:cb - B.c0] = v
                us.append(up)
                vs.append(vp)
    if not us:
        dev = _dev_of(A)
        z = torch.zeros((m, 0), dtype=torch.complex128, device=dev)
        return z, torch.zeros((n, 0), dtype=torch.complex128, device=dev)
    U, V = torch.cat([t.mT for t in us], 0).mT, torch.cat([t.mT for t in vs], 0).mT
    return _trunc(ar, U, V) if U.shape[1] > _AGGLO_MAX else (U, V)


def _addmul(ar, C, A, B, alpha=-1.0):
    """C <- C + alpha A B (formatted, truncation eps_LU on low-rank targets)."""
    if isinstance(A, LowRank) and isinstance(B, LowRank):
        # rank min(r_A, r_B) through the r_A x r_B core A.v^H B.u
        _flush(ar, A)
        _flush(ar, B)
        core = A.v.mH @ B.u
        if A.rank <= B.rank:
            _add_lr(ar, C, alpha * A.u, B.v @ core.mH)
        else:
            _add_lr(ar, C, alpha * (A.u @ core), B.v)
        return
    if isinstance(A, LowRank):
        _flush(ar, A)
        if A.rank:
            _add_lr(ar, C, alpha * A.u, _mulh(ar, B, A.v))
        return
    if isinstance(B, LowRank):
        _flush(ar, B)
        if B.rank:
            _add_lr(ar, C, alpha * _mul(ar, A, B.u), B.v)
        return
    if isinstance(C, Sub):
        if C.r1 - C.r0 <= _DENSE_T and C.c1 - C.c0 <= _DENSE_T:
            # small hierarchical target: the exact product by one GEMM on the operands' dense
            # images, scattered into the target's leaves (oracle decision 8)
            M = _dense_op(ar, A) @ _dense_op(ar, B)
            _add_dense(ar, C, M if alpha == 1.0 else M.mul_(alpha))
            return
        Kp = A.cs if isinstance(A, Sub) else (B.rs if isinstance(B, Sub) else [(A.c0, A.c1)])
        for i, (ra, rb) in enumerate(C.rs):
            for j, (ca, cb) in enumerate(C.cs):
                for k, (ka, kb) in enumerate(Kp):
                    _addmul(ar, C.ch[i][j], _part(ar, A, i, k, ra, rb, ka, kb),
                            _part(ar, B, k, j, ka, kb, ca, cb), alpha)
        return
    if isinstance(C, Dense):
        if isinstance(A, Dense) and isinstance(B, Dense):
            C.a.addmm_(A.a, B.a, alpha=alpha)
        else:
            C.a.add_(_mul(ar, A, _dense(ar, B)), alpha=alpha)
        return
    u, v = _prod_lr(ar, A, B)
    if u.shape[1]:
        _pend(ar, C, alpha * u, v)


# --------------------------------------------------------------------------------------------
# LU and triangular solves
# --------------------------------------------------------------------------------------------
def _lu(ar, x, path):
    torch = _torch()
    if isinstance(x, Dense):
        ar.n_getrf += 1
        lu, piv, info = torch.linalg.lu_factor_ex(x.a)
        P, L, U = torch.lu_unpack(lu, piv)
        d = U.diagonal().abs()
        dmax = float(d.max()) if d.numel() else 0.0
        if int(info) != 0 or d.numel() == 0 or float(d.min()) <= 1e-14 * max(dmax, 1e-300):
            raise FactorizationError(f"hlu: singular dense diagonal leaf at block path {path} "
                                     f"(rows [{x.r0}, {x.r1}))")
        x.L, x.U = L, U
        x.pidx = P.real.argmax(0)   # P^T X = X[pidx]
        x.pinv = P.real.argmax(1)   # P X = X[pinv]
        x.a = None
        return
    if not isinstance(x, Sub) or x.rs != x.cs:
        raise ValueError("hlu: diagonal block is not square / hierarchical")
    p = len(x.rs)
    for k in range(p):
        _lu(ar, x.ch[k][k], path + (k,))
        for j in range(k + 1, p):
            _solve_lower(ar, x.ch[k][k], x.ch[k][j])
        for i in range(k + 1, p):
            _solve_upper_right(ar, x.ch[k][k], x.ch[i][k])
        for j in range(k + 1, p):
            _finalize(x.ch[k][j])
            _finalize(x.ch[j][k])
        for i in range(k + 1, p):
            for j in range(k + 1, p):
                _addmul(ar, x.ch[i][j], x.ch[i][k], x.ch[k][j], -1.0)
        _flush_batch(ar, [x.ch[i][j] for i in range(k + 1, p) for j in range(k + 1, p)])


def _lsolve(ar, L, X):
    """L^{-1} X for a dense multivector (L = factored diagonal node)."""
    torch = _torch()
    if isinstance(L, Dense):
        return torch.linalg.solve_triangular(L.L, X[L.pidx], upper=False, unitriangular=True)
    X = X.clone()
    for k, (a, b) in enumerate(L.rs):
        xk = _lsolve(ar, L.ch[k][k], X[a - L.r0:b - L.r0])
        X[a - L.r0:b - L.r0] = xk
        for i in range(k + 1, len(L.rs)):
            c, e = L.rs[i]
            X[c - L.r0:e - L.r0] -= _mul(ar, L.ch[i][k], xk)
    return X


def _usolve(ar, U, X):
    """U^{-1} X for a dense multivector."""
    torch = _torch()
    if isinstance(U, Dense):
        return torch.linalg.solve_triangular(U.U, X, upper=True)
    X = X.clone()
    for k in range(len(U.rs) - 1, -1, -1):
        a, b = U.rs[k]
        xk = _usolve(ar, U.ch[k][k], X[a - U.r0:b - U.r0])
        X[a - U.r0:b - U.r0] = xk
        for i in range(k):
            c, e = U.rs[i]
            X[c - U.r0:e - U.r0] -= _mul(ar, U.ch[i][k], xk)
    return X


def _rsolve(ar, U, Y):
    """Y U^{-1} for a dense multivector Y (columns = U's columns)."""
    torch = _torch()
    if isinstance(U, Dense):
        return torch.linalg.solve_triangular(U.U, Y, upper=True, left=False)
    Y = Y.clone()
    for k, (a, b) in enumerate(U.cs):
        yk = _rsolve(ar, U.ch[k][k], Y[:, a - U.c0:b - U.c0])
        Y[:, a - U.c0:b - U.c0] = yk
        for j in range(k + 1, len(U.cs)):
            c, e = U.cs[j]
            Y[:, c - U.c0:e - U.c0] -= _mulh(ar, U.ch[k][j], yk.mH).mH
    return Y


def _solve_lower(ar, L, B):
    """B <- L^{-1} B (B any format, same row cluster as L)."""
    if isinstance(B, Dense):
        B.a = _lsolve(ar, L, B.a)
    elif isinstance(B, LowRank):
        _flush(ar, B)
        if B.rank:
            B.u = _lsolve(ar, L, B.u)
    elif isinstance(L, Sub):
        p, q = len(L.rs), len(B.cs)
        for k in range(p):
            for j in range(q):
                _solve_lower(ar, L.ch[k][k], B.ch[k][j])
            for j in range(q):
                for i in range(k + 1, p):
                    _addmul(ar, B.ch[i][j], L.ch[i][k], B.ch[k][j], -1.0)
            _flush_batch(ar, [B.ch[i][j] for i in range(k + 1, p) for j in range(q)])
    else:
        for j in range(len(B.cs)):
            _solve_lower(ar, L, B.ch[0][j])


def _solve_upper_right(ar, U, B):
    """B <- B U^{-1} (B any format, same column cluster as U)."""
    if isinstance(B, Dense):
        B.a = _rsolve(ar, U, B.a)
    elif isinstance(B, LowRank):
        _flush(ar, B)
        if B.rank:
            B.v = _rsolve(ar, U, B.v.mH).mH
    elif isinstance(U, Sub):
        p, q = len(U.cs), len(B.rs)
        for k in range(p):
            for i in range(q):
                _solve_upper_right(ar, U.ch[k][k], B.ch[i][k])
            for i in range(q):
                for j in range(k + 1, p):
                    _addmul(ar, B.ch[i][j], B.ch[i][k], U.ch[k][j], -1.0)
            _flush_batch(ar, [B.ch[i][j] for i in range(q) for j in range(k + 1, p)])
    else:
        for i in range(len(B.rs)):
            _solve_upper_right(ar, U, B.ch[i][0])


def _lmul(ar, L, X):
    """L X (unit-lower factor incl. the leaf permutations)."""
    if isinstance(L, Dense):
        return (L.L @ X)[L.pinv]
    out = X.new_zeros(X.shape)
    for i, (a, b) in enumerate(L.rs):
        acc = _lmul(ar, L.ch[i][i], X[a - L.r0:b - L.r0])
        for j in range(i):
            c, e = L.rs[j]
            acc = acc + _mul(ar, L.ch[i][j], X[c - L.r0:e - L.r0])
        out[a - L.r0:b - L.r0] = acc
    return out


def _umul(ar, U, X):
    if isinstance(U, Dense):
        return U.U @ X
    out = X.new_zeros(X.shape)
    for i, (a, b) in enumerate(U.rs):
        acc = _umul(ar, U.ch[i][i], X[a - U.r0:b - U.r0])
        for j in range(i + 1, len(U.rs)):
            c, e = U.rs[j]
            acc = acc + _mul(ar, U.ch[i][j], X[c - U.r0:e - U.r0])
        out[a - U.r0:b - U.r0] = acc
    return out


def _drop_images(x):
    if isinstance(x, Sub):
        x.dc = None
        for row in x.ch:
            for c in row:
                _drop_images(c)


def _walk(x):
    if isinstance(x, Sub):
        for row in x.ch:
            for c in row:
                yield from _walk(c)
    else:
        yield x


# --------------------------------------------------------------------------------------------
# construction
# --------------------------------------------------------------------------------------------
class _CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<c16", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _build(root, d, leaf_of, make_leaf):
    def rec(node):
        if isinstance(node, (DenseLeaf, AdmissibleLeaf)):
            return make_leaf(leaf_of[(node.row.index, node.col.index)])
        r, c = node.row, node.col
        rk = (r,) if r.is_leaf else r.children
        ck = (c,) if c.is_leaf else c.children
        kids = [rec(k) for k in node.children]
        grid = [kids[i * len(ck):(i + 1) * len(ck)] for i in range(len(rk))]
        return Sub(d * r.start, d * r.stop, d * c.start, d * c.stop,
                   [(d * q.start, d * q.stop) for q in rk], [(d * q.start, d * q.stop) for q in ck], grid)

    return rec(root)


def _leaf_index(bt):
    return {(int(t[5]), int(t[6])): b for b, t in enumerate(bt.table)}


def _own_copy(view):
    """A private contiguous copy of a view of the assembly's HBM streams.  ``.contiguous()`` is not
    enough: torch returns the view itself when it is already contiguous (a 1-row or 1-column block),
    and the in-place Schur updates would then write into the immutable source H."""
    out = _torch().empty(view.shape, dtype=view.dtype, device=view.device)
    out.copy_(view)
    return out


def copy_hmatrix(h, block_tree=None):
    """Device node tree holding a private copy of every leaf of the assembled H
    (zero-copy views of the HBM streams, cloned)."""
    torch = _torch()
    bt = block_tree if block_tree is not None else h.block_tree
    if bt is None:
        raise ValueError("hlu needs the H-matrix's block tree")
    nb = len(h.table)
    moff = np.empty(nb, np.int64)
    ld = np.empty(nb, np.int64)
    voff = np.empty(nb, np.int64)
    bufs = np.empty(4, np.uint64)
    _lib.check(_lib.lib().hmx_hmatrix_device_layout(h.handle, _lib.ptr(moff), _lib.ptr(ld), _lib.ptr(voff),
                                                    _lib.ptr(bufs)), "hmx_hmatrix_device_layout")
    dev = torch.device("cuda", h.device)
    R = torch.as_tensor(_CAI(bufs[0], bufs[1]), device=dev)
    Vs = torch.as_tensor(_CAI(bufs[2], bufs[3]), device=dev) if bufs[3] else None
    ranks = h.block_info()["rank_after"]
    d = h.d
    tab = np.asarray(h.table)

    def make_leaf(b):
        k, r0, r1, c0, c1 = (int(t) for t in tab[b][:5])
        dm, dn = d * (r1 - r0), d * (c1 - c0)
        o, l = int(moff[b]), int(ld[b])
        if k == 0:
            a = _own_copy(R[o:o + l * dn].view(dn, l)[:, :dm].transpose(0, 1))
            return Dense(d * r0, d * r1, d * c0, d * c1, a)
        r = int(ranks[b])
        if r == 0:
            u = torch.zeros((dm, 0), dtype=torch.complex128, device=dev)
            v = torch.zeros((dn, 0), dtype=torch.complex128, device=dev)
        else:
            u = _own_copy(R[o:o + l * r].view(r, l)[:, :dm].transpose(0, 1))
            vo = int(voff[b])
            v = _own_copy(Vs[vo:vo + dn * r].view(r, dn).transpose(0, 1))
        return LowRank(d * r0, d * r1, d * c0, d * c1, u, v)

    return _build(bt.root, d, _leaf_index(bt), make_leaf)


def from_dense(bt, d, A, eps, rule="frobenius", device=0):
    """Node tree of a dense (tree-ordered) matrix on the block partition ``bt``:
    dense leaves copied, admissible leaves compressed by truncated SVD with ``eps``
    (test / formatted_addmul operands)."""
    torch = _torch()
    dev = torch.device("cuda", device)
    At = torch.as_tensor(np.ascontiguousarray(A), dtype=torch.complex128, device=dev)
    ar = Arith(eps, rule)
    tab = bt.table

    def make_leaf(b):
        k, r0, r1, c0, c1 = (int(t) for t in tab[b][:5])
        blk = At[d * r0:d * r1, d * c0:d * c1]
        if k == 0:
            return Dense(d * r0, d * r1, d * c0, d * c1, blk.clone())
        u, v = _dense_to_lr(ar, blk)
        return LowRank(d * r0, d * r1, d * c0, d * c1, u.contiguous(), v.contiguous())

    return _build(bt.root, d, _leaf_index(bt), make_leaf)


def to_dense(x, ar=None):
    """Dense (tree-ordered) device matrix of a node tree."""
    return _dense(ar or Arith(0.0), x)


def formatted_addmul(target, a, b, eps_lu, rule="frobenius"):
    """target <- target + a b in the H-format of ``target`` (
    PAPER.md 3.2 "A''' <- A + A' A''", the 27 format cases); low-rank targets
    are truncated with ``eps_lu``.  Returns the updated target."""
    if (a.r0, a.r1) != (target.r0, target.r1) or (b.c0, b.c1) != (target.c0, target.c1) or \
            (a.c0, a.c1) != (b.r0, b.r1):
        raise ValueError("formatted_addmul: non-conformal ranges")
    ar = Arith(eps_lu, rule)
    _addmul(ar, target, a, b, 1.0)
    _flush_batch(ar, [target])
    return target


# --------------------------------------------------------------------------------------------
# public API: hlu / triangular_solve / solve_direct
# --------------------------------------------------------------------------------------------
@dataclass
class _Tri:
    """``LUFactors.lower`` / ``.upper``: a triangular view of the in-place factor tree."""

    root: object
    lower: bool


@dataclass
class LUFactors:
    """L_H (unit lower by block convention, leaf pivots folded
    in), U_H (upper), eps_LU.  Both views share the in-place factor tree."""

    lower: _Tri
    upper: _Tri
    eps_lu: float
    d: int
    perm: np.ndarray
    n: int
    stats: dict = field(default_factory=dict)

    @property
    def root(self):
        return self.lower.root

    def storage(self):
        """Complex entries stored by the factors (dense leaves count dm x dn)."""
        tot = 0
        for x in _walk(self.root):
            if isinstance(x, Dense):
                tot += (x.r1 - x.r0) * (x.c1 - x.c0)
            else:
                tot += x.rank * ((x.r1 - x.r0) + (x.c1 - x.c0))
        return tot


def hlu(h, eps_lu, rule="frobenius", block_tree=None):
    """Recursive H-LU of an assembled square H-matrix: steps
    (1) LU(A11), (2) U12 = L11^{-1} A12, (3) L21 = A21 U11^{-1}, (4) A22 -= L21 U12
    by ``formatted_addmul`` with truncation ``eps_lu``, recurse; dense leaves by
    pivoted LU.  Raises ``FactorizationError`` on a singular diagonal leaf."""
    torch = _torch()
    if h.block_tree is None and block_tree is None:
        raise ValueError("hlu needs the H-matrix's block tree")
    bt = block_tree if block_tree is not None else h.block_tree
    if bt.rows is not bt.cols and not np.array_equal(bt.rows.permutation, bt.cols.permutation):
        raise ValueError("hlu: row and column trees differ")
    torch.cuda.set_device(h.device)
    free, total = torch.cuda.mem_get_info(h.device)
    if free < total // 4:
        # hand the context's cached blocks to torch's allocator (dense images) only when HBM is
        # short: the cache is what the truncation calls below reuse instead of cudaMalloc / cudaFree
        _lib.release_cached(h.device)
    t0 = time.perf_counter()
    root = copy_hmatrix(h, bt)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ar = Arith(float(eps_lu), rule)
    _lu(ar, root, ())
    _flush_batch(ar, [root])
    _drop_images(root)   # the dense operand images were factorisation workspace, not factor storage
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    f = LUFactors(lower=_Tri(root, True), upper=_Tri(root, False), eps_lu=float(eps_lu), d=h.d,
                  perm=np.asarray(h.perm), n=h.d * h.n_points)
    f.stats = {"copy_s": t1 - t0, "factor_s": t2 - t1, "n_truncations": ar.n_trunc,
               "n_truncate_calls": ar.n_trunc_calls, "truncate_s": ar.t_trunc, "dense_image_GB": ar.dc_bytes / 1e9,
               "truncate_kmax_p50_p90_max": ([int(q) for q in np.percentile(ar.k_hist, [50, 90, 100])]
                                             if ar.k_hist else []),
               "n_getrf": ar.n_getrf, "max_rank": ar.max_rank}
    return f


def _to_tree(f, b):
    torch = _torch()
    d = f.d
    idx = torch.as_tensor((d * f.perm[:, None] + np.arange(d)[None, :]).reshape(-1), device=_dev_of(f.root))
    return idx


def _as_dev(f, b):
    torch = _torch()
    dev = _dev_of(f.root)
    if hasattr(b, "is_cuda"):
        bt = b.to(device=dev, dtype=torch.complex128)
        host = False
    else:
        b = np.asarray(b, dtype=np.complex128)
        bt = torch.as_tensor(b, device=dev)
        host = True
    if bt.shape[0] != f.n:
        raise ValueError("dimension mismatch")
    return bt, host


def triangular_solve(f, b):
    """x0 = U_H^{-1} L_H^{-1} b; b, x0 in original point order
    (numpy in -> numpy out; CUDA tensor in -> CUDA tensor out)."""
    bt, host = _as_dev(f, b)
    idx = _to_tree(f, b)
    vec = bt.dim() == 1
    X = bt.reshape(f.n, -1)[idx]
    ar = Arith(f.eps_lu)
    X = _usolve(ar, f.root, _lsolve(ar, f.root, X))
    out = X.new_empty(X.shape)
    out[idx] = X
    out = out.reshape(-1) if vec else out
    return out.cpu().numpy() if host else out


def lu_matvec(f, x):
    """L_H U_H x (original point order) -- the consistency product of SPEC.md:417, 443."""
    bt, host = _as_dev(f, x)
    idx = _to_tree(f, x)
    vec = bt.dim() == 1
    X = bt.reshape(f.n, -1)[idx]
    ar = Arith(f.eps_lu)
    Y = _lmul(ar, f.root, _umul(ar, f.root, X))
    out = Y.new_empty(Y.shape)
    out[idx] = Y
    out = out.reshape(-1) if vec else out
    return out.cpu().numpy() if host else out


def solve_direct(h, b, eps_lu, rule="frobenius"):
    """factorise once with ``hlu(h, eps_lu)`` and solve;
    returns (x0, LUFactors) so the factors can be reused for more right-hand sides."""
    f = hlu(h, eps_lu, rule)
    return triangular_solve(f, b), f
