"""Formatted H-arithmetic and the recursive H-LU -- the reference's
``hmatx.hmatrix`` operations ``formatted_addmul``, ``hlu``, ``triangular_solve``
and ``hmatx.solve.solve_direct`` (section 3.2,
"the LU factorization is classically decomposed into 4 steps").  The reference
module is absent from the mount; SURVEY 8(f) row 4.

This module is the host-side mirror of that interface.  The arithmetic itself --
the factor tree, the 27 format cases of ``formatted_addmul``, the recursive LU,
the block triangular solves and every truncation -- runs in ``libhmx.so``
(``csrc/hlu.cu``: C++ recursion over cuBLAS / cuSOLVER and the assembly's own
recompression kernels, one stream-ordered memory pool, one truncation batch per
elimination step).  Python only describes trees to the engine and wraps what
comes back:

* ``HTree`` owns an ``hmx_hlu`` handle: a device factor tree over the block tree
  of ``BlockTree.root`` (``geometry.py:277-295``) -- dense (dm x dn), low-rank
  (U dm x r, V dn x r, block = U V^H) and hierarchical nodes, complex128
  column-major in HBM, index ranges in dofs, tree order.
* ``HTree.from_hmatrix`` hands the engine the assembled H-matrix's leaves as
  pointers into its HBM streams (``hmx_hmatrix_device_layout``); the engine copies
  them, so the source H stays immutable.
* ``HTree.nodes()`` is a read-only Python view of the engine's tree (``Dense`` /
  ``LowRank`` / ``Sub`` with torch tensors aliasing the engine's storage): what the
  snapshot writer and the parity tests walk.

The LU is in place: ``LUFactors.lower`` / ``.upper`` are the strictly lower /
upper blocks plus the unit-lower / upper factors of the diagonal leaves of the
same tree; a factored diagonal leaf holds the packed LU of
``getrf`` and its row permutation as an index vector.
"""

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import AdmissibleLeaf, DenseLeaf

_RULES = {"frobenius": 0, "spectral": 1}
_DESC_W, _PAY_W = 8, 5
_DENSE, _LOWRANK, _SUB, _LOWRANK_FROM_DENSE = 0, 1, 2, 3

_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("hlu: a CUDA device is required (no CPU fallback)")
        _TORCH = torch
    return _TORCH


def _rule(rule):
    if rule not in _RULES:
        raise ValueError(f"unknown truncation rule {rule!r}")
    return _RULES[rule]


def _eps(eps):
    eps = float(eps)
    if not eps >= 0:
        raise ValueError("eps_lu must be >= 0")
    return eps


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _colmajor_view(ptr, m, n, ld, dev, keep):
    """(m, n) torch view of an engine matrix (complex128 column-major, leading dimension ld)."""
    torch = _torch()
    if m == 0 or n == 0 or not ptr:
        return torch.zeros((m, n), dtype=torch.complex128, device=dev)
    flat = torch.as_tensor(_CAI(ptr, ld * (n - 1) + m, "<c16"), device=dev)
    t = torch.as_strided(flat, (m, n), (1, ld))
    t._hmx_keep = keep   # the engine tree that owns the storage
    return t


def _colmajor(t):
    """Device tensor (m, n) -> (column-major copy, pointer, ld)."""
    c = t.mT.contiguous()   # (n, m) row-major = m x n column-major
    return c, c.data_ptr(), max(int(t.shape[0]), 1)


# --------------------------------------------------------------------------------------------
# read-only node views of an engine tree
# --------------------------------------------------------------------------------------------
class Dense:
    """Dense leaf.  ``a`` is the block -- or, once ``factored``, the packed LU of getrf
    (unit lower L~ below the diagonal, U on and above it) with ``pidx``: P^T X = X[pidx]."""

    __slots__ = ("r0", "r1", "c0", "c1", "a", "factored", "pidx")

    def __init__(self, r0, r1, c0, c1, a, factored=False, pidx=None):
        self.r0, self.r1, self.c0, self.c1, self.a, self.factored, self.pidx = r0, r1, c0, c1, a, factored, pidx

    @property
    def L(self):
        if not self.factored:
            return None
        torch = _torch()
        return torch.tril(self.a, -1) + torch.eye(self.a.shape[0], dtype=self.a.dtype, device=self.a.device)

    @property
    def U(self):
        return _torch().triu(self.a) if self.factored else None


class LowRank:
    __slots__ = ("r0", "r1", "c0", "c1", "u", "v")

    def __init__(self, r0, r1, c0, c1, u, v):
        self.r0, self.r1, self.c0, self.c1, self.u, self.v = r0, r1, c0, c1, u, v

    @property
    def rank(self):
        return int(self.u.shape[1])


class Sub:
    __slots__ = ("r0", "r1", "c0", "c1", "rs", "cs", "ch")

    def __init__(self, r0, r1, c0, c1, rs, cs, ch):
        self.r0, self.r1, self.c0, self.c1, self.rs, self.cs, self.ch = r0, r1, c0, c1, rs, cs, ch


def _walk(x):
    """Leaves of a node view in the engine's order (preorder, grids row-major)."""
    if isinstance(x, Sub):
        for row in x.ch:
            for c in row:
                yield from _walk(c)
    else:
        yield x


# --------------------------------------------------------------------------------------------
# tree descriptors (include/hmx.h: hmx_hlu_build)
# --------------------------------------------------------------------------------------------
def _describe_block_tree(bt, d, leaf_row):
    """Descriptor / payload arrays of the block tree ``bt`` in the engine's preorder;
    ``leaf_row(b)`` -> (kind, extra, p0, ld0, p1, ld1) for leaf ``b`` of ``bt.table``."""
    leaf_of = {(int(t[5]), int(t[6])): b for b, t in enumerate(bt.table)}
    desc, pay = [], []

    def rec(node):
        r, c = node.row, node.col
        box = (d * r.start, d * r.stop, d * c.start, d * c.stop)
        if isinstance(node, (DenseLeaf, AdmissibleLeaf)):
            kind, extra, p0, ld0, p1, ld1 = leaf_row(leaf_of[(r.index, c.index)])
            desc.append((kind,) + box + (0, 0, extra))
            pay.append((p0, ld0, p1, ld1, 0))
            return
        nr = 1 if r.is_leaf else len(r.children)
        nc = 1 if c.is_leaf else len(c.children)
        desc.append((_SUB,) + box + (nr, nc, 0))
        for k in node.children:
            rec(k)

    rec(bt.root)
    return (np.ascontiguousarray(desc, dtype=np.int64).reshape(-1, _DESC_W),
            np.ascontiguousarray(pay, dtype=np.uint64).reshape(-1, _PAY_W))


def _describe_nodes(root, keep):
    """Descriptor / payload of a Python node tree holding device tensors (snapshot load)."""
    desc, pay = [], []

    def rec(x):
        box = (x.r0, x.r1, x.c0, x.c1)
        if isinstance(x, Sub):
            desc.append((_SUB,) + box + (len(x.rs), len(x.cs), 0))
            for row in x.ch:
                for c in row:
                    rec(c)
        elif isinstance(x, Dense):
            a, p, ld = _colmajor(x.a)
            keep.append(a)
            pp = 0
            if x.factored:
                pi = x.pidx.to(dtype=_torch().int64).contiguous()
                keep.append(pi)
                pp = pi.data_ptr()
            desc.append((_DENSE,) + box + (0, 0, int(x.factored)))
            pay.append((p, ld, 0, 0, pp))
        else:
            r = x.rank
            if r:
                u, pu, ldu = _colmajor(x.u)
                v, pv, ldv = _colmajor(x.v)
                keep.extend((u, v))
            else:
                pu = pv = 0
                ldu = ldv = 1
            desc.append((_LOWRANK,) + box + (0, 0, r))
            pay.append((pu, ldu, pv, ldv, 0))

    rec(root)
    return (np.ascontiguousarray(desc, dtype=np.int64).reshape(-1, _DESC_W),
            np.ascontiguousarray(pay, dtype=np.uint64).reshape(-1, _PAY_W))


class HTree:
    """A device factor tree owned by the H-LU engine (``hmx_hlu``, include/hmx.h)."""

    def __init__(self, handle, device):
        self.handle = handle
        self.device = int(device)
        self._nodes = None

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.lib().hmx_hlu_free(h)
            except Exception:
                pass

    # ---- construction ----
    @classmethod
    def _build(cls, device, desc, pay, eps=0.0, rule="frobenius", finished=False):
        _lib.bind_torch_stream(device)
        h = C.c_void_p()
        _lib.check(_lib.lib().hmx_hlu_build(_lib.context(device), len(desc), _lib.ptr(desc), _lib.ptr(pay),
                                            _eps(eps), _rule(rule), int(finished), C.byref(h)), "hmx_hlu_build")
        return cls(h, device)

    @classmethod
    def from_hmatrix(cls, h, block_tree=None):
        """Engine copy of every leaf of the assembled H (pointers into its HBM streams)."""
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
        rbase, vbase = int(bufs[0]), int(bufs[2])
        ranks = h.block_info()["rank_after"]
        d = h.d
        tab = np.asarray(h.table)

        def leaf_row(b):
            k, c0, c1 = int(tab[b][0]), int(tab[b][3]), int(tab[b][4])
            p0 = rbase + 16 * int(moff[b])
            if k == 0:
                return _DENSE, 0, p0, int(ld[b]), 0, 0
            r = int(ranks[b])
            if r == 0:
                return _LOWRANK, 0, 0, 1, 0, 1
            return _LOWRANK, r, p0, int(ld[b]), vbase + 16 * int(voff[b]), d * (c1 - c0)

        desc, pay = _describe_block_tree(bt, d, leaf_row)
        return cls._build(h.device, desc, pay)

    @classmethod
    def from_dense(cls, bt, d, A, eps, rule="frobenius", device=0):
        """Tree of a dense (tree-ordered) matrix on the block partition ``bt``: dense leaves
        copied, admissible leaves compressed by truncated SVD with ``eps``."""
        torch = _torch()
        dev = torch.device("cuda", device)
        A = np.asarray(A, dtype=np.complex128)
        n = A.shape[0]
        At = torch.as_tensor(np.ascontiguousarray(A.T), device=dev)   # row-major A^T = column-major A
        base = At.data_ptr()
        tab = np.asarray(bt.table)

        def leaf_row(b):
            k, r0, c0 = int(tab[b][0]), int(tab[b][1]), int(tab[b][3])
            p = base + 16 * (d * c0 * n + d * r0)
            return (_DENSE if k == 0 else _LOWRANK_FROM_DENSE), 0, p, max(n, 1), 0, 0

        desc, pay = _describe_block_tree(bt, d, leaf_row)
        return cls._build(device, desc, pay, eps, rule)

    @classmethod
    def from_nodes(cls, root, device, finished=True):
        keep = []
        desc, pay = _describe_nodes(root, keep)
        t = cls._build(device, desc, pay, finished=finished)
        del keep
        return t

    # ---- inspection ----
    def structure(self):
        """(descriptor, payload) of the engine's tree (payload pointers alias its storage)."""
        nn, nl = C.c_int64(), C.c_int64()
        L = _lib.lib()
        _lib.check(L.hmx_hlu_count(self.handle, C.byref(nn), C.byref(nl)), "hmx_hlu_count")
        desc = np.zeros((nn.value, _DESC_W), np.int64)
        pay = np.zeros((max(nl.value, 1), _PAY_W), np.uint64)
        _lib.check(L.hmx_hlu_export(self.handle, _lib.ptr(desc), _lib.ptr(pay)), "hmx_hlu_export")
        return desc, pay[:nl.value]

    def nodes(self):
        """Read-only node view (rebuilt after every operation that modifies the tree)."""
        if self._nodes is None:
            torch = _torch()
            dev = torch.device("cuda", self.device)
            desc, pay = self.structure()
            it = iter(range(len(desc)))
            leaf = iter(range(len(pay)))

            def rec():
                k, r0, r1, c0, c1, nr, nc, extra = (int(t) for t in desc[next(it)])
                if k == _SUB:
                    kids = [[rec() for _ in range(nc)] for _ in range(nr)]
                    return Sub(r0, r1, c0, c1, [(row[0].r0, row[0].r1) for row in kids],
                               [(c.c0, c.c1) for c in kids[0]], kids)
                q = [int(t) for t in pay[next(leaf)]]
                dm, dn = r1 - r0, c1 - c0
                if k == _DENSE:
                    a = _colmajor_view(q[0], dm, dn, q[1], dev, self)
                    pidx = None
                    if extra:
                        pidx = torch.as_tensor(_CAI(q[4], dm, "<i8"), device=dev)
                        pidx._hmx_keep = self
                    return Dense(r0, r1, c0, c1, a, bool(extra), pidx)
                return LowRank(r0, r1, c0, c1, _colmajor_view(q[0], dm, extra, q[1], dev, self),
                               _colmajor_view(q[2], dn, extra, q[3], dev, self))

            self._nodes = rec()
        return self._nodes

    @property
    def shape(self):
        root = self.structure()[0][0]
        return int(root[2] - root[1]), int(root[4] - root[3])

    def to_dense(self):
        """Dense (tree-ordered) device matrix."""
        torch = _torch()
        m, n = self.shape
        out = torch.empty((n, max(m, 1)), dtype=torch.complex128, device=torch.device("cuda", self.device))
        _lib.bind_torch_stream(self.device)
        _lib.check(_lib.lib().hmx_hlu_to_dense(self.handle, C.c_void_p(out.data_ptr()), max(m, 1)), "hmx_hlu_to_dense")
        return out[:, :m].mT

    # ---- arithmetic ----
    def factor(self, eps_lu, rule="frobenius"):
        """In-place recursive H-LU; returns the engine's counters."""
        st = _lib.HmxHluStats()
        self._nodes = None
        _lib.bind_torch_stream(self.device)
        _lib.check(_lib.lib().hmx_hlu_factor(self.handle, _eps(eps_lu), _rule(rule), C.byref(st)), "hmx_hlu_factor")
        return st.as_dict()

    def apply(self, X, mode):
        """mode 0: U_H^{-1} L_H^{-1} X; mode 1: L_H U_H X.  X: device (n, nrhs) tensor, tree order."""
        torch = _torch()
        n, nrhs = X.shape
        xc = X.mT.contiguous()
        yc = torch.empty_like(xc)
        _lib.bind_torch_stream(self.device)
        _lib.check(_lib.lib().hmx_hlu_apply(self.handle, int(mode), C.c_void_p(xc.data_ptr()),
                                            C.c_void_p(yc.data_ptr()), n, nrhs), "hmx_hlu_apply")
        return yc.mT


def from_dense(bt, d, A, eps, rule="frobenius", device=0):
    """``HTree`` of a dense (tree-ordered) matrix (test / formatted_addmul operands)."""
    return HTree.from_dense(bt, d, A, eps, rule, device)


def to_dense(x):
    """Dense (tree-ordered) device matrix of an ``HTree``."""
    return x.to_dense()


def formatted_addmul(target, a, b, eps_lu, rule="frobenius", alpha=1.0):
    """target <- target + alpha a b in the H-format of ``target`` (
    PAPER.md 3.2 "A''' <- A + A' A''", the 27 format cases); low-rank targets
    are truncated with ``eps_lu``.  Returns the updated target."""
    target._nodes = None
    _lib.bind_torch_stream(target.device)
    _lib.check(_lib.lib().hmx_hlu_addmul(target.handle, a.handle, b.handle, float(alpha), _eps(eps_lu), _rule(rule)),
               "formatted_addmul")
    return target


def truncate_pairs(items, eps, rule="frobenius"):
    """The engine's truncation (recompress rule) of factor pairs: list of
    device (U dm x K, V dn x K) -> list of truncated (U', V') with U' V'^H ~ U V^H."""
    torch = _torch()
    if not items:
        return []
    dev = items[0][0].device
    device = dev.index or 0
    n = len(items)
    dm = np.array([u.shape[0] for u, _ in items], np.int64)
    dn = np.array([v.shape[0] for _, v in items], np.int64)
    K = np.array([u.shape[1] for u, _ in items], np.int64)
    ptrs = np.zeros((4, n), np.uint64)
    keep, outs = [], []
    for i, (u, v) in enumerate(items):
        uc, vc = u.mT.contiguous(), v.mT.contiguous()
        uo, vo = torch.empty_like(uc), torch.empty_like(vc)
        keep += [uc, vc]
        outs.append((uo, vo))
        ptrs[:, i] = (uc.data_ptr(), vc.data_ptr(), uo.data_ptr(), vo.data_ptr())
    ranks = np.zeros(n, np.int64)
    _lib.bind_torch_stream(device)
    _lib.check(_lib.lib().hmx_hlu_truncate(_lib.context(device), n, _lib.ptr(dm), _lib.ptr(dn), _lib.ptr(K),
                                           _lib.ptr(ptrs[0]), _lib.ptr(ptrs[1]), _lib.ptr(ptrs[2]), _lib.ptr(ptrs[3]),
                                           _eps(eps), _rule(rule), _lib.ptr(ranks)), "hmx_hlu_truncate")
    return [(uo[:int(r)].mT, vo[:int(r)].mT) for (uo, vo), r in zip(outs, ranks)]


# --------------------------------------------------------------------------------------------
# public API: hlu / triangular_solve / solve_direct
# --------------------------------------------------------------------------------------------
@dataclass
class _Tri:
    """``LUFactors.lower`` / ``.upper``: a triangular view of the in-place factor tree."""

    tree: HTree
    lower: bool

    @property
    def root(self):
        return self.tree.nodes()


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
    def tree(self):
        return self.lower.tree

    @property
    def root(self):
        return self.tree.nodes()

    def storage(self):
        """Complex entries stored by the factors (dense leaves count dm x dn)."""
        desc, _ = self.tree.structure()
        dm, dn = desc[:, 2] - desc[:, 1], desc[:, 4] - desc[:, 3]
        dense, lr = desc[:, 0] == _DENSE, desc[:, 0] == _LOWRANK
        return int((dm * dn)[dense].sum() + (desc[:, 7] * (dm + dn))[lr].sum())


def _factors(tree, eps_lu, d, perm, n, stats=None):
    return LUFactors(lower=_Tri(tree, True), upper=_Tri(tree, False), eps_lu=float(eps_lu), d=int(d),
                     perm=np.asarray(perm), n=int(n), stats=stats or {})


def hlu(h, eps_lu, rule="frobenius", block_tree=None):
    """Recursive H-LU of an assembled square H-matrix: steps
    (1) LU(A11), (2) U12 = L11^{-1} A12, (3) L21 = A21 U11^{-1}, (4) A22 -= L21 U12
    by ``formatted_addmul`` with truncation ``eps_lu``, recurse; dense leaves by
    pivoted LU.  Raises ``FactorizationError`` on a singular diagonal leaf."""
    _torch()
    eps_lu, _ = _eps(eps_lu), _rule(rule)
    bt = block_tree if block_tree is not None else h.block_tree
    if bt is None:
        raise ValueError("hlu needs the H-matrix's block tree")
    if bt.rows is not bt.cols and not np.array_equal(bt.rows.permutation, bt.cols.permutation):
        raise ValueError("hlu: row and column trees differ")
    t0 = time.perf_counter()
    tree = HTree.from_hmatrix(h, bt)
    t1 = time.perf_counter()
    st = tree.factor(eps_lu, rule)
    t2 = time.perf_counter()
    stats = {"copy_s": t1 - t0, "factor_s": t2 - t1, "n_truncations": st["n_truncations"],
             "n_truncate_calls": st["n_truncate_calls"], "truncate_s": st["t_truncate_s"],
             "dense_image_GB": st["dense_image_bytes"] / 1e9,
             "truncate_kmax_p50_p90_max": [st["k_p50"], st["k_p90"], st["k_max"]] if st["n_truncate_calls"] else [],
             "n_getrf": st["n_getrf"], "max_rank": st["max_rank"], "engine_factor_s": st["t_factor_s"]}
    return _factors(tree, eps_lu, h.d, h.perm, h.d * h.n_points, stats)


def _io(f, b):
    torch = _torch()
    dev = torch.device("cuda", f.tree.device)
    host = not hasattr(b, "is_cuda")
    bt = torch.as_tensor(np.asarray(b, dtype=np.complex128), device=dev) if host else \
        b.to(device=dev, dtype=torch.complex128)
    if bt.shape[0] != f.n:
        raise ValueError("dimension mismatch")
    d = f.d
    idx = torch.as_tensor((d * f.perm[:, None] + np.arange(d)[None, :]).reshape(-1), device=dev)
    return bt, host, idx


def _apply(f, b, mode):
    bt, host, idx = _io(f, b)
    vec = bt.dim() == 1
    Y = f.tree.apply(bt.reshape(f.n, -1)[idx], mode)
    out = Y.new_empty(Y.shape)
    out[idx] = Y
    out = out.reshape(-1) if vec else out
    return out.cpu().numpy() if host else out


def triangular_solve(f, b):
    """x0 = U_H^{-1} L_H^{-1} b; b, x0 in original point order
    (numpy in -> numpy out; CUDA tensor in -> CUDA tensor out)."""
    return _apply(f, b, 0)


def lu_matvec(f, x):
    """L_H U_H x (original point order) -- the consistency product of SPEC.md:417, 443."""
    return _apply(f, x, 1)


def solve_direct(h, b, eps_lu, rule="frobenius"):
    """factorise once with ``hlu(h, eps_lu)`` and solve;
    returns (x0, LUFactors) so the factors can be reused for more right-hand sides."""
    f = hlu(h, eps_lu, rule)
    return triangular_solve(f, b), f
