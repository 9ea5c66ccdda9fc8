"""Oracle: formatted H-arithmetic, recursive H-LU, triangular solves (CPU, numpy/scipy).
TEST INFRASTRUCTURE -- only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
leg may import this module.

Restates SPEC.md:401-429 and 487-495 (``formatted_addmul``, ``hlu``,
``triangular_solve``, ``solve_direct``; section 3.2 "the LU factorization is
classically decomposed into 4 steps ... results into 27 cases").  The reference
``hmatx/hmatrix.py`` / ``hmatx/solve.py`` are absent from the mount, so there is no
reference output to pin against: **parity unpinned** beyond SPEC's own examples
(all-dense addmul exact, rank bound of a low-rank sum, 10 eps_LU consistency of
L_H U_H against A_H, 1-leaf dense LU at machine precision, b = L U y recovers y,
identity solve, cross-solver agreement with GMRES).

Decisions (shared with the device implementation ``paper_1706_09384_b200/hierarchical_lu.py``):
1. block structure = ``BlockTree.root`` (``geometry.py:277-295``), leaves in tree order,
   dof ranges d * point ranges;
2. dense diagonal leaves: partial-pivoting LU (LAPACK getrf), L = P L~;
3. a low-rank operand multiplies through its thin factors; hierarchical x hierarchical
   recurses over the cluster children; leaves meeting a finer partition are sliced;
4. low-rank targets collect addends and truncate once when next read: QR(U), QR(V),
   SVD(R_U R_V^H), Frobenius-tail rule of ``lowrank.truncation_rank`` (decision 8 of
   oracle/lowrank.py) with eps_LU;
5. a product with no low-rank operand landing on a low-rank target is formed per child
   block (a dense leaf pair A B as the untruncated pair (A, B^H)) and agglomerated by
   concatenating padded factors, truncated only above AGGLO_MAX columns;
6. a singular dense diagonal leaf (|u_ii| <= 1e-14 max |u_jj|) raises with its block path;
7. truncation points: a target holding more than PEND_FLUSH columns; every low-rank leaf
   of the trailing blocks after each elimination step of the LU and of the block
   triangular solves (the device batches each such set into one kernel call); a block
   read as an operand; the end of hlu / formatted_addmul;
8. a product (no low-rank operand) landing on a hierarchical target of at most DENSE_T rows and
   columns is formed exactly as one dense product and scattered into the target's leaves: dense
   leaves add it, low-rank leaves accumulate it densely and are truncated at their next truncation
   point as the pair (X, I), X = U V^H + pending addends + the dense addend.
"""

import numpy as np
import scipy.linalg as sla

from .lowrank import truncation_rank

DENSE, LOWRANK, SUB = 0, 1, 2
PEND_FLUSH = 400     # decision 7: pending columns on one target before an early truncation
AGGLO_MAX = 512      # decision 5: agglomerated product columns before an intermediate truncation
DENSE_T = 512        # decision 8: hierarchical targets up to this many rows / columns take products densely


class Node:
    __slots__ = ("kind", "r0", "r1", "c0", "c1", "a", "u", "v", "pend", "acc", "rs", "cs", "ch",
                 "lu", "piv")

    def __init__(self, kind, r0, r1, c0, c1):
        self.kind, self.r0, self.r1, self.c0, self.c1 = kind, r0, r1, c0, c1
        self.a = self.u = self.v = self.rs = self.cs = self.ch = self.lu = self.piv = None
        self.pend = []
        self.acc = None


class Ctx:
    def __init__(self, eps, rule="frobenius"):
        self.eps, self.rule = eps, rule
        self.n_trunc = 0


def _trunc(cx, u, v):
    if u.shape[1] == 0:
        return u, v
    cx.n_trunc += 1
    qu, ru = np.linalg.qr(u)
    qv, rv = np.linalg.qr(v)
    p, s, lh = np.linalg.svd(ru @ rv.conj().T, full_matrices=False)
    r = truncation_rank(s, cx.eps, cx.rule)
    root = np.sqrt(s[:r])
    return (qu @ p[:, :r]) * root, (qv @ lh.conj().T[:, :r]) * root


def _compress(cx, m):
    cx.n_trunc += 1
    p, s, lh = np.linalg.svd(m, full_matrices=False)
    r = truncation_rank(s, cx.eps, cx.rule)
    root = np.sqrt(s[:r])
    return p[:, :r] * root, lh.conj().T[:, :r] * root


def _flush(cx, x):
    if x.acc is not None:
        X = x.acc
        for u, v in [(x.u, x.v)] + x.pend:
            X = X + u @ v.conj().T
        x.acc, x.pend = None, []
        x.u, x.v = _trunc(cx, X, np.eye(X.shape[1], dtype=np.complex128))
    elif x.pend:
        u = np.concatenate([x.u] + [p[0] for p in x.pend], axis=1)
        v = np.concatenate([x.v] + [p[1] for p in x.pend], axis=1)
        x.pend = []
        x.u, x.v = _trunc(cx, u, v)


def flush_all(cx, x):
    if x.kind == LOWRANK:
        _flush(cx, x)
    elif x.kind == SUB:
        for row in x.ch:
            for c in row:
                flush_all(cx, c)


def leaves(x):
    if x.kind == SUB:
        for row in x.ch:
            for c in row:
                yield from leaves(c)
    else:
        yield x


# ---- construction -----------------------------------------------------------------------
def build(bt, d, make_leaf):
    """Node tree over ``bt.root``; ``make_leaf(b)`` returns the leaf node of table row b."""
    leaf_of = {(int(t[5]), int(t[6])): b for b, t in enumerate(bt.table)}

    def rec(node):
        if not hasattr(node, "children"):
            return make_leaf(leaf_of[(node.row.index, node.col.index)])
        r, c = node.row, node.col
        rk = (r,) if r.is_leaf else r.children
        ck = (c,) if c.is_leaf else c.children
        kids = [rec(k) for k in node.children]
        x = Node(SUB, d * r.start, d * r.stop, d * c.start, d * c.stop)
        x.rs = [(d * q.start, d * q.stop) for q in rk]
        x.cs = [(d * q.start, d * q.stop) for q in ck]
        x.ch = [kids[i * len(ck):(i + 1) * len(ck)] for i in range(len(rk))]
        return x

    return rec(bt.root)


def from_payload(bt, d, payload):
    """Node tree of an oracle H (``oracle.hmatrix.OracleH.payload`` in table order); copies."""
    def mk(b):
        k, r0, r1, c0, c1 = (int(t) for t in bt.table[b][:5])
        x = Node(DENSE if k == 0 else LOWRANK, d * r0, d * r1, d * c0, d * c1)
        if k == 0:
            x.a = np.array(payload[b], dtype=np.complex128)
        else:
            x.u = np.array(payload[b][0], dtype=np.complex128)
            x.v = np.array(payload[b][1], dtype=np.complex128)
        return x
    return build(bt, d, mk)


def from_dense(bt, d, A, eps, rule="frobenius"):
    cx = Ctx(eps, rule)

    def mk(b):
        k, r0, r1, c0, c1 = (int(t) for t in bt.table[b][:5])
        x = Node(DENSE if k == 0 else LOWRANK, d * r0, d * r1, d * c0, d * c1)
        blk = A[d * r0:d * r1, d * c0:d * c1]
        if k == 0:
            x.a = np.array(blk)
        else:
            x.u, x.v = _compress(cx, blk)
        return x
    return build(bt, d, mk)


# ---- products with dense multivectors -----------------------------------------------------
def mul(cx, x, X):
    if x.kind == DENSE:
        return x.a @ X
    if x.kind == LOWRANK:
        _flush(cx, x)
        return x.u @ (x.v.conj().T @ X)
    out = np.zeros((x.r1 - x.r0, X.shape[1]), np.complex128)
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            out[a - x.r0:b - x.r0] += mul(cx, x.ch[i][j], X[c - x.c0:e - x.c0])
    return out


def mulh(cx, x, X):
    if x.kind == DENSE:
        return x.a.conj().T @ X
    if x.kind == LOWRANK:
        _flush(cx, x)
        return x.v @ (x.u.conj().T @ X)
    out = np.zeros((x.c1 - x.c0, X.shape[1]), np.complex128)
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            out[c - x.c0:e - x.c0] += mulh(cx, x.ch[i][j], X[a - x.r0:b - x.r0])
    return out


def dense(cx, x):
    if x.kind == DENSE:
        return x.a
    if x.kind == LOWRANK:
        _flush(cx, x)
        return x.u @ x.v.conj().T
    out = np.zeros((x.r1 - x.r0, x.c1 - x.c0), np.complex128)
    for i, (a, b) in enumerate(x.rs):
        for j, (c, e) in enumerate(x.cs):
            out[a - x.r0:b - x.r0, c - x.c0:e - x.c0] = dense(cx, x.ch[i][j])
    return out


def _part(cx, x, i, k, r0, r1, c0, c1):
    if x.kind == SUB:
        ch = x.ch[i][k]
        assert (ch.r0, ch.r1, ch.c0, ch.c1) == (r0, r1, c0, c1), "non-conformal partitions"
        return ch
    if (x.r0, x.r1, x.c0, x.c1) == (r0, r1, c0, c1):
        return x
    y = Node(x.kind, r0, r1, c0, c1)
    if x.kind == DENSE:
        y.a = x.a[r0 - x.r0:r1 - x.r0, c0 - x.c0:c1 - x.c0]
    else:
        _flush(cx, x)
        y.u, y.v = x.u[r0 - x.r0:r1 - x.r0], x.v[c0 - x.c0:c1 - x.c0]
    return y


# ---- formatted add / multiply -------------------------------------------------------------
def _pend(cx, C, U, V):
    C.pend.append((U, V))
    if C.u.shape[1] + sum(p[0].shape[1] for p in C.pend) > PEND_FLUSH:
        _flush(cx, C)


def _add_lr(cx, C, U, V):
    if U.shape[1] == 0:
        return
    if C.kind == DENSE:
        C.a += U @ V.conj().T
    elif C.kind == LOWRANK:
        _pend(cx, C, U, V)
    else:
        for i, (a, b) in enumerate(C.rs):
            for j, (c, e) in enumerate(C.cs):
                _add_lr(cx, C.ch[i][j], U[a - C.r0:b - C.r0], V[c - C.c0:e - C.c0])


def _add_dense(cx, C, M):
    if C.kind == DENSE:
        C.a += M
    elif C.kind == LOWRANK:
        C.acc = M.copy() if C.acc is None else C.acc + M
    else:
        for i, (a, b) in enumerate(C.rs):
            for j, (c, e) in enumerate(C.cs):
                _add_dense(cx, C.ch[i][j], M[a - C.r0:b - C.r0, c - C.c0:e - C.c0])


def _prod_lr(cx, A, B):
    if A.kind == LOWRANK:
        _flush(cx, A)
        return A.u, mulh(cx, B, A.v)
    if B.kind == LOWRANK:
        _flush(cx, B)
        return mul(cx, A, B.u), B.v
    if A.kind == DENSE and B.kind == DENSE:
        return A.a, B.a.conj().T
    m, n = A.r1 - A.r0, B.c1 - B.c0
    Rp = A.rs if A.kind == SUB else [(A.r0, A.r1)]
    Cp = B.cs if B.kind == SUB else [(B.c0, B.c1)]
    Kp = A.cs if A.kind == SUB else B.rs
    us, vs = [], []
    for i, (ra, rb) in enumerate(Rp):
        for j, (ca, cb) in enumerate(Cp):
            for k, (ka, kb) in enumerate(Kp):
                u, v = _prod_lr(cx, _part(cx, A, i, k, ra, rb, ka, kb), _part(cx, B, k, j, ka, kb, ca, cb))
                if u.shape[1] == 0:
                    continue
                up = np.zeros((m, u.shape[1]), np.complex128)
                vp = np.zeros((n, v.shape[1]), np.complex128)
                up[ra - A.r0:rb - A.r0] = u
                vp[ca - B.c0:cb - B.c0] = v
                us.append(up)
                vs.append(vp)
    if not us:
        return np.zeros((m, 0), np.complex128), np.zeros((n, 0), np.complex128)
    U, V = np.concatenate(us, 1), np.concatenate(vs, 1)
    return _trunc(cx, U, V) if U.shape[1] > AGGLO_MAX else (U, V)


def addmul(cx, C, A, B, alpha=-1.0):
    """C <- C + alpha A B."""
    if A.kind == LOWRANK and B.kind == LOWRANK:
        # rank min(r_A, r_B) through the r_A x r_B core A.v^H B.u
        _flush(cx, A)
        _flush(cx, B)
        core = A.v.conj().T @ B.u
        if A.u.shape[1] <= B.u.shape[1]:
            _add_lr(cx, C, alpha * A.u, B.v @ core.conj().T)
        else:
            _add_lr(cx, C, alpha * (A.u @ core), B.v)
        return
    if A.kind == LOWRANK:
        _flush(cx, A)
        if A.u.shape[1]:
            _add_lr(cx, C, alpha * A.u, mulh(cx, B, A.v))
        return
    if B.kind == LOWRANK:
        _flush(cx, B)
        if B.u.shape[1]:
            _add_lr(cx, C, alpha * mul(cx, A, B.u), B.v)
        return
    if C.kind == SUB:
        if C.r1 - C.r0 <= DENSE_T and C.c1 - C.c0 <= DENSE_T:
            _add_dense(cx, C, alpha * (dense(cx, A) @ dense(cx, B)))
            return
        Kp = A.cs if A.kind == SUB else (B.rs if B.kind == SUB else [(A.c0, A.c1)])
        for i, (ra, rb) in enumerate(C.rs):
            for j, (ca, cb) in enumerate(C.cs):
                for k, (ka, kb) in enumerate(Kp):
                    addmul(cx, C.ch[i][j], _part(cx, A, i, k, ra, rb, ka, kb),
                           _part(cx, B, k, j, ka, kb, ca, cb), alpha)
        return
    if C.kind == DENSE:
        C.a += alpha * mul(cx, A, dense(cx, B))
        return
    u, v = _prod_lr(cx, A, B)
    if u.shape[1]:
        _pend(cx, C, alpha * u, v)


def formatted_addmul(target, a, b, eps_lu, rule="frobenius"):
    cx = Ctx(eps_lu, rule)
    addmul(cx, target, a, b, 1.0)
    flush_all(cx, target)
    return target


# ---- LU and solves --------------------------------------------------------
def lu(cx, x, path=()):
    if x.kind == DENSE:
        lu_, piv = sla.lu_factor(x.a, check_finite=False)
        dg = np.abs(np.diag(lu_))
        if dg.size == 0 or dg.min() <= 1e-14 * max(dg.max(), 1e-300):
            raise ArithmeticError(f"singular dense diagonal leaf at block path {path}")
        x.lu, x.piv, x.a = lu_, piv, None
        return
    assert x.kind == SUB and x.rs == x.cs
    p = len(x.rs)
    for k in range(p):
        lu(cx, x.ch[k][k], path + (k,))
        for j in range(k + 1, p):
            solve_lower(cx, x.ch[k][k], x.ch[k][j])
        for i in range(k + 1, p):
            solve_upper_right(cx, x.ch[k][k], x.ch[i][k])
        for i in range(k + 1, p):
            for j in range(k + 1, p):
                addmul(cx, x.ch[i][j], x.ch[i][k], x.ch[k][j], -1.0)
        for i in range(k + 1, p):
            for j in range(k + 1, p):
                flush_all(cx, x.ch[i][j])


def _perm_T(x, X):
    """P^T X for the leaf's getrf pivots (row interchanges in order)."""
    X = X.copy()
    for i, p in enumerate(x.piv):
        if p != i:
            X[[i, p]] = X[[p, i]]
    return X


def _perm(x, X):
    X = X.copy()
    for i in range(len(x.piv) - 1, -1, -1):
        p = x.piv[i]
        if p != i:
            X[[i, p]] = X[[p, i]]
    return X


def lsolve(cx, L, X):
    if L.kind == DENSE:
        return sla.solve_triangular(L.lu, _perm_T(L, X), lower=True, unit_diagonal=True)
    X = X.copy()
    for k, (a, b) in enumerate(L.rs):
        xk = lsolve(cx, L.ch[k][k], X[a - L.r0:b - L.r0])
        X[a - L.r0:b - L.r0] = xk
        for i in range(k + 1, len(L.rs)):
            c, e = L.rs[i]
            X[c - L.r0:e - L.r0] -= mul(cx, L.ch[i][k], xk)
    return X


def usolve(cx, U, X):
    if U.kind == DENSE:
        return sla.solve_triangular(U.lu, X, lower=False)
    X = X.copy()
    for k in range(len(U.rs) - 1, -1, -1):
        a, b = U.rs[k]
        xk = usolve(cx, U.ch[k][k], X[a - U.r0:b - U.r0])
        X[a - U.r0:b - U.r0] = xk
        for i in range(k):
            c, e = U.rs[i]
            X[c - U.r0:e - U.r0] -= mul(cx, U.ch[i][k], xk)
    return X


def rsolve(cx, U, Y):
    """Y U^{-1} = (U^{-H} Y^H)^H."""
    if U.kind == DENSE:
        return sla.solve_triangular(U.lu, Y.conj().T, lower=False, trans="C").conj().T
    Y = Y.copy()
    for k, (a, b) in enumerate(U.cs):
        yk = rsolve(cx, U.ch[k][k], Y[:, a - U.c0:b - U.c0])
        Y[:, a - U.c0:b - U.c0] = yk
        for j in range(k + 1, len(U.cs)):
            c, e = U.cs[j]
            Y[:, c - U.c0:e - U.c0] -= mulh(cx, U.ch[k][j], yk.conj().T).conj().T
    return Y


def solve_lower(cx, L, B):
    if B.kind == DENSE:
        B.a = lsolve(cx, L, B.a)
    elif B.kind == LOWRANK:
        _flush(cx, B)
        if B.u.shape[1]:
            B.u = lsolve(cx, L, B.u)
    elif L.kind == SUB:
        p, q = len(L.rs), len(B.cs)
        for k in range(p):
            for j in range(q):
                solve_lower(cx, L.ch[k][k], B.ch[k][j])
            for j in range(q):
                for i in range(k + 1, p):
                    addmul(cx, B.ch[i][j], L.ch[i][k], B.ch[k][j], -1.0)
            for i in range(k + 1, p):
                for j in range(q):
                    flush_all(cx, B.ch[i][j])
    else:
        for j in range(len(B.cs)):
            solve_lower(cx, L, B.ch[0][j])


def solve_upper_right(cx, U, B):
    if B.kind == DENSE:
        B.a = rsolve(cx, U, B.a)
    elif B.kind == LOWRANK:
        _flush(cx, B)
        if B.u.shape[1]:
            B.v = rsolve(cx, U, B.v.conj().T).conj().T
    elif U.kind == SUB:
        p, q = len(U.cs), len(B.rs)
        for k in range(p):
            for i in range(q):
                solve_upper_right(cx, U.ch[k][k], B.ch[i][k])
            for i in range(q):
                for j in range(k + 1, p):
                    addmul(cx, B.ch[i][j], B.ch[i][k], U.ch[k][j], -1.0)
            for i in range(q):
                for j in range(k + 1, p):
                    flush_all(cx, B.ch[i][j])
    else:
        for i in range(len(B.rs)):
            solve_upper_right(cx, U, B.ch[i][0])


def lmul(cx, L, X):
    if L.kind == DENSE:
        Lm = np.tril(L.lu, -1) + np.eye(L.lu.shape[0])
        return _perm(L, Lm @ X)
    out = np.zeros_like(X)
    for i, (a, b) in enumerate(L.rs):
        acc = lmul(cx, L.ch[i][i], X[a - L.r0:b - L.r0])
        for j in range(i):
            c, e = L.rs[j]
            acc = acc + mul(cx, L.ch[i][j], X[c - L.r0:e - L.r0])
        out[a - L.r0:b - L.r0] = acc
    return out


def umul(cx, U, X):
    if U.kind == DENSE:
        return np.triu(U.lu) @ X
    out = np.zeros_like(X)
    for i, (a, b) in enumerate(U.rs):
        acc = umul(cx, U.ch[i][i], X[a - U.r0:b - U.r0])
        for j in range(i + 1, len(U.rs)):
            c, e = U.rs[j]
            acc = acc + mul(cx, U.ch[i][j], X[c - U.r0:e - U.r0])
        out[a - U.r0:b - U.r0] = acc
    return out


def hlu(root, eps_lu, rule="frobenius"):
    """In-place H-LU of a node tree; returns the context (truncation count)."""
    cx = Ctx(eps_lu, rule)
    lu(cx, root)
    flush_all(cx, root)
    return cx


def solve_tree(root, b_tree):
    cx = Ctx(0.0)
    X = b_tree.reshape(b_tree.shape[0], -1)
    return usolve(cx, root, lsolve(cx, root, X)).reshape(b_tree.shape)


def lu_apply_tree(root, x_tree):
    cx = Ctx(0.0)
    X = x_tree.reshape(x_tree.shape[0], -1)
    return lmul(cx, root, umul(cx, root, X)).reshape(x_tree.shape)


def tree_index(perm, d):
    """Tree-order dof -> original dof (x_tree = x[idx])."""
    return (d * np.asarray(perm)[:, None] + np.arange(d)[None, :]).reshape(-1)
