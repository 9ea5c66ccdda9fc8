"""Oracle: restarted GMRES (CPU).  TEST INFRASTRUCTURE.

Restates ``solve_gmres`` (reference ``solve.py`` is
absent from the mount) with the decisions of SURVEY 8(c) item 10 pinned, and
mirrored by the device GMRES in ``csrc/gmres.cu``:

* x0 = 0; b = 0 -> (0, 0 iterations, []);
* Arnoldi with modified Gram-Schmidt, complex Givens rotations
  G = [[c, s], [-conj(s), c]], c real;
* after every inner step the Arnoldi residual estimate |g_{j+1}| / ||b|| is
  appended to ``history``; stop when it is <= tol;
* ``iters`` = total inner steps (= H-matvecs, not counting the explicit
  residual b - A x recomputed at each restart);
* ``max_iters`` reached -> returned with ``converged = False``.
"""

import numpy as np


def givens(a, b):
    """(c, s, r) with [[c, s], [-conj(s), c]] @ [a, b] = [r, 0]."""
    if b == 0:
        return 1.0, 0.0j, a
    if a == 0:
        return 0.0, np.conj(b) / abs(b), complex(abs(b))
    t = np.hypot(abs(a), abs(b))
    ph = a / abs(a)
    return abs(a) / t, ph * np.conj(b) / t, ph * t


def gmres(apply, b, tol=1e-4, restart=50, max_iters=1000):
    """Returns (x, iters, history, converged)."""
    b = np.asarray(b, dtype=complex)
    x = np.zeros_like(b)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, [], True
    history = []
    iters = 0
    r = b.copy()
    beta = bnorm
    while True:
        m = restart
        Vb = [r / beta]
        H = np.zeros((m + 1, m), complex)
        cs = np.zeros(m)
        sn = np.zeros(m, complex)
        g = np.zeros(m + 1, complex)
        g[0] = beta
        k = 0
        done = False
        for j in range(m):
            w = apply(Vb[j])
            iters += 1
            for i in range(j + 1):
                h = np.vdot(Vb[i], w)
                H[i, j] = h
                w = w - h * Vb[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            for i in range(j):
                t0 = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t0
            c, s, rr = givens(H[j, j], H[j + 1, j])
            cs[j], sn[j] = c, s
            H[j, j] = rr
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            res = abs(g[j + 1])
            history.append(res / bnorm)
            k = j + 1
            if res <= tol * bnorm:
                done = True
                break
            if iters >= max_iters or hn == 0.0:
                break
            Vb.append(w / hn)
        y = np.zeros(k, complex)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1 : k] @ y[i + 1 : k]) / H[i, i]
        for i in range(k):
            x = x + y[i] * Vb[i]
        if done:
            return x, iters, history, True
        if iters >= max_iters:
            return x, iters, history, False
        r = b - apply(x)
        beta = float(np.linalg.norm(r))
        if beta <= tol * bnorm:
            return x, iters, history, True
