"""Oracle: Green's-tensor entry evaluation (CPU, numpy).  TEST INFRASTRUCTURE.

Restates the reference kernel core ``/root/reference/pkg/src/hmatx/
_kernelcore_np.py`` (the numpy backend of the reference's kernel-core seam):

* ``pair_geometry``   -- ``_kernelcore_np.py:17-20`` (differences and r)
* ``radial_series``   -- ``_kernelcore_np.py:23-34`` (d^q/dr^q e^{ikr}/(4 pi r))
* ``navier_coeffs``   -- ``_kernelcore_np.py:52-71`` (A, B, A', B')
* ``scalar_block``    -- ``_kernelcore_np.py:37-49``
* ``elasto_u_block``  -- ``_kernelcore_np.py:89-102``
* ``elasto_t_block``  -- ``_kernelcore_np.py:105-130``
* ``point_major``     -- ``_kernelcore_np.py:74-77`` ((m,n,3,3) -> (3m,3n))

Every arithmetic step uses the same numpy operation (and therefore the same
rounding) as the reference, so the results are bit-identical to it on the same
host; ``tests/test_oracle_pins.py`` asserts exactly that against the live
reference module (when ``/root/reference`` is mounted) and against
``tests/golden/kernels.npz``.

Return convention (reference seam): a new C-contiguous complex128
array, or ``None`` when an exact r == 0 pair exists and ``self_shift`` is None.
"""

import numpy as np

_4PI = 4.0 * np.pi


def pair_geometry(X, Y):
    """Differences Z[i,j] = X[i]-Y[j] and distances r (``_kernelcore_np.py:17-20``)."""
    diff = X[:, None, :] - Y[None, :, :]
    dist = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
    return diff, dist


def radial_series(kappa, r, nder):
    """[g, g', ..., g^(nder)] of g(r) = e^{i kappa r}/(4 pi r) (``_kernelcore_np.py:23-34``)."""
    g0 = np.exp(1j * kappa * r) / (_4PI * r)
    ik = 1j * kappa
    series = [g0]
    if nder > 0:
        series.append(g0 * (ik - 1.0 / r))
    if nder > 1:
        series.append(g0 * (-(kappa**2) - 2.0 * ik / r + 2.0 / r**2))
    if nder > 2:
        series.append(
            g0 * (-ik * kappa**2 + 3.0 * kappa**2 / r + 6.0 * ik / r**2 - 6.0 / r**3)
        )
    return series


def navier_coeffs(kp, ks, scale, r, with_derivs):
    """A, B (and A', B') of U = A I + B zz^T (``_kernelcore_np.py:52-71``).

    f = G_ks - G_kp; A = s (ks^2 G_ks + f'/r); B = s (f'' - f'/r);
    A' = s (ks^2 G_ks' + (f'' r - f')/r^2); B' = s (f''' - (f'' r - f')/r^2).
    """
    nder = 3 if with_derivs else 2
    s_ser = radial_series(ks, r, nder)
    p_ser = radial_series(kp, r, nder)
    f1 = s_ser[1] - p_ser[1]
    f2 = s_ser[2] - p_ser[2]
    A = scale * (ks**2 * s_ser[0] + f1 / r)
    B = scale * (f2 - f1 / r)
    if not with_derivs:
        return A, B
    f3 = s_ser[3] - p_ser[3]
    Ap = scale * (ks**2 * s_ser[1] + (f2 * r - f1) / r**2)
    Bp = scale * (f3 - (f2 * r - f1) / r**2)
    return A, B, Ap, Bp


def point_major(tensor):
    """(m, n, 3, 3) per-pair tensors -> (3m, 3n), row 3i+a, col 3j+b (``_kernelcore_np.py:74-77``)."""
    m, n = tensor.shape[:2]
    return np.ascontiguousarray(tensor.transpose(0, 2, 1, 3).reshape(3 * m, 3 * n))


def _self_rule(tensor, coincident, self_shift):
    """Coincident pairs -> self_shift * I_3; None when no rule (``_kernelcore_np.py:80-86``)."""
    if not coincident.any():
        return tensor
    if self_shift is None:
        return None
    tensor[coincident] = self_shift * np.eye(3)
    return tensor


def scalar_block(kappa, X, Y, self_shift=None):
    """(m, n) Helmholtz/Laplace matrix e^{i kappa r}/(4 pi r) (``_kernelcore_np.py:37-49``)."""
    _, r = pair_geometry(X, Y)
    coincident = r == 0.0
    if coincident.any():
        if self_shift is None:
            return None
        r = np.where(coincident, 1.0, r)
        vals = np.exp(1j * kappa * r) / (_4PI * r)
        vals[coincident] = self_shift
        return np.ascontiguousarray(vals)
    return np.ascontiguousarray(np.exp(1j * kappa * r) / (_4PI * r))


def _unit_dirs(X, Y):
    Z, r = pair_geometry(X, Y)
    coincident = r == 0.0
    r = np.where(coincident, 1.0, r)
    return Z / r[..., None], r, coincident


def elasto_u_block(kp, ks, scale, X, Y, self_shift=None):
    """(3m, 3n) displacement tensor U (``_kernelcore_np.py:89-102``)."""
    zh, r, coincident = _unit_dirs(X, Y)
    A, B = navier_coeffs(kp, ks, scale, r, False)
    zz = zh[..., :, None] * zh[..., None, :]
    tensor = A[..., None, None] * np.eye(3) + B[..., None, None] * zz
    tensor = _self_rule(tensor, coincident, self_shift)
    return None if tensor is None else point_major(tensor)


def elasto_t_block(kp, ks, lam, mu, scale, X, Y, NY, self_shift=None):
    """(3m, 3n) traction tensor T with column-point normals NY (``_kernelcore_np.py:105-130``).

    T = -lam D (n z^T) - mu A' (c I + z n^T) - 2 mu B' c z z^T
        - mu (B/r) (2 n z^T + z n^T + c I - 4 c z z^T),  D = A' + B' + 2B/r, c = n.z
    """
    zh, r, coincident = _unit_dirs(X, Y)
    A, B, Ap, Bp = navier_coeffs(kp, ks, scale, r, True)
    nrm = np.broadcast_to(NY[None, :, :], zh.shape)
    c = np.einsum("ijk,ijk->ij", nrm, zh)
    D = Ap + Bp + 2.0 * B / r
    eye = np.eye(3)
    cI = c[..., None, None] * eye
    nz = nrm[..., :, None] * zh[..., None, :]
    zn = zh[..., :, None] * nrm[..., None, :]
    zz = zh[..., :, None] * zh[..., None, :]
    tensor = (
        -lam * D[..., None, None] * nz
        - mu * Ap[..., None, None] * (cI + zn)
        - 2.0 * mu * (Bp * c)[..., None, None] * zz
        - mu * (B / r)[..., None, None] * (2.0 * nz + zn + cI - 4.0 * c[..., None, None] * zz)
    )
    tensor = _self_rule(tensor, coincident, self_shift)
    return None if tensor is None else point_major(tensor)


def block(kind, params, X, Y, NY=None, self_shift=None):
    """Dispatch on kind in {"H","U","T"} with ``params`` = kernel parameter dict."""
    if kind == "H":
        return scalar_block(params["kappa"], X, Y, self_shift)
    if kind == "U":
        return elasto_u_block(params["kp"], params["ks"], params["scale"], X, Y, self_shift)
    if kind == "T":
        return elasto_t_block(
            params["kp"], params["ks"], params["lam"], params["mu"], params["scale"],
            X, Y, NY, self_shift,
        )
    raise ValueError(f"unknown kernel kind {kind!r}")
