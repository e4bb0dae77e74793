"""Seeded synthetic problems for the BASELINE.json configurations.

Host-side problem *setup* only (the reference builds its problems on the host
too: matio.py:278-307, tests/conftest.py:33-46); nothing here is on the solve
path.  Every generator returns a `ProblemInstance` whose matrix is a sorted
int32-index CSR `SparseMatrix`, exactly the boundary contract of
`adaptive_solve` (adaptive.py:111).  BASELINE configs name no public dataset:
all inputs are synthetic and seeded (`np.random.default_rng(seed)`).

  c1  2-D Poisson 5-point, 64x64 (N=4096), x* ~ U[-1,1], b = A x*
  c2  Strakos diagonal N=1e4, lambda in [1e-3, 1e2], rho=0.9, b ~ N(0,1)/||.||
  c3  3-D Poisson 7-point, 128^3, x* ~ U[-1,1], b = A x*
  c4  3-D variable-coefficient 27-point, 192^3, lognormal(0,1.5) cells,
      harmonic-mean face weights / |offset|^2, Dirichlet, b ~ N(0,1)/||.||
  c5  3-D Poisson 7-point, 512^3 (or 256x256x(256 P) weak-scaled), b = A x*
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from .types import ProblemInstance, SparseMatrix


def _sparse(n, indptr, indices, data):
    indptr = np.ascontiguousarray(indptr)
    if indptr[-1] < 2**31:
        indptr = indptr.astype(np.int32)
    a = SparseMatrix(
        n=n,
        row_ptr=indptr,
        col_idx=np.ascontiguousarray(indices, dtype=np.int32),
        values=np.ascontiguousarray(data, dtype=np.float64),
        n_a=int(np.diff(indptr).max()) if n else 0,
    )
    return a


def stencil7(nx, ny, nz):
    """7-point Dirichlet Laplacian kron(I,I,T)+kron(I,T,I)+kron(T,I,I), x fastest.

    Columns of each row are emitted in ascending order (-z, -y, -x, 0, +x, +y, +z)
    without building COO temporaries, so 256^3 (117M nnz) builds in seconds.
    """
    n = nx * ny * nz
    i = np.arange(n, dtype=np.int64)
    ix = i % nx
    iy = (i // nx) % ny
    iz = i // (nx * ny)
    offs = [(-nx * ny, iz > 0), (-nx, iy > 0), (-1, ix > 0), (0, None),
            (1, ix < nx - 1), (nx, iy < ny - 1), (nx * ny, iz < nz - 1)]
    counts = np.ones(n, dtype=np.int64)
    for off, m in offs:
        if m is not None:
            counts += m
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int32)
    data = np.empty(nnz, dtype=np.float64)
    pos = indptr[:-1].copy()
    for off, m in offs:
        if m is None:
            indices[pos] = i.astype(np.int32)
            data[pos] = 6.0
            pos += 1
        else:
            rows = np.nonzero(m)[0]
            indices[pos[rows]] = (rows + off).astype(np.int32)
            data[pos[rows]] = -1.0
            pos[rows] += 1
    del pos, i, ix, iy, iz
    return _sparse(n, indptr, indices, data)


def stencil5(nx, ny):
    """2-D 5-point Dirichlet Laplacian kron(I,T)+kron(T,I) (x fastest)."""
    t = sp.diags([-np.ones(nx - 1), 2 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1])
    ty = sp.diags([-np.ones(ny - 1), 2 * np.ones(ny), -np.ones(ny - 1)], [-1, 0, 1])
    a = (sp.kron(sp.identity(ny), t) + sp.kron(ty, sp.identity(nx))).tocsr()
    a.sum_duplicates()
    a.sort_indices()
    return _sparse(a.shape[0], a.indptr, a.indices, a.data)


def _lap_eigs_1d(n):
    k = np.arange(1, n + 1)
    return 2.0 - 2.0 * np.cos(k * np.pi / (n + 1))


def _problem(a, b, norm_a, norm_abs_a, kappa_a, label):
    return ProblemInstance(a=a, b=np.ascontiguousarray(b, dtype=np.float64),
                           x0=np.zeros(a.n), norm_a=float(norm_a),
                           norm_abs_a=float(norm_abs_a), kappa_a=float(kappa_a),
                           label=label)


def spmv_host(a, x):
    """b = A x* for problem setup (scipy; same as the reference's own setup)."""
    m = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    return m @ x


def poisson2d(n=64, seed=0):
    """c1: 2-D Poisson 64x64."""
    a = stencil5(n, n)
    rng = np.random.default_rng(seed)
    xs = rng.uniform(-1.0, 1.0, a.n)
    b = spmv_host(a, xs)
    e = _lap_eigs_1d(n)
    lmax, lmin = 2 * e[-1], 2 * e[0]
    return _problem(a, b, lmax, 4.0 + 4.0 * math.cos(math.pi / (n + 1)), lmax / lmin,
                    f"poisson2d-{n}")


def poisson3d(nx, ny=None, nz=None, seed=0):
    """c3 / c5: 3-D Poisson 7-point on nx*ny*nz, b = A x*, x* ~ U[-1,1]."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    a = stencil7(nx, ny, nz)
    rng = np.random.default_rng(seed)
    xs = rng.uniform(-1.0, 1.0, a.n)
    b = spmv_host(a, xs)
    lmax = _lap_eigs_1d(nx)[-1] + _lap_eigs_1d(ny)[-1] + _lap_eigs_1d(nz)[-1]
    lmin = _lap_eigs_1d(nx)[0] + _lap_eigs_1d(ny)[0] + _lap_eigs_1d(nz)[0]
    nabs = sum(2.0 + 2.0 * math.cos(math.pi / (m + 1)) for m in (nx, ny, nz))
    return _problem(a, b, lmax, nabs, lmax / lmin, f"poisson3d-{nx}x{ny}x{nz}")


def strakos(n=10_000, l1=1e-3, ln=1e2, rho=0.9, seed=0):
    """c2: Strakos diagonal lambda_i = l1 + (i-1)/(n-1) (ln-l1) rho^(n-i)."""
    i = np.arange(1, n + 1, dtype=np.float64)
    lam = l1 + (i - 1.0) / (n - 1.0) * (ln - l1) * rho ** (n - i)
    indptr = np.arange(n + 1, dtype=np.int64)
    a = _sparse(n, indptr, np.arange(n, dtype=np.int32), lam)
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(n)
    b = b / np.linalg.norm(b)
    return _problem(a, b, lam.max(), lam.max(), lam.max() / lam.min(), f"strakos-{n}")


def varcoef27(n=192, sigma_ln=1.5, seed=0):
    """c4: 27-point variable-coefficient diffusion on n^3 (SURVEY.md 8(d) rule).

    k ~ exp(N(0, sigma_ln^2)) per cell; each of the 26 neighbour offsets o has
    weight 1/|o|^2 times the harmonic mean 2 k_i k_j / (k_i + k_j);
    A_ij = -w, A_ii = sum of in-domain w plus out-of-domain w_o k_i (Dirichlet).
    Exactly symmetric, SPD, ~27 nnz/row; b ~ N(0,1) normalised.
    """
    rng = np.random.default_rng(seed)
    k = np.exp(rng.normal(0.0, sigma_ln, (n, n, n)))  # [z, y, x]
    nn = n ** 3
    offsets = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    # per-row entries in ascending column order == lexicographic (dz, dy, dx)
    counts = np.zeros(nn, dtype=np.int64)
    diag = np.zeros((n, n, n))
    masks = {}
    idx = np.arange(n)
    for (dz, dy, dx) in offsets:
        if (dz, dy, dx) == (0, 0, 0):
            counts += 1
            continue
        mz = (idx + dz >= 0) & (idx + dz < n)
        my = (idx + dy >= 0) & (idx + dy < n)
        mx = (idx + dx >= 0) & (idx + dx < n)
        m = mz[:, None, None] & my[None, :, None] & mx[None, None, :]
        masks[(dz, dy, dx)] = m
        counts += m.ravel()
        w0 = 1.0 / (dz * dz + dy * dy + dx * dx)
        shifted = np.zeros_like(k)
        sz = slice(max(0, -dz), n - max(0, dz))
        sy = slice(max(0, -dy), n - max(0, dy))
        sx = slice(max(0, -dx), n - max(0, dx))
        tz = slice(max(0, dz), n - max(0, -dz))
        ty = slice(max(0, dy), n - max(0, -dy))
        tx = slice(max(0, dx), n - max(0, -dx))
        shifted[sz, sy, sx] = k[tz, ty, tx]
        h = np.where(m, 2.0 * k * shifted / np.where(m, k + shifted, 1.0), 0.0)
        diag += np.where(m, w0 * h, w0 * k)
    indptr = np.zeros(nn + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int32)
    data = np.empty(nnz, dtype=np.float64)
    pos = indptr[:-1].copy()
    rows_all = np.arange(nn, dtype=np.int64)
    for (dz, dy, dx) in offsets:
        if (dz, dy, dx) == (0, 0, 0):
            indices[pos] = rows_all.astype(np.int32)
            data[pos] = diag.ravel()
            pos += 1
            continue
        m = masks[(dz, dy, dx)].ravel()
        rows = np.nonzero(m)[0]
        off = dz * n * n + dy * n + dx
        w0 = 1.0 / (dz * dz + dy * dy + dx * dx)
        kr = k.ravel()
        kc = kr[rows + off]
        ki = kr[rows]
        indices[pos[rows]] = (rows + off).astype(np.int32)
        data[pos[rows]] = -(w0 * (2.0 * ki * kc / (ki + kc)))
        pos[rows] += 1
    a = _sparse(nn, indptr, indices, data)
    b = rng.standard_normal(nn)
    b = b / np.linalg.norm(b)
    # norms only feed the full-bound c; Gershgorin bounds are adequate here
    gersh = float(np.max(2.0 * np.abs(diag)))
    return _problem(a, b, gersh, gersh, math.inf, f"varcoef27-{n}")


def varcoef27_jacobi(n=192, seed=0):
    """c4 with the paper's two-sided Jacobi scaling (matio.py
    jacobi_precondition): A_hat = D^-1/2 A D^-1/2, the same b.  SURVEY.md H6:
    BASELINE.json does not pin the scaling; the literal c4 is the primary run,
    this the secondary one."""
    from .matio import jacobi_precondition
    base = varcoef27(n, seed=seed)
    a_hat, _ = jacobi_precondition(base.a)
    # |A_hat| <= Gershgorin of the scaled rows (unit diagonal)
    rs = np.add.reduceat(np.abs(np.asarray(a_hat.values)), np.asarray(a_hat.row_ptr)[:-1])
    g = float(rs.max())
    return _problem(a_hat, base.b, g, g, math.inf, f"varcoef27-jacobi-{n}")


CONFIGS = {
    "c1": dict(desc="2D Poisson 64^2, sigma=8 Newton, 1e-10", sigma=8, eps_star=1e-10,
               basis_kind="newton"),
    "c2": dict(desc="Strakos 1e4, sigma=10 Chebyshev, 1e-8", sigma=10, eps_star=1e-8,
               basis_kind="chebyshev"),
    "c2n": dict(desc="Strakos 1e4, sigma=10 Newton, 1e-8", sigma=10, eps_star=1e-8,
                basis_kind="newton"),
    "c3": dict(desc="3D Poisson 128^3, sigma=10 Chebyshev, 1e-10", sigma=10,
               eps_star=1e-10, basis_kind="chebyshev"),
    "c4": dict(desc="27-pt var-coef 192^3, sigma=10 Newton, 1e-8", sigma=10, eps_star=1e-8,
               basis_kind="newton"),
    "c4j": dict(desc="27-pt var-coef 192^3, Jacobi-scaled, sigma=10 Newton, 1e-8", sigma=10,
                eps_star=1e-8, basis_kind="newton"),
    "c5": dict(desc="3D Poisson 512^3, sigma=12 Newton, 1e-10", sigma=12, eps_star=1e-10,
               basis_kind="newton"),
    "c5w": dict(desc="3D Poisson 256^3 per GPU (weak), sigma=12 Newton, 1e-10", sigma=12,
                eps_star=1e-10, basis_kind="newton"),
}


def make_problem(name, seed=0, scale=None, world=1):
    """Build the named BASELINE config (scale overrides the grid edge for tests)."""
    if name == "c1":
        return poisson2d(scale or 64, seed)
    if name in ("c2", "c2n"):
        return strakos(scale or 10_000, seed=seed)
    if name == "c3":
        return poisson3d(scale or 128, seed=seed)
    if name == "c4":
        return varcoef27(scale or 192, seed=seed)
    if name == "c4j":
        return varcoef27_jacobi(scale or 192, seed=seed)
    if name == "c5":
        return poisson3d(scale or 512, seed=seed)
    if name == "c5w":
        e = scale or 256
        return poisson3d(e, e, e * world, seed=seed)
    raise KeyError(name)
