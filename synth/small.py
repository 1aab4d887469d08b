"""Tiny seeded test matrices (inputs only; no method arithmetic).

All return CSR triples (indptr int32, indices int32, data) so both the oracle
and the CUDA path consume the same bits.
"""
from __future__ import annotations

import numpy as np


def dense_to_csr(M):
    M = np.asarray(M)
    n = M.shape[0]
    mask = M != 0
    counts = mask.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(counts, out=indptr[1:])
    rows, cols = np.nonzero(mask)
    return indptr, cols.astype(np.int32), M[rows, cols].copy()


def random_sparse(n, density=0.05, seed=0, complex_=False, shift=3.0):
    """Nonsymmetric sparse matrix with a dominant diagonal `shift`
    plus a random off-diagonal pattern (well conditioned)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    M = np.zeros((n, n), dtype=np.complex128 if complex_ else np.float64)
    mask = rng.random((n, n)) < density
    vals = rng.standard_normal((n, n))
    if complex_:
        vals = vals + 1j * rng.standard_normal((n, n))
    M[mask] = vals[mask] / np.sqrt(max(1.0, density * n))
    M[np.arange(n), np.arange(n)] = shift + rng.uniform(0, 1, n)
    return dense_to_csr(M)


def spd_sparse(n, seed=0):
    """Sparse SPD matrix: 1-D Laplacian plus a random diagonal shift."""
    rng = np.random.Generator(np.random.PCG64(seed))
    M = np.zeros((n, n))
    i = np.arange(n)
    M[i, i] = 2.0 + rng.uniform(0.1, 1.0, n)
    M[i[:-1], i[:-1] + 1] = -1.0
    M[i[1:], i[1:] - 1] = -1.0
    return dense_to_csr(M)


def deflation_matrix(n, k, seed=0, complex_=False, cond_s=10.0):
    """A = S diag(0.01*(1..k), linspace(1,10,n-k)) S^{-1} with a seeded,
    well-conditioned non-orthogonal S.  Returns the dense A,
    its eigenvalues and S (columns = right eigenvectors)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lam = np.concatenate([0.01 * np.arange(1, k + 1),
                          np.linspace(1.0, 10.0, n - k)])
    # S = I + E with ||E||_2 small enough that kappa(S) <= cond_s
    E = rng.standard_normal((n, n))
    if complex_:
        E = E + 1j * rng.standard_normal((n, n))
    E *= (1.0 - 2.0 / (1.0 + cond_s)) / np.linalg.norm(E, 2)
    S = np.eye(n) + E
    A = S @ np.diag(lam) @ np.linalg.inv(S)
    return A, lam, S


def vec(n, seed, complex_=False, dist="uniform"):
    rng = np.random.Generator(np.random.PCG64(seed))
    if dist == "uniform":
        v = rng.uniform(-1.0, 1.0, n)
        if complex_:
            v = v + 1j * rng.uniform(-1.0, 1.0, n)
    else:
        v = rng.standard_normal(n)
        if complex_:
            v = v + 1j * rng.standard_normal(n)
    return v
