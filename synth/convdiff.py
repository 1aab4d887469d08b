"""Finite-difference convection-diffusion operators in CSR (inputs only).

Discretisation of  -Δu + β·∇u = f  on the unit square / cube, following the
reading SURVEY.md Q9 (the paper's own coefficient field, is not
given in its text):

* N interior points per axis, h = 1/(N+1), homogeneous Dirichlet boundary;
* lexicographic ordering, x fastest (row = x + N*y + N^2*z);
* every row multiplied by h^2;
* central differences: diagonal 2d, neighbour along axis a is
  -1 + β_a h/2 (forward neighbour) and -1 - β_a h/2 (backward neighbour);
* first-order upwind: diagonal 2d + Σ_a |β_a| h, upstream neighbour
  -1 - |β_a| h, downstream neighbour -1 (upstream = backward when β_a > 0).

Column indices are strictly increasing within each row.  P17 pins the grid
size rule against the paper's "h = 1/64 ... 3969 unknowns".
"""
from __future__ import annotations

import numpy as np


def convdiff_nnz(N: int, d: int) -> int:
    """Structural nonzeros of the (2d+1)-point stencil: (2d+1)n - 2d N^(d-1)."""
    n = N ** d
    return (2 * d + 1) * n - 2 * d * N ** (d - 1)


def _coefficients(beta, h, scheme):
    """Per-axis (backward, forward) neighbour coefficients and the diagonal."""
    d = len(beta)
    back, fwd = [], []
    diag = 2.0 * d
    for b in beta:
        b = float(b)
        if scheme == "central":
            back.append(-1.0 - b * h / 2.0)
            fwd.append(-1.0 + b * h / 2.0)
        elif scheme == "upwind":
            diag += abs(b) * h
            if b >= 0.0:
                back.append(-1.0 - abs(b) * h)
                fwd.append(-1.0)
            else:
                back.append(-1.0)
                fwd.append(-1.0 - abs(b) * h)
        else:
            raise ValueError(f"unknown scheme {scheme!r}")
    return diag, back, fwd


def convdiff_csr(N: int, d: int, beta, scheme: str = "central"):
    """Return (indptr int32[n+1], indices int32[nnz], data float64[nnz], n)."""
    if d not in (2, 3):
        raise ValueError("d must be 2 or 3")
    if len(beta) != d:
        raise ValueError("beta must have d components")
    n = N ** d
    h = 1.0 / (N + 1)
    diag, back, fwd = _coefficients(beta, h, scheme)

    rows = np.arange(n, dtype=np.int64)
    coords = []
    rem = rows.copy()
    for _ in range(d):
        coords.append(rem % N)
        rem //= N
    strides = [N ** a for a in range(d)]

    # Entries in ascending column order: backward neighbours from the slowest
    # axis to the fastest, the diagonal, then forward neighbours fastest to
    # slowest.
    slots = []  # list of (mask, column offset, value)
    for a in reversed(range(d)):
        slots.append((coords[a] > 0, -strides[a], back[a]))
    slots.append((np.ones(n, dtype=bool), 0, diag))
    for a in range(d):
        slots.append((coords[a] < N - 1, strides[a], fwd[a]))

    counts = np.zeros(n, dtype=np.int64)
    for m, _, _ in slots:
        counts += m
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    assert nnz == convdiff_nnz(N, d)
    indices = np.empty(nnz, dtype=np.int32)
    data = np.empty(nnz, dtype=np.float64)
    pos = indptr[:-1].copy()
    for m, off, val in slots:
        r = rows[m]
        p = pos[m]
        indices[p] = (r + off).astype(np.int32)
        data[p] = val
        pos[m] += 1
    return indptr.astype(np.int32), indices, data, n


def laplacian_offdiag_positions(N: int, d: int = 3):
    """CSR of the unscaled 7-point Laplacian L (diag 2d, off-diagonal -1) and a
    boolean mask of its off-diagonal entries in CSR order (rows ascending,
    columns ascending) -- the draw order of the C4 perturbation."""
    indptr, indices, _, n = convdiff_csr(N, d, [0.0] * d, "central")
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    offmask = indices != rows
    return indptr, indices, offmask, n
