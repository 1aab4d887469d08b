"""Split preconditioning for (R)BiCG -- test-infrastructure
oracle.  Plain NumPy/SciPy, step by step; shares no code with the CUDA path.

The paper's experiments split-precondition every system with a Crout ILUT
(drop tolerance 0.05 for the convection-diffusion runs, PAPER.md:1330-1331;
ILUTP with per-problem drop tolerances for IRKA), and the
recycle spaces "pertain to the preconditioned linear systems"
(PAPER.md:1332-1333).  With M = L U ≈ A:

    primal  (L^{-1} A U^{-1}) x̂ = L^{-1} b,        x = U^{-1} x̂
    dual    (L^{-1} A U^{-1})^* x̂~ = U^{-*} b~,    x~ = L^{-*} x̂~

since (L^{-1}AU^{-1})^* = U^{-*}A^*L^{-*} and A^* x~ = b~ <=> U^{-*}A^*L^{-*}
(L^* x~) = U^{-*} b~.  Algorithm 2 runs unchanged on Â = L^{-1}AU^{-1}
(reading Q33: the stop test and Q2's true residuals are those of the
preconditioned pair, the only residuals the iteration sees).

ILUC (Crout ILU with threshold; Saad, "Iterative Methods for Sparse Linear
Systems", 2nd ed., Alg. 10.8 / Li, Saad & Chow 2003), in the order the paper's
Matlab `ilu(A, struct('type','crout','droptol',t))` documents its result
(reading Q34): at step k the row z = A[k, k:] - L[k, :k] U[:k, k:] and the
column w = A[k+1:, k] - L[k+1:, :k] U[:k, k] are formed from the finished
rows of U and columns of L; off-diagonal entries with |z_j| < t ||A[:, j]||
(U) or |w_i| < t ||A[:, k]|| (L, tested before the scaling by the pivot)
are dropped; the diagonal is kept; U[k, k:] = z, L[k+1:, k] = w / z_k.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def iluc(A, droptol):
    """Crout ILU with threshold of a sparse A (no pivoting).  Returns
    (L, U) as CSR: L unit lower triangular (diagonal stored), U upper
    triangular.  droptol = 0 keeps every entry: L U = A exactly."""
    A = sp.csc_matrix(A)
    n = A.shape[0]
    dt = A.dtype
    colnorm = np.sqrt(np.asarray(abs(A).power(2).sum(axis=0))).ravel()
    Ar = sp.csr_matrix(A)
    Ucols = [dict() for _ in range(n)]   # U by column: Ucols[j][i] = U[i, j] (i <= j)
    Urows = [dict() for _ in range(n)]   # U by row
    Lrows = [dict() for _ in range(n)]   # L by row: Lrows[i][k] = L[i, k] (k < i)
    Lcols = [dict() for _ in range(n)]   # L by column
    for k in range(n):
        # z = A[k, k:] - sum_{i<k, L[k,i] != 0} L[k, i] U[i, k:]
        z = {}
        row = Ar.getrow(k)
        for j, v in zip(row.indices, row.data):
            if j >= k:
                z[j] = z.get(j, 0) + v
        for i, lki in Lrows[k].items():
            for j, uij in Urows[i].items():
                if j >= k:
                    z[j] = z.get(j, 0) - lki * uij
        # w = A[k+1:, k] - sum_{i<k, U[i,k] != 0} U[i, k] L[k+1:, i]
        w = {}
        col = A.getcol(k)
        for i, v in zip(col.indices, col.data):
            if i > k:
                w[i] = w.get(i, 0) + v
        for i, uik in Ucols[k].items():
            if i >= k:
                continue
            for r, lri in Lcols[i].items():
                if r > k:
                    w[r] = w.get(r, 0) - uik * lri
        piv = z.get(k, 0)
        if piv == 0:
            raise ZeroDivisionError(f"zero pivot at row {k}")
        for j, v in z.items():
            if j == k or abs(v) >= droptol * colnorm[j]:
                Urows[k][j] = v
                Ucols[j][k] = v
        for r, v in w.items():
            if abs(v) >= droptol * colnorm[k]:
                lv = v / piv
                Lrows[r][k] = lv
                Lcols[k][r] = lv
    Li, Lj, Lv, Ui, Uj, Uv = [], [], [], [], [], []
    for i in range(n):
        for k, v in Lrows[i].items():
            Li.append(i), Lj.append(k), Lv.append(v)
        Li.append(i), Lj.append(i), Lv.append(1.0)
        for j, v in Urows[i].items():
            Ui.append(i), Uj.append(j), Uv.append(v)
    L = sp.csr_matrix((np.array(Lv, dtype=dt), (Li, Lj)), shape=(n, n))
    U = sp.csr_matrix((np.array(Uv, dtype=dt), (Ui, Uj)), shape=(n, n))
    L.sort_indices()
    U.sort_indices()
    return L, U


class SplitOperator:
    """Â = L^{-1} A U^{-1} as an operator (vectors and n x k blocks), with
    its adjoint U^{-*} A^* L^{-*} (``adjoint_op``), for oracle.rbicg."""

    def __init__(self, A, L, U, adjoint=False):
        self.A, self.L, self.U, self.adj = sp.csr_matrix(A), sp.csr_matrix(L), sp.csr_matrix(U), adjoint
        self.shape = A.shape
        self.dtype = np.result_type(A.dtype, L.dtype, U.dtype)

    def _tri(self, M, v, lower):
        return spla.spsolve_triangular(M, v, lower=lower)

    def __matmul__(self, v):
        v = np.asarray(v)
        if not self.adj:   # L^{-1} (A (U^{-1} v))
            y = self._tri(self.U, v, lower=False)
            return self._tri(self.L, self.A @ y, lower=True)
        # U^{-*} (A^* (L^{-*} v))
        y = self._tri(self.L.conj().T.tocsr(), v, lower=False)
        return self._tri(self.U.conj().T.tocsr(), self.A.conj().T @ y, lower=True)

    def adjoint_op(self):
        return SplitOperator(self.A, self.L, self.U, adjoint=not self.adj)

    def toarray(self):
        """Dense Â (small n only; tests)."""
        return self @ np.eye(self.shape[0], dtype=self.dtype)


def solve_dual_split(A, L, U, b, bt, x_m1=None, xt_m1=None, Ur=None, Utr=None, **kw):
    """Split-preconditioned RBiCG on the dual pair (module docstring):
    Algorithm 2 on Â = L^{-1}AU^{-1} with b̂ = L^{-1}b, b̂~ = U^{-*}b~ and
    x̂_{-1} = U x_{-1}, x̂~_{-1} = L^* x~_{-1}; returns (x, x~, result) with
    x = U^{-1}x̂, x~ = L^{-*}x̂~ and the result of the preconditioned solve
    (its recycle space belongs to Â)."""
    from .rbicg import solve_dual
    n = A.shape[0]
    Ah = SplitOperator(A, L, U)
    Lc, Uc = sp.csr_matrix(L), sp.csr_matrix(U)
    bh = spla.spsolve_triangular(Lc, b, lower=True)
    bth = spla.spsolve_triangular(Uc.conj().T.tocsr(), bt, lower=True)
    xh0 = None if x_m1 is None else Uc @ x_m1
    xth0 = None if xt_m1 is None else Lc.conj().T @ xt_m1
    res = solve_dual(Ah, bh, bth, xh0, xth0, Ur, Utr, **kw)
    x = spla.spsolve_triangular(Uc, res.x, lower=False)
    xt = spla.spsolve_triangular(Lc.conj().T.tocsr(), res.xt, lower=False)
    assert x.shape == (n,)
    return x, xt, res
