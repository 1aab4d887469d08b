"""Pins of the split-preconditioning oracle (oracle/precond.py, SURVEY §8(f)
NEXT-4), CPU only.

* ILUC with droptol = 0 is the exact LU without pivoting: L U = A (a
  textbook identity, checked against a dense elimination), L unit lower, U
  upper; on a tridiagonal A (no fill) every droptol below the entries gives
  the exact LU too.
* Every kept off-diagonal factor entry satisfies the documented drop rule
  (reading Q34).
* Â = L^{-1} A U^{-1}: the operator equals the dense product and its adjoint
  is the conjugate transpose ((u, Â v) = (Â^* u, v)).
* With the exact LU (droptol 0) the preconditioned solve converges in one
  iteration to A^{-1} b and A^{-*} b~.
* solve_dual_split equals Algorithm 2 run on the explicitly formed dense Â
  (an independent route to the same iteration).
* Repeated-solve protocol on a split-preconditioned 2-D
  conv-diff system: the recycled runs need fewer iterations.
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import precond as PC
from oracle import rbicg as R
from synth import convdiff_csr
from synth.small import vec


def _convdiff(N, beta):
    ip, ix, dv = convdiff_csr(N, 2, (beta, beta), "central")[:3]
    return sp.csr_matrix((dv, ix, ip), shape=(N * N, N * N))


def _dense_lu_nopivot(M):
    M = np.array(M, dtype=float)
    n = M.shape[0]
    L = np.eye(n)
    U = M.copy()
    for k in range(n - 1):
        L[k + 1:, k] = U[k + 1:, k] / U[k, k]
        U[k + 1:, :] -= np.outer(L[k + 1:, k], U[k, :])
    return L, np.triu(U)


def test_iluc_droptol0_is_exact_lu():
    A = _convdiff(9, 5.0)
    L, U = PC.iluc(A, 0.0)
    Ld, Ud = _dense_lu_nopivot(A.toarray())
    np.testing.assert_allclose(L.toarray(), Ld, atol=1e-13)
    np.testing.assert_allclose(U.toarray(), Ud, atol=1e-12)
    assert sp.triu(L, 1).nnz == 0 and sp.tril(U, -1).nnz == 0
    np.testing.assert_array_equal(L.diagonal(), 1.0)


def test_iluc_tridiagonal_has_no_fill():
    n = 40
    A = sp.diags([np.full(n - 1, -1.2), np.full(n, 4.0), np.full(n - 1, -0.7)], [-1, 0, 1],
                 format="csr")
    L, U = PC.iluc(A, 0.1)
    assert abs(L @ U - A).max() <= 1e-14 * abs(A).max()


def test_iluc_drop_rule():
    A = _convdiff(12, 30.0)
    t = 0.05
    L, U = PC.iluc(A, t)
    cn = np.sqrt(np.asarray(abs(A).power(2).sum(axis=0))).ravel()
    Uc = sp.coo_matrix(U)
    off = Uc.row != Uc.col
    assert np.all(np.abs(Uc.data[off]) >= t * cn[Uc.col[off]] * (1 - 1e-12))
    Lc = sp.coo_matrix(L)
    off = Lc.row != Lc.col
    piv = U.diagonal()
    # tested before the division by the pivot: |l * u_kk| >= t ||A(:, k)||
    assert np.all(np.abs(Lc.data[off] * piv[Lc.col[off]]) >= t * cn[Lc.col[off]] * (1 - 1e-12))
    assert abs(L @ U - A).max() > 0   # something was dropped
    assert np.any(np.abs(Lc.data[off]) > 0)


def test_split_operator_dense_and_adjoint():
    A = _convdiff(8, 10.0)
    L, U = PC.iluc(A, 0.05)
    op = PC.SplitOperator(A, L, U)
    dense = np.linalg.solve(L.toarray(), A.toarray() @ np.linalg.inv(U.toarray()))
    v, u = vec(64, 3, False), vec(64, 4, False)
    np.testing.assert_allclose(op @ v, dense @ v, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(op.adjoint_op() @ u, dense.conj().T @ u, rtol=1e-12, atol=1e-13)
    assert abs(np.vdot(u, op @ v) - np.vdot(op.adjoint_op() @ u, v)) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(v) * 10


def test_exact_lu_converges_in_one_iteration():
    A = _convdiff(10, 8.0)
    L, U = PC.iluc(A, 0.0)
    b, bt = vec(100, 5, False), vec(100, 6, False)
    x, xt, res = PC.solve_dual_split(A, L, U, b, bt, k=0, s=10, tol=1e-10, max_itn=20)
    assert res.status == R.OK and res.iterations == 1
    np.testing.assert_allclose(x, spla.spsolve(A.tocsc(), b), rtol=1e-10)
    np.testing.assert_allclose(xt, spla.spsolve(A.conj().T.tocsc(), bt), rtol=1e-10)


def test_split_solve_equals_algorithm2_on_dense_ahat():
    A = _convdiff(12, 20.0)
    L, U = PC.iluc(A, 0.1)
    n = A.shape[0]
    b, bt = vec(n, 7, False), vec(n, 8, False)
    # 12 iterations, one cycle end (beyond ~20 iterations BiCG's rounding
    # amplification separates any two routes to the same iteration)
    kw = dict(k=4, s=8, tol=1e-10, max_itn=40, force_iters=12, trunc_tol=1e-6)
    x, xt, res = PC.solve_dual_split(A, L, U, b, bt, **kw)
    Ad = np.linalg.solve(L.toarray(), A.toarray() @ np.linalg.inv(U.toarray()))
    bh = sla.solve_triangular(L.toarray(), b, lower=True)
    bth = sla.solve_triangular(U.toarray().conj().T, bt, lower=True)
    ref = R.solve_dual(sp.csr_matrix(Ad), bh, bth, **kw)
    np.testing.assert_allclose(res.hist["alpha"], ref.hist["alpha"], rtol=1e-8)
    np.testing.assert_allclose(res.x, ref.x, rtol=1e-8, atol=1e-10 * np.abs(ref.x).max())
    assert res.basis_out.k == ref.basis_out.k > 0
    Q1 = np.linalg.qr(res.basis_out.U)[0]
    Q2 = np.linalg.qr(ref.basis_out.U)[0]
    assert np.linalg.svd(Q1.T @ Q2, compute_uv=False).min() >= 1 - 1e-8


def test_repeated_solve_protocol_preconditioned():
    """PAPER.md:1321-1327 with split ILUT preconditioning on a 2-D conv-diff
    operator (h = 1/64, the paper's grid; drop tolerance 0.2 so
    that a solve spans more than one cycle of s = 40): the second run with the
    first run's recycle space is >= 15 % shorter."""
    A = _convdiff(63, 40.0)
    L, U = PC.iluc(A, 0.2)
    n = A.shape[0]
    b, bt = vec(n, 1, False, dist="uniform"), vec(n, 2, False, dist="uniform")
    its, Ur, Utr = [], None, None
    for _ in range(2):
        x, xt, res = PC.solve_dual_split(A, L, U, b, bt, Ur=Ur, Utr=Utr, k=10, s=40, tol=1e-8,
                                         max_itn=2000, trunc_tol=1e-6)
        assert res.status == R.OK and np.linalg.norm(b - A @ x) <= 1e-6 * np.linalg.norm(b)
        its.append(res.iterations)
        Ur, Utr = res.basis_out.U, res.basis_out.Ut
    assert its[1] <= 0.85 * its[0], its
