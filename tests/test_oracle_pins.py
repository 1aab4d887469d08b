"""Pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md §8(c) P1-P18).  All CPU-only (``-m "not gpu"``)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import rbicg as R
from oracle.bicg import bicg
from synth import CONFIGS, system_sequence, convdiff_csr
from synth.small import (dense_to_csr, random_sparse, spd_sparse,
                         deflation_matrix, vec)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "worked_examples.json")))


def csr(t, n=None):
    indptr, indices, data = t[:3]
    n = len(indptr) - 1
    return sp.csr_matrix((data, indices, indptr), shape=(n, n))


def cosines(X, Y):
    Q1, _ = np.linalg.qr(X)
    Q2, _ = np.linalg.qr(Y)
    return np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False)


# --------------------------------------------------------------- P13, P17
def test_p17_grid_size_from_paper():
    g = GOLD["convdiff_h_1_64"]
    _, _, _, n = convdiff_csr(g["N"], g["d"], [1.0, 1.0])
    assert n == g["n"]
    assert 1.0 / (g["N"] + 1) == 1.0 / 64


def test_p13_identity_one_iteration():
    g = GOLD["bicg_identity"]
    n = g["n"]
    A = sp.identity(n, format="csr")
    b = np.ones(n)
    res = bicg(A, b, b, np.zeros(n), np.zeros(n), 1e-12, 10)
    assert res["iterations"] == g["iterations"]
    np.testing.assert_allclose(res["x"], g["x"], rtol=1e-15)
    r2 = R.solve_dual(A, b, b, k=0, tol=1e-12, max_itn=10)
    assert r2.iterations == 1
    np.testing.assert_allclose(r2.x, g["x"], rtol=1e-15)


def test_p13_diag12():
    g = GOLD["bicg_diag12"]
    A = sp.diags(g["diag"]).tocsr()
    b, bt = np.array(g["b"]), np.array(g["bt"])
    res = bicg(A, b, bt, np.zeros(2), np.zeros(2), 1e-14, 10)
    assert res["iterations"] <= g["max_iterations"]
    np.testing.assert_allclose(res["x"], g["x"], rtol=1e-13)
    r2 = R.solve_dual(A, b, bt, k=0, tol=1e-14, max_itn=10)
    np.testing.assert_allclose(r2.x, g["x"], rtol=1e-13)


def test_p13_tridiag_from_one_alpha():
    g = GOLD["tridiag_alpha2"]
    L = R.LanczosData()
    L.alpha[1] = g["alpha1"]
    assert L.T(1, 1) == g["T"][0][0]


def test_p13_first_cycle_eigvecs():
    g = GOLD["first_cycle_T1"]
    W, Wt, lam = R.solve_tridiag_first(np.array(g["T"]), g["k"], real=True)
    assert lam.shape == (1,)
    assert abs(lam[0] - g["lambda"]) < 1e-14
    w = W[:, 0] / W[0, 0]
    np.testing.assert_allclose(w, g["w"], atol=1e-14)


def test_p13_diagonal_pencil_selection():
    g = GOLD["pencil_diag"]
    W, Wt, lam = R.solve_pencil(np.diag(g["P"]), np.eye(3), g["k"], True)
    np.testing.assert_allclose(lam.real, g["lambda"], rtol=1e-14)


def test_p13_biorth_cases():
    n = 20
    A = sp.identity(n, format="csr")
    # C~^*C = diag(2,1) (already bi-orthogonal)
    U = np.zeros((n, 2)); U[0, 0] = 2.0; U[1, 1] = 1.0
    Ut = np.zeros((n, 2)); Ut[0, 0] = 1.0; Ut[1, 1] = 1.0
    B = R.biorthogonalize(A, A, U, Ut, 1e-6)
    assert B.k == GOLD["biorth_diag"]["p"]
    assert cosines(B.U, U).min() > 1 - 1e-14
    # rank-1 Gram -> p = 1
    U2 = np.zeros((n, 2)); U2[0, :] = 1.0; U2[1, 1] = 1.0
    Ut2 = np.zeros((n, 2)); Ut2[0, :] = 1.0; Ut2[5, 1] = 1.0
    B2 = R.biorthogonalize(A, A, U2, Ut2, 1e-6)
    assert B2.k == GOLD["biorth_rank1"]["p"]


def test_p13_spmv_adjoint_example():
    g = GOLD["spmv_adjoint_shift"]
    A = sp.csr_matrix(np.array(g["A"]))
    np.testing.assert_array_equal(R.adjoint(A) @ np.array(g["x"]), g["AHx"])


# --------------------------------------------------------------- P1 k=0 == BiCG
@pytest.mark.parametrize("cplx", [False, True])
def test_p1_k0_is_bicg(cplx):
    A = csr(random_sparse(120, 0.05, seed=1, complex_=cplx))
    b, bt = vec(120, 2, cplx), vec(120, 3, cplx)
    ref = bicg(A, b, bt, np.zeros_like(b), np.zeros_like(b), 1e-10, 500)
    res = R.solve_dual(A, b, bt, k=0, tol=1e-10, max_itn=500,
                       update_recycle=False)
    assert res.iterations == ref["iterations"]
    np.testing.assert_allclose(res.hist["alpha"], ref["hist"]["alpha"],
                               rtol=1e-12)
    np.testing.assert_allclose(res.hist["beta"], ref["hist"]["beta"],
                               rtol=1e-12)
    np.testing.assert_allclose(res.x, ref["x"], rtol=1e-12)


# --------------------------------------------------------------- P2 CG
def test_p2_spd_is_cg():
    """Real SPD A, b~ = b, x~ = x: BiCG iterates are CG iterates (scipy cg
    callback iterates as an independent library cross-check)."""
    A = csr(spd_sparse(80, seed=4))
    b = vec(80, 5)
    res = bicg(A, b, b, np.zeros(80), np.zeros(80), 1e-10, 20,
               force_iters=12)
    iters = []
    spla.cg(A, b, rtol=1e-30, maxiter=12,
            callback=lambda xk: iters.append(xk.copy()))
    # oracle x_i after i iterations vs scipy's i-th iterate
    for i in (3, 7, 12):
        r = bicg(A, b, b, np.zeros(80), np.zeros(80), 1e-10, 20,
                 force_iters=i)
        np.testing.assert_allclose(r["x"], iters[i - 1], rtol=1e-10,
                                   atol=1e-12)
        np.testing.assert_allclose(r["xt"], r["x"], rtol=1e-12)


# --------------------------------------------------------------- P3 / P15
def _recycled_problem(cplx=False, n=150, k=4, seed=7):
    A, lam, S = deflation_matrix(n, k, seed=seed, complex_=cplx)
    As = sp.csr_matrix(A)
    b, bt = vec(n, seed + 1, cplx), vec(n, seed + 2, cplx)
    first = R.solve_dual(As, b, bt, k=k, s=12, tol=1e-10, max_itn=600,
                         trunc_tol=1e-6)
    return As, b, bt, first


@pytest.mark.parametrize("cplx", [False, True])
def test_p3_invariants(cplx):
    As, b, bt, first = _recycled_problem(cplx)
    U, Ut = first.basis_out.U, first.basis_out.Ut
    assert U.shape[1] >= 2
    b2, bt2 = vec(len(b), 91, cplx), vec(len(b), 92, cplx)
    r0n = None
    for m in (0, 1, 5, 12):
        res = R.solve_dual(As, b2, bt2, U=U, Ut=Ut, k=4, s=12, tol=1e-10,
                           max_itn=600, force_iters=m, update_recycle=False,
                           trunc_tol=1e-6)
        B = res.basis_in
        if r0n is None:
            r0n = np.linalg.norm(res.r)
            rt0n = np.linalg.norm(res.rt)
            # D_c real positive diagonal; Ĉ^*C = I
            G = B.Ct.conj().T @ B.C
            np.testing.assert_allclose(G, np.diag(B.d), atol=1e-10 * B.d.max())
            assert np.all(B.d > 0)
            np.testing.assert_allclose((B.Ct / B.d).conj().T @ B.C,
                                       np.eye(B.k), atol=1e-10)
        cn = np.linalg.norm(B.Ct, axis=0)
        assert np.max(np.abs(B.Ct.conj().T @ res.r) / cn) <= 1e-10 * r0n
        assert np.max(np.abs(B.C.conj().T @ res.rt)
                      / np.linalg.norm(B.C, axis=0)) <= 1e-10 * rt0n


def test_p3_p15_lanczos_biorthogonality():
    As, b, bt, first = _recycled_problem()
    res = R.solve_dual(As, vec(150, 11), vec(150, 12), U=first.basis_out.U,
                       Ut=first.basis_out.Ut, k=4, s=12, tol=1e-10,
                       max_itn=12, force_iters=12, keep_pencils=True,
                       trunc_tol=1e-6)
    info = res.pencils[0]
    V, Vt = info["V"], info["Vt"]
    Dv = Vt.conj().T @ V
    # (v_i, ṽ_i) = 1 scaling and ṽ_i ⊥ v_m
    np.testing.assert_allclose(np.diag(Dv), 1.0, atol=1e-8)
    off = Dv - np.diag(np.diag(Dv))
    assert np.abs(off).max() <= 1e-8
    np.testing.assert_allclose(np.linalg.norm(V, axis=0), 1.0, rtol=1e-12)
    # Petrov-Galerkin: [C V] ⊥_b [C~ Ṽ] (biorth; P15)
    B = res.basis_in
    assert np.abs(B.Ct.conj().T @ V).max() <= 1e-9
    assert np.abs(B.C.conj().T @ Vt).max() <= 1e-9 * np.abs(Vt).max() * 10


# --------------------------------------------------------------- P4 dense LU
@pytest.mark.parametrize("cplx", [False, True])
def test_p4_dense_lu(cplx):
    n = 200
    A = csr(random_sparse(n, 0.03, seed=21, complex_=cplx))
    b, bt = vec(n, 22, cplx), vec(n, 23, cplx)
    Ad = A.toarray()
    xs = np.linalg.solve(Ad, b)
    xts = np.linalg.solve(Ad.conj().T, bt)
    kappa = np.linalg.cond(Ad)
    tol = 1e-10
    U = Ut = None
    for _ in range(3):
        res = R.solve_dual(A, b, bt, U=U, Ut=Ut, k=4, s=15, tol=tol,
                           max_itn=800, trunc_tol=1e-6)
        U, Ut = res.basis_out.U, res.basis_out.Ut
        assert res.status in (0, 4)
        assert np.linalg.norm(res.x - xs) <= 2 * kappa * tol * np.linalg.norm(xs)
        assert np.linalg.norm(res.xt - xts) <= 2 * kappa * tol * np.linalg.norm(xts)


# --------------------------------------------------------------- P5 Table 1 pattern
def test_p5_recycle_space_converges():
    n, k = 200, 4
    A, lam, S = deflation_matrix(n, k, seed=3)
    As = sp.csr_matrix(A)
    b, bt = vec(n, 1), vec(n, 2)
    left = np.linalg.inv(S).conj().T
    U = Ut = None
    prev = np.zeros(k)
    prevt = np.zeros(k)
    its = []
    for run in range(5):
        res = R.solve_dual(As, b, bt, U=U, Ut=Ut, k=k, s=15, tol=1e-10,
                           max_itn=800, trunc_tol=1e-6)
        U, Ut = res.basis_out.U, res.basis_out.Ut
        its.append(res.iterations)
        c = np.sort(cosines(U, S[:, :k]))[::-1]
        ct = np.sort(cosines(Ut, left[:, :k]))[::-1]
        assert np.all(c >= prev - 1e-3)
        assert np.all(ct >= prevt - 1e-3)
        prev, prevt = c, ct
    assert prev[:k - 1].min() >= 0.99 and prevt[:k - 1].min() >= 0.99
    assert its[-1] < its[0]


# --------------------------------------------------------------- P6 / P6b / R8
@pytest.mark.parametrize("cplx", [False, True])
def test_p6_T_from_scalars_matches_explicit(cplx):
    n = 100
    A = csr(random_sparse(n, 0.05, seed=31, complex_=cplx))
    b, bt = vec(n, 32, cplx), vec(n, 33, cplx)
    res = R.solve_dual(A, b, bt, k=3, s=10, tol=1e-12, max_itn=10,
                       force_iters=10, keep_pencils=True)
    info = res.pencils[0]
    V, Vt, Gam, Gamt, Ups, Upst = (info[x] for x in
                                   ("V", "Vt", "Gam", "Gamt", "Ups", "Upst"))
    T_explicit = Vt.conj().T @ (A @ V)            # Ṽ^* A V (k_in = 0)
    np.testing.assert_allclose(Gam[:10], T_explicit, atol=1e-10 *
                               np.abs(T_explicit).max())
    # T~ = T^*
    Tt_explicit = V.conj().T @ (A.conj().T @ Vt)
    np.testing.assert_allclose(Gamt[:10], Tt_explicit, atol=1e-10 *
                               np.abs(T_explicit).max())
    # extended relation A V_1 = V̲_1 T̲_1 (augBiLanExtend with C = 0)
    np.testing.assert_allclose(A @ V, Ups @ Gam, atol=1e-10 * np.abs(A @ V).max())


@pytest.mark.parametrize("cplx", [False, True])
def test_p6b_B_from_zeta_and_R8(cplx):
    As, b, bt, first = _recycled_problem(cplx, n=120)
    res = R.solve_dual(As, vec(120, 41, cplx), vec(120, 42, cplx),
                       U=first.basis_out.U, Ut=first.basis_out.Ut, k=4, s=12,
                       tol=1e-12, max_itn=24, force_iters=24,
                       keep_pencils=True, trunc_tol=1e-6)
    for info in res.pencils:
        if info["B"] is None:
            continue
        L, j, s = info["L"], info["j"], 12
        B_id = np.stack([(L["zeta"][m] - L["beta"][m - 1] *
                          (L["zeta"][m - 1] if m > 1 else 0))
                         / L["rnorm"][m - 1]
                         for m in range((j - 1) * s + 1, j * s + 1)], axis=1)
        np.testing.assert_allclose(B_id, info["B"], atol=1e-10 *
                                   np.abs(info["B"]).max())
        Bt_id = np.stack([(L["zetat"][m] - np.conj(L["beta"][m - 1]) *
                           (L["zetat"][m - 1] if m > 1 else 0))
                          * L["rnorm"][m - 1] / np.conj(L["rho"][m - 1])
                          for m in range((j - 1) * s + 1, j * s + 1)], axis=1)
        np.testing.assert_allclose(Bt_id, info["Bt"], atol=1e-10 *
                                   np.abs(info["Bt"]).max())
        # R8: C~_j^*C_j = W~^* P W  (A Φ = Ψ H)
        AH = As.conj().T
        G = (AH @ info["Utnew"]).conj().T @ (As @ info["Unew"])
        G8 = info["Wt"].conj().T @ info["P"] @ info["W"]
        np.testing.assert_allclose(G, G8, atol=1e-9 * np.abs(G).max())


# --------------------------------------------------------------- P7 harmonic Ritz
def test_p7_harmonic_ritz_residuals():
    n = 100
    A = csr(random_sparse(n, 0.06, seed=51, complex_=True, shift=1.0))
    b, bt = vec(n, 52, True), vec(n, 53, True)
    first = R.solve_dual(A, b, bt, k=4, s=10, tol=1e-12, max_itn=10,
                         force_iters=10, trunc_tol=1e-6)
    res = R.solve_dual(A, vec(n, 54, True), vec(n, 55, True),
                       U=first.basis_out.U, Ut=first.basis_out.Ut, k=4, s=10,
                       tol=1e-12, max_itn=10, force_iters=10,
                       keep_pencils=True, trunc_tol=1e-6)
    info = res.pencils[0]
    AH = A.conj().T
    Phi, Phit = info["Phi"], info["Phit"]
    nA = sla.norm(A.toarray(), 2)
    for i, lam in enumerate(info["lam"]):
        u = Phi @ info["W"][:, i]
        ut = Phit @ info["Wt"][:, i]
        g = (AH @ Phit).conj().T @ (A @ u - lam * u)
        assert np.linalg.norm(g) <= 1e-8 * nA * np.linalg.norm(u) * \
            np.linalg.norm(AH @ Phit)
        gt = (A @ Phi).conj().T @ (AH @ ut - np.conj(lam) * ut)
        assert np.linalg.norm(gt) <= 1e-8 * nA * np.linalg.norm(ut) * \
            np.linalg.norm(A @ Phi)


def test_q11_real_pairs_kept_together():
    # real pencil whose 3 smallest |λ| are a pair straddling k = 2 plus ...
    P = np.diag([0.5, 2.0, 3.0])
    P[1:, 1:] = [[1.0, 1.0], [-1.0, 1.0]]   # eigenvalues 1 ± i (|λ| = 1.414)
    W, Wt, lam = R.solve_pencil(P, np.eye(3), 2, True)
    assert lam.shape == (1,) and abs(lam[0] - 0.5) < 1e-14   # k-1 taken
    W, Wt, lam = R.solve_pencil(P, np.eye(3), 3, True)
    assert W.shape == (3, 3) and np.isrealobj(W)
    assert np.linalg.matrix_rank(W) == 3


# --------------------------------------------------------------- P8 exact invariant
def test_p8_diagonal_exact_invariant():
    n, k = 60, 3
    d = np.linspace(0.5, 5.0, n)
    A = sp.diags(d).tocsr()
    b, bt = vec(n, 61), vec(n, 62)
    E = np.eye(n)[:, :k]
    res = R.solve_dual(A, b, bt, U=E, Ut=E, k=k, s=10, tol=1e-12,
                       max_itn=200, update_recycle=False)
    ref = bicg(sp.diags(d[k:]).tocsr(), b[k:], bt[k:], np.zeros(n - k),
               np.zeros(n - k), 1e-12 * np.linalg.norm(b) /
               np.linalg.norm(b[k:]), 200)
    assert abs(res.iterations - ref["iterations"]) <= 0
    # identical up to rounding (ζ ~ 1e-16 each step, amplified by BiCG)
    np.testing.assert_allclose(res.hist["alpha"], ref["hist"]["alpha"],
                               rtol=1e-9)
    np.testing.assert_allclose(res.x[:k], b[:k] / d[:k], rtol=1e-14)


# --------------------------------------------------------------- P9
def test_p9_residual_in_range_of_C():
    n = 50
    A = csr(random_sparse(n, 0.1, seed=71))
    AH = A.conj().T.tocsr()
    U, Ut = vec(n * 3, 72).reshape(n, 3), vec(n * 3, 73).reshape(n, 3)
    B = R.biorthogonalize(A, AH, U, Ut, 1e-12)
    b = B.C @ np.array([1.0, -2.0, 0.5])
    x0, xt0, r0, rt0 = R.project_initial(A, AH, B, b, vec(n, 74),
                                         np.zeros(n), np.zeros(n))
    assert np.linalg.norm(r0) <= 1e-12 * np.linalg.norm(b)
    np.testing.assert_allclose(A @ x0, b, atol=1e-12 * np.linalg.norm(b))


# --------------------------------------------------------------- P10 invariance
def test_p10_scaling_invariance():
    n = 150
    A = csr(random_sparse(n, 0.04, seed=81))
    b, bt = vec(n, 82), vec(n, 83)
    r1 = R.solve_dual(A, b, bt, k=3, s=10, tol=1e-10, max_itn=600)
    r2 = R.solve_dual(4.0 * A, b, bt, k=3, s=10, tol=1e-10, max_itn=600)
    assert r1.iterations == r2.iterations
    np.testing.assert_allclose(r2.x, r1.x / 4.0, rtol=1e-9)


# --------------------------------------------------------------- P11 / P12
def test_p12_bilinear_dense_and_quadratic_bound():
    n = 200
    A = csr(random_sparse(n, 0.03, seed=91, complex_=True))
    u, w = vec(n, 92, True), vec(n, 93, True)
    exact = np.vdot(u, np.linalg.solve(A.toarray(), w))
    val, res = R.bilinear(A, u, w, k=4, s=15, tol=1e-10, max_itn=800)
    assert abs(val - exact) <= 1e-8 * abs(exact)
    r = w - A @ res.x
    rt = u - A.conj().T @ res.xt
    Ainv = np.linalg.norm(np.linalg.inv(A.toarray()), 2)
    assert abs(val - exact) <= np.linalg.norm(rt) * Ainv * np.linalg.norm(r) \
        * (1 + 1e-6) + 1e-14 * abs(exact)


def test_p11_conjugate_shift_symmetry():
    cfg = CONFIGS["C4"].scaled(8, systems=2, s=10)
    items = list(system_sequence(cfg, lam_r=0.0))   # slots 0/1: σ, σ̄
    A0 = csr((items[0]["indptr"], items[0]["indices"], items[0]["data"]))
    A1 = csr((items[1]["indptr"], items[1]["indices"], items[1]["data"]))
    assert abs(items[0]["sigma"] - np.conj(items[1]["sigma"])) == 0
    v0, r0 = R.bilinear(A0, items[0]["bt"], items[0]["b"], k=0, tol=1e-10,
                        max_itn=500)
    v1, r1 = R.bilinear(A1, items[1]["bt"], items[1]["b"], k=0, tol=1e-10,
                        max_itn=500)
    assert abs(v1 - np.conj(v0)) <= 1e-8 * abs(v0)
    np.testing.assert_allclose(r1.x, np.conj(r0.x), rtol=1e-7)


# --------------------------------------------------------------- P14 / P18
def test_p14_finite_termination():
    n = 25
    A = csr(random_sparse(n, 0.3, seed=101, shift=2.0))
    b, bt = vec(n, 102), vec(n, 103)
    res = bicg(A, b, bt, np.zeros(n), np.zeros(n), 1e-12, 4 * n)
    assert res["status"] == 0 and res["iterations"] <= n + 3


def test_p18_step7_true_vs_recursive():
    As, b, bt, first = _recycled_problem(n=150)
    res = R.solve_dual(As, vec(150, 111), vec(150, 112), U=first.basis_out.U,
                       Ut=first.basis_out.Ut, k=4, s=12, tol=1e-10,
                       max_itn=600, trunc_tol=1e-6)
    b2 = vec(150, 111)
    assert res.status in (0, 4)
    # after step 7, b - A x equals the recursive residual up to the gap
    np.testing.assert_allclose(b2 - As @ res.x, res.r,
                               atol=1e-12 * np.linalg.norm(b2))
    assert res.relres_true <= 1e-10 and res.relres_dual_true <= 1e-10


# --------------------------------------------------------------- generators
def test_convdiff_stencil_values():
    """Q9 coefficients on a 3x3 grid, checked entry by entry."""
    indptr, indices, data, n = convdiff_csr(3, 2, [8.0, 0.0], "central")
    A = sp.csr_matrix((data, indices, indptr), shape=(n, n)).toarray()
    h = 0.25
    assert A[4, 4] == 4.0
    assert A[4, 5] == -1.0 + 8.0 * h / 2 and A[4, 3] == -1.0 - 8.0 * h / 2
    assert A[4, 7] == -1.0 and A[4, 1] == -1.0
    indptr, indices, data, n = convdiff_csr(3, 2, [8.0, -4.0], "upwind")
    A = sp.csr_matrix((data, indices, indptr), shape=(n, n)).toarray()
    assert A[4, 4] == 4.0 + 8 * h + 4 * h
    assert A[4, 3] == -1.0 - 8 * h and A[4, 5] == -1.0
    assert A[4, 7] == -1.0 - 4 * h and A[4, 1] == -1.0
    for c in ("C1", "C2", "C3", "C5"):
        cfg = CONFIGS[c]
        assert cfg.nnz == (2 * cfg.d + 1) * cfg.n - 2 * cfg.d * cfg.N ** (cfg.d - 1)


# --------------------------------------------------------------- NEXT-1 study variant
@pytest.mark.parametrize("variant", ["single_reduction", "lookahead"])
def test_next1_single_reduction_spd_is_cg(variant):
    """The re-associated variants (single reduction, oracle only;
    lookahead ρ, the fused GPU iteration) on real SPD A with b~ = b, k = 0:
    their iterates are scipy's CG iterates."""
    A = csr(spd_sparse(80, seed=4))
    b = vec(80, 5)
    iters = []
    spla.cg(A, b, rtol=1e-30, maxiter=12, callback=lambda xk: iters.append(xk.copy()))
    for i in (3, 7, 12):
        r = R.solve_dual(A, b, b, k=0, s=20, tol=1e-10, max_itn=20, force_iters=i,
                         variant=variant)
        np.testing.assert_allclose(r.x, iters[i - 1], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("variant", ["single_reduction", "lookahead"])
@pytest.mark.parametrize("cplx", [False, True])
def test_next1_single_reduction_matches_algorithm2(cplx, variant):
    """With a recycle space (k = 4 requested from a first solve of a
    diagonally shifted random sparse matrix) the re-associated recurrences
    reproduce Algorithm 2 as written: the same iteration count, σ_i = (p~_i,
    q_i) histories to 1e-8 (of the largest |σ|), the α_i of the first 12
    iterations to 1e-8, the same solution, the dense-LU solution
    (P4).  (On near-breakdown problems the recurrence σ_{i+1} = δ_i -
    β_iρ_i/α_i cancels and the variants part -- the DESIGN §6 study.)"""
    n = 300
    As = csr(random_sparse(n, 0.03, seed=5, shift=3.0, complex_=cplx))
    first = R.solve_dual(As, vec(n, 1, cplx), vec(n, 2, cplx), k=4, s=12, tol=1e-12,
                         max_itn=300, trunc_tol=1e-8)
    assert first.basis_out.k >= 2
    kw = dict(U=first.basis_out.U, Ut=first.basis_out.Ut, k=4, s=12, tol=1e-12,
              max_itn=300, trunc_tol=1e-8)
    b2, bt2 = vec(n, 3, cplx), vec(n, 4, cplx)
    ref = R.solve_dual(As, b2, bt2, **kw)
    got = R.solve_dual(As, b2, bt2, variant=variant, **kw)
    assert got.basis_in.k >= 2
    assert got.iterations == ref.iterations and got.status == ref.status
    sg, sr = np.array(got.hist["sigma"]), np.array(ref.hist["sigma"])
    np.testing.assert_allclose(sg, sr, rtol=1e-8, atol=1e-10 * np.abs(sr).max())
    np.testing.assert_allclose(got.hist["alpha"][:12], ref.hist["alpha"][:12], rtol=1e-8)
    np.testing.assert_allclose(got.x, ref.x, rtol=1e-8)
    xd = np.linalg.solve(As.toarray(), b2)
    assert np.linalg.norm(got.x - xd) <= 1e-9 * np.linalg.norm(xd)


# ------------------------------------------------------------------ Q3 / Q11 pins
def test_q3_serious_breakdown_at_start_and_redraw():
    """(r~_0, r_0) = 0 exactly (b = e_1, b~ = e_2, x_{-1} = 0): Algorithm 1/2
    step 3 -- without a re-draw vector the solve reports a
    serious breakdown at iteration 0 (Q3, Q4); with one (used once) it runs
    and converges to the dense solution."""
    from oracle import rbicg as R
    n = 6
    A = sp.csr_matrix(np.diag(np.arange(1.0, n + 1)) + np.diag(np.full(n - 1, 0.3), 1)
                      + np.diag(np.full(n - 1, -0.2), -1))
    b, bt = np.eye(n)[0], np.eye(n)[1]
    res = R.solve_dual(A, b, bt, k=0, s=5, tol=1e-12, max_itn=50)
    assert res.status == R.BREAKDOWN_SERIOUS and res.iterations == 0
    res2 = R.solve_dual(A, b, bt, k=0, s=5, tol=1e-12, max_itn=50,
                        xt_redraw=np.linspace(-1, 1, n))
    assert res2.status == R.OK
    np.testing.assert_allclose(res2.x, np.linalg.solve(A.toarray(), b), rtol=1e-10, atol=1e-12)


def test_q3_second_kind_breakdown():
    """σ_1 = (p~_1, A p_1) = 0 with ρ_0 ≠ 0: A = [[0, 1], [1, 0]], b = b~ = e_1
    (p_1 = e_1, A p_1 = e_2 ⊥ e_1) -- the textbook zero-curvature failure of
    CG on an indefinite matrix; BiCG reports a breakdown of the second kind
    before its first update (Q3)."""
    from oracle import rbicg as R
    from oracle.bicg import bicg, BREAKDOWN_SECOND
    A = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    e1 = np.array([1.0, 0.0])
    res = R.solve_dual(A, e1, e1, k=0, s=5, tol=1e-12, max_itn=10)
    assert res.status == R.BREAKDOWN_SECOND and res.iterations == 0
    out = bicg(A, e1, e1, np.zeros(2), np.zeros(2), 1e-12, 10)
    assert out["status"] == BREAKDOWN_SECOND


def test_q3_breakdown_predicate():
    from oracle.bicg import breakdown
    assert breakdown(0.0, 1.0, 1.0, 0.0)              # exact zero (the paper's "= 0")
    assert breakdown(float("nan"), 1.0, 1.0, 0.0)     # non-finite
    assert breakdown(float("inf"), 1.0, 1.0, 0.0)
    assert not breakdown(1e-300, 1.0, 1.0, 0.0)       # tiny but nonzero passes at eps = 0
    assert breakdown(1e-15, 1.0, 1.0, 1e-14) and not breakdown(1e-13, 1.0, 1.0, 1e-14)


def test_q11_infinite_eigenvalues_excluded():
    """Q11: the pencil's infinite eigenvalues (β_QZ = 0, a singular Q) are not
    'nearest the origin' candidates: P = diag(1, 2, 3, 4), Q = diag(1, 0, 1, 1)
    has eigenvalues {1, ∞, 3, 4}; the two nearest the origin are 1 and 3."""
    from oracle import rbicg as R
    P = np.diag([1.0, 2.0, 3.0, 4.0])
    Q = np.diag([1.0, 0.0, 1.0, 1.0])
    W, Wt, lam = R.solve_pencil(P, Q, 2, real=True)
    np.testing.assert_allclose(np.sort(lam.real), [1.0, 3.0], rtol=1e-12)
    # the selected right vectors span e_1, e_3
    assert np.abs(W[[1, 3], :]).max() < 1e-12
