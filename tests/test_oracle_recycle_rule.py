"""Pins of the truncation rule (Q13) and of the Petrov-Galerkin maintenance
(Q32), CPU only.

* Q32 is an exact-arithmetic no-op: on a well-conditioned recycled problem
  (recycle space = exact invariant subspace of a diagonalisable A with
  κ(S) <= 10) the scalars and iterates with and without it agree
  to rounding.
* With it, the Petrov-Galerkin condition r_i ⊥ C~, r~_i ⊥ C ((orth),
  PAPER.md:306-312) holds to BASELINE's 1e-10 (reading Q22) at the end of
  every solve of an ill-conditioned conv-diff sequence.
* The conv-diff C3 family sequences converge under the paper's rule (1e-6,
  PAPER.md:694, :1405) -- without Q32 one of them stagnates (the measured
  mechanism of DESIGN §3: the oblique component CĈ^*r is never touched by
  the projected updates).
* Repeated-solve protocol on the C3 operator at 12^3:
  the iterations fall and the recycle spaces converge to the right/left
  invariant subspaces of the smallest-|λ| eigenvalues, more directions with
  each run -- Table 1's pattern.
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import rbicg as R
from oracle.sequence import csr_matrix, run_sequence
from synth.configs import CONFIGS, system_sequence
from synth.small import deflation_matrix, vec


def _cosines(U, V):
    """Cosines of the principal angles between range(U) and range(V)."""
    Qu = np.linalg.qr(U)[0]
    Qv = np.linalg.qr(V)[0]
    return np.linalg.svd(Qv.conj().T @ Qu, compute_uv=False)


def test_q32_is_exact_arithmetic_noop():
    n, k = 150, 4
    A, lam, S = deflation_matrix(n, k, seed=3)
    Sinv = np.linalg.inv(S)
    U, Ut = S[:, :k], Sinv[:k, :].conj().T    # exact right / left eigenvectors
    A = sp.csr_matrix(A)
    b, bt = vec(n, 1, False), vec(n, 2, False)
    kw = dict(U=U, Ut=Ut, k=k, s=20, tol=1e-10, max_itn=400, trunc_tol=1e-6,
              update_recycle=False)
    on = R.solve_dual(A, b, bt, reproject=True, **kw)
    off = R.solve_dual(A, b, bt, reproject=False, **kw)
    assert on.basis_in.k == k and on.status == off.status == R.OK
    assert on.iterations == off.iterations
    np.testing.assert_allclose(on.hist["alpha"], off.hist["alpha"], rtol=1e-9)
    assert np.linalg.norm(on.x - off.x) <= 1e-9 * np.linalg.norm(off.x)


def test_c3_family_sequences_converge_under_rule():
    """C3@24^3 (8 systems; the sequence that stagnated at 1e-6 before Q32)
    and C3@16^3: every system converges, true residuals <= tol (Q2), and a
    recycle space is in use on most systems."""
    for N in (16, 24):
        cfg = CONFIGS["C3"].scaled(N, systems=8, max_itn=1500)
        assert cfg.trunc_tol == 1e-6
        res = run_sequence(cfg, list(system_sequence(cfg)))
        for r in res:
            assert r.status in (R.OK, R.RECYCLE_EMPTY), (N, r.status, r.iterations)
            assert r.relres_true <= cfg.tol and r.relres_dual_true <= cfg.tol
        assert sum(r.basis_in.k > 0 for r in res) >= 5
        # Petrov-Galerkin maintained ((orth), Q22: normalised by ||r_0||)
        for r in res:
            if r.basis_in.k:
                B = r.basis_in
                pg = np.abs(B.Ct.conj().T @ r.r).max() / np.linalg.norm(r.hist["rnorm"][0])
                pgt = np.abs(B.C.conj().T @ r.rt).max() / np.linalg.norm(r.hist["rtnorm"][0])
                assert pg <= 1e-10 and pgt <= 1e-10, (pg, pgt)


def test_without_q32_a_c3_sequence_stagnates():
    """The mechanism Q32 removes: with reproject=False the same C3@24^3
    sequence (paper's rule) reaches max_itn on some system while the
    recursive residual stalls far above tol."""
    cfg = CONFIGS["C3"].scaled(24, systems=3, max_itn=600)
    items = list(system_sequence(cfg))
    U = Ut = None
    stalled = False
    for item in items:
        A = csr_matrix(item)
        r = R.solve_dual(A, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                         tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol,
                         reproject=False)
        stalled |= r.status == R.MAXITER and r.relres_rec > 1e3 * cfg.tol
        U, Ut = r.basis_out.U, r.basis_out.Ut
    assert stalled


def test_repeated_solve_protocol_table1_pattern():
    """PAPER.md:1321-1327 on the C3 operator at 12^3 (k = 10, s = 40, tol
    1e-8): solve the same dual pair repeatedly, passing the recycle space on.
    Iterations fall by >= 10 % from run 1 to run 2 and never rise above run
    1; the number of principal cosines >= 0.99 between U (Ũ) and the right
    (left) eigenvectors of the same number of smallest-|λ| eigenvalues grows
    to >= 5 (Table 1: more directions converge with each run)."""
    cfg = CONFIGS["C3"].scaled(12, systems=1)
    item = next(iter(system_sequence(cfg)))
    A = csr_matrix(item)
    lam, VL, VR = sla.eig(A.toarray(), left=True, right=True)
    o = np.argsort(np.abs(lam))
    U = Ut = None
    its, good_r, good_l = [], [], []
    for run in range(5):
        res = R.solve_dual(A, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                           tol=cfg.tol, max_itn=1000, trunc_tol=cfg.trunc_tol)
        assert res.status == R.OK
        its.append(res.iterations)
        U, Ut = res.basis_out.U, res.basis_out.Ut
        kk = U.shape[1]
        good_r.append(int(np.sum(_cosines(U, VR[:, o[:kk]]) >= 0.99)))
        good_l.append(int(np.sum(_cosines(Ut, VL[:, o[:kk]]) >= 0.99)))
    assert its[1] <= 0.9 * its[0] and max(its[1:]) <= its[0], its
    assert good_r[-1] >= 5 and good_l[-1] >= 5, (good_r, good_l)
    assert good_r[-1] > good_r[0] and good_l[-1] > good_l[0], (good_r, good_l)
