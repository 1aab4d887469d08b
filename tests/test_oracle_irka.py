"""Pins of the IRKA oracle (oracle/irka.py, Algorithm 3),
all CPU (-m "not gpu").

* scalar model: G(s) = 1/(s - a) has the single pole a, so IRKA's fixed point
  is σ = -a after one update (Theorem 3.2's mirror-image condition,
  PAPER.md:1083-1091);
* Theorem 3.1: the projected model of V_r, W_r built
  from the RBiCG dual solves Hermite-interpolates G at every shift --
  checked against dense direct solves;
* fixed point at convergence: σ_i = -λ_i(A_r, E_r) to the shift tolerance;
* an independent textbook IRKA with dense LU solves reaches the same shifts;
* BiCG and RBiCG (recycling strategy 1) give the same shift trajectory
  (SPEC.md:453).
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import irka as I
from synth.convdiff import convdiff_csr
from synth.small import vec


def _model(N=8):
    """A stable nonsymmetric state matrix: minus the 2-D conv-diff operator
    (its eigenvalues have positive real parts), b, c seeded."""
    indptr, indices, data = convdiff_csr(N, 2, (10.0, 10.0), "central")[:3]
    n = N * N
    A = -sp.csr_matrix((data, indices, indptr), shape=(n, n))
    return A, vec(n, 71, dist="normal"), vec(n, 72, dist="normal")


def _G(A, b, c, s):
    M = s * np.eye(A.shape[0]) - A.toarray()
    y = np.linalg.solve(M, b)
    return np.vdot(c, y), -np.vdot(c, np.linalg.solve(M, y))


def test_scalar_model_fixed_point():
    a = -2.5
    A = sp.csr_matrix(np.array([[a]]))
    res = I.irka(A, np.ones(1), np.ones(1), [0.3], k=0, tol=1e-14, shift_tol=1e-12)
    assert res.converged
    assert abs(res.shifts[0] - (-a)) <= 1e-12
    assert res.steps <= 2


def test_theorem_3_1_hermite_interpolation():
    A, b, c = _model()
    sig = I.order_shifts([0.05, 0.4, 2.0])
    res = I.irka(A, b, c, sig, k=4, s=10, tol=1e-13, max_steps=0)   # steps 2-3 and 5 only
    for si in res.shifts:
        g, dg = _G(A, b, c, si)
        gr, dgr = I.transfer(res.Ar, res.Er, res.br, res.cr, si)
        assert abs(gr - g) <= 1e-8 * abs(g)
        assert abs(dgr - dg) <= 1e-6 * abs(dg)
    # an interpolation point it was NOT built for is not matched (the check has teeth)
    g, _ = _G(A, b, c, 1.0)
    gr, _ = I.transfer(res.Ar, res.Er, res.br, res.cr, 1.0)
    assert abs(gr - g) > 1e-6 * abs(g)


def _dense_irka(A, b, c, sig, tol=1e-6, steps=60):
    """Textbook IRKA with dense LU solves (an independent implementation)."""
    Ad = A.toarray().astype(np.complex128)
    n = Ad.shape[0]
    sig = I.order_shifts(sig)
    for _ in range(steps):
        V = np.column_stack([np.linalg.solve(s * np.eye(n) - Ad, b) for s in sig])
        W = np.column_stack([np.linalg.solve((s * np.eye(n) - Ad).conj().T, c) for s in sig])
        lam = sla.eigvals(W.conj().T @ Ad @ V, W.conj().T @ V)
        new = I.order_shifts(-lam)
        done = np.max(np.abs(new - sig) / np.abs(sig)) < tol
        sig = new
        if done:
            break
    return sig


def test_converged_fixed_point_and_dense_reference():
    A, b, c = _model()
    res = I.irka(A, b, c, [0.05, 0.4, 2.0], k=4, s=10, tol=1e-12, shift_tol=1e-8,
                 max_steps=60)
    assert res.converged
    lam = sla.eigvals(res.Ar, res.Er)
    np.testing.assert_allclose(I.order_shifts(-lam), res.shifts, rtol=1e-6)
    ref = _dense_irka(A, b, c, [0.05, 0.4, 2.0], tol=1e-8)
    np.testing.assert_allclose(res.shifts, ref, rtol=1e-6)
    # Theorem 3.2: Hermite interpolation at the mirrored reduced poles
    for si in res.shifts:
        g, dg = _G(A, b, c, si)
        gr, dgr = I.transfer(res.Ar, res.Er, res.br, res.cr, si)
        assert abs(gr - g) <= 1e-7 * abs(g) and abs(dgr - dg) <= 1e-5 * abs(dg)


def test_bicg_and_rbicg_trajectories_agree():
    A, b, c = _model()
    kw = dict(s=10, tol=1e-12, shift_tol=1e-8, max_steps=8)
    r1 = I.irka(A, b, c, [0.05, 0.4, 2.0], k=4, recycle=True, **kw)
    r0 = I.irka(A, b, c, [0.05, 0.4, 2.0], k=0, recycle=False, **kw)
    assert len(r1.history) == len(r0.history)
    for s1, s0 in zip(r1.history, r0.history):
        np.testing.assert_allclose(s1, s0, rtol=1e-6)


def test_pick_space_rule():
    """Strategy 3's choice: smallest relative shift
    change below the tolerance, first on ties, none above it."""
    pool = [(1.0, "a"), (2.0 + 0.1j, "b"), (2.1, "c"), (2.1, "d")]
    assert I.pick_space(pool, 2.0, np.inf) == "b"          # |0.1j|/2 = 0.05 < 0.1/2
    assert I.pick_space(pool, 2.1, np.inf) == "c"          # exact match, first of the tie
    assert I.pick_space(pool, 2.0, 0.01) is None           # nothing within 1 %
    assert I.pick_space([], 2.0, np.inf) is None


@pytest.mark.parametrize("strategy", [2, 3])
def test_strategies_reach_the_same_fixed_point(strategy):
    """Recycling changes how the dual pairs are solved, not what they solve:
    strategies 2 and 3 converge to the shifts of strategy 1 and of the dense
    textbook IRKA."""
    A, b, c = _model()
    kw = dict(k=4, s=10, tol=1e-12, shift_tol=1e-8, max_steps=60)
    ref = I.irka(A, b, c, [0.05, 0.4, 2.0], strategy=1, **kw)
    got = I.irka(A, b, c, [0.05, 0.4, 2.0], strategy=strategy, **kw)
    assert got.converged and ref.converged
    np.testing.assert_allclose(got.shifts, ref.shifts, rtol=1e-6)
    np.testing.assert_allclose(got.shifts, _dense_irka(A, b, c, [0.05, 0.4, 2.0], tol=1e-8),
                               rtol=1e-6)


def test_strategy3_zero_tolerance_is_plain_bicg():
    """Strategy 3 with reuse_tol = 0 never hands a space to a solve: every
    solve is BiCG (Algorithm 1 = Algorithm 2 with k = 0), so the iteration
    counts equal those of the non-recycling run."""
    A, b, c = _model()
    kw = dict(s=10, tol=1e-12, shift_tol=1e-8, max_steps=5)
    r3 = I.irka(A, b, c, [0.05, 0.4, 2.0], k=4, strategy=3, reuse_tol=0.0, **kw)
    r0 = I.irka(A, b, c, [0.05, 0.4, 2.0], k=0, recycle=False, **kw)
    assert r3.iterations == r0.iterations
