"""Pins of the §4.4 pencil assembly (oracle.rbicg.fast_grams, PAPER.md:709-958,
SURVEY §8(f) NEXT-2), CPU only.

§4.4 replaces the Grams Ψ~_j^*Ψ_j and Ψ~_j^*Φ_j of the pencil
(finalGenEigValue) by recurrences that hold in exact arithmetic.  The pins:
* every block of the recurrence-built Grams equals the explicit product of the
  stored vectors (the plain assembly) to the level the Lanczos vectors' own
  bi-orthogonality holds, in all three cases of §4.2 that use the pencil
  (first system j >= 2; first cycle of a later system; the general case),
  real and complex -- a wrong block, index, transpose or conjugate is an O(1)
  difference;
* on the C4-family workload (shifted, near-normal: its recycle spaces are
  well conditioned) the solver with the fast assembly converges like the
  plain one (same systems, iteration counts within a few, true residuals
  below tol).  On the C1 family the Lanczos vectors lose bi-orthogonality
  within a cycle, so the recurrences (exact-arithmetic identities) and the
  explicit products select different spaces there (Q31).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import rbicg as R
from oracle.sequence import run_sequence
from synth.configs import CONFIGS, system_sequence
from synth.small import deflation_matrix, vec


def _cfg(name):
    return CONFIGS[name] if isinstance(CONFIGS, dict) else \
        [c for c in CONFIGS if c.name == name][0]


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_fast_grams_equal_explicit_products(cplx):
    n, k, s = 120, 4, 12
    A, _, _ = deflation_matrix(n, k, seed=7, complex_=cplx)
    A = sp.csr_matrix(A)
    kw = dict(k=k, s=s, tol=1e-12, trunc_tol=1e-2, keep_pencils=True, pencil="fast")
    first = R.solve_dual(A, vec(n, 8, cplx), vec(n, 9, cplx), max_itn=48,
                         force_iters=48, **kw)
    second = R.solve_dual(A, vec(n, 41, cplx), vec(n, 42, cplx),
                          U=first.basis_out.U, Ut=first.basis_out.Ut,
                          max_itn=48, force_iters=48, **kw)
    cases = set()
    for res in (first, second):
        for info in res.pencils:
            if info["case"] != "pencil" or info["j"] > 3:
                continue
            cases.add((info["kc"] > 0, info["kp"] > 0))
            assert _rel(info["G1"], info["G1_plain"]) <= 1e-6, info["j"]
            assert _rel(info["G2"], info["G2_plain"]) <= 1e-6, info["j"]
    # all three pencil cases of §4.2 were exercised
    assert cases == {(False, True), (True, False), (True, True)}


def test_fast_grams_identity_blocks():
    """The blocks §4.4 sets from identities are the identities: C~^*C = D_c,
    Ῡ_j^*Υ_j = I, C~^*Υ_j = 0 -- read back from the fast Grams."""
    n, k, s = 120, 4, 12
    A, _, _ = deflation_matrix(n, k, seed=7, complex_=True)
    A = sp.csr_matrix(A)
    first = R.solve_dual(A, vec(n, 8, True), vec(n, 9, True), k=k, s=s, tol=1e-12,
                         max_itn=48, force_iters=48, trunc_tol=1e-2)
    res = R.solve_dual(A, vec(n, 41, True), vec(n, 42, True), U=first.basis_out.U,
                       Ut=first.basis_out.Ut, k=k, s=s, tol=1e-12, max_itn=12,
                       force_iters=12, trunc_tol=1e-2, keep_pencils=True, pencil="fast")
    info = res.pencils[0]
    kc = res.basis_in.k
    assert info["kc"] == kc and info["kp"] == 0 and kc > 0
    G1 = info["G1"]
    np.testing.assert_array_equal(np.diag(G1[:kc, :kc]).real, res.basis_in.d)
    np.testing.assert_array_equal(G1[kc:, kc:], np.eye(G1.shape[0] - kc))
    assert not G1[:kc, kc:].any() and not G1[kc:, :kc].any()


def test_fast_pencil_c4_sequence_converges_like_plain():
    cfg = _cfg("C4").scaled(10, systems=8)
    items = list(system_sequence(cfg, lam_r=0.0))
    plain = run_sequence(cfg, items)
    fast = run_sequence(cfg, items, pencil="fast")
    for a, b in zip(plain, fast):
        assert b.status == a.status
        assert abs(a.iterations - b.iterations) <= 4
        assert b.relres_true <= cfg.tol and b.relres_dual_true <= cfg.tol
        assert b.basis_in.k == a.basis_in.k and b.basis_out.k == a.basis_out.k
