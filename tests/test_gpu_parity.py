"""CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances are BASELINE.json's: per-call SpMV / projection 1e-12 relative
(norm-wise, reading Q25), iterations within max(2, 3%), solutions 1e-7
relative at matched iteration counts (Q27), true residuals <= tol, bilinear
1e-8 relative.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from synth import CONFIGS, system_sequence
from synth.small import random_sparse, deflation_matrix, vec, dense_to_csr

pytestmark = pytest.mark.gpu


def _csr(t):
    indptr, indices, data = t[:3]
    n = len(indptr) - 1
    return sp.csr_matrix((data, indices, indptr), shape=(n, n))


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1010_0762_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def iters_close(a, b):
    return abs(a - b) <= max(2, 0.03 * max(a, b))


# ------------------------------------------------------------------ per call
@pytest.mark.parametrize("cplx,n", [(False, 1000), (True, 777), (False, 33),
                                    (True, 1)])
def test_spmv_pair_parity(ctx, cplx, n):
    t = random_sparse(n, min(1.0, 8.0 / n), seed=n, complex_=cplx)
    A = _csr(t)
    M = ctx.matrix(*t)
    p, pt = vec(n, 1, cplx), vec(n, 2, cplx)
    z, zt = ctx.spmv_pair(M, p, pt)
    zr, ztr = A @ p, A.conj().T @ pt
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)
    assert np.linalg.norm(zt - ztr) <= 1e-12 * np.linalg.norm(ztr)


def test_spmv_pair_unsorted_and_empty_rows(ctx):
    n = 300
    rng = np.random.default_rng(5)
    D = np.zeros((n, n))
    for i in range(n):
        if i % 7 == 3:
            continue                      # empty row
        cols = rng.choice(n, size=rng.integers(1, 40), replace=False)
        D[i, cols] = rng.standard_normal(len(cols))
    indptr, indices, data = dense_to_csr(D)
    # shuffle column order inside each row
    for i in range(n):
        a, b = indptr[i], indptr[i + 1]
        perm = rng.permutation(b - a)
        indices[a:b] = indices[a:b][perm]
        data[a:b] = data[a:b][perm]
    M = ctx.matrix(indptr, indices, data)
    p, pt = vec(n, 3), vec(n, 4)
    z, zt = ctx.spmv_pair(M, p, pt)
    assert np.linalg.norm(z - D @ p) <= 1e-12 * np.linalg.norm(D @ p)
    assert np.linalg.norm(zt - D.T @ pt) <= 1e-12 * np.linalg.norm(D.T @ pt)


@pytest.mark.parametrize("cplx", [False, True])
def test_projection_parity(ctx, cplx):
    from oracle import rbicg as R
    n, k = 500, 6
    t = random_sparse(n, 0.02, seed=11, complex_=cplx)
    A = _csr(t)
    AH = A.conj().T.tocsr()
    U = vec(n * k, 12, cplx).reshape(n, k)
    Ut = vec(n * k, 13, cplx).reshape(n, k)
    B = R.biorthogonalize(A, AH, U, Ut, 1e-6)
    M = ctx.matrix(*t)
    rec = ctx.recycle(n, k, cplx)
    rec.import_(U, Ut)
    z, zt = vec(n, 14, cplx), vec(n, 15, cplx)
    out = ctx.project(M, rec, z, zt, 1e-6)
    assert out["k"] == B.k
    np.testing.assert_allclose(out["d"], B.d, rtol=1e-12)
    # gauge-invariant: C ζ = C D^{-1} C~^* z (Q25 / SURVEY "never column by column")
    ref = B.C @ ((B.Ct / B.d).conj().T @ z)
    got = out["C"] @ out["zeta"]
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(z) * \
        np.linalg.norm(B.C) / B.d.min()
    reft = B.Ct @ ((B.C / B.d).conj().T @ zt)
    gott = out["Ct"] @ out["zetat"]
    assert np.linalg.norm(gott - reft) <= 1e-12 * np.linalg.norm(zt) * \
        np.linalg.norm(B.Ct) / B.d.min()
    # bi-orthogonality of the device basis
    G = out["Ct"].conj().T @ out["C"]
    np.testing.assert_allclose(G, np.diag(out["d"]), atol=1e-10 * out["d"].max())


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("n,k", [(1000, 1), (1000, 3), (4099, 8), (4099, 9), (1000, 16), (4099, 17),
                                 (1000, 25), (4099, 32)])
def test_projection_parity_widths(ctx, cplx, n, k):
    """The refresh's bi-orthogonalisation Gram (norms of C, C~ and C~^*C) at every
    tile width of the fp64 tensor-core form (k_gram_cc_mma, 8-column tiles: KT = 1..4,
    k odd and even) and row counts that end in a partial 128-row stage; complex data
    runs the FFMA form.  Against the oracle's biorthogonalize:
    the singular values D_c to 1e-12 and the gauge-invariant projection C D^{-1} C~^*z."""
    from oracle import rbicg as R
    t = random_sparse(n, 6.0 / n, seed=100 + k, complex_=cplx)
    A = _csr(t)
    AH = A.conj().T.tocsr()
    U = vec(n * k, 200 + k, cplx).reshape(n, k)
    Ut = vec(n * k, 300 + k, cplx).reshape(n, k)
    B = R.biorthogonalize(A, AH, U, Ut, 1e-6)
    M = ctx.matrix(*t)
    rec = ctx.recycle(n, k, cplx)
    rec.import_(U, Ut)
    z, zt = vec(n, 14, cplx), vec(n, 15, cplx)
    out = ctx.project(M, rec, z, zt, 1e-6)
    assert out["k"] == B.k
    np.testing.assert_allclose(out["d"], B.d, rtol=1e-12)
    ref = B.C @ ((B.Ct / B.d).conj().T @ z)
    got = out["C"] @ out["zeta"]
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(z) * \
        np.linalg.norm(B.C) / B.d.min()


# ------------------------------------------------------------------ solves
def _solve_both(ctx, A, Ad, b, bt, U=None, Ut=None, **kw):
    from oracle import rbicg as R
    ref = R.solve_dual(Ad, b, bt, U=U, Ut=Ut, **kw)
    n = Ad.shape[0]
    cplx = np.iscomplexobj(b)
    rec = ctx.recycle(n, max(kw.get("k", 0), 1), cplx)
    if U is not None and U.shape[1]:
        rec.import_(U, Ut)
    x, xt, res, _ = ctx.solve_dual(A, b, bt, R=rec, **kw)
    return ref, (x, xt, res), rec


@pytest.mark.parametrize("cplx", [False, True])
def test_bicg_k0_parity(ctx, cplx):
    n = 400
    t = random_sparse(n, 0.02, seed=21, complex_=cplx)
    Ad = _csr(t)
    M = ctx.matrix(*t)
    b, bt = vec(n, 22, cplx), vec(n, 23, cplx)
    ref, (x, xt, res), _ = _solve_both(ctx, M, Ad, b, bt, k=0, s=10, tol=1e-10,
                                       max_itn=2000)
    assert res["status"] == ref.status == 0
    assert res["iterations"] == ref.iterations
    np.testing.assert_allclose(x, ref.x, rtol=0, atol=1e-9 * np.linalg.norm(ref.x))
    assert res["relres_true"] <= 1e-10 and res["relres_dual_true"] <= 1e-10


def _cosines(X, Y):
    if X.shape[1] == 0 or Y.shape[1] == 0:
        return np.zeros(0)
    Q1, _ = np.linalg.qr(X)
    Q2, _ = np.linalg.qr(Y)
    return np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False)


def _oracle_ensemble(R, Ad, item, x0, xt0, U, Ut, k, s, tol, max_itn, trunc, size=8):
    """Oracle iteration counts under rounding-level perturbations of b
    (relative 1e-15, seeded): the spread of equally correct counts (Q28)."""
    rng = np.random.default_rng(12345)
    b = item["b"]
    cnt = []
    for _ in range(size):
        bp = b * (1 + 1e-15 * rng.standard_normal(b.shape))
        r = R.solve_dual(Ad, bp, item["bt"], x0, xt0, U=U, Ut=Ut, k=k, s=s, tol=tol,
                         max_itn=max_itn, trunc_tol=trunc, update_recycle=False)
        cnt.append(r.iterations)
    return min(cnt), max(cnt)


def _forced_spread(R, Ad, item, ref, **kw):
    """Relative distance between the oracle's forced iterates and those of
    the oracle on b perturbed by relative 1e-15 (seeded): the rounding
    sensitivity of the iterates at this count (reading Q27/Q28).  On the
    BASELINE conv-diff operators BiCG's near-breakdowns amplify rounding by
    ~1e3 within 40 iterations, so the oracle's own 1-vs-8-thread runs differ
    by ~1e-6 at C3's m = s + 3."""
    rng = np.random.default_rng(4321)
    bp = item["b"] * (1 + 1e-15 * rng.standard_normal(item["b"].shape))
    alt = R.solve_dual(Ad, bp, item["bt"], **kw)
    return (np.linalg.norm(alt.x - ref.x) / np.linalg.norm(ref.x),
            np.linalg.norm(alt.xt - ref.xt) / np.linalg.norm(ref.xt))


def _residual_bound_check(Ad, item, x, xt, ref):
    """x - x_ref = A^{-1}(r_ref - r_gpu): both solutions within
    ||A^{-1}|| (||r|| + ||r_ref||) of each other (dense, small n only)."""
    A = Ad.toarray()
    nrm_inv = 1.0 / np.linalg.svd(A, compute_uv=False)[-1]
    for xs, xr, rhs, M in ((x, ref.x, item["b"], A), (xt, ref.xt, item["bt"], A.conj().T)):
        bound = nrm_inv * (np.linalg.norm(rhs - M @ xs) + np.linalg.norm(rhs - M @ xr))
        assert np.linalg.norm(xs - xr) <= 1.01 * bound + 1e-14 * np.linalg.norm(xr)


def _carry_from_oracle(ctx, cfg_k, cfg_s, tol, trunc, items, csr_of, max_itn,
                       lam_slots=False, check_space=0.0, pencil="plain"):
    """Q27 protocol: every system is solved by both sides from the ORACLE's
    input recycle space; iterations within max(2, 3%), solutions 1e-7 at
    matched counts (re-running the oracle with force_iters = m_gpu when the
    counts differ), true residuals <= tol, output spaces compared by
    principal angles."""
    from oracle import rbicg as R
    U = Ut = None
    prev = {}
    its = []
    for item in items:
        Ad = csr_of(item)
        x0, xt0 = prev.get(item.get("slot", -1), (None, None))
        ref = R.solve_dual(Ad, item["b"], item["bt"], x0, xt0, U=U, Ut=Ut,
                           k=cfg_k, s=cfg_s, tol=tol, max_itn=max_itn,
                           trunc_tol=trunc, pencil=pencil)
        cplx = np.iscomplexobj(item["b"])
        rec = ctx.recycle(Ad.shape[0], max(cfg_k, 1), cplx)
        if U is not None and U.shape[1]:
            rec.import_(U, Ut)
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], x0, xt0, R=rec,
                                       k=cfg_k, s=cfg_s, tol=tol,
                                       max_itn=max_itn, trunc_tol=trunc,
                                       pencil=pencil)
        its.append((res["iterations"], ref.iterations))
        assert res["status"] == ref.status, (res, ref.status)
        assert res["relres_true"] <= tol and res["relres_dual_true"] <= tol
        assert res["k_in"] == ref.basis_in.k
        m = res["iterations"]
        if not iters_close(m, ref.iterations):
            # DESIGN.md reading Q28: a system whose iteration count the
            # oracle itself does not reproduce under rounding-level input
            # perturbations is judged against that ensemble, and its solution
            # by the residual bound instead of at a matched count.
            lo, hi = _oracle_ensemble(R, Ad, item, x0, xt0, U, Ut, cfg_k, cfg_s, tol,
                                      max_itn, trunc)
            assert hi - lo > max(2, 0.03 * hi), (its, lo, hi)   # really chaotic
            assert lo - 2 <= m <= hi + 2, (its, lo, hi)
            if Ad.shape[0] <= 5000:   # dense ||A^{-1}|| only at small n
                _residual_bound_check(Ad, item, x, xt, ref)
        elif m != ref.iterations:
            ref_m = R.solve_dual(Ad, item["b"], item["bt"], x0, xt0, U=U, Ut=Ut,
                                 k=cfg_k, s=cfg_s, tol=tol, max_itn=max_itn,
                                 trunc_tol=trunc, force_iters=m,
                                 update_recycle=False)
            xr = ref_m.x
        else:
            xr = ref.x
        if iters_close(m, ref.iterations):
            assert np.linalg.norm(x - xr) <= 1e-7 * np.linalg.norm(xr), its
        if check_space and ref.basis_out.k:
            Ug, Utg = rec.export()
            assert Ug.shape[1] == ref.basis_out.k
            # leading k-2 directions: the trailing ones of a space still
            # converging (Table 1) are ill-determined -- their D_c entries are
            # ~1e-3 on the C4 family, so rounding-level differences in the
            # Lanczos data move them by up to ~1e-3 in cosine
            kk = max(1, ref.basis_out.k - 2)
            assert np.sort(_cosines(Ug, ref.basis_out.U))[::-1][:kk].min() >= check_space
            assert np.sort(_cosines(Utg, ref.basis_out.Ut))[::-1][:kk].min() >= check_space
        if lam_slots:
            prev[item["slot"]] = (ref.x, ref.xt)
        U, Ut = ref.basis_out.U, ref.basis_out.Ut
    return its


@pytest.mark.parametrize("cplx", [False, True])
def test_rbicg_repeated_solves(ctx, cplx):
    """P5-type repeated solves of one system (the paper's §6.1 protocol,
    PAPER.md:1321-1327) on a well-conditioned deflation matrix; recycle spaces
    must agree with the oracle's (principal angles) and iterations drop."""
    n, k = 300, 4
    A, lam, S = deflation_matrix(n, k, seed=3, complex_=cplx)
    t = dense_to_csr(A)
    b, bt = vec(n, 1, cplx), vec(n, 2, cplx)
    items = [dict(indptr=t[0], indices=t[1], data=t[2], b=b, bt=bt)] * 4
    its = _carry_from_oracle(ctx, k, 15, 1e-10, 1e-6, items, lambda it: _csr(t),
                             1000, check_space=0.999)
    assert its[-1][0] < its[0][0]


def test_rbicg_matched_iterations(ctx):
    """Q27 protocol: run both sides for exactly m iterations (stop test off)
    from the same recycle input and compare iterates."""
    from oracle import rbicg as R
    n, k = 250, 4
    A, lam, S = deflation_matrix(n, k, seed=41)
    Ad = sp.csr_matrix(A)
    M = ctx.matrix(*dense_to_csr(A))
    b, bt = vec(n, 42), vec(n, 43)
    first = R.solve_dual(Ad, b, bt, k=k, s=10, tol=1e-10, max_itn=1000,
                         trunc_tol=1e-6)
    U, Ut = first.basis_out.U, first.basis_out.Ut
    b2, bt2 = vec(n, 44), vec(n, 45)
    for m in (1, 7, 10, 23):
        ref = R.solve_dual(Ad, b2, bt2, U=U, Ut=Ut, k=k, s=10, tol=1e-10,
                           max_itn=1000, trunc_tol=1e-6, force_iters=m)
        rec = ctx.recycle(n, k)
        rec.import_(U, Ut)
        x, xt, res, h = ctx.solve_dual(M, b2, bt2, R=rec, k=k, s=10, tol=1e-10,
                                       max_itn=1000, trunc_tol=1e-6,
                                       force_iters=m, history=True)
        assert res["iterations"] == m
        assert np.linalg.norm(x - ref.x) <= 1e-9 * np.linalg.norm(ref.x)
        assert np.linalg.norm(xt - ref.xt) <= 1e-9 * np.linalg.norm(ref.xt)
        np.testing.assert_allclose(h[:, 2], np.real(ref.hist["alpha"]), rtol=1e-8)


@pytest.mark.parametrize("pencil", ["plain", "fast"])
def test_c1_sequence_parity(ctx, pencil):
    cfg = CONFIGS["C1"]
    items = list(system_sequence(cfg))
    _carry_from_oracle(ctx, cfg.k, cfg.s, cfg.tol, cfg.trunc_tol, items,
                       lambda it: _csr((it["indptr"], it["indices"], it["data"])),
                       cfg.max_itn, pencil=pencil)


@pytest.mark.parametrize("pencil", ["plain", "fast"])
def test_c4_small_complex_sequence(ctx, pencil):
    cfg = CONFIGS["C4"].scaled(12, systems=12, s=20)
    items = list(system_sequence(cfg, lam_r=0.0))
    _carry_from_oracle(ctx, cfg.k, cfg.s, cfg.tol, cfg.trunc_tol, items,
                       lambda it: _csr((it["indptr"], it["indices"], it["data"])),
                       cfg.max_itn, lam_slots=True, check_space=0.9999, pencil=pencil)


def test_c4_small_complex_sequence_wide_k(ctx):
    """A complex sequence with a wide recycle space (k = 24 > 16: the complex
    pencil's X side exceeds 64 columns -> the FFMA Gram, the U F GEMM falls back
    to the panel kernel, the C~^*C Gram runs 64-row stages) against the oracle
    under the Q27 protocol."""
    cfg = CONFIGS["C4"].scaled(10, systems=4, s=24, k=24)
    items = list(system_sequence(cfg, lam_r=0.0))
    _carry_from_oracle(ctx, cfg.k, cfg.s, cfg.tol, cfg.trunc_tol, items,
                       lambda it: _csr((it["indptr"], it["indices"], it["data"])),
                       cfg.max_itn, lam_slots=True, check_space=0.99)


@pytest.mark.parametrize("cplx", [False, True])
def test_fast_pencil_output_space(ctx, cplx):
    """§4.4 assembly (rbicg_opts.pencil = 1): the
    pencil only decides the space handed to the next system, so the
    check is on that space.  A later system run for m iterations (Q27) over
    three cycles -- the first cycle of a later system, then two general-case
    cycles whose Grams come from the recurrences -- from the oracle's input
    space: the exported U_j, Ũ_j span the oracle's (pencil="fast") to
    principal-angle cosines >= 1 - 1e-8, and the iterates are unchanged."""
    from oracle import rbicg as R
    n, k, s, m = 250, 4, 10, 30
    A, _, _ = deflation_matrix(n, k, seed=41, complex_=cplx)
    Ad = sp.csr_matrix(A)
    M = ctx.matrix(*dense_to_csr(A))
    first = R.solve_dual(Ad, vec(n, 42, cplx), vec(n, 43, cplx), k=k, s=s, tol=1e-10,
                         max_itn=1000, trunc_tol=1e-2)
    U, Ut = first.basis_out.U, first.basis_out.Ut
    assert U.shape[1] >= 2
    b2, bt2 = vec(n, 44, cplx), vec(n, 45, cplx)
    ref = R.solve_dual(Ad, b2, bt2, U=U, Ut=Ut, k=k, s=s, tol=1e-10, max_itn=1000,
                       trunc_tol=1e-2, force_iters=m, pencil="fast", keep_pencils=True)
    assert [(i["kc"] > 0, i["kp"] > 0) for i in ref.pencils][:2] == [(True, False), (True, True)]
    rec = ctx.recycle(n, k, cplx)
    rec.import_(U, Ut)
    x, xt, res, _ = ctx.solve_dual(M, b2, bt2, R=rec, k=k, s=s, tol=1e-10, max_itn=1000,
                                   trunc_tol=1e-2, force_iters=m, pencil="fast")
    assert res["iterations"] == m and res["cycles"] == m // s
    assert np.linalg.norm(x - ref.x) <= 1e-9 * np.linalg.norm(ref.x)
    Ug, Utg = rec.export()
    assert Ug.shape[1] == ref.basis_out.k > 0
    assert _cosines(Ug, ref.basis_out.U).min() >= 1 - 1e-8
    assert _cosines(Utg, ref.basis_out.Ut).min() >= 1 - 1e-8


def test_gpu_own_chain_c4(ctx):
    """The GPU carries its own recycle space through a C4-like sequence (no
    oracle input); per-system iterations still track the oracle's chain."""
    from oracle.sequence import run_sequence
    cfg = CONFIGS["C4"].scaled(12, systems=8, s=20)
    items = list(system_sequence(cfg, lam_r=0.0))
    ref = run_sequence(cfg, items)
    rec = ctx.recycle(cfg.n, cfg.k, True)
    prev = {}
    its = []
    for item, r in zip(items, ref):
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x0, xt0 = prev.get(item["slot"], (None, None))
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], x0, xt0, R=rec,
                                       k=cfg.k, s=cfg.s, tol=cfg.tol,
                                       max_itn=cfg.max_itn,
                                       trunc_tol=cfg.trunc_tol)
        prev[item["slot"]] = (x, xt)
        its.append(res["iterations"])
        assert res["relres_true"] <= cfg.tol and res["relres_dual_true"] <= cfg.tol
    # Q28 for a chain (tests/chain_ensemble.py)
    from chain_ensemble import oracle_chain_counts, within_ensemble
    ok, info = within_ensemble(its, oracle_chain_counts(cfg, items))
    assert ok, info


def test_bilinear_parity(ctx):
    from oracle import rbicg as R
    n = 300
    t = random_sparse(n, 0.02, seed=51, complex_=True)
    Ad = _csr(t)
    M = ctx.matrix(*t)
    u, w = vec(n, 52, True), vec(n, 53, True)
    val_o, _ = R.bilinear(Ad, u, w, k=4, s=10, tol=1e-10, max_itn=1000)
    val_g, res = ctx.bilinear(M, u, w, k=4, s=10, tol=1e-10, max_itn=1000)
    assert abs(val_g - val_o) <= 1e-8 * abs(val_o)
    exact = np.vdot(u, np.linalg.solve(Ad.toarray(), w))
    assert abs(val_g - exact) <= 1e-8 * abs(exact)


def test_deterministic(ctx):
    n = 2000
    t = random_sparse(n, 0.003, seed=61)
    M = ctx.matrix(*t)
    b, bt = vec(n, 62), vec(n, 63)
    outs = []
    for _ in range(2):
        rec = ctx.recycle(n, 4)
        x, xt, res, _ = ctx.solve_dual(M, b, bt, R=rec, k=4, s=10, tol=1e-10,
                                       max_itn=3000)
        x2, _, res2, _ = ctx.solve_dual(M, b, bt, R=rec, k=4, s=10, tol=1e-10,
                                        max_itn=3000)
        outs.append((x.copy(), x2.copy(), res["iterations"], res2["iterations"]))
    assert outs[0][2:] == outs[1][2:]
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_edge_cases(ctx):
    # identity: one iteration
    n = 64
    t = dense_to_csr(np.eye(n))
    M = ctx.matrix(*t)
    b = np.ones(n)
    x, xt, res, _ = ctx.solve_dual(M, b, b, k=0, s=4, tol=1e-12, max_itn=10)
    assert res["iterations"] == 1 and np.allclose(x, 1.0, rtol=1e-15)
    # max_itn = 0 and an exact initial guess
    x, xt, res, _ = ctx.solve_dual(M, b, b, b.copy(), b.copy(), k=0, s=4,
                                   tol=1e-12, max_itn=0)
    assert res["iterations"] == 0 and res["status"] == 0
    # orthogonal initial residuals -> step-3 redraw
    e1, e2 = np.zeros(n), np.zeros(n)
    e1[0], e2[1] = 1.0, 1.0
    x, xt, res, _ = ctx.solve_dual(M, e1, e2, k=0, s=4, tol=1e-12, max_itn=10)
    assert res["status"] == 2
    x, xt, res, _ = ctx.solve_dual(M, e1, e2, k=0, s=4, tol=1e-12, max_itn=10,
                                   xt_redraw=vec(n, 7))
    assert res["status"] == 0


# ------------------------------------------------------------------ full size
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_spmv_pair(ctx, name):
    """BASELINE sizes (C2: n = 1,048,576; C3: n = 7,077,888; C4: n = 10^6
    complex; C5: n = 56,623,104, nnz = 395,476,992): the SpMV pair of the
    device SELL store vs scipy, 1e-12 norm-wise."""
    cfg = CONFIGS[name]
    if name == "C5":
        import psutil
        if psutil.virtual_memory().available < 24 * 2**30:
            pytest.skip("C5 host-side reference needs ~12 GB of host memory (+ margin)")
    it = next(system_sequence(cfg, systems=[0], lam_r=0.0) if cfg.kind == "irka"
              else system_sequence(cfg, systems=[0]))
    A = _csr((it["indptr"], it["indices"], it["data"]))
    M = ctx.matrix(it["indptr"], it["indices"], it["data"])
    p, pt = it["b"], it["bt"]
    z, zt = ctx.spmv_pair(M, p, pt)
    zr, ztr = A @ p, A.conj().T @ pt
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)
    assert np.linalg.norm(zt - ztr) <= 1e-12 * np.linalg.norm(ztr)
    M.free()


def test_full_size_c2_matched_iterations(ctx):
    """C2 system 0 at full size in the bench configuration: both sides run
    exactly 2s + 3 iterations (two cycle ends, Q27 force_iters), then
    compare iterates, the recycle space they build, and the recursive vs
    true residual relation; then the next system from that space."""
    from oracle import rbicg as R
    cfg = CONFIGS["C2"]
    items = list(system_sequence(cfg, systems=[0, 1]))
    m = 2 * cfg.s + 3
    rec = ctx.recycle(cfg.n, cfg.k)
    U = Ut = None
    for item in items:
        A = _csr((item["indptr"], item["indices"], item["data"]))
        ref = R.solve_dual(A, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                           tol=cfg.tol, max_itn=m, trunc_tol=cfg.trunc_tol,
                           force_iters=m)
        if U is not None and U.shape[1]:
            rec.import_(U, Ut)
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k,
                                       s=cfg.s, tol=cfg.tol, max_itn=m,
                                       trunc_tol=cfg.trunc_tol, force_iters=m,
                                       history=True)
        assert res["iterations"] == m and res["cycles"] == ref.cycles == 2
        sp_x, sp_xt = _forced_spread(R, A, item, ref, U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                                     tol=cfg.tol, max_itn=m, trunc_tol=cfg.trunc_tol,
                                     force_iters=m)
        assert np.linalg.norm(x - ref.x) <= max(1e-7, 10 * sp_x) * np.linalg.norm(ref.x)
        assert np.linalg.norm(xt - ref.xt) <= max(1e-7, 10 * sp_xt) * np.linalg.norm(ref.xt)
        np.testing.assert_allclose(h[:, 0], np.array(ref.hist["rnorm"][1:]) /
                                   np.linalg.norm(item["b"]), rtol=max(1e-6, 20 * sp_x))
        assert res["k_out"] == ref.basis_out.k
        U, Ut = ref.basis_out.U, ref.basis_out.Ut
        M.free()


def test_full_size_c3_matched_iterations(ctx):
    """C3 system 0 (n = 7,077,888, 3-D) at full size: s + 3 iterations with
    one cycle end, iterates and residual histories vs the oracle."""
    from oracle import rbicg as R
    cfg = CONFIGS["C3"]
    item = next(system_sequence(cfg, systems=[0]))
    m = cfg.s + 3
    A = _csr((item["indptr"], item["indices"], item["data"]))
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol,
                       max_itn=m, trunc_tol=cfg.trunc_tol, force_iters=m)
    rec = ctx.recycle(cfg.n, cfg.k)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k,
                                   s=cfg.s, tol=cfg.tol, max_itn=m,
                                   trunc_tol=cfg.trunc_tol, force_iters=m,
                                   history=True)
    assert res["iterations"] == m and res["cycles"] == ref.cycles == 1
    sp_x, sp_xt = _forced_spread(R, A, item, ref, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                 max_itn=m, trunc_tol=cfg.trunc_tol, force_iters=m)
    assert np.linalg.norm(x - ref.x) <= max(1e-7, 10 * sp_x) * np.linalg.norm(ref.x)
    assert np.linalg.norm(xt - ref.xt) <= max(1e-7, 10 * sp_xt) * np.linalg.norm(ref.xt)
    np.testing.assert_allclose(h[:, 0], np.array(ref.hist["rnorm"][1:]) /
                               np.linalg.norm(item["b"]), rtol=max(1e-6, 20 * sp_x))
    assert res["k_out"] == ref.basis_out.k
    M.free()


def test_c5_family_k20_sequence(ctx):
    """C5's solver parameters (k = 20, s = 50: the widest recycle space of the
    five configs, cycle-end GEMMs wider than one 32-column launch) on the C5
    operator family at 24^3, three systems in sequence (Q27 protocol)."""
    cfg = CONFIGS["C5"].scaled(24, systems=3)
    items = list(system_sequence(cfg))
    its = _carry_from_oracle(ctx, cfg.k, cfg.s, cfg.tol, cfg.trunc_tol, items,
                             lambda it: _csr((it["indptr"], it["indices"], it["data"])),
                             cfg.max_itn, check_space=0.99)
    assert len(its) == 3


def _c5_host_ok(extra_gb):
    import psutil
    return psutil.virtual_memory().available >= extra_gb * 2**30


def test_full_size_c5_matched_iterations(ctx):
    """C5 system 0 at full size (n = 56,623,104, nnz = 395,476,992, k = 20,
    s = 50) on ONE GPU: 12 forced iterations vs the oracle (iterates 1e-7,
    residual histories 1e-6)."""
    from oracle import rbicg as R
    if not _c5_host_ok(48):
        pytest.skip("the C5 oracle run needs ~40 GB of host memory")
    cfg = CONFIGS["C5"]
    item = next(system_sequence(cfg, systems=[0]))
    m = 12
    A = _csr((item["indptr"], item["indices"], item["data"]))
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol,
                       max_itn=m, trunc_tol=cfg.trunc_tol, force_iters=m)
    rec = ctx.recycle(cfg.n, cfg.k)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k,
                                   s=cfg.s, tol=cfg.tol, max_itn=m,
                                   trunc_tol=cfg.trunc_tol, force_iters=m,
                                   history=True)
    assert res["iterations"] == m
    assert np.linalg.norm(x - ref.x) <= 1e-7 * np.linalg.norm(ref.x)
    assert np.linalg.norm(xt - ref.xt) <= 1e-7 * np.linalg.norm(ref.xt)
    np.testing.assert_allclose(h[:, 0], np.array(ref.hist["rnorm"][1:]) /
                               np.linalg.norm(item["b"]), rtol=1e-6)
    M.free()


def test_full_size_c5_sequence_converges(ctx):
    """C5 systems 0 and 1 at full size on ONE GPU, the GPU's own recycle
    chain: both converge (status 0 or recycle_empty, P:702 footnote) and the
    true residuals recomputed on the host with scipy are <= tol = 1e-8."""
    if not _c5_host_ok(24):
        pytest.skip("host-side residuals need ~16 GB of host memory")
    cfg = CONFIGS["C5"]
    rec = ctx.recycle(cfg.n, cfg.k)
    for item in system_sequence(cfg, systems=[0, 1]):
        A = _csr((item["indptr"], item["indices"], item["data"]))
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k,
                                       s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn,
                                       trunc_tol=cfg.trunc_tol)
        M.free()
        assert res["status_name"] in ("ok", "recycle_empty"), res
        for rhs, op, v in ((item["b"], A, x), (item["bt"], A.conj().T, xt)):
            assert np.linalg.norm(rhs - op @ v) <= cfg.tol * np.linalg.norm(rhs)


def test_full_size_c4_bilinear_conjugate_pair(ctx):
    """C4 operator at 100^3 (complex128, n = 1,000,000), the first conjugate
    shift pair (slots 0, 1; λ_R taken as 0 -- the shifts stay right of the
    spectrum): converged solves to tol, G(σ) = c^*A^{-1}b within
    1e-8 of the oracle, and G(σ̄) = conj G(σ) (P11)."""
    from oracle import rbicg as R
    cfg = CONFIGS["C4"]
    items = list(system_sequence(cfg, systems=[0, 1], lam_r=0.0))
    vals = []
    for item in items:
        A = _csr((item["indptr"], item["indices"], item["data"]))
        val_o, ref = R.bilinear(A, item["bt"], item["b"], k=0, s=cfg.s,
                                tol=cfg.tol, max_itn=cfg.max_itn)
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        val_g, res = ctx.bilinear(M, item["bt"], item["b"], k=0, s=cfg.s,
                                  tol=cfg.tol, max_itn=cfg.max_itn)
        assert res["status"] == 0
        assert iters_close(res["iterations"], ref.iterations)
        assert abs(val_g - val_o) <= 1e-8 * abs(val_o)
        vals.append(val_g)
        M.free()
    assert abs(vals[1] - np.conj(vals[0])) <= 1e-8 * abs(vals[0])


@pytest.mark.parametrize("strategy,reuse_tol", [(1, np.inf), (2, np.inf), (3, 0.5)])
def test_irka_gpu_matches_oracle(ctx, strategy, reuse_tol):
    """NEXT-3: IRKA (Algorithm 3) with the dual solves on the GPU vs the IRKA
    oracle on a stable conv-diff model: same number of IRKA steps, shift
    trajectories to 1e-6, the same per-solve iterations (max(2, 3%)), and the
    GPU's reduced model Hermite-interpolates G at its final shifts
    (Theorem 3.1, dense check); recycling strategies 1, 2 and 3
    (PAPER.md:1196-1235)."""
    from oracle import irka as OI
    from paper_1010_0762_b200 import irka as GI
    from synth.convdiff import convdiff_csr
    indptr, indices, data = convdiff_csr(8, 2, (10.0, 10.0), "central")[:3]
    n = 64
    A = -sp.csr_matrix((data, indices, indptr), shape=(n, n))
    A.sort_indices()
    b, c = vec(n, 81, dist="normal"), vec(n, 82, dist="normal")
    kw = dict(k=4, s=10, tol=1e-12, shift_tol=1e-8, max_steps=40, strategy=strategy,
              reuse_tol=reuse_tol)
    ref = OI.irka(A, b, c, [0.05, 0.4, 2.0], **kw)
    got = GI.irka(ctx, A.indptr, A.indices, A.data, b, c, [0.05, 0.4, 2.0], **kw)
    assert ref.converged and got.converged and got.steps == ref.steps
    for sg, so in zip(got.history, ref.history):
        np.testing.assert_allclose(sg, so, rtol=1e-6)
    # per-solve counts: each slot carries its own recycle chain across the
    # IRKA steps, so the counts are judged against IRKA oracle runs with b
    # perturbed by relative 1e-15 (Q28 for a chain, tests/chain_ensemble.py)
    rng = np.random.default_rng(91)
    ens = [ref.iterations]
    for _ in range(5):
        bp = b * (1 + 1e-15 * rng.standard_normal(n))
        alt = OI.irka(A, bp, c, [0.05, 0.4, 2.0], **kw)
        if alt.steps == ref.steps:
            ens.append(alt.iterations)
    for step, ig in enumerate(got.iterations):
        for slot, m in enumerate(ig):
            col = [e[step][slot] for e in ens]
            lo, hi = min(col), max(col)
            assert lo - max(2, 0.03 * lo) <= m <= hi + max(2, 0.03 * hi), (step, slot, m, col)
    Ad = A.toarray()
    for si in got.shifts:
        M = si * np.eye(n) - Ad
        y = np.linalg.solve(M, b)
        g, dg = np.vdot(c, y), -np.vdot(c, np.linalg.solve(M, y))
        gr, dgr = OI.transfer(got.Ar, got.Er, got.br, got.cr, si)
        assert abs(gr - g) <= 1e-8 * abs(g) and abs(dgr - dg) <= 1e-6 * abs(dg)


@pytest.mark.parametrize("env", ["RBICG_NO_SHARED_COLS", "RBICG_NO_SYM_T", "RBICG_NO_DCOLS"])
def test_shared_column_array_bitwise(ctx, monkeypatch, env):
    """A structurally symmetric A (the conv-diff stencils) keeps one SELL
    column array for A and A^* (matrix.cu share_cols) and gets A^*'s values
    by the search-based transpose (k_sym_transpose), and the fused kernel
    streams int16 column deltas: the solve must be bitwise identical to the
    one with two column arrays / the sorted transpose / int32 columns."""
    cfg = CONFIGS["C3"].scaled(20, systems=1)
    item = next(system_sequence(cfg))
    outs = []
    for off in (False, True):
        if off:
            monkeypatch.setenv(env, "1")
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        kt = ctx.time_kernels(M, None, k=0, s=cfg.s, iters=3)
        assert kt["shared_cols"] == (not off or env != "RBICG_NO_SHARED_COLS")
        if env == "RBICG_NO_DCOLS":
            assert kt["dcols"] == (not off)
        rec = ctx.recycle(cfg.n, cfg.k)
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s,
                                       tol=cfg.tol, max_itn=cfg.max_itn,
                                       trunc_tol=cfg.trunc_tol)
        outs.append((x, xt, res["iterations"]))
        M.free()
    assert outs[0][2] == outs[1][2]
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


# ------------------------------------------------------------------ fused iteration
@pytest.mark.parametrize("name,N", [("C1", 0), ("C3", 20), ("C4", 10), ("C5", 16)])
def test_fused_iteration_matches_lookahead_oracle(ctx, name, N):
    """First systems (no recycle space) run the fused one-kernel iteration
    (DESIGN §6): against the oracle's "lookahead" variant -- the same
    arithmetic -- iterations within max(2, 3 %) and the same status (the same
    count, recycle width and residual history (1e-5) when they agree),
    solutions at matched counts to 1e-8."""
    from oracle import rbicg as R
    cfg = CONFIGS[name].scaled(N, systems=1) if N else CONFIGS[name]
    item = next(system_sequence(cfg, **({"lam_r": 0.0} if cfg.kind == "irka" else {})))
    A = _csr((item["indptr"], item["indices"], item["data"]))
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    kt = ctx.time_kernels(M, None, k=0, s=cfg.s, iters=3)
    assert kt["fused_ms"] > 0 and kt["fused_done_flag"] == 0
    rec = ctx.recycle(cfg.n, cfg.k, cfg.complex)
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s,
                                   tol=cfg.tol, max_itn=cfg.max_itn,
                                   trunc_tol=cfg.trunc_tol, history=True)
    M.free()
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol,
                       max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, variant="lookahead")
    m = res["iterations"]
    assert iters_close(m, ref.iterations) and res["status"] == ref.status, (m, ref.iterations)
    if m != ref.iterations:   # Q27: the oracle at the GPU's count
        ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol,
                           max_itn=m, trunc_tol=cfg.trunc_tol, force_iters=m,
                           variant="lookahead")
    else:
        assert res["k_out"] == ref.basis_out.k
        np.testing.assert_allclose(h[:, 0], np.array(ref.hist["rnorm"][1:]) /
                                   np.linalg.norm(item["b"]), rtol=1e-5, atol=1e-11)
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    assert np.linalg.norm(xt - ref.xt) <= 1e-8 * np.linalg.norm(ref.xt)
    assert res["relres_true"] <= cfg.tol and res["relres_dual_true"] <= cfg.tol


def test_fused_and_two_kernel_forms_agree(ctx, monkeypatch):
    """The fused iteration vs the two-kernel iteration (RBICG_FUSED=0) on a
    3-D conv-diff system: the same iteration count and solutions to 1e-8
    (they differ only in how β_i's ρ_i is formed), and the fused
    form also at the bench configuration's cycle length with forced
    iterations across two cycle ends (Q27) against the lookahead oracle."""
    from oracle import rbicg as R
    cfg = CONFIGS["C3"].scaled(24, systems=1)
    item = next(system_sequence(cfg))
    outs = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("RBICG_FUSED", "0")
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        rec = ctx.recycle(cfg.n, cfg.k)
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s,
                                       tol=cfg.tol, max_itn=cfg.max_itn,
                                       trunc_tol=cfg.trunc_tol)
        outs.append((x, xt, res["iterations"]))
        M.free()
    assert outs[0][2] == outs[1][2]
    assert np.linalg.norm(outs[0][0] - outs[1][0]) <= 1e-8 * np.linalg.norm(outs[1][0])
    monkeypatch.delenv("RBICG_FUSED")
    m = 2 * cfg.s + 3
    A = _csr((item["indptr"], item["indices"], item["data"]))
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=m,
                       trunc_tol=cfg.trunc_tol, force_iters=m, variant="lookahead")
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    rec = ctx.recycle(cfg.n, cfg.k)
    x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s,
                                   tol=cfg.tol, max_itn=m, trunc_tol=cfg.trunc_tol,
                                   force_iters=m)
    M.free()
    assert res["iterations"] == m and res["cycles"] == ref.cycles == 2
    assert np.linalg.norm(x - ref.x) <= 1e-9 * np.linalg.norm(ref.x)
    assert res["k_out"] == ref.basis_out.k


# ------------------------------------------------------------------ full size, k > 0
def _seeded_space(cfg, k, seed_off=777):
    rng = np.random.default_rng(cfg.seed + seed_off)
    shp = (cfg.n, k)
    if cfg.complex:
        return (rng.standard_normal(shp) + 1j * rng.standard_normal(shp),
                rng.standard_normal(shp) + 1j * rng.standard_normal(shp))
    return rng.standard_normal(shp), rng.standard_normal(shp)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_full_size_projection_parity(ctx, name):
    """Per-call projection parity at BASELINE size with a live recycle space
    (Q25, 1e-12): the device refresh of a seeded k-column space for system 1
    (C = AU, C~ = A^*Ũ, unit columns, SVD, truncation at the paper's 1e-6,
    P:690-705) and ζ = D_c^{-1}C~^*z, ζ~ = D_c^{-1}C^*z~ against the oracle
    on the gauge-invariant C ζ; D_c to 1e-12; the device basis bi-orthogonal."""
    from oracle import rbicg as R
    cfg = CONFIGS[name]
    item = next(system_sequence(cfg, systems=[1]))
    A = _csr((item["indptr"], item["indices"], item["data"]))
    U, Ut = _seeded_space(cfg, cfg.k)
    B = R.biorthogonalize(A, R.adjoint(A), U, Ut, cfg.trunc_tol)
    assert B.k > 0
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    rec = ctx.recycle(cfg.n, cfg.k)
    rec.import_(U, Ut)
    z, zt = item["b"], item["bt"]
    out = ctx.project(M, rec, z, zt, cfg.trunc_tol)
    assert out["k"] == B.k
    np.testing.assert_allclose(out["d"], B.d, rtol=1e-12)
    ref = B.C @ ((B.Ct / B.d).conj().T @ z)
    got = out["C"] @ out["zeta"]
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(z) * \
        np.linalg.norm(B.C) / B.d.min()
    reft = B.Ct @ ((B.C / B.d).conj().T @ zt)
    gott = out["Ct"] @ out["zetat"]
    assert np.linalg.norm(gott - reft) <= 1e-12 * np.linalg.norm(zt) * \
        np.linalg.norm(B.Ct) / B.d.min()
    G = out["Ct"].conj().T @ out["C"]
    np.testing.assert_allclose(G, np.diag(out["d"]), atol=1e-10 * out["d"].max())
    M.free()


def _robust_prefix(ref_hist, alt_hist, rel=1e-8):
    """Length of the leading stretch where the oracle and the oracle on
    1e-15-perturbed b agree to `rel` (before BiCG's rounding amplification,
    Q27/Q28, makes the histories differ)."""
    a, b = np.abs(np.asarray(ref_hist)), np.asarray(alt_hist)
    dev = np.abs(np.asarray(ref_hist) - b) > rel * np.maximum(a, 1e-300)
    return int(np.argmax(dev)) if dev.any() else len(a)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_full_size_k_matched_iterations(ctx, name):
    """Algorithm 2 with the projections active at BASELINE size:
    system 1 from a recycle space -- C3: the oracle's own, built by its cycle
    end after s + 3 iterations of system 0 (harmonic Ritz vectors of T_1,
    P:614-628); C2: a seeded k-column space (C2's own spaces are truncated to
    p = 0) -- both sides forced to m = s + 3 iterations (Q27)
    across one cycle end of the "later system, cycle 1" case.
    The α and ‖r‖ histories agree to 1e-6 over the stretch where the oracle
    agrees with itself under a 1e-15 perturbation of b (BiCG's rounding
    amplification, Q28) and that stretch is >= 3 iterations; x, x~ agree to
    1e-7 or 10x the oracle's own spread; k_in equal, k_out within one
    (borderline σ at the 1e-6 cut); leading output directions agree."""
    from oracle import rbicg as R
    cfg = CONFIGS[name]
    items = list(system_sequence(cfg, systems=[0, 1]))
    m = cfg.s + 3
    if name == "C3":
        A0 = _csr((items[0]["indptr"], items[0]["indices"], items[0]["data"]))
        first = R.solve_dual(A0, items[0]["b"], items[0]["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol,
                             max_itn=m, trunc_tol=cfg.trunc_tol, force_iters=m)
        U, Ut = first.basis_out.U, first.basis_out.Ut
        del A0, first
    else:
        U, Ut = _seeded_space(cfg, cfg.k)
    item = items[1]
    A = _csr((item["indptr"], item["indices"], item["data"]))
    kw = dict(U=U, Ut=Ut, k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=m,
              trunc_tol=cfg.trunc_tol, force_iters=m)
    ref = R.solve_dual(A, item["b"], item["bt"], **kw)
    assert ref.basis_in.k > 0 and ref.cycles == 1
    rng = np.random.default_rng(4321)
    alt = R.solve_dual(A, item["b"] * (1 + 1e-15 * rng.standard_normal(cfg.n)), item["bt"], **kw)
    sp_x = np.linalg.norm(alt.x - ref.x) / np.linalg.norm(ref.x)
    sp_xt = np.linalg.norm(alt.xt - ref.xt) / np.linalg.norm(ref.xt)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    rec = ctx.recycle(cfg.n, cfg.k)
    rec.import_(U, Ut)
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s,
                                   tol=cfg.tol, max_itn=m, trunc_tol=cfg.trunc_tol,
                                   force_iters=m, history=True)
    assert res["iterations"] == m and res["cycles"] == 1
    assert res["k_in"] == ref.basis_in.k and abs(res["k_out"] - ref.basis_out.k) <= 1
    assert np.linalg.norm(x - ref.x) <= max(1e-7, 10 * sp_x) * np.linalg.norm(ref.x)
    assert np.linalg.norm(xt - ref.xt) <= max(1e-7, 10 * sp_xt) * np.linalg.norm(ref.xt)
    # the stretch where a 1e-15 perturbation moves the oracle's α by < 1e-10:
    # beyond it the ~1e-16 differences of the device's reduction order, which
    # the near-singular projections (D_c down to 1e-6) amplify more than a
    # perturbation of b, have grown past 1e-6
    na = _robust_prefix(np.real(ref.hist["alpha"]), np.real(alt.hist["alpha"]), rel=1e-10)
    assert na >= 3, na
    np.testing.assert_allclose(h[:na, 2], np.real(ref.hist["alpha"])[:na], rtol=1e-6)
    rn = np.array(ref.hist["rnorm"][1:]) / np.linalg.norm(item["b"])
    np.testing.assert_allclose(h[:na, 0], rn[:na], rtol=1e-6)
    kk = min(res["k_out"], ref.basis_out.k) - 2
    if kk > 0:
        Ug, Utg = rec.export()
        assert np.sort(_cosines(Ug, ref.basis_out.U))[::-1][:kk].min() >= 0.99
        assert np.sort(_cosines(Utg, ref.basis_out.Ut))[::-1][:kk].min() >= 0.99
    M.free()


def test_full_size_c4_sweep(ctx):
    """One full IRKA-like sweep of C4 at BASELINE size (n = 10^6 complex,
    k = 8, s = 40, the paper's truncation 1e-6): six shifted dual systems,
    each solved by both sides from the oracle's input recycle space (Q27
    protocol: iterations max(2, 3 %) or the Q28 ensemble, solutions 1e-7 at
    matched counts, true residuals <= tol, same k_in).  Shifts placed right of
    0 (lam_r = 0) instead of the ARPACK estimate of max Re λ(K) (~50 s of
    host time), the same on both sides."""
    cfg = CONFIGS["C4"].scaled(100, systems=6)
    items = list(system_sequence(cfg, lam_r=0.0))
    its = _carry_from_oracle(ctx, cfg.k, cfg.s, cfg.tol, cfg.trunc_tol, items,
                             lambda it: _csr((it["indptr"], it["indices"], it["data"])),
                             cfg.max_itn, lam_slots=True)
    assert len(its) == 6


def test_full_size_c2_fused_count_vs_algorithm2(ctx):
    """The default k = 0 iteration (one kernel per iteration, β from the
    one-step expansion of ρ) against Algorithm 2 AS WRITTEN
    (oracle variant="standard") on C2 system 0 at full size
    (n = 1,048,576, ~3,300 iterations): iteration counts within BASELINE's
    max(2, 3 %), both converged, true residuals <= tol.  (Measured here:
    oracle 3,352; look-ahead oracle 3,339; GPU 3,313.)"""
    from oracle import rbicg as R
    cfg = CONFIGS["C2"]
    item = next(system_sequence(cfg, systems=[0]))
    A = _csr((item["indptr"], item["indices"], item["data"]))
    ref = R.solve_dual(A, item["b"], item["bt"], k=0, s=cfg.s, tol=cfg.tol,
                       max_itn=cfg.max_itn, variant="standard")
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], k=0, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn)
    assert ref.status == 0 and res["status"] == 0
    assert iters_close(res["iterations"], ref.iterations), (res["iterations"], ref.iterations)
    assert res["relres_true"] <= cfg.tol and res["relres_dual_true"] <= cfg.tol
    M.free()


@pytest.mark.parametrize("cplx", [False, True])
def test_fusedk_matches_lookahead_oracle(ctx, monkeypatch, cplx):
    """The opt-in fused iteration with a recycle space (k_fusedk,
    RBICG_FUSEDK_MAXK): one kernel per iteration with the neighbours' Cγ
    term through A C, eager x and β from the expansion of ρ_i including the
    Q32 terms -- the oracle's variant="lookahead" with projections.  A
    recycled problem (deflation matrix, k = 4 from a first solve) forced to
    m iterations across cycle ends: iterates and α to 1e-8; then the full
    solve converges with the standard oracle's count (max(2, 3 %))."""
    from oracle import rbicg as R
    monkeypatch.setenv("RBICG_FUSEDK_MAXK", "8")
    n, k = 250, 4
    A, _, _ = deflation_matrix(n, k, seed=41, complex_=cplx)
    Ad = sp.csr_matrix(A)
    M = ctx.matrix(*dense_to_csr(A))
    first = R.solve_dual(Ad, vec(n, 42, cplx), vec(n, 43, cplx), k=k, s=10, tol=1e-10,
                         max_itn=1000, trunc_tol=1e-6)
    U, Ut = first.basis_out.U, first.basis_out.Ut
    b2, bt2 = vec(n, 44, cplx), vec(n, 45, cplx)
    for m in (7, 23):
        ref = R.solve_dual(Ad, b2, bt2, U=U, Ut=Ut, k=k, s=10, tol=1e-10, max_itn=1000,
                           trunc_tol=1e-6, force_iters=m, variant="lookahead")
        rec = ctx.recycle(n, k, cplx)
        rec.import_(U, Ut)
        x, xt, res, h = ctx.solve_dual(M, b2, bt2, R=rec, k=k, s=10, tol=1e-10, max_itn=1000,
                                       trunc_tol=1e-6, force_iters=m, history=True)
        assert res["iterations"] == m and res["k_in"] == ref.basis_in.k > 0
        assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
        assert np.linalg.norm(xt - ref.xt) <= 1e-8 * np.linalg.norm(ref.xt)
        np.testing.assert_allclose(h[:, 2], np.real(ref.hist["alpha"]), rtol=1e-8)
    std = R.solve_dual(Ad, b2, bt2, U=U, Ut=Ut, k=k, s=10, tol=1e-10, max_itn=1000, trunc_tol=1e-6)
    rec = ctx.recycle(n, k, cplx)
    rec.import_(U, Ut)
    x, xt, res, _ = ctx.solve_dual(M, b2, bt2, R=rec, k=k, s=10, tol=1e-10, max_itn=1000,
                                   trunc_tol=1e-6)
    assert res["status"] == 0 and iters_close(res["iterations"], std.iterations)
    assert res["relres_true"] <= 1e-10 and res["relres_dual_true"] <= 1e-10
