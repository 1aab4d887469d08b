"""Recycling BiCG (Algorithm 2 + §4) -- test-infrastructure oracle.

Plain fp64 / complex128, step by step in the paper's order and notation.
Every function cites the passage it follows; the readings Qn are those of
SURVEY.md §8(c), restated in DESIGN.md §3.

R1 refresh / R6 bi-orthogonalisation   PAPER.md:687-705  (+Q13)
R2 initial projection (minusXR)         PAPER.md:418-426, :449-452 (+Q4, Q5)
R3 loop                                 PAPER.md:453-473 (+Q1, Q2, Q3, Q23)
R4 Lanczos data (T from scalars, Υ, Γ)
R5 pencil (finalGenEigValue), cases     PAPER.md:552-684 (+Q11, Q12, Q15)
R7 step 7 and true residuals            PAPER.md:476-477 (+Q2, Q18)
bilinear form u^*A^{-1}w                PAPER.md:63-67 (+Q19)

The pencil is assembled with plain explicit products (Q15): B_j = Ĉ^*AV_j is
formed by explicit sparse products of the stored Lanczos vectors, and
P = H~^*(Ψ~^*Ψ)H, Q = H~^*(Ψ~^*Φ) by dense products.  ``pencil="fast"``
 takes Ψ~^*Ψ and Ψ~^*Φ from the §4.4 recurrences instead
(fast_grams): the paper's exact-arithmetic identities, so
the two agree while the Lanczos vectors stay bi-orthogonal (pinned against
the plain products in tests/test_oracle_fast_pencil.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from .bicg import (inner, breakdown, OK, MAXITER, BREAKDOWN_SERIOUS,
                   BREAKDOWN_SECOND, BREAKDOWN_EPS)

RECYCLE_EMPTY = 4
STATUS_NAMES = {OK: "ok", MAXITER: "maxiter", BREAKDOWN_SERIOUS: "breakdown_serious",
                BREAKDOWN_SECOND: "breakdown_second", RECYCLE_EMPTY: "recycle_empty"}


@dataclass
class Basis:
    """Recycle basis (U, Ũ, C = AU, C~ = A^*Ũ, D_c = C~^*C diagonal)."""
    U: np.ndarray
    Ut: np.ndarray
    C: np.ndarray
    Ct: np.ndarray
    d: np.ndarray          # real positive diagonal of D_c

    @property
    def k(self):
        return self.U.shape[1]


def empty_basis(n, dtype):
    z = np.zeros((n, 0), dtype=dtype)
    return Basis(z, z.copy(), z.copy(), z.copy(), np.zeros(0))


def adjoint(A):
    """Explicit conjugate transpose A^* (BASELINE.json (1)); an operator
    (oracle.precond.SplitOperator, NEXT-4) supplies its own adjoint."""
    if hasattr(A, "adjoint_op"):
        return A.adjoint_op()
    return A.conj().T.tocsr()


# ----------------------------------------------------------------------------
# R1 / R6: bi-orthogonal C, C~, truncation reading Q13
# ----------------------------------------------------------------------------
def biorthogonalize(A, AH, U, Ut, trunc_tol, return_maps=False):
    """C = AU, C~ = A^*Ũ; scale column pairs to unit norm (Q13); SVD
    C~^*C = M Σ N^* (equationSVD); keep σ_i >= trunc_tol (absolute);
    U <- U N_p, Ũ <- Ũ M_p, C <- C N_p, C~ <- C~ M_p (equationForUC,
    PAPER.md:695-700); D_c = Σ_p.

    return_maps=True also returns the column maps (T, T~) with U_out = U T,
    Ũ_out = Ũ T~ (the §4.4 recurrences carry them)."""
    n = U.shape[0]
    kin = U.shape[1]
    dt = np.result_type(U.dtype, Ut.dtype, A.dtype)
    none = (np.zeros((kin, 0), dt), np.zeros((kin, 0), dt))
    if kin == 0:
        return (empty_basis(n, dt), none) if return_maps else empty_basis(n, dt)
    C = np.asarray(A @ U, dtype=dt)
    Ct = np.asarray(AH @ Ut, dtype=dt)
    nc = np.linalg.norm(C, axis=0)
    nct = np.linalg.norm(Ct, axis=0)
    keep = (nc > 0) & (nct > 0)
    U, Ut, C, Ct = U[:, keep], Ut[:, keep], C[:, keep], Ct[:, keep]
    nc, nct = nc[keep], nct[keep]
    if U.shape[1] == 0:
        return (empty_basis(n, dt), none) if return_maps else empty_basis(n, dt)
    U = U / nc
    C = C / nc
    Ut = Ut / nct
    Ct = Ct / nct
    G = Ct.conj().T @ C
    M, S, Nh = np.linalg.svd(G)
    N = Nh.conj().T
    # "pick p such that σ_p >= tol > σ_{p+1}": absolute test on
    # the Gram of unit-norm columns, i.e. on cosines (reading Q13)
    p = int(np.sum(S >= trunc_tol))
    out = Basis(U @ N[:, :p], Ut @ M[:, :p], C @ N[:, :p], Ct @ M[:, :p],
                S[:p].copy())
    if not return_maps:
        return out
    Tm = np.zeros((kin, p), dt)
    Ttm = np.zeros((kin, p), dt)
    Tm[keep, :] = N[:, :p] / nc[:, None]
    Ttm[keep, :] = M[:, :p] / nct[:, None]
    return out, (Tm, Ttm)


# ----------------------------------------------------------------------------
# R2: initial projection (minusXR)
# ----------------------------------------------------------------------------
def project_initial(A, AH, basis, b, bt, x_m1, xt_m1):
    """x_0 = x_{-1} + UĈ^*r_{-1}, r_0 = (I - CĈ^*)r_{-1} and the duals with
    Č; Ĉ = C~D_c^{-1}, Č = C D_c^{-1} (eq:CcheckChat)."""
    r_m1 = b - A @ x_m1
    rt_m1 = bt - AH @ xt_m1
    if basis.k == 0:
        return x_m1.copy(), xt_m1.copy(), r_m1, rt_m1
    Chat = basis.Ct / basis.d          # Ĉ = C~ D_c^{-1}  (D_c real, Q6)
    Ccheck = basis.C / basis.d         # Č = C D_c^{-1}
    g = Chat.conj().T @ r_m1
    gt = Ccheck.conj().T @ rt_m1
    x0 = x_m1 + basis.U @ g
    r0 = r_m1 - basis.C @ g
    xt0 = xt_m1 + basis.Ut @ gt
    rt0 = rt_m1 - basis.Ct @ gt
    return x0, xt0, r0, rt0


# ----------------------------------------------------------------------------
# R4: Lanczos data
# ----------------------------------------------------------------------------
class LanczosData:
    """Scalars and residual columns recorded by the loop.

    Global Lanczos index m >= 1: v_m = r_{m-1}/||r_{m-1}||,
    ṽ_m = r~_{m-1}/(v_m, r~_{m-1}) = r~_{m-1} ||r_{m-1}|| / conj(ρ_{m-1})
    (scalingfactor)."""

    def __init__(self):
        self.alpha = {}     # α_m, m >= 1
        self.beta = {0: 0.0}  # β_m, β_0 = 0
        self.rho = {}       # ρ_m = (r~_m, r_m), m >= 0
        self.rnorm = {}     # ||r_m||, m >= 0
        self.zeta = {}      # ζ_m, m >= 1
        self.zetat = {}     # ζ~_m
        self.r = {}         # r_m (kept for the current cycle window)
        self.rt = {}

    def v(self, m):
        return self.r[m - 1] / self.rnorm[m - 1]

    def vt(self, m):
        return self.rt[m - 1] * (self.rnorm[m - 1] / np.conj(self.rho[m - 1]))

    def T(self, a, b):
        """Entry (a, b) of the tridiagonal T from the iteration scalars
        (PAPER.md:513-524); 1-based Lanczos indices."""
        al, be, rn = self.alpha, self.beta, self.rnorm
        if a == b:
            return 1.0 / al[a] + (be[a - 1] / al[a - 1] if a > 1 else 0.0)
        if a == b + 1:
            return -(rn[b] / rn[b - 1]) / al[b]
        if b == a + 1:
            return -(rn[a - 1] / rn[a]) * be[a] / al[a]
        return 0.0

    def forget_before(self, m):
        for key in [q for q in self.r if q < m]:
            del self.r[key]
            del self.rt[key]


def cycle_blocks(L: LanczosData, j, s, dtype):
    """Υ_j, Ῡ_j, Γ_j, Γ~_j, V_j, Ṽ_j for cycle j (augBiLanExtend,
    PAPER.md:527-550).  In cycle 1 the top row and v_0 are absent
    (V̲_1, T̲_1)."""
    cols = list(range((j - 1) * s + 1, j * s + 1))
    rows = ([(j - 1) * s] if j > 1 else []) + cols + [j * s + 1]
    Ups = np.stack([L.v(m) for m in rows], axis=1).astype(dtype)
    Upst = np.stack([L.vt(m) for m in rows], axis=1).astype(dtype)
    Gam = np.array([[L.T(a, b) for b in cols] for a in rows], dtype=dtype)
    # T~ = T^* under the scaling: Γ~[a,b] = conj(T[b,a])
    Gamt = np.array([[np.conj(L.T(b, a)) for b in cols] for a in rows],
                    dtype=dtype)
    off = 1 if j > 1 else 0
    V = Ups[:, off:off + s]
    Vt = Upst[:, off:off + s]
    return Ups, Upst, Gam, Gamt, V, Vt


# ----------------------------------------------------------------------------
# R5: harmonic Ritz selection (Q11, Q12)
# ----------------------------------------------------------------------------
def select_eigvecs(alpha_qz, beta_qz, VR, VL, k, real, qnorm):
    """Pick the k eigenpairs of the pencil nearest the origin.
    Q11: sort by |λ|, then arg λ, then index; exclude infinite/NaN
    (|β_QZ| <= 1e-14 ||Q||).  For real problems keep conjugate pairs together
    as [Re w, Im w]; if the k-th would split a pair, take k-1.
    Q12: W~ = left eigenvectors of the same pencil."""
    m = len(alpha_qz)
    finite = np.abs(beta_qz) > 1e-14 * qnorm
    lam = np.full(m, np.inf, dtype=np.complex128)
    lam[finite] = alpha_qz[finite] / beta_qz[finite]
    finite &= np.isfinite(lam)
    order = sorted((i for i in range(m) if finite[i]),
                   key=lambda i: (abs(lam[i]), np.angle(lam[i]), i))
    if not real:
        sel = order[:k]
        return VR[:, sel], VL[:, sel], lam[sel]
    # real pencil: eigenvalues with nonzero imaginary part come in conjugate
    # pairs; represent each pair once by its +Im member.
    W, Wt, lams, used = [], [], [], set()
    count = 0
    for i in order:
        if i in used:
            continue
        if lam[i].imag == 0.0:
            if count + 1 > k:
                break
            W.append(VR[:, i].real)
            Wt.append(VL[:, i].real)
            lams.append(lam[i])
            used.add(i)
            count += 1
        else:
            # partner: the conjugate eigenvalue (LAPACK stores pairs adjacent)
            partner = i + 1 if lam[i].imag > 0 else i - 1
            if count + 2 > k:
                break
            ip = i if lam[i].imag > 0 else partner
            W += [VR[:, ip].real, VR[:, ip].imag]
            Wt += [VL[:, ip].real, VL[:, ip].imag]
            lams += [lam[ip], np.conj(lam[ip])]
            used |= {i, partner}
            count += 2
    if not W:
        z = np.zeros((VR.shape[0], 0))
        return z, z.copy(), np.zeros(0, dtype=np.complex128)
    return np.stack(W, 1), np.stack(Wt, 1), np.array(lams)


def solve_pencil(P, Q, k, real):
    """Generalised eigenproblem P w = λ Q w with left and right vectors
    (finalGenEigValue), LAPACK ggev via scipy."""
    if real:
        P = P.real
        Q = Q.real
    (a, b), VL, VR = sla.eig(P, Q, left=True, right=True,
                             homogeneous_eigvals=True)
    return select_eigvecs(a, b, VR, VL, k, real, np.linalg.norm(Q))


def solve_tridiag_first(Tm, k, real):
    """First cycle without any recycle data: T_1 w = λ w, left and right
    eigenvectors of T_1."""
    if real:
        Tm = Tm.real
    lam, VL, VR = sla.eig(Tm, left=True, right=True)
    return select_eigvecs(lam, np.ones_like(lam), VR, VL, k, real, 1.0)


# ----------------------------------------------------------------------------
# One dual pair: Algorithm 2 with the §4 recycle-space update
# ----------------------------------------------------------------------------
@dataclass
class SolveResult:
    x: np.ndarray
    xt: np.ndarray
    status: int
    iterations: int
    cycles: int
    basis_out: Basis
    basis_in: Basis
    relres_rec: float
    relres_dual_rec: float
    relres_true: float
    relres_dual_true: float
    hist: dict = field(default_factory=dict)
    pencils: list = field(default_factory=list)
    r: np.ndarray = None      # recursive residuals at exit
    rt: np.ndarray = None


def solve_dual(A, b, bt, x_m1=None, xt_m1=None, U=None, Ut=None, *, k=10,
               s=40, tol=1e-8, max_itn=20000, trunc_tol=1e-6,
               xt_redraw=None, update_recycle=True, force_iters=None,
               keep_pencils=False, breakdown_tol=BREAKDOWN_EPS,
               variant="standard", pencil="plain", reproject=True):
    """Solve A x = b and A^* x~ = b~ with RBiCG (Algorithm 2)
    using the recycle space (U, Ũ) (may be None/empty: first system), and
    build the recycle space for the next system (§4).

    variant="single_reduction": the same
    iteration re-associated so that one batch of inner products per iteration
    yields both β_i and α_{i+1}.  With w_i = A r_i and ω_i = Ĉ^*w_i (exact
    arithmetic, using z_{i+1} = w_i + β_i z_i, C~^*r_i = 0, C^*r~_i = 0 and the
    bi-orthogonality of the residuals):
        ζ_{i+1} = ω_i + β_i ζ_i,   q_{i+1} = (w_i - Cω_i) + β_i q_i,
        δ_i = (r~_i, w_i - Cω_i),  σ_{i+1} = δ_i - β_i ρ_i / α_i,
    and the duals with ω~_i = Č^*A^*r~_i, β̄_i.  Every other step (x, r, the
    stop test, ζ_c, the recycle-space update) is Algorithm 2's.  The
    second-kind breakdown test (σ_{i+1} = 0, Q3) is taken at the end of
    iteration i, before its cycle end.

    reproject=True (reading Q32): keep the Petrov-Galerkin
    condition r_i ⊥ C~, r~_i ⊥ C ((orth)) explicitly.  At the
    start of iteration i, g_{i-1} = Ĉ^*r_{i-1}, g~_{i-1} = Č^*r~_{i-1} (zero in
    exact arithmetic); the update becomes r_i = r_{i-1} - α_i q_i - C g_{i-1},
    ζ_c += α_i ζ_i - g_{i-1} (so b - A(x_i - Uζ_c) = r_i still holds exactly,
    C = AU), and the duals alike.  Without it the oblique component CĈ^*r --
    left untouched by every later update because q_i ∈ null(Ĉ^*) -- keeps the
    rounding injected while ||r|| is large (minusXR can inflate ||r_0|| by
    1/σ_min) and the recursion stagnates at ≈ eps·max||r_i||/σ_min.

    variant="lookahead" (the fused single-kernel iteration of the
    GPU path): Algorithm 2 except that β_i is
    formed from the one-step expansion of ρ_i = (r~_i, r_i) with r_i = r_{i-1}
    - α_i q_i,
        ρ_i ≈ ρ_{i-1} - α_i (r~_{i-1}, q_i) - α_i (q~_i, r_{i-1}) + α_i² (q~_i, q_i),
    (with a recycle space and Q32 also - (r~_{i-1}, C g) - (C~ g~, r_{i-1})
    + (C~ g~, C g)), whose inner products belong to iteration i's first
    reduction (on the GPU: C^*r~, C~^*r, C~^*z, C^*z~ and scalars); ρ_i itself
    (for α_{i+1}, the breakdown test) and the norms stay exact -- on the GPU
    they complete one kernel later, which does not change the arithmetic.
    """
    if variant not in ("standard", "single_reduction", "lookahead"):
        raise ValueError(variant)
    if pencil not in ("plain", "fast"):
        raise ValueError(pencil)
    pipe = variant == "single_reduction"
    look = variant == "lookahead"
    n = A.shape[0]
    AH = adjoint(A)
    dt = np.result_type(A.dtype, b.dtype, bt.dtype)
    real = not np.iscomplexobj(np.zeros(0, dtype=dt))
    b = np.asarray(b, dtype=dt)
    bt = np.asarray(bt, dtype=dt)
    x_m1 = np.zeros(n, dt) if x_m1 is None else np.asarray(x_m1, dt).copy()
    xt_m1 = np.zeros(n, dt) if xt_m1 is None else np.asarray(xt_m1, dt).copy()
    bn, btn = np.linalg.norm(b), np.linalg.norm(bt)

    # Step 1 + per-system refresh
    if U is None or U.shape[1] == 0:
        basis = empty_basis(n, dt)
    else:
        basis = biorthogonalize(A, AH, np.asarray(U, dt), np.asarray(Ut, dt),
                                trunc_tol)
    kc = basis.k

    # Step 2-3: initial projection, re-randomise x~_{-1} once (Q4)
    x, xt, r, rt = project_initial(A, AH, basis, b, bt, x_m1, xt_m1)
    rho = inner(rt, r)
    if breakdown(rho, np.linalg.norm(r), np.linalg.norm(rt), breakdown_tol) \
            and xt_redraw is not None:
        xt_m1 = np.asarray(xt_redraw, dt).copy()
        x, xt, r, rt = project_initial(A, AH, basis, b, bt, x_m1, xt_m1)
        rho = inner(rt, r)

    L = LanczosData()
    L.rho[0] = rho
    L.rnorm[0] = np.linalg.norm(r)
    L.r[0], L.rt[0] = r.copy(), rt.copy()
    hist = dict(rnorm=[np.linalg.norm(r)], rtnorm=[np.linalg.norm(rt)],
                alpha=[], beta=[], rho=[rho], sigma=[])

    # Step 4: p_0 = p~_0 = 0, β_0 = 0; ζ_c = ζ~_c = 0 (Q5)
    p = np.zeros(n, dt)
    pt = np.zeros(n, dt)
    beta = 0.0
    zc = np.zeros(kc, dt)
    ztc = np.zeros(kc, dt)

    # recycle-space update state
    cand = None           # (U_j, Ũ_j, C_j, C~_j) from the last full cycle
    # pencil="fast" (§4.4): the blocks carried from cycle to
    # cycle; C~^*U "must be computed at most once per linear system"
    fast = None
    if pencil == "fast":
        fast = dict(prev=None,
                    CtU=basis.Ct.conj().T @ basis.U if kc else None)
    cycles = 0
    pencils = []

    status = MAXITER
    it = 0
    tol_rec = tol
    retried = False
    rn, rtn = np.linalg.norm(r), np.linalg.norm(rt)
    if force_iters is None and rn <= tol * bn and rtn <= tol * btn:
        status = OK
        n_iter = 0
    elif breakdown(rho, rn, rtn, breakdown_tol):
        status = BREAKDOWN_SERIOUS
        n_iter = 0
    else:
        n_iter = max_itn if force_iters is None else force_iters

    Chat = basis.Ct / basis.d if kc else None
    Ccheck = basis.C / basis.d if kc else None

    def project_w(w, wt):
        """ω = Ĉ^*w, ω~ = Č^*w~ and the projected w - Cω, w~ - C~ω~."""
        if not kc:
            return np.zeros(0, dt), np.zeros(0, dt), w, wt
        om = Chat.conj().T @ w
        omt = Ccheck.conj().T @ wt
        return om, omt, w - basis.C @ om, wt - basis.Ct @ omt

    if pipe and n_iter > 0:
        # prologue: w_0 = A r_0, σ_1 = δ_0 = (r~_0, (I - CĈ^*) A r_0)
        w, wt = A @ r, AH @ rt
        om, omt, wp, wtp = project_w(w, wt)
        sigma_next = inner(rt, wp)
        zeta_next, zetat_next = om, omt
        q = np.zeros(n, dt)
        qt = np.zeros(n, dt)
    i = 0
    while i < n_iter:
        i += 1
        # Step 5
        reproj = reproject and kc and not pipe
        if reproj:   # Q32: g_{i-1} = Ĉ^*r_{i-1}, g~_{i-1} = Č^*r~_{i-1}
            g = Chat.conj().T @ r
            gt = Ccheck.conj().T @ rt
        p = r + beta * p
        pt = rt + np.conj(beta) * pt
        if pipe:
            zeta, zetat = zeta_next, zetat_next        # ζ_i = ω_{i-1} + β_{i-1}ζ_{i-1}
            q = wp + beta * q                          # q_i = (w_{i-1} - Cω_{i-1}) + β q_{i-1}
            qt = wtp + np.conj(beta) * qt
            sigma = sigma_next                         # σ_i (recurrence)
        else:
            z = A @ p
            zt = AH @ pt
            if kc:
                zeta = Chat.conj().T @ z          # ζ_i = Ĉ^* z_i
                zetat = Ccheck.conj().T @ zt      # ζ~_i = Č^* z~_i
                q = z - basis.C @ zeta
                qt = zt - basis.Ct @ zetat
            else:
                zeta = np.zeros(0, dt)
                zetat = np.zeros(0, dt)
                q, qt = z, zt
            sigma = inner(pt, q)                  # (p~_i, q_i)  (Q23)
            if breakdown(sigma, np.linalg.norm(pt), np.linalg.norm(q),
                         breakdown_tol):
                status = BREAKDOWN_SECOND
                i -= 1
                break
        alpha = rho / sigma
        zc = zc + alpha * zeta
        ztc = ztc + np.conj(alpha) * zetat
        x = x + alpha * p
        xt = xt + np.conj(alpha) * pt
        if look:   # ρ_i from iteration i's first reduction (before the update)
            rho_ext = rho - alpha * inner(rt, q) - alpha * inner(qt, r) \
                + alpha * alpha * inner(qt, q)
            if reproj:
                # the Q32 terms of (r~_i, r_i) with r_i = r - α q - C g: (r~, Cg),
                # (C~g~, r), (C~g~, Cg); (q~, Cg) = (C~g~, q) = 0 exactly (C^*q~ = 0,
                # C~^*q = 0 by the projections) and are left out
                Cg, Ctg = basis.C @ g, basis.Ct @ gt
                rho_ext = rho_ext - inner(rt, Cg) - inner(Ctg, r) + inner(Ctg, Cg)
        r = r - alpha * q
        rt = rt - np.conj(alpha) * qt
        if reproj:   # Q32: r_i ⊥ C~, r~_i ⊥ C ((orth))
            r = r - basis.C @ g
            rt = rt - basis.Ct @ gt
            zc = zc - g
            ztc = ztc - gt
        it = i
        rn, rtn = np.linalg.norm(r), np.linalg.norm(rt)
        L.alpha[i] = alpha
        L.rnorm[i] = rn
        L.zeta[i], L.zetat[i] = zeta, zetat
        L.r[i], L.rt[i] = r.copy(), rt.copy()
        hist["alpha"].append(alpha)
        hist["sigma"].append(sigma)
        hist["rnorm"].append(rn)
        hist["rtnorm"].append(rtn)
        converged = force_iters is None and rn <= tol_rec * bn \
            and rtn <= tol_rec * btn
        # ρ_i = (r~_i, r_i); also needed for ṽ_{i+1} when the
        # loop stops at a cycle boundary
        rho_new = inner(rt, r)
        beta_new = rho_new / rho          # β_i
        if look:
            beta_new = rho_ext / rho
        L.rho[i] = rho_new
        L.beta[i] = beta_new              # Γ~_j's bottom row needs β_{js}
        hist["rho"].append(rho_new)
        serious = breakdown(rho_new, rn, rtn, breakdown_tol)
        second = False
        if pipe:
            # the one batch of inner products of iteration i: ρ_i, the norms,
            # and δ_i, ω_i, ω~_i from w_i = A r_i, w~_i = A^* r~_i
            w, wt = A @ r, AH @ rt
            om, omt, wp, wtp = project_w(w, wt)
            delta = inner(rt, wp)
            sigma_next = delta - beta_new * rho_new / alpha
            zeta_next = om + beta_new * zeta
            zetat_next = omt + np.conj(beta_new) * zetat
            second = not converged and not serious and i < n_iter and \
                breakdown(sigma_next, 1.0, 1.0, breakdown_tol)
        if second:   # σ_{i+1} = 0: iteration i+1 cannot start
            status = BREAKDOWN_SECOND
            break
        # cycle end (full cycles only, Q14)
        if update_recycle and k > 0 and i % s == 0 and (converged or not serious):
            j = i // s
            cand = _cycle_end(A, AH, L, j, s, basis, cand, k, trunc_tol, dt,
                              real, pencils if keep_pencils else None, fast)
            cycles += 1
            L.forget_before((j * s) - 1)
        if converged:
            # Step 7 + true residual confirmation (Q2)
            xf = x - basis.U @ zc if kc else x.copy()
            xtf = xt - basis.Ut @ ztc if kc else xt.copy()
            tr = np.linalg.norm(b - A @ xf) / bn
            trt = np.linalg.norm(bt - AH @ xtf) / btn
            if (tr > tol or trt > tol) and not retried:
                retried = True
                tol_rec = 0.1 * tol
            else:
                status = OK
                break
        if serious:
            status = BREAKDOWN_SERIOUS
            break
        beta = beta_new
        hist["beta"].append(beta)
        rho = rho_new
    else:
        if force_iters is not None:
            status = OK

    # Step 7
    if kc:
        x = x - basis.U @ zc
        xt = xt - basis.Ut @ ztc
    tr = np.linalg.norm(b - A @ x) / bn
    trt = np.linalg.norm(bt - AH @ xt) / btn
    if not update_recycle:
        out = basis
    elif cand is not None:
        out = cand
    else:
        out = basis  # Q18: refreshed input when no full cycle completed
    if status == OK and update_recycle and k > 0 and cand is not None and cand.k == 0:
        status = RECYCLE_EMPTY  # p = 0 after truncation (PAPER.md:702 footnote)
    return SolveResult(x=x, xt=xt, status=status, iterations=it, cycles=cycles,
                       basis_out=out, basis_in=basis,
                       relres_rec=np.linalg.norm(r) / bn,
                       relres_dual_rec=np.linalg.norm(rt) / btn,
                       relres_true=tr, relres_dual_true=trt, hist=hist,
                       pencils=pencils, r=r, rt=rt)


def _lanczos_biorth(rows_a, rows_b, dt):
    """Ῡ_a^*Υ_b in exact arithmetic: ṽ_m^*v_l = δ_ml, the bi-orthogonality of
    the Lanczos vectors under the scaling (scalingfactor) of PAPER.md:506-512
    -- the shifted identities of PAPER.md:853-868 and :883-897."""
    return np.array([[1.0 if ra == rb else 0.0 for rb in rows_b] for ra in rows_a],
                    dtype=dt).reshape(len(rows_a), len(rows_b))


def fast_grams(j, s, basis, cand, fast, Upst, X0, dt):
    """Ψ~_j^*Ψ_j and Ψ~_j^*Φ_j by the recurrences of §4.4.

    Ψ_j = [C, C_{j-1}, Υ_j] and Φ_j = [X0, V_j] with X0 = U_{j-1} (or U in the
    first cycle of a later system); blocks absent in a case are dropped.  With
    AΦ_{j-1} = Ψ_{j-1}H_{j-1} and U_{j-1} = Φ_{j-1}F_{j-1} (F = W_{j-1}N_{j-1}
    incl. the Q13 column scaling), every block follows from cycle j-1's small
    matrices (carried in ``fast["prev"]``) and the exact relations
    C~^*Υ_j = 0, Ῡ_j^*C = 0 (the residuals are kept ⊥ C~, ⊥ C),
    C~_{j-2} ⊥ Υ_j, C_{j-2} ⊥ Ῡ_j (biorthj), Ῡ^*Υ = shifted
    identities, C~^*C = D_c, C~_{j-1}^*C_{j-1} = Σ_{j-1}:
      C~^*C_{j-1}      = [C~^*C_{j-2}, D_cB_{j-1}] W_{j-1}N_{j-1}
      C~_{j-1}^*C      = N~^*W~^*[C~_{j-2}^*C; B~^*D_c]
      C~_{j-1}^*Υ_j    = N~^*W~^*[0; Γ~_{j-1}^*Ῡ_{j-1}^*Υ_j]
      Ῡ_j^*C_{j-1}     = [0, Ῡ_j^*Υ_{j-1}Γ_{j-1}] W_{j-1}N_{j-1}
      C~^*U_{j-1}      = [C~^*U_{j-2}, 0] W_{j-1}N_{j-1}
      C~_{j-1}^*U_{j-1} = N~^*W~^*[[C~_{j-2}^*U_{j-2}, C~_{j-2}^*V_{j-1}],
                                  [Ṽ_{j-1}^*C_{j-2}, T~_{j-1}]] W N
    written here in the compact form F~^*H~^*(Ψ~_{j-1}^*·) and (·Ψ_{j-1})HF
    of the same products.  The one O(n) product is Ῡ_j^*X0; C~^*U in
    the first cycle of a later system is the once-per-system block."""
    kc = basis.k
    have_prev = cand is not None and cand.k > 0
    ps = fast["prev"] if have_prev else None
    kp = cand.k if have_prev else 0
    rows = list(fast["rows"])
    cols = list(fast["cols"])
    nr = len(rows)
    top = 1 if j > 1 else 0
    kx = X0.shape[1]
    iC = slice(0, kc)
    iP = slice(kc, kc + kp)
    iU = slice(kc + kp, kc + kp + nr)
    m = kc + kp + nr
    G1 = np.zeros((m, m), dt)
    G2 = np.zeros((m, kx + s), dt)
    if kc:
        G1[iC, iC] = np.diag(basis.d)                       # D_c
    G1[iU, iU] = np.eye(nr)                                 # Ῡ_j^*Υ_j = I
    if have_prev:
        pC = slice(0, ps["kc"])
        pU = slice(ps["kc"] + ps["kp"], ps["m"])
        HF = ps["H"] @ ps["F"]                              # C_{j-1} = Ψ_{j-1}(H F)
        HFt = ps["Ht"] @ ps["Ft"]                           # C~_{j-1} = Ψ~_{j-1}(H~ F~)
        if kc:
            G1[iC, iP] = ps["G1"][pC, :] @ HF               # C~^*C_{j-1}
            G1[iP, iC] = HFt.conj().T @ ps["G1"][:, pC]     # C~_{j-1}^*C
            G2[iC, :kx] = ps["G2"][pC, :] @ ps["F"]         # C~^*U_{j-1}
        G1[iP, iP] = np.diag(cand.d)                        # Σ_{j-1}
        Z = np.zeros((ps["m"], nr), dt)                     # Ψ~_{j-1}^*Υ_j
        Z[pU, :] = _lanczos_biorth(ps["rows"], rows, dt)
        G1[iP, iU] = HFt.conj().T @ Z                       # C~_{j-1}^*Υ_j
        Zt = np.zeros((nr, ps["m"]), dt)                    # Ῡ_j^*Ψ_{j-1}
        Zt[:, pU] = _lanczos_biorth(rows, ps["rows"], dt)
        G1[iU, iP] = Zt @ HF                                # Ῡ_j^*C_{j-1}
        G2[iP, :kx] = HFt.conj().T @ ps["G2"] @ ps["F"]     # C~_{j-1}^*U_{j-1}
        G2[iP, kx:] = G1[iP, iU][:, top:top + s]            # C~_{j-1}^*V_j
    elif kc:
        G2[iC, :kx] = fast["CtU"]                           # C~^*U (once per system)
    G2[iU, :kx] = Upst.conj().T @ X0                        # Ῡ_j^*X0: the O(n) product
    G2[iU, kx:] = _lanczos_biorth(rows, cols, dt)           # Ῡ_j^*V_j = I with zero rows
    return G1, G2


def _cycle_end(A, AH, L, j, s, basis, cand, k, trunc_tol, dt, real, pencils,
               fast=None):
    """Build U_j, Ũ_j at the end of cycle j (R5/R6); with
    ``fast`` the pencil's Grams come from fast_grams (§4.4)."""
    Ups, Upst, Gam, Gamt, V, Vt = cycle_blocks(L, j, s, dt)
    kc = basis.k
    have_prev = cand is not None and cand.k > 0
    cols = list(range((j - 1) * s + 1, j * s + 1))
    rows = ([(j - 1) * s] if j > 1 else []) + cols + [j * s + 1]
    if fast is not None:
        fast["rows"], fast["cols"] = rows, cols
    if not have_prev and kc == 0:
        # first system, no recycle data: eigenvectors of T_j
        top = 1 if j > 1 else 0
        Tj = Gam[top:top + s, :]
        W, Wt, lam = solve_tridiag_first(Tj, k, real)
        Phi, Phit = V, Vt
        info = dict(j=j, case="T", P=Tj, Q=np.eye(s), lam=lam, W=W, Wt=Wt)
        # for the next cycle's recurrences: AV_j = Υ_jΓ_j, Ῡ_j^*Υ_j = I
        H, Ht = Gam, Gamt
        G1 = np.eye(len(rows), dtype=dt)
        G2 = _lanczos_biorth(rows, cols, dt)
        kcb = kpb = 0
    else:
        if kc:
            # B_j = Ĉ^*AV_j, B~_j = Č^*A^*Ṽ_j by explicit products
            B = (basis.Ct / basis.d).conj().T @ (A @ V)
            Bt = (basis.C / basis.d).conj().T @ (AH @ Vt)
        if have_prev:
            Uprev, Utprev, Cprev, Ctprev = cand.U, cand.Ut, cand.C, cand.Ct
            kp = cand.k
            Phi = np.hstack([Uprev, V])
            Phit = np.hstack([Utprev, Vt])
            if kc:
                # general case
                Psi = np.hstack([basis.C, Cprev, Ups])
                Psit = np.hstack([basis.Ct, Ctprev, Upst])
                H = _blk([[np.zeros((kc, kp)), B],
                          [np.eye(kp), np.zeros((kp, s))],
                          [np.zeros((Gam.shape[0], kp)), Gam]], dt)
                Ht = _blk([[np.zeros((kc, kp)), Bt],
                           [np.eye(kp), np.zeros((kp, s))],
                           [np.zeros((Gamt.shape[0], kp)), Gamt]], dt)
            else:
                # first system, later cycles
                Psi = np.hstack([Cprev, Ups])
                Psit = np.hstack([Ctprev, Upst])
                H = _blk([[np.eye(kp), np.zeros((kp, s))],
                          [np.zeros((Gam.shape[0], kp)), Gam]], dt)
                Ht = _blk([[np.eye(kp), np.zeros((kp, s))],
                           [np.zeros((Gamt.shape[0], kp)), Gamt]], dt)
        else:
            # first cycle of a later system; Φ = [U V_j]
            Phi = np.hstack([basis.U, V])
            Phit = np.hstack([basis.Ut, Vt])
            Psi = np.hstack([basis.C, Ups])
            Psit = np.hstack([basis.Ct, Upst])
            H = _blk([[np.eye(kc), B],
                      [np.zeros((Gam.shape[0], kc)), Gam]], dt)
            Ht = _blk([[np.eye(kc), Bt],
                       [np.zeros((Gamt.shape[0], kc)), Gamt]], dt)
        # finalGenEigValue
        kcb, kpb = kc, (cand.k if have_prev else 0)
        if fast is None:
            G1 = Psit.conj().T @ Psi
            G2 = Psit.conj().T @ Phi
        else:
            X0 = Phi[:, :Phi.shape[1] - s]
            G1, G2 = fast_grams(j, s, basis, cand, fast, Upst, X0, dt)
        P = Ht.conj().T @ G1 @ H
        Q = Ht.conj().T @ G2
        W, Wt, lam = solve_pencil(P, Q, k, real)
        info = dict(j=j, case="pencil", P=P, Q=Q, lam=lam, W=W, Wt=Wt,
                    B=B if kc else None, Bt=Bt if kc else None, G1=G1, G2=G2,
                    kc=kcb, kp=kpb)
        if fast is not None and pencils is not None:   # the plain Grams, for the pins
            info.update(G1_plain=Psit.conj().T @ Psi, G2_plain=Psit.conj().T @ Phi)
    Unew = Phi @ W.astype(dt)
    Utnew = Phit @ Wt.astype(dt)
    # §4.3: C_j = AU_j, C~_j = A^*Ũ_j, SVD, truncation
    out, (Tm, Ttm) = biorthogonalize(A, AH, Unew, Utnew, trunc_tol, return_maps=True)
    if fast is not None:
        fast["prev"] = dict(G1=G1, G2=G2, H=np.asarray(H, dt), Ht=np.asarray(Ht, dt),
                            F=W.astype(dt) @ Tm, Ft=Wt.astype(dt) @ Ttm,
                            kc=kcb, kp=kpb, m=G1.shape[0], rows=rows)
    if pencils is not None:
        info.update(Phi=Phi, Phit=Phit, Unew=Unew, Utnew=Utnew, Gam=Gam,
                    Gamt=Gamt, V=V, Vt=Vt, Ups=Ups, Upst=Upst,
                    L=dict(alpha=dict(L.alpha), beta=dict(L.beta),
                           rho=dict(L.rho), rnorm=dict(L.rnorm),
                           zeta=dict(L.zeta), zetat=dict(L.zetat)))
        pencils.append(info)
    return out


def _blk(rows, dt):
    return np.block([[np.asarray(m, dtype=dt) for m in row] for row in rows])


# ----------------------------------------------------------------------------
# Bilinear form, estimator Q19
# ----------------------------------------------------------------------------
def bilinear(A, u, w, U=None, Ut=None, **kw):
    """u^*A^{-1}w from the dual pair A x = w, A^* x~ = u:
    estimate u^*x + x~^*(w - Ax) (error r~^*A^{-1}r, quadratic)."""
    res = solve_dual(A, w, u, U=U, Ut=Ut, **kw)
    r = w - A @ res.x
    value = inner(u, res.x) + inner(res.xt, r)
    return value, res
