"""IRKA (Algorithm 3) driving the dual solves --
test-infrastructure oracle (see oracle/__init__.py).

The model is the SISO LTI system G(s) = c^*(sE - A)^{-1} b of
(equation:orginalModel), with E = I (the IRKA-like C4
family; PAPER.md:1186-1194 discusses E = I).  Step by step:

1. initial shifts σ_1..σ_r;
2./3. V_r = [(σ_i E - A)^{-1} b], W_r = [(σ_i E - A)^{-*} c]: ONE dual pair per
   shift, (σ_i I - A) v_i = b and (σ_i I - A)^* w_i = c, solved by RBiCG
   (oracle.rbicg.solve_dual) -- recycling strategy 1:
   shift slot i carries its recycle space and its previous solutions from one
   IRKA step to the next;
4. while not converged: A_r = W_r^* A V_r and E_r = W_r^* E V_r (reading Q20:
   the paper's "E_r = W_r^*AV_r" is a typo for W_r^*EV_r),
   σ_i ← -λ_i(A_r, E_r), new V_r, W_r;
5. A_r, E_r, b_r = W_r^* b, c_r = V_r^* c (reading: the paper's "c_r = V_r^*c_r"
   is a typo for V_r^* c, (red_projection) PAPER.md:1004-1007).

Recycling strategies, ``strategy=``:
1. slot i of step m+1 recycles the space of slot i of step m;
2. within a step, each solve recycles the space of the previous solve (the
   chain continues across steps: column 1 of step m+1 takes the last column's
   space of step m);
3. each solve picks, from the spaces of sigma^(m)_1..r and sigma^(m+1)_1..i-1,
   the one whose shift has the smallest relative change |sigma' - sigma_i| /
   |sigma_i|, if that change is below ``reuse_tol`` (else no recycle space).
In all three the initial guesses are the previous step's solutions of the
same slot.

Readings for what the paper leaves open (Q29):
* convergence: max_i |σ_i^new - σ_i| / |σ_i| < shift_tol (relative change of
  the shifts, 10^-6), at most max_steps steps;
* pairing of slots across steps (strategy 1, "the i-th column to the i-th
  column"): both shift sets sorted by (|σ|, arg σ) -- SPEC.md:456's magnitude
  sort, ties broken by the argument so conjugate pairs keep their slots;
* the reduced model uses the V_r, W_r of the LAST solves (the model whose
  Hermite interpolation Theorem 3.1 guarantees at the current shifts).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import rbicg as R


def order_shifts(sig):
    """Slot order of a shift set: by |σ| (rounded to 10 significant digits so a
    conjugate pair ties), then arg σ (reading Q29)."""
    sig = np.asarray(sig, dtype=np.complex128)
    mag = np.abs(sig)
    key = np.round(mag / max(float(mag.max()), 1e-300), 10) if len(sig) else mag
    return sig[np.lexsort((np.angle(sig), key))]


def reduced_model(A, V, W, b, c):
    """(red_projection), with E = I."""
    Ar = W.conj().T @ (A @ V)
    Er = W.conj().T @ V
    br = W.conj().T @ b
    cr = V.conj().T @ c
    return Ar, Er, br, cr


def transfer(Ar, Er, br, cr, s):
    """G_r(s) = c_r^*(s E_r - A_r)^{-1} b_r and G_r'(s)."""
    M = s * Er - Ar
    y = np.linalg.solve(M, br)
    g = np.vdot(cr, y)
    dg = -np.vdot(cr, np.linalg.solve(M, Er @ y))
    return g, dg


@dataclass
class IrkaResult:
    shifts: np.ndarray                 # final shifts (the last solves' σ)
    steps: int                         # IRKA steps (shift updates) performed
    converged: bool
    history: list = field(default_factory=list)     # shift set per step
    iterations: list = field(default_factory=list)  # per step: iterations per slot
    V: np.ndarray = None
    W: np.ndarray = None
    Ar: np.ndarray = None
    Er: np.ndarray = None
    br: np.ndarray = None
    cr: np.ndarray = None


def pick_space(pool, si, reuse_tol):
    """Strategy 3: the pool entry (sigma', space) with the smallest relative
    shift change below reuse_tol (first such entry on ties), else None."""
    best, bd = None, reuse_tol
    for sp_, sp in pool:
        d = abs(sp_ - si) / abs(si)
        if d < bd:
            best, bd = sp, d
    return best


def irka(A, b, c, shifts0, *, k=8, s=40, tol=1e-10, max_itn=20000, trunc_tol=1e-6,
         shift_tol=1e-6, max_steps=30, recycle=True, strategy=1, reuse_tol=np.inf):
    """Algorithm 3 with E = I; A is the (sparse) state matrix of the model."""
    A = sp.csr_matrix(A, dtype=np.complex128)
    n = A.shape[0]
    I = sp.identity(n, dtype=np.complex128, format="csr")
    b = np.asarray(b, dtype=np.complex128)
    c = np.asarray(c, dtype=np.complex128)
    sig = order_shifts(shifts0)
    r = len(sig)
    slots = [dict(U=None, Ut=None, x=None, xt=None) for _ in range(r)]
    res = IrkaResult(shifts=sig, steps=0, converged=False)
    chain = [None]       # strategy 2: the last solve's space
    prev_pool = []       # strategy 3: (sigma, space) of the previous step

    def solve_all(sig):
        V = np.zeros((n, r), np.complex128)
        W = np.zeros((n, r), np.complex128)
        its = []
        cur_pool = []
        for i, si in enumerate(sig):
            st = slots[i]
            if strategy == 1:
                space = (st["U"], st["Ut"])
            elif strategy == 2:
                space = chain[0]
            else:
                space = pick_space(prev_pool + cur_pool, si, reuse_tol)
            U0, Ut0 = space if (recycle and space is not None) else (None, None)
            out = R.solve_dual(si * I - A, b, c, st["x"], st["xt"], U=U0, Ut=Ut0,
                               k=k if recycle else 0, s=s, tol=tol, max_itn=max_itn,
                               trunc_tol=trunc_tol)
            V[:, i], W[:, i] = out.x, out.xt
            st["x"], st["xt"] = out.x, out.xt          # previous solution
            st["U"], st["Ut"] = out.basis_out.U, out.basis_out.Ut
            chain[0] = (out.basis_out.U, out.basis_out.Ut)
            cur_pool.append((si, (out.basis_out.U, out.basis_out.Ut)))
            its.append(out.iterations)
        prev_pool[:] = cur_pool
        return V, W, its

    V, W, its = solve_all(sig)                          # steps 2-3
    res.history.append(sig.copy())
    res.iterations.append(its)
    for step in range(max_steps):                       # step 4
        Ar, Er, _, _ = reduced_model(A, V, W, b, c)
        lam = sla.eigvals(Ar, Er)
        new = order_shifts(-lam)
        change = np.max(np.abs(new - sig) / np.abs(sig))
        sig = new
        res.steps = step + 1
        V, W, its = solve_all(sig)
        res.history.append(sig.copy())
        res.iterations.append(its)
        if change < shift_tol:
            res.converged = True
            break
    res.shifts = sig
    res.V, res.W = V, W
    res.Ar, res.Er, res.br, res.cr = reduced_model(A, V, W, b, c)   # step 5
    return res
