"""IRKA (Algorithm 3) over the B200 RBiCG library.

The model is G(s) = c^*(sE - A)^{-1} b with E = I (PAPER.md:963-977,
:1186-1194).  Every dual pair (σ_i I - A) v_i = b, (σ_i I - A)^* w_i = c runs
through ``Context.solve_dual`` (the sm_100a hot path) with recycling strategy
1: shift slot i keeps its recycle handle and its previous
solutions from one IRKA step to the next.  Everything of size n stays on
the device: the CSR of A, b, c and the solutions V, W (torch CUDA tensors);
each shifted store σ_i I - A is formed by the library from A's CSR
(rbicg_matrix_shifted_csr) and the reduced model A_r = W_r^*AV_r,
E_r = W_r^*V_r (reading Q20: E_r = W_r^*EV_r), W_r^*b, V_r^*c by its SpMV
and Gram kernels (rbicg_reduced_model).  Only the r x r eigenproblem and the
shift update σ_i ← -λ_i(A_r, E_r) are host control work (as the cycle-end
pencil is for the solver).  Readings (Q29): convergence on the
relative shift change, slots paired by sorting shifts by (|σ|, arg σ).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


def pick_space(pool, si, reuse_tol):
    """Strategy 3: the pool entry with the smallest relative shift change below
    reuse_tol (first on ties), else None (the oracle's rule)."""
    best, bd = None, reuse_tol
    for sp_, h in pool:
        d = abs(sp_ - si) / abs(si)
        if d < bd:
            best, bd = h, d
    return best


def order_shifts(sig):
    """Slot order: by |σ| (10 significant digits, so conjugate pairs tie),
    then arg σ."""
    sig = np.asarray(sig, dtype=np.complex128)
    mag = np.abs(sig)
    key = np.round(mag / max(float(mag.max()), 1e-300), 10) if len(sig) else mag
    return sig[np.lexsort((np.angle(sig), key))]


@dataclass
class IrkaRun:
    shifts: np.ndarray
    steps: int
    converged: bool
    history: list = field(default_factory=list)      # shift set per step
    iterations: list = field(default_factory=list)   # per step: RBiCG iterations per slot
    Ar: np.ndarray = None
    Er: np.ndarray = None
    br: np.ndarray = None
    cr: np.ndarray = None


def irka(ctx, indptr, indices, data, b, c, shifts0, *, k=8, s=40, tol=1e-10,
         max_itn=20000, trunc_tol=1e-6, shift_tol=1e-6, max_steps=30, recycle=True,
         strategy=1, reuse_tol=np.inf):
    """Algorithm 3 on the GPU; (indptr, indices, data) is the CSR of A.
    strategy 1/2/3: the recycling strategies of PAPER.md:1196-1235 (see
    oracle/irka.py for the readings); strategies 2 and 3 copy the chosen
    space into the solve's own handle on the device (Recycle.copy_from)."""
    import torch
    A = sp.csr_matrix((np.asarray(data, np.complex128), indices, indptr))
    n = A.shape[0]
    if np.any(A.diagonal() == 0) or not A.has_sorted_indices:   # setup only: every row
        Ac = A.tocoo()                                          # holds its diagonal once
        ii = np.arange(n)
        A = sp.csr_matrix((np.concatenate([Ac.data, np.zeros(n, np.complex128)]),
                           (np.concatenate([Ac.row, ii]), np.concatenate([Ac.col, ii]))),
                          shape=(n, n))
        A.sum_duplicates()
        A.sort_indices()
    dev = torch.device("cuda", ctx.device)
    Ad = [torch.from_numpy(np.ascontiguousarray(a)).to(dev)
          for a in (A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data)]
    MA = ctx.matrix(*Ad)                                   # for the products A v_i
    b = torch.from_numpy(np.asarray(b, np.complex128).copy()).to(dev)
    c = torch.from_numpy(np.asarray(c, np.complex128).copy()).to(dev)
    sig = order_shifts(shifts0)
    r = len(sig)
    slots = [dict(R=ctx.recycle(n, max(k, 1), True), x=None, xt=None) for _ in range(r)]
    run = IrkaRun(shifts=sig, steps=0, converged=False)
    chain = [None]       # strategy 2: handle holding the last solve's space
    prev_pool = []       # strategy 3: (sigma, handle) of the previous step
    spare = []           # handles of the pool two steps back, reused

    def solve_all(sig):
        V = torch.zeros((r, n), dtype=torch.complex128, device=dev)
        W = torch.zeros((r, n), dtype=torch.complex128, device=dev)
        its = []
        cur_pool = []
        for i, si in enumerate(sig):
            st = slots[i]
            if strategy == 1:
                Rh = st["R"]
            else:
                Rh = spare.pop() if spare else ctx.recycle(n, max(k, 1), True)
                src = chain[0] if strategy == 2 else \
                    pick_space(prev_pool + cur_pool, si, reuse_tol)
                if src is not None:
                    Rh.copy_from(src)
                else:
                    Rh.clear()
            M = ctx.matrix(*Ad, shift=si)                  # σ_i I - A on the device
            x, xt, res, _ = ctx.solve_dual(M, b, c, st["x"], st["xt"],
                                           R=Rh if recycle else None,
                                           k=k if recycle else 0, s=s, tol=tol,
                                           max_itn=max_itn, trunc_tol=trunc_tol)
            M.free()
            V[i], W[i] = x, xt
            st["x"], st["xt"] = x, xt                     # previous solution
            if strategy == 2 and chain[0] is not None:
                spare.append(chain[0])
            chain[0] = Rh
            cur_pool.append((si, Rh))
            its.append(res["iterations"])
        if strategy == 3:
            spare.extend(h for _, h in prev_pool)
            prev_pool[:] = cur_pool
        return V, W, its

    def reduced(V, W):
        return ctx.reduced_model(MA, V, W, b, c)

    V, W, its = solve_all(sig)
    run.history.append(sig.copy())
    run.iterations.append(its)
    for step in range(max_steps):
        Ar, Er, _, _ = reduced(V, W)
        new = order_shifts(-sla.eigvals(Ar, Er))
        change = np.max(np.abs(new - sig) / np.abs(sig))
        sig = new
        run.steps = step + 1
        V, W, its = solve_all(sig)
        run.history.append(sig.copy())
        run.iterations.append(its)
        if change < shift_tol:
            run.converged = True
            break
    run.shifts = sig
    run.Ar, run.Er, run.br, run.cr = reduced(V, W)
    MA.free()
    return run
