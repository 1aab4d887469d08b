"""Algorithm 1: BiCG -- test-infrastructure oracle.

Readings:
* Q1  (u, v) = u^* v (conjugate-linear in the first argument), np.vdot.
* Q2  stop when ||r_i|| <= tol ||b|| and ||r~_i|| <= tol ||b~|| (relative).
* Q3  serious breakdown |rho_i| <= eps ||r_i|| ||r~_i||; second kind
      |(p~_i, q_i)| <= eps ||p~_i|| ||q_i||, with eps = ``breakdown_tol``
      (default 0: the paper's literal "= 0"; a positive
      threshold such as SURVEY's 1e-14 stops the conv-diff configs at
      rounding-level near-breakdowns that BiCG passes through).
      Non-finite scalars are also reported as breakdowns.  Not cured.
* Q4  step 2's "(r_0, r~_0) = 0" uses the Q3 test; the random x~_0 is an
      input (``xt_redraw``), used at most once.
* Pre-loop: if both initial residuals already meet the stop test, zero
  iterations are performed (the paper's loop tests only after an update).
"""
from __future__ import annotations

import numpy as np

OK, MAXITER, BREAKDOWN_SERIOUS, BREAKDOWN_SECOND = 0, 1, 2, 3
BREAKDOWN_EPS = 0.0   # Q3 (revised): the paper's literal "= 0"


def inner(u, v):
    """Standard inner product (u, v) = u^* v (reading Q1)."""
    return np.vdot(u, v)


def breakdown(val, na, nb, eps):
    """Q3: |val| <= eps * na * nb, or val not finite."""
    return (not np.isfinite(val)) or abs(val) <= eps * na * nb


def bicg(A, b, bt, x0, xt0, tol, max_itn, xt_redraw=None, force_iters=None,
         breakdown_tol=BREAKDOWN_EPS):
    """Run Algorithm 1 on the dual pair A x = b, A^* x~ = b~.

    A is a scipy.sparse matrix (real or complex).  Returns a dict with the
    final iterates, status, iteration count and per-iteration scalars."""
    AH = A.conj().T.tocsr()
    dt = np.result_type(A.dtype, b.dtype, bt.dtype)
    x = np.array(x0, dtype=dt)
    xt = np.array(xt0, dtype=dt)
    bn, btn = np.linalg.norm(b), np.linalg.norm(bt)
    # 1. r_0 = b - A x_0, r~_0 = b~ - A^* x~_0
    r = b - A @ x
    rt = bt - AH @ xt
    rho = inner(rt, r)
    # 2. if (r_0, r~_0) = 0 then initialise x~_0 to a random vector
    if breakdown(rho, np.linalg.norm(r), np.linalg.norm(rt), breakdown_tol):
        if xt_redraw is not None:
            xt = np.array(xt_redraw, dtype=dt)
            rt = bt - AH @ xt
            rho = inner(rt, r)
    hist = dict(alpha=[], beta=[], rho=[rho], rnorm=[np.linalg.norm(r)],
                rtnorm=[np.linalg.norm(rt)])
    status = MAXITER
    it = 0
    if force_iters is None and np.linalg.norm(r) <= tol * bn \
            and np.linalg.norm(rt) <= tol * btn:
        return dict(x=x, xt=xt, r=r, rt=rt, iterations=0, status=OK,
                    hist=hist)
    if breakdown(rho, np.linalg.norm(r), np.linalg.norm(rt), breakdown_tol):
        return dict(x=x, xt=xt, r=r, rt=rt, iterations=0,
                    status=BREAKDOWN_SERIOUS, hist=hist)
    # 3. p_0 = p~_0 = 0, beta_0 = 0
    p = np.zeros_like(r)
    pt = np.zeros_like(rt)
    beta = 0.0
    n_iter = max_itn if force_iters is None else force_iters
    for i in range(1, n_iter + 1):
        p = r + beta * p
        pt = rt + np.conj(beta) * pt
        q = A @ p
        qt = AH @ pt
        sigma = inner(pt, q)
        if breakdown(sigma, np.linalg.norm(pt), np.linalg.norm(q),
                     breakdown_tol):
            status = BREAKDOWN_SECOND
            break
        alpha = rho / sigma
        x = x + alpha * p
        xt = xt + np.conj(alpha) * pt
        r = r - alpha * q
        rt = rt - np.conj(alpha) * qt
        it = i
        rn, rtn = np.linalg.norm(r), np.linalg.norm(rt)
        hist["alpha"].append(alpha)
        hist["rnorm"].append(rn)
        hist["rtnorm"].append(rtn)
        if force_iters is None and rn <= tol * bn and rtn <= tol * btn:
            status = OK
            break
        rho_new = inner(rt, r)
        hist["rho"].append(rho_new)
        if breakdown(rho_new, rn, rtn, breakdown_tol):
            status = BREAKDOWN_SERIOUS
            break
        beta = rho_new / rho
        hist["beta"].append(beta)
        rho = rho_new
    else:
        status = OK if force_iters is not None else MAXITER
    return dict(x=x, xt=xt, r=r, rt=rt, iterations=it, status=status,
                hist=hist)
