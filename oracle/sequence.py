"""Sequence driver for the oracle: system j -> j+1.

The recycle space (U, Ũ) is the only state carried between systems; the next
system's Step 1 re-establishes C = A^{(j+1)}U, C~ = A^{(j+1)*}Ũ (refresh).
Initial guesses follow reading Q7: zeros for the conv-diff configs; for the
IRKA-like config the previous sweep's solution of the same shift slot.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .rbicg import solve_dual


def csr_matrix(item):
    n = item["n"]
    return sp.csr_matrix((item["data"], item["indices"], item["indptr"]),
                         shape=(n, n))


def run_sequence(cfg, items, k=None, s=None, tol=None, max_itn=None,
                 recycle=True, callback=None, force_iters=None, pencil="plain"):
    """Solve every system in ``items`` (dicts from synth.system_sequence) in
    order, carrying the recycle space.  Returns a list of SolveResult."""
    from synth import redraw_vector  # inputs only
    k = cfg.k if k is None else k
    s = cfg.s if s is None else s
    tol = cfg.tol if tol is None else tol
    max_itn = cfg.max_itn if max_itn is None else max_itn
    U = Ut = None
    prev_x = {}
    results = []
    for idx, item in enumerate(items):
        A = csr_matrix(item)
        n = item["n"]
        x0 = xt0 = None
        if cfg.kind == "irka" and item["slot"] in prev_x:
            x0, xt0 = prev_x[item["slot"]]
        fi = None if force_iters is None else force_iters[idx]
        res = solve_dual(A, item["b"], item["bt"], x0, xt0,
                         U if recycle else None, Ut if recycle else None,
                         k=k if recycle else 0, s=s, tol=tol, max_itn=max_itn,
                         trunc_tol=cfg.trunc_tol,
                         xt_redraw=redraw_vector(cfg, item["j"], n),
                         update_recycle=recycle and k > 0, force_iters=fi,
                         pencil=pencil)
        if recycle:
            U, Ut = res.basis_out.U, res.basis_out.Ut
        if cfg.kind == "irka":
            prev_x[item["slot"]] = (res.x, res.xt)
        results.append(res)
        if callback is not None:
            callback(idx, item, res)
    return results
