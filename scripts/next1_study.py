"""NEXT-1 study: the single-reduction (re-associated) RBiCG
iteration and the look-ahead-ρ iteration of the fused GPU kernel vs
Algorithm 2 as written, on the BASELINE operator families at
oracle-size grids -- iteration counts, statuses, recycle widths and true
residuals per system.  Oracle only (CPU); the table is quoted in DESIGN §6.

    python scripts/next1_study.py            # all families
    python scripts/next1_study.py C2 128 3   # one family, grid, systems
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scipy.sparse as sp  # noqa: E402

from oracle import rbicg as R  # noqa: E402
from synth import CONFIGS, system_sequence  # noqa: E402


def run(name, N, nsys):
    cfg = CONFIGS[name].scaled(N, systems=nsys) if N else CONFIGS[name]
    kw = {"lam_r": 0.0} if cfg.kind == "irka" else {}
    for var in ("standard", "single_reduction", "lookahead"):
        U = Ut = None
        out = []
        for item in system_sequence(cfg, **kw):
            A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]))
            r = R.solve_dual(A, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                             tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol,
                             variant=var)
            out.append((r.iterations, R.STATUS_NAMES.get(r.status, r.status), r.basis_in.k,
                        r.basis_out.k, float("%.1e" % r.relres_true)))
            U, Ut = r.basis_out.U, r.basis_out.Ut
        print(cfg.name, var, out, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
    else:
        for args in (("C1", 0, 4), ("C2", 128, 3), ("C3", 24, 3), ("C4", 12, 6), ("C5", 24, 3)):
            run(*args)
