"""GPU vs oracle per system with the ORACLE's input basis imported (Q27)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from paper_1010_0762_b200 import api
from oracle import rbicg as R
from oracle.sequence import run_sequence, csr_matrix
from synth import CONFIGS, system_sequence
from synth.small import deflation_matrix, dense_to_csr, vec

def cosines(X, Y):
    if X.shape[1] == 0 or Y.shape[1] == 0: return np.zeros(0)
    Q1, _ = np.linalg.qr(X); Q2, _ = np.linalg.qr(Y)
    return np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False)

ctx = api.Context(0)
for name, cfg in [("C1", CONFIGS["C1"]), ("C1tt6", CONFIGS["C1"].scaled(32, trunc_tol=1e-6, tol=1e-8)),
                  ("C4@12", CONFIGS["C4"].scaled(12, systems=6, s=20))]:
    items = list(system_sequence(cfg, lam_r=0.0) if cfg.kind == "irka" else system_sequence(cfg))
    U = Ut = None
    for item in items:
        Ad = csr_matrix(item)
        r = R.solve_dual(Ad, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s, tol=cfg.tol,
                         max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, keep_pencils=True)
        rec = ctx.recycle(cfg.n, cfg.k, cfg.complex)
        if U is not None and U.shape[1]:
            rec.import_(U, Ut)
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                       max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, history=True)
        Ug, Utg = rec.export()
        bo = r.basis_out
        cs = cosines(Ug, bo.U); cst = cosines(Utg, bo.Ut)
        bn = np.linalg.norm(item["b"])
        m = min(len(h), len(r.hist["rnorm"]) - 1)
        orn = np.array(r.hist["rnorm"][1:m + 1]) / bn
        d = np.abs(h[:m, 0] - orn) / orn
        first = int(np.argmax(d > 1e-6)) if (d > 1e-6).any() else None
        lam = [np.round(np.sort(np.abs(pc["lam"]))[:cfg.k + 2], 5) for pc in r.pencils[-1:]]
        print(name, item["j"], "gpu", res["status"], res["iterations"], res["k_in"], res["k_out"], "| or", r.status, r.iterations,
              r.basis_in.k, bo.k, "| x err %.1e" % (np.linalg.norm(x - r.x) / np.linalg.norm(r.x)),
              "| first>1e-6:", first, "| cos U", np.round(cs, 6), "Ut", np.round(cst, 6), "lam", lam)
        U, Ut = bo.U, bo.Ut
