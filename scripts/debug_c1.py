"""Debug: C1 sequence, GPU from the oracle's input spaces: residuals."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence
from oracle import rbicg as R
cfg = CONFIGS["C1"]
ctx = api.Context(0)
U = Ut = None
for item in system_sequence(cfg):
    A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]), shape=(cfg.n, cfg.n))
    ref = R.solve_dual(A, item["b"], item["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s, tol=cfg.tol,
                       max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    rec = ctx.recycle(cfg.n, cfg.k)
    if U is not None and U.shape[1]:
        rec.import_(U, Ut)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, history=True)
    tr = np.linalg.norm(item["b"] - A @ x) / np.linalg.norm(item["b"])
    print(item["j"], "it", res["iterations"], ref.iterations, "st", res["status_name"], ref.status,
          "kin", res["k_in"], "true lib %.2e host %.2e oracle %.2e" % (res["relres_true"], tr, ref.relres_true),
          "rec %.2e %.2e" % (res["relres_rec"], ref.relres_rec), "last hist %.2e" % h[-1, 0], flush=True)
    U, Ut = ref.basis_out.U, ref.basis_out.Ut
