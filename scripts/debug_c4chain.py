"""Debug: C4@12^3 (s = 20) chain, GPU vs oracle from the same input spaces."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence
from oracle import rbicg as R

def cos(U, V):
    Qu = np.linalg.qr(U)[0]; Qv = np.linalg.qr(V)[0]
    return np.linalg.svd(Qv.conj().T @ Qu, compute_uv=False)

trunc = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
cfg = CONFIGS["C4"].scaled(12, systems=8, s=20)
items = list(system_sequence(cfg, lam_r=0.0))
ctx = api.Context(0)
U = Ut = None
prev = {}
recg = ctx.recycle(cfg.n, cfg.k, True)   # the GPU's own chain
prevg = {}
for item in items:
    A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]), shape=(cfg.n, cfg.n))
    x0, xt0 = prev.get(item["slot"], (None, None))
    ref = R.solve_dual(A, item["b"], item["bt"], x0, xt0, U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                       tol=cfg.tol, max_itn=2000, trunc_tol=trunc)
    rec = ctx.recycle(cfg.n, cfg.k, True)
    if U is not None and U.shape[1]:
        rec.import_(U, Ut)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], x0, xt0, R=rec, k=cfg.k, s=cfg.s,
                                   tol=cfg.tol, max_itn=2000, trunc_tol=trunc)
    g0, gt0 = prevg.get(item["slot"], (None, None))
    xg, xtg, resg, _ = ctx.solve_dual(M, item["b"], item["bt"], g0, gt0, R=recg, k=cfg.k,
                                      s=cfg.s, tol=cfg.tol, max_itn=2000, trunc_tol=trunc)
    prevg[item["slot"]] = (xg, xtg)
    Ug, Utg = rec.export()
    c = cos(Ug, ref.basis_out.U) if ref.basis_out.k and Ug.shape[1] == ref.basis_out.k else []
    print(item["j"], "oracle", ref.iterations, "gpu", res["iterations"], "gpu-own", resg["iterations"],
          "kin", ref.basis_in.k, res["k_in"], "kout", ref.basis_out.k, res["k_out"],
          "d", np.round(ref.basis_in.d, 6) if ref.basis_in.k else "",
          "cos", np.round(c, 6), flush=True)
    prev[item["slot"]] = (ref.x, ref.xt)
    U, Ut = ref.basis_out.U, ref.basis_out.Ut
    M.free()
