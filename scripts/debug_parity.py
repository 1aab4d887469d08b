"""Debug helper: print GPU vs oracle per-solve numbers for the parity cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from paper_1010_0762_b200 import api
from oracle import rbicg as R
from oracle.sequence import run_sequence
from synth import CONFIGS, system_sequence, redraw_vector
from synth.small import deflation_matrix, dense_to_csr, vec

ctx = api.Context(0)
n, k = 300, 4
A, lam, S = deflation_matrix(n, k, seed=31)
Ad = sp.csr_matrix(A)
M = ctx.matrix(*dense_to_csr(A))
b, bt = vec(n, 32), vec(n, 33)
rec = ctx.recycle(n, k)
U = Ut = None
for run in range(4):
    ref = R.solve_dual(Ad, b, bt, U=U, Ut=Ut, k=k, s=15, tol=1e-10, max_itn=1000, trunc_tol=1e-6)
    x, xt, res, h = ctx.solve_dual(M, b, bt, R=rec, k=k, s=15, tol=1e-10, max_itn=1000, trunc_tol=1e-6, history=True)
    U, Ut = ref.basis_out.U, ref.basis_out.Ut
    print("P5 run", run, "gpu it", res["iterations"], "rec %.2e true %.2e host-true %.2e" % (res["relres_rec"], res["relres_true"], np.linalg.norm(b - Ad @ x) / np.linalg.norm(b)),
          "| oracle it", ref.iterations, "rec %.2e true %.2e" % (ref.relres_rec, ref.relres_true), "kin", res["k_in"], ref.basis_in.k, "kout", res["k_out"], ref.basis_out.k)
    print("   gpu hist relres last5", h[-5:, 0], " oracle", np.array(ref.hist["rnorm"][-5:]) / np.linalg.norm(b))

cfg = CONFIGS["C1"]
items = list(system_sequence(cfg))
ref = run_sequence(cfg, items)
rec = ctx.recycle(cfg.n, cfg.k)
for item, r in zip(items, ref):
    Mi = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, h = ctx.solve_dual(Mi, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, history=True)
    print("C1 sys", item["j"], "gpu", res["status"], res["iterations"], res["k_in"], res["k_out"], "%.2e %.2e" % (res["relres_rec"], res["relres_true"]),
          "| oracle", r.status, r.iterations, r.basis_in.k, r.basis_out.k, "%.2e %.2e" % (r.relres_rec, r.relres_true))
    m = min(len(h), len(r.hist["rnorm"]) - 1)
    d = np.abs(h[:m, 0] - np.array(r.hist["rnorm"][1:m + 1]) / np.linalg.norm(item["b"])) / (np.array(r.hist["rnorm"][1:m + 1]) / np.linalg.norm(item["b"]))
    print("   first iteration with rel diff > 1e-6:", int(np.argmax(d > 1e-6)) if (d > 1e-6).any() else None, " diff at 10, 50:", d[min(10, m-1)], d[min(50, m-1)])
