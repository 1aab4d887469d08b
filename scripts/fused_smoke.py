import sys, os; sys.path.insert(0, '/root/repo')
import numpy as np, scipy.sparse as sp
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api
from oracle import rbicg as R
ctx = api.Context(0)
for name, N in (("C2", 96), ("C3", 20), ("C4", 10), ("C1", 0)):
    cfg = CONFIGS[name].scaled(N, systems=1) if N else CONFIGS[name]
    item = next(system_sequence(cfg, **({"lam_r": 0.0} if cfg.kind == "irka" else {})))
    A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]))
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    kt = ctx.time_kernels(M, None, k=0, s=cfg.s, iters=5)
    rec = ctx.recycle(cfg.n, cfg.k, cfg.complex)
    x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol, variant="lookahead")
    ref0 = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    print(name, N, "fused_ms", kt["fused_ms"], kt["fused_done_flag"], "gpu", res["iterations"], res["status_name"], res["k_out"], "%.2e %.2e" % (res["relres_true"], res["relres_dual_true"]),
          "| oracle lookahead", ref.iterations, ref.status, ref.basis_out.k, "| standard", ref0.iterations, ref0.basis_out.k,
          "| dx", np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x), flush=True)
    M.free()
