"""Debug: C_j from the bi-Lanczos relation vs explicit SpMM (RBICG_C_CHECK=1)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api
for name, N in (("C1", 32), ("C2", 128), ("C3", 24), ("C4", 12)):
    cfg = CONFIGS[name].scaled(N, systems=1)
    it = next(system_sequence(cfg, lam_r=0.0) if cfg.kind == "irka" else system_sequence(cfg))
    ctx = api.Context(0)
    A = ctx.matrix(it["indptr"], it["indices"], it["data"])
    R = ctx.recycle(cfg.n, cfg.k, cfg.complex)
    x, xt, res, _ = ctx.solve_dual(A, it["b"], it["bt"], R=R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    print(name, N, res["iterations"], res["status_name"], res["k_out"], flush=True)
