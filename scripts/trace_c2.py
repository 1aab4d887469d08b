"""Trace one C2 system solve phase by phase (RBICG_TRACE=1)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RBICG_TRACE"] = "1"
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ctx = api.Context(0)
R = ctx.recycle(cfg.n, cfg.k)
for it in system_sequence(cfg, systems=[0, 1]):
    A = ctx.matrix(it["indptr"], it["indices"], it["data"])
    x, xt, res, _ = ctx.solve_dual(A, it["b"], it["bt"], R=R, k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    print({k: res[k] for k in ("iterations", "cycles", "k_in", "k_out", "t_loop_ms", "t_cycle_dev_ms", "t_host_eig_ms", "t_total_ms", "status_name")}, flush=True)
