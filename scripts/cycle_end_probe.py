"""Target of an ncu capture of the cycle-end kernels (never timed): system 1
of a BASELINE config from a seeded N(0,1) k-column input space (truncation at
the config's rule), forced to s + 3 iterations so one general-case cycle end
(C, C_{j-1}, Υ_j Grams, U_j GEMM, C_j SpMM, SVD Gram) runs in
stream order (RBICG_SYNC_CYCLE=1 recommended).  Prints the solve's phase
times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

name = sys.argv[1]
pencil = sys.argv[2] if len(sys.argv) > 2 else "plain"
cfg = CONFIGS[name]
kw = dict(lam_r=0.0) if cfg.kind == "irka" else {}
item = next(system_sequence(cfg, systems=[1], **kw))
ctx = api.Context(0)
d = {q: torch.from_numpy(np.ascontiguousarray(item[q])).cuda()
     for q in ("indptr", "indices", "data", "b", "bt")}
A = ctx.matrix(d["indptr"], d["indices"], d["data"])
rng = np.random.default_rng(cfg.seed + 777)
shp = (cfg.n, cfg.k)
if cfg.complex:
    U = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
    Ut = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
else:
    U, Ut = rng.standard_normal(shp), rng.standard_normal(shp)
R = ctx.recycle(cfg.n, cfg.k, cfg.complex)
R.import_(U, Ut)
m = 2 * cfg.s + 3
x, xt, res, _ = ctx.solve_dual(A, d["b"], d["bt"], None, None, R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                               max_itn=m, force_iters=m, trunc_tol=cfg.trunc_tol, pencil=pencil)
print({q: res[q] for q in ("iterations", "k_in", "k_out", "cycles", "t_loop_ms", "t_cycle_dev_ms",
                           "t_host_eig_ms", "t_refresh_ms", "t_total_ms")})
