"""Debug: system 0 of a BASELINE config at full size, m = s + 3 forced
iterations, GPU vs oracle: x error and the per-iteration residual history."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence
from oracle import rbicg as R
cfg = CONFIGS[sys.argv[1]]
truncs = [float(t) for t in sys.argv[2:]] or [cfg.trunc_tol]
item = next(system_sequence(cfg, systems=[0]))
m = cfg.s + 3
A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]), shape=(cfg.n, cfg.n))
ctx = api.Context(0)
M = ctx.matrix(item["indptr"], item["indices"], item["data"])
for trunc in truncs:
    ref = R.solve_dual(A, item["b"], item["bt"], k=cfg.k, s=cfg.s, tol=cfg.tol, max_itn=m,
                       trunc_tol=trunc, force_iters=m)
    rec = ctx.recycle(cfg.n, cfg.k)
    x, xt, res, h = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                   max_itn=m, trunc_tol=trunc, force_iters=m, history=True)
    rn = np.array(ref.hist["rnorm"][1:]) / np.linalg.norm(item["b"])
    rel = np.abs(h[:, 0] - rn) / rn
    print("trunc", trunc, "xerr %.2e" % (np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)),
          "kout", res["k_out"], ref.basis_out.k, "hist rel by iteration:",
          " ".join("%.0e" % v for v in rel), flush=True)
