"""Target of the in-run ncu traffic capture of bench.py (never timed): the
hot-loop kernels of one BASELINE system for a few iterations, with a k-column
recycle space (seeded N(0,1) columns, truncation off: only k matters for the
bytes a launch moves) or none (k = 0: the fused iteration kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

name, k, j = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = CONFIGS[name]
kw = dict(lam_r=0.0) if cfg.kind == "irka" else {}
item = next(system_sequence(cfg, systems=[j], **kw))
ctx = api.Context(0)
d = {q: torch.from_numpy(np.ascontiguousarray(item[q])).cuda() for q in ("indptr", "indices", "data")}
A = ctx.matrix(d["indptr"], d["indices"], d["data"])
R = None
if k > 0:
    rng = np.random.default_rng(cfg.seed + 777)
    shp = (cfg.n, k)
    if cfg.complex:
        U = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
        Ut = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
    else:
        U, Ut = rng.standard_normal(shp), rng.standard_normal(shp)
    R = ctx.recycle(cfg.n, k, cfg.complex)
    R.import_(U, Ut)
iters = int(os.environ.get("KT_ITERS", "3"))
kt = ctx.time_kernels(A, R, k=max(k, 1), s=cfg.s, iters=iters, trunc_tol=1e-300)
print(kt)
