"""Graph-timed iteration kernels against problem size (fixed launch cost vs
streaming rate): python scripts/pass_scaling.py C4 8 60 80 100 126"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

name, k = sys.argv[1], int(sys.argv[2])
ctx = api.Context(0)
for N in map(int, sys.argv[3:]):
    cfg = CONFIGS[name].scaled(N, systems=1)
    kw = dict(lam_r=0.0) if cfg.kind == "irka" else {}
    item = next(system_sequence(cfg, systems=[0], **kw))
    d = {q: torch.from_numpy(np.ascontiguousarray(item[q])).cuda() for q in ("indptr", "indices", "data")}
    A = ctx.matrix(d["indptr"], d["indices"], d["data"])
    R = None
    if k > 0:
        rng = np.random.default_rng(5)
        shp = (cfg.n, k)
        U = rng.standard_normal(shp) + (1j * rng.standard_normal(shp) if cfg.complex else 0)
        Ut = rng.standard_normal(shp) + (1j * rng.standard_normal(shp) if cfg.complex else 0)
        R = ctx.recycle(cfg.n, k, cfg.complex)
        R.import_(U, Ut)
    kt = ctx.time_kernels(A, R, k=max(k, 1), s=cfg.s, iters=20, trunc_tol=1e-300)
    print(json.dumps(dict(N=N, n=cfg.n, nnz=int(item["indptr"][-1]), p1=kt["pass1_graph_ms"],
                          p2=kt["pass2_graph_ms"], fused=kt["fused_ms"], it=kt["graph_iter_ms"])),
          flush=True)
    A.free()
    if R is not None:
        R.free()
