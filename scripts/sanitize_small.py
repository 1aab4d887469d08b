"""Small end-to-end solves for compute-sanitizer (memcheck / racecheck /
synccheck runs, one tool per call): C1 sequence (recycling, cycle ends,
relation GEMMs), a complex C4-family system, 2 virtual ranks."""
import sys, os, threading, uuid
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api

ctx = api.Context(0)
cfg = CONFIGS["C1"].scaled(16, systems=2, s=8)
R = ctx.recycle(cfg.n, cfg.k)
for it in system_sequence(cfg):
    A = ctx.matrix(it["indptr"], it["indices"], it["data"])
    x, xt, res, _ = ctx.solve_dual(A, it["b"], it["bt"], R=R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
    print("C1", res["iterations"], res["status_name"], flush=True)
cfg4 = CONFIGS["C4"].scaled(6, systems=1, s=8)
it = next(system_sequence(cfg4, lam_r=0.0))
A = ctx.matrix(it["indptr"], it["indices"], it["data"])
R4 = ctx.recycle(cfg4.n, cfg4.k, True)
x, xt, res, _ = ctx.solve_dual(A, it["b"], it["bt"], R=R4, k=cfg4.k, s=cfg4.s, tol=cfg4.tol,
                               max_itn=cfg4.max_itn, trunc_tol=cfg4.trunc_tol)
print("C4", res["iterations"], res["status_name"], flush=True)
key = uuid.uuid4().bytes * 8
it = next(system_sequence(cfg))
out = [None, None]
def body(q):
    c = api.Context(0, dist=dict(rank=q, nranks=2, mode=1, key=key))
    n = cfg.n; r0, r1 = (n * q) // 2, (n * (q + 1)) // 2
    M = c.matrix(it["indptr"], it["indices"], it["data"])
    Rq = c.recycle(r1 - r0, cfg.k)
    out[q] = c.solve_dual(M, it["b"][r0:r1].copy(), it["bt"][r0:r1].copy(), R=Rq, k=cfg.k,
                          s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)[2]
th = [threading.Thread(target=body, args=(q,)) for q in range(2)]
[t.start() for t in th]; [t.join() for t in th]
print("dist", out[0]["iterations"], out[0]["status_name"], flush=True)
