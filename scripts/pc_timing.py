"""NEXT-4 timing: split-preconditioned (Crout ILUT) dual solves of a 2-D
conv-diff operator on ONE GPU -- factorisation (host) time, iterations with
and without preconditioning, per-iteration device time."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp

from paper_1010_0762_b200 import api
from synth import convdiff_csr
from synth.small import vec

ctx = api.Context(0)
for N, beta, t in [(int(a.split(":")[0]), float(a.split(":")[1]), float(a.split(":")[2]))
                   for a in (sys.argv[1:] or ["255:40:0.05", "511:40:0.05", "1023:50:0.05"])]:
    ip, ix, dv = convdiff_csr(N, 2, (beta, beta), "central")[:3]
    n = N * N
    b, bt = vec(n, 1), vec(n, 2)
    t0 = time.perf_counter()
    P = ctx.precond_ilut(ip, ix, dv, t)
    t_fac = time.perf_counter() - t0
    M = ctx.matrix(ip, ix, dv)
    rec = ctx.recycle(n, 10)
    row = dict(N=N, n=n, droptol=t, factor_s=round(t_fac, 3))
    for name, pc in (("bicg_plain", None), ("rbicg_ilut", P), ("rbicg_ilut_run2", P)):
        t0 = time.perf_counter()
        x, xt, res, _ = ctx.solve_dual(M, b, bt, R=rec if pc else None, k=10 if pc else 0, s=40,
                                       tol=1e-8, max_itn=20000, M=pc)
        el = time.perf_counter() - t0
        row[name] = dict(it=res["iterations"], k_in=res["k_in"], status=res["status_name"],
                         wall_ms=round(1e3 * el, 1), loop_ms=round(res["t_loop_ms"], 1),
                         ms_per_it=round(res["t_loop_ms"] / max(1, res["iterations"]), 4))
    print(json.dumps(row), flush=True)
    M.free()
    P.free()
