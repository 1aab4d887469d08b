"""Full-size sequence of a BASELINE config on ONE GPU under the recycle rule
(Q13 + Q32): per system the RBiCG iterations, k_in/k_out, status, true
residuals (library), and the same systems as plain BiCG (k = 0) for the
DESIGN table.  Usage: python scripts/seq_table.py C3 [nsys] [--no-bicg]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

name = sys.argv[1]
nsys = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else None
cfg = CONFIGS[name]
if nsys:
    cfg = cfg.scaled(cfg.N, systems=nsys)
do_bicg = "--no-bicg" not in sys.argv
pencil = "fast" if "--fast" in sys.argv else "plain"
ctx = api.Context(0)
R = ctx.recycle(cfg.n, cfg.k, complex_=cfg.complex)
rows = []
prev = {}
for item in system_sequence(cfg):
    d = {k: torch.from_numpy(np.ascontiguousarray(item[k])).cuda()
         for k in ("indptr", "indices", "data", "b", "bt")}
    A = ctx.matrix(d["indptr"], d["indices"], d["data"])
    x0 = xt0 = None
    if cfg.kind == "irka" and item["slot"] in prev:
        x0, xt0 = prev[item["slot"]]
    row = dict(j=item["j"])
    if do_bicg:
        torch.cuda.synchronize()
        t = time.time()
        _, _, rb, _ = ctx.solve_dual(A, d["b"], d["bt"], x0, xt0, None, k=0, s=cfg.s,
                                     tol=cfg.tol, max_itn=cfg.max_itn)
        torch.cuda.synchronize()
        row.update(bicg_it=rb["iterations"], bicg_status=rb["status_name"],
                   bicg_s=round(time.time() - t, 3))
    torch.cuda.synchronize()
    t = time.time()
    x, xt, res, _ = ctx.solve_dual(A, d["b"], d["bt"], x0, xt0, R, k=cfg.k, s=cfg.s,
                                   tol=cfg.tol, max_itn=cfg.max_itn,
                                   trunc_tol=cfg.trunc_tol, pencil=pencil)
    torch.cuda.synchronize()
    if cfg.kind == "irka":
        prev[item["slot"]] = (x, xt)
    row.update(it=res["iterations"], status=res["status_name"], k_in=res["k_in"],
               k_out=res["k_out"], cycles=res["cycles"],
               relres_true=res["relres_true"], relres_dual_true=res["relres_dual_true"],
               s=round(time.time() - t, 3), loop_ms=round(res["t_loop_ms"], 1))
    rows.append(row)
    print(json.dumps(row), flush=True)
    A.free()
print(json.dumps(dict(config=name, n=cfg.n, k=cfg.k, s=cfg.s, trunc_tol=cfg.trunc_tol,
                      systems=rows)))
