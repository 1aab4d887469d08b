"""C5 (384^3, n = 56.6M, k = 20, s = 50) on ONE GPU: system 0 solved through
the C ABI; iterations, it/s, true residuals recomputed on the host."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp, torch
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api
cfg = CONFIGS["C5"]
t0 = time.time()
it = next(system_sequence(cfg, systems=[0]))
print("gen", round(time.time() - t0, 1), "s", flush=True)
ctx = api.Context(0)
d = {k: torch.from_numpy(np.ascontiguousarray(it[k])).cuda() for k in ("indptr", "indices", "data", "b", "bt")}
A = ctx.matrix(d["indptr"], d["indices"], d["data"])
del d["indptr"], d["indices"], d["data"]
torch.cuda.empty_cache()
print("free GB after matrix", torch.cuda.mem_get_info()[0] / 2**30, flush=True)
R = ctx.recycle(cfg.n, cfg.k)
torch.cuda.synchronize()
t = time.time()
x, xt, res, _ = ctx.solve_dual(A, d["b"], d["bt"], R=R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                               max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
torch.cuda.synchronize()
el = time.time() - t
x, xt = x.cpu().numpy(), xt.cpu().numpy()
M = sp.csr_matrix((it["data"], it["indices"], it["indptr"]), shape=(cfg.n, cfg.n))
rt = np.linalg.norm(it["b"] - M @ x) / np.linalg.norm(it["b"])
rtt = np.linalg.norm(it["bt"] - M.T @ xt) / np.linalg.norm(it["bt"])
out = dict(config="C5", n=cfg.n, nnz=int(len(it["indices"])), iterations=res["iterations"],
           status=res["status_name"], k_out=res["k_out"], cycles=res["cycles"],
           wall_s=el, it_per_s=res["iterations"] / el, loop_ms=res["t_loop_ms"],
           cycle_end_ms=res["t_cycle_dev_ms"], host_eig_ms=res["t_host_eig_ms"],
           relres_true_host=rt, relres_dual_true_host=rtt,
           relres_true_lib=res["relres_true"], relres_dual_true_lib=res["relres_dual_true"])
print(json.dumps(out), flush=True)
