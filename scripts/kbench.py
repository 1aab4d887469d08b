"""Kernel micro-benchmark: pass1/pass2 CUDA-event times on C2 (or --config)
for k = 0 and k = cfg.k with a random recycle space."""
import sys, os, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C2"); ap.add_argument("--N", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.config]
if args.N: cfg = cfg.scaled(args.N, systems=1)
it = next(system_sequence(cfg, systems=[0], lam_r=0.0) if cfg.kind == "irka" else system_sequence(cfg, systems=[0]))
ctx = api.Context(0)
A = ctx.matrix(it["indptr"], it["indices"], it["data"])
w = 16 if cfg.complex else 8
n, nnz = cfg.n, len(it["indices"])
for k in (0, cfg.k):
    R = ctx.recycle(n, max(k, 1), cfg.complex)
    if k:
        rng = np.random.default_rng(0)
        U = rng.standard_normal((n, k)); Ut = rng.standard_normal((n, k))
        if cfg.complex: U = U + 1j * rng.standard_normal((n, k)); Ut = Ut + 1j * rng.standard_normal((n, k))
        R.import_(U, Ut)
    t = ctx.time_kernels(A, R if k else None, k=k, s=cfg.s, iters=30, trunc_tol=1e-12)
    mat = 2 * (nnz * (w + 4) + 4 * (n + 1)) - (4 * nnz if t["shared_cols"] else 0)
    kk = t["k"]
    b1 = mat + 2 * kk * n * w + 8 * n * w
    b2 = 2 * kk * n * w + (6 if t["lazy_x"] else 12) * n * w
    print(json.dumps(dict(config=cfg.name, k=kk, pass1_ms=t["pass1_ms"], pass2_ms=t["pass2_ms"],
                          pass1_GBps=b1 / t["pass1_ms"] / 1e6, pass2_GBps=b2 / t["pass2_ms"] / 1e6,
                          iter_GBps=(b1 + b2) / (t["pass1_ms"] + t["pass2_ms"]) / 1e6, done=t["done_flag"],
                          graph_iter_ms=t["graph_iter_ms"], graph_GBps=(b1 + b2) / t["graph_iter_ms"] / 1e6,
                          graph_done=t["graph_done_flag"], loop_iter_ms=t["loop_iter_ms"],
                          p1g=t["pass1_graph_ms"], p2g=t["pass2_graph_ms"],
                          loop_GBps=(b1 + b2) / t["loop_iter_ms"] / 1e6 if t["loop_iter_ms"] > 0 else None,
                          loop_done=t["loop_done_flag"], fused_ms=t["fused_ms"],
                          fused_GBps=(mat + 12 * n * w) / t["fused_ms"] / 1e6 if t["fused_ms"] > 0 else None)))
