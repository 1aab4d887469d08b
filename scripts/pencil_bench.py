"""Cycle-end cost with the plain vs the §4.4 pencil assembly (rbicg_opts.pencil,
SURVEY §8(f) NEXT-2) at full BASELINE sizes.

Under reading Q13 the BASELINE workloads truncate every cycle's space to p = 0,
so their cycle ends never take the recycle-space branch that §4.4 changes.  To
measure that branch at full size this script runs the config's operator with a
small truncation threshold (``--trunc``, default 1e-12) so that spaces survive:
system 0 builds U, system 1 runs ``--cycles`` full cycles (force_iters, Q27)
from it, once per pencil mode, cycle ends in stream order (RBICG_SYNC_CYCLE=1)
so their device time is not shared with the loop.  Prints one JSON line:
per-cycle cycle-end time, the O(n) columns read by the pencil Grams, and the
principal-angle cosines between the two modes' output spaces.
"""
import argparse, json, os, sys
os.environ.setdefault("RBICG_SYNC_CYCLE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--trunc", type=float, default=1e-12)
ap.add_argument("--cycles", type=int, default=8)
a = ap.parse_args()
cfg = CONFIGS[a.config]
items = list(system_sequence(cfg, systems=[0, 1]))
cplx = np.iscomplexobj(items[0]["b"])
ctx = api.Context(0)
it0 = items[0]
M0 = ctx.matrix(it0["indptr"], it0["indices"], it0["data"])
R0 = ctx.recycle(cfg.n, cfg.k, cplx)
_, _, r0, _ = ctx.solve_dual(M0, it0["b"], it0["bt"], R=R0, k=cfg.k, s=cfg.s, tol=cfg.tol,
                             max_itn=cfg.max_itn, trunc_tol=a.trunc)
M0.free()
U0, Ut0 = R0.export()
it1 = items[1]
M1 = ctx.matrix(it1["indptr"], it1["indices"], it1["data"])
out = dict(config=a.config, trunc_tol=a.trunc, k=cfg.k, s=cfg.s, n=cfg.n,
           system0=dict(iterations=r0["iterations"], k_out=r0["k_out"]))
spaces = {}
m = a.cycles * cfg.s
for mode in ("plain", "fast", "plain", "fast"):   # second pass is the timed one
    R = ctx.recycle(cfg.n, cfg.k, cplx)
    R.import_(U0, Ut0)
    _, _, r, _ = ctx.solve_dual(M1, it1["b"], it1["bt"], R=R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                max_itn=m + 1, trunc_tol=a.trunc, force_iters=m, pencil=mode)
    spaces[mode] = R.export()
    out[mode] = dict(k_in=r["k_in"], k_out=r["k_out"], cycles=r["cycles"],
                     cycle_ms=r["t_cycle_dev_ms"] / max(1, r["cycles"]),
                     host_eig_ms=r["t_host_eig_ms"] / max(1, r["cycles"]),
                     loop_ms=r["t_loop_ms"])
    R.free()


def cosines(X, Y):
    if X.shape[1] == 0 or Y.shape[1] == 0:
        return []
    Q1, _ = np.linalg.qr(X)
    Q2, _ = np.linalg.qr(Y)
    return np.linalg.svd(Q1.conj().T @ Q2, compute_uv=False).tolist()


out["cos_U_plain_fast"] = cosines(spaces["plain"][0], spaces["fast"][0])
k, s = cfg.k, cfg.s
nr = s + 2
# columns per side read by the pencil Grams in the general case (kc = kp = k)
out["gram_cols_plain"] = (k + k + nr) + (k + k + nr + k)   # Ψ~ and [Ψ, X0] (+ the C_{j-1} SpMM)
out["gram_cols_fast"] = nr + k                              # Ῡ_j and X0
print(json.dumps(out))
