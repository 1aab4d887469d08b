"""IRKA (Algorithm 3) on the GPU with and without Krylov-subspace recycling:
the C4 operator family K = -L + 0.1 xi at N^3 as the state
matrix, r = 6 initial shifts from the C4 schedule (sweep 0), strategies 1
and 3 vs plain BiCG (k = 0).  Prints one JSON line:
IRKA steps, final shifts' agreement, total and per-step dual-solve
iterations, GPU wall time.  The paper's own IRKA savings are
context, not a target: its model, preconditioner and shift mix differ."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from paper_1010_0762_b200 import api, irka as GI  # noqa: E402
from synth import CONFIGS  # noqa: E402
from synth.configs import irka_operator, irka_shift  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
model = sys.argv[2] if len(sys.argv) > 2 else "c4"
cfg = CONFIGS["C4"].scaled(N, systems=6)
if model == "c4":   # K = -L + 0.1 xi on N^3, the C4 schedule's sweep-0 shifts
    op = irka_operator(cfg, lam_r=0.0)
    n = op["n"]
    A = sp.csr_matrix((op["kdata"], op["indices"], op["indptr"]), shape=(n, n))
    b, c = op["b"], op["c"]
    shifts0 = [irka_shift(op, 0, i) for i in range(6)]
else:               # stable 2-D conv-diff model -A (tests' IRKA model) at N^2
    from synth.convdiff import convdiff_csr
    from synth.small import vec
    indptr, indices, data = convdiff_csr(N, 2, (10.0, 10.0), "central")[:3]
    n = N * N
    A = -sp.csr_matrix((data, indices, indptr), shape=(n, n))
    b, c = vec(n, 81, dist="normal"), vec(n, 82, dist="normal")
    shifts0 = [0.05, 0.4, 2.0, 10.0]
A.sort_indices()
ctx = api.Context(0)
out = dict(workload=f"IRKA, model {model} n={n}, r={len(shifts0)}, k={cfg.k}, s={cfg.s}, "
                    f"tol={cfg.tol}", runs={})
for name, kw in (("bicg", dict(recycle=False, k=0)), ("strategy1", dict(strategy=1)),
                 ("strategy3", dict(strategy=3, reuse_tol=0.5))):
    base = dict(k=cfg.k, s=cfg.s, tol=cfg.tol, trunc_tol=cfg.trunc_tol, shift_tol=1e-6,
                max_steps=30)
    base.update(kw)
    t0 = time.perf_counter()
    run = GI.irka(ctx, A.indptr, A.indices, A.data, b, c, shifts0, **base)
    el = time.perf_counter() - t0
    its = [int(sum(s)) for s in run.iterations]
    out["runs"][name] = dict(steps=run.steps, converged=run.converged, total_iterations=int(sum(its)),
                             iterations_per_step=its, wall_s=round(el, 2),
                             shifts=[[round(z.real, 8), round(z.imag, 8)] for z in run.shifts])
ref = np.array([complex(*z) for z in out["runs"]["bicg"]["shifts"]])
for name, r in out["runs"].items():
    sh = np.array([complex(*z) for z in r["shifts"]])
    r["max_rel_shift_diff_vs_bicg"] = float(np.max(np.abs(sh - ref) / np.abs(ref)))
print(json.dumps(out))
