"""GPU iteration counts of system 0 of a BASELINE config (k = 0) on b
perturbed by relative 1e-15 (seeds 1..4; 0 = unperturbed) -- the GPU side of
the Q28 spread (scripts/fullsize_count_ensemble.py is the oracle side).
RBICG_FUSED=0 in the environment selects the two-kernel iteration (exact ρ,
Algorithm 2's form) instead of the fused look-ahead-ρ kernel.

    python scripts/gpu_count_ensemble.py C3
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from synth import CONFIGS, system_sequence          # noqa: E402
from paper_1010_0762_b200 import api                 # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = CONFIGS[name]
item = next(system_sequence(cfg, systems=[0]))
ctx = api.Context(0)
M = ctx.matrix(item["indptr"], item["indices"], item["data"])
out = []
for seed in range(5):
    b = item["b"]
    if seed:
        b = b * (1 + 1e-15 * np.random.default_rng(seed).standard_normal(b.shape))
    _, _, res, _ = ctx.solve_dual(M, b, item["bt"], k=0, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn)
    out.append({"seed": seed, "iterations": res["iterations"], "status": res["status"],
                "relres_true": res["relres_true"]})
M.free()
print(json.dumps({"config": name, "form": "two-kernel (RBICG_FUSED=0)" if os.environ.get("RBICG_FUSED") == "0"
                  else "fused (look-ahead rho)", "runs": out}))
