"""Full-size iteration counts of the default k = 0 iteration (k_fused, β from
the one-step expansion of ρ) against Algorithm 2 AS WRITTEN
(oracle variant="standard") on system 0 of a BASELINE config.

Too slow for the GPU suite at C3 size (the oracle needs minutes); run once per
kernel change and keep the JSON line under profiles/:

    python scripts/fullsize_count_check.py C3
"""
import json
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from synth import CONFIGS, system_sequence          # noqa: E402
from oracle import rbicg as R                        # noqa: E402  (checker, not the product)
from paper_1010_0762_b200 import api                 # noqa: E402


def main(name):
    cfg = CONFIGS[name]
    item = next(system_sequence(cfg, systems=[0]))
    n = len(item["indptr"]) - 1
    A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]), shape=(n, n))
    ctx = api.Context(0)
    M = ctx.matrix(item["indptr"], item["indices"], item["data"])
    x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], k=0, s=cfg.s, tol=cfg.tol,
                                   max_itn=cfg.max_itn)
    M.free()
    t0 = time.time()
    ref = R.solve_dual(A, item["b"], item["bt"], k=0, s=cfg.s, tol=cfg.tol,
                       max_itn=cfg.max_itn, variant="standard")
    t_or = time.time() - t0
    a, b = res["iterations"], ref.iterations
    ok = abs(a - b) <= max(2, 0.03 * max(a, b))
    ex = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
    print(json.dumps({"config": name, "n": n, "gpu_iterations": a, "oracle_standard_iterations": b,
                      "within_max2_3pct": bool(ok), "gpu_status": res["status"],
                      "oracle_status": int(ref.status),
                      "gpu_relres_true": res["relres_true"],
                      "gpu_relres_dual_true": res["relres_dual_true"],
                      "x_rel_diff_vs_oracle": float(ex), "oracle_seconds": round(t_or, 1)}))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1] if len(sys.argv) > 1 else "C3"))
