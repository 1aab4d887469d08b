"""Rounding spread of the oracle's iteration count at full size (reading Q28):
Algorithm 2 as written (variant="standard") on b perturbed by relative 1e-15
(seeded), and the look-ahead-ρ variant, on system 0 of a BASELINE config.
CPU only (oracle); compared with the GPU count of scripts/fullsize_count_check.py.

    python scripts/fullsize_count_ensemble.py C3 standard 0     # seed 0 = unperturbed
    python scripts/fullsize_count_ensemble.py C3 lookahead 0
"""
import json
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from synth import CONFIGS, system_sequence          # noqa: E402
from oracle import rbicg as R                        # noqa: E402

name, variant, seed = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = CONFIGS[name]
item = next(system_sequence(cfg, systems=[0]))
n = len(item["indptr"]) - 1
A = sp.csr_matrix((item["data"], item["indices"], item["indptr"]), shape=(n, n))
b = item["b"]
if seed:
    b = b * (1 + 1e-15 * np.random.default_rng(seed).standard_normal(b.shape))
ref = R.solve_dual(A, b, item["bt"], k=0, s=cfg.s, tol=cfg.tol, max_itn=cfg.max_itn, variant=variant)
print(json.dumps({"config": name, "variant": variant, "b_perturb_seed": seed,
                  "iterations": ref.iterations, "status": int(ref.status)}))
