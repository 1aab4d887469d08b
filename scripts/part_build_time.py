"""Partitioned matrix build time per rank (virtual ranks on one GPU, blocks of
a BASELINE matrix passed as local rows with global columns): first build
(plan + value halo) and a rebuild of the same pattern (cached plan)."""
import json
import os
import sys
import threading
import time
import uuid

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

name, P = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
item = next(system_sequence(cfg, systems=[0]))
n = cfg.n
key = uuid.uuid4().bytes * 8
out = [None] * P


def body(q):
    r0, r1 = (n * q) // P, (n * (q + 1)) // P
    ip = item["indptr"]
    a, b = int(ip[r0]), int(ip[r1])
    loc = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in
           (ip[r0:r1 + 1] - ip[r0], item["indices"][a:b], item["data"][a:b])]
    ctx = api.Context(0, dist=dict(rank=q, nranks=P, mode=1, key=key))
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        M = ctx.matrix(*loc)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
        M.free()
    out[q] = ts


th = [threading.Thread(target=body, args=(q,)) for q in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
print(json.dumps(dict(config=name, ranks=P, rows_per_rank=n // P,
                      build_ms_first=[round(o[0], 1) for o in out],
                      build_ms_cached=[round(min(o[1:]), 1) for o in out],
                      note="virtual ranks share one GPU: the ranks' builds run concurrently on it")))
