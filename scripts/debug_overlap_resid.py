"""Diagnosis (not a test): the forced-overlap NCCL one-rank sequence of
tests/test_gpu_dist.py::test_nccl_one_rank_forced_overlap_in_graph, printing
per system the iterations, k_in/k_out, recursive and true residuals of the
plain and the partitioned context (RBICG_* switches from the environment)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RBICG_FORCE_HALO_SPLIT", "1")
from paper_1010_0762_b200 import api
from synth import CONFIGS, system_sequence

cfg = CONFIGS["C1"].scaled(40, systems=3, s=10)
items = list(system_sequence(cfg))
plain = api.Context(0)
part = api.Context(0, dist=dict(rank=0, nranks=1, mode=0, key=api.nccl_unique_id(), force_partition=1))
for name, ctx in (("plain", plain), ("part", part)):
    rec = ctx.recycle(cfg.n, cfg.k)
    for j, item in enumerate(items):
        M = ctx.matrix(item["indptr"], item["indices"], item["data"])
        x, xt, res, _ = ctx.solve_dual(M, item["b"], item["bt"], R=rec, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                       max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
        print(name, j, {q: res[q] for q in ("iterations", "status_name", "k_in", "k_out", "relres_rec", "relres_dual_rec",
                                            "relres_true", "relres_dual_true")}, flush=True)
