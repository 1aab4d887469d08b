"""C4 sequence with one chained recycle handle vs per-slot handles (IRKA
recycling strategy 1): iterations, k_in per system."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import CONFIGS, system_sequence
from paper_1010_0762_b200 import api
cfg = CONFIGS["C4"]
nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 18
items = list(system_sequence(cfg, systems=list(range(nsys))))
ctx = api.Context(0)
out = {}
for mode in ("chain", "slots"):
    R1 = ctx.recycle(cfg.n, cfg.k, True)
    Rs = {}
    prev = {}
    its, kin, st = [], [], []
    for it in items:
        slot = it["slot"]
        R = R1 if mode == "chain" else Rs.setdefault(slot, ctx.recycle(cfg.n, cfg.k, True))
        M = ctx.matrix(it["indptr"], it["indices"], it["data"])
        x0, xt0 = prev.get(slot, (None, None))
        x, xt, res, _ = ctx.solve_dual(M, it["b"], it["bt"], x0, xt0, R=R, k=cfg.k, s=cfg.s, tol=cfg.tol,
                                       max_itn=cfg.max_itn, trunc_tol=cfg.trunc_tol)
        M.free()
        prev[slot] = (x, xt)
        its.append(res["iterations"]); kin.append(res["k_in"]); st.append(res["status_name"])
    out[mode] = dict(iterations=its, total=sum(its), k_in=kin, status=st)
print(json.dumps(out))
