"""Debug: single-GPU vs P virtual ranks on the same RBiCG inputs (history)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, scipy.sparse as sp
from synth.small import deflation_matrix, vec, dense_to_csr, random_sparse
from oracle import rbicg as R
from paper_1010_0762_b200 import api
from test_gpu_dist import _solve_group
np.set_printoptions(precision=6, linewidth=200)
kind = sys.argv[1] if len(sys.argv) > 1 else "defl"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if kind == "defl":
    n, k = 240, 4
    A, lam, S = deflation_matrix(n, k, seed=43)
    t = dense_to_csr(A)
else:
    n, k = 400, 4
    t = random_sparse(n, 0.02, seed=9)
    A = sp.csr_matrix((t[2], t[1], t[0]), shape=(n, n)).toarray()
Ad = sp.csr_matrix(A)
first = R.solve_dual(Ad, vec(n, 44), vec(n, 45), k=k, s=10, tol=1e-10, max_itn=1000, trunc_tol=1e-6)
U, Ut = first.basis_out.U, first.basis_out.Ut
b, bt = vec(n, 46), vec(n, 47)
m = int(sys.argv[3]) if len(sys.argv) > 3 else 7
ref = R.solve_dual(Ad, b, bt, U=U, Ut=Ut, k=k, s=10, tol=1e-10, max_itn=1000, trunc_tol=1e-6, force_iters=m)
ctx = api.Context(0)
M = ctx.matrix(*t)
rec = ctx.recycle(n, k); rec.import_(U, Ut)
x1, xt1, res1, h1 = ctx.solve_dual(M, b, bt, R=rec, k=k, s=10, tol=1e-10, max_itn=1000, trunc_tol=1e-6, force_iters=m, history=True)
x2, xt2, res2, h2, _, _ = _solve_group(P, t, b, bt, k, 10, 1e-10, 1000, 1e-6, U, Ut, force=m, history=True)
print("oracle alpha", np.real(ref.hist["alpha"])[:m])
print("gpu1   alpha", h1[:, 2])
print("gpuP   alpha", h2[:, 2])
print("gpu1 relres", h1[:, 0])
print("gpuP relres", h2[:, 0])
print("res1", {k_: res1[k_] for k_ in ("iterations", "k_in", "relres_rec", "relres_true")})
print("resP", {k_: res2[k_] for k_ in ("iterations", "k_in", "relres_rec", "relres_true")})
print("x err 1", np.linalg.norm(x1 - ref.x) / np.linalg.norm(ref.x), "P", np.linalg.norm(x2 - ref.x) / np.linalg.norm(ref.x))
