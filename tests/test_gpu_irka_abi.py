"""IRKA entry points of the C ABI (NEXT-3; include/rbicg.h): the shifted
store σI - A formed on the device (rbicg_matrix_shifted_csr, the shifted
systems of Algorithm 3) and the reduced model
W^*AV, W^*V, W^*b, V^*c (rbicg_reduced_model) against
SciPy/NumPy on the same inputs, 1e-12 relative (BASELINE's per-call bar)."""
import numpy as np
import pytest
import scipy.sparse as sp

from synth import CONFIGS
from synth.small import random_sparse, vec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1010_0762_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def _with_diag(t):
    ip, ix, dv = t[:3]
    n = len(ip) - 1
    A = sp.csr_matrix((dv, ix, ip), shape=(n, n))
    A = (A + sp.identity(n, dtype=A.dtype, format="csr") * 0.5).tocsr()
    A.sort_indices()
    return A


@pytest.mark.parametrize("cplx,sigma", [(False, 0.7), (True, 0.3 + 1.1j), (True, -2.0)])
def test_shifted_store_matches_scipy(ctx, cplx, sigma):
    A = _with_diag(random_sparse(700, 0.02, seed=31, complex_=cplx))
    M = ctx.matrix(A.indptr, A.indices, A.data, shift=sigma)
    S = (sigma * sp.identity(A.shape[0], dtype=A.dtype) - A).tocsr()
    p, pt = vec(700, 32, cplx), vec(700, 33, cplx)
    z, zt = ctx.spmv_pair(M, p, pt)
    ez, ezt = S @ p, S.conj().T @ pt
    assert np.linalg.norm(z - ez) <= 1e-12 * np.linalg.norm(ez)
    assert np.linalg.norm(zt - ezt) <= 1e-12 * np.linalg.norm(ezt)
    M.free()


def test_shifted_store_c4_operator_device_arrays(ctx):
    """C4's K at 24^3 (synth.irka_operator) given as CUDA tensors: σI - K
    matches SciPy's SpMV pair."""
    import torch
    from synth.configs import irka_operator
    cfg = CONFIGS["C4"].scaled(24, systems=1)
    op = irka_operator(cfg, lam_r=0.0)
    n = op["n"]
    K = sp.csr_matrix((op["kdata"].astype(np.complex128), op["indices"], op["indptr"]),
                      shape=(n, n))
    sig = 0.25 + 0.5j
    d = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
         for a in (K.indptr.astype(np.int32), K.indices.astype(np.int32), K.data)]
    M = ctx.matrix(*d, shift=sig)
    p = torch.from_numpy(vec(n, 5, True)).cuda()
    z, zt = ctx.spmv_pair(M, p, p)
    S = (sig * sp.identity(n, dtype=np.complex128) - K).tocsr()
    ez, ezt = S @ p.cpu().numpy(), S.conj().T @ p.cpu().numpy()
    assert np.linalg.norm(z.cpu().numpy() - ez) <= 1e-12 * np.linalg.norm(ez)
    assert np.linalg.norm(zt.cpu().numpy() - ezt) <= 1e-12 * np.linalg.norm(ezt)
    M.free()


def test_shifted_store_rejects_missing_diagonal(ctx):
    from paper_1010_0762_b200._lib import RBiCGError
    A = sp.csr_matrix(np.array([[0.0, 1.0], [2.0, 3.0]]))
    A.eliminate_zeros()
    with pytest.raises(RBiCGError):
        ctx.matrix(A.indptr, A.indices, A.data, shift=1.0)
    with pytest.raises(RBiCGError):   # a complex shift of a real matrix
        ctx.matrix(A.indptr, A.indices, A.data + 1.0, shift=1j)


@pytest.mark.parametrize("cplx,r,n", [(True, 6, 3001), (False, 3, 999), (True, 1, 5000)])
@pytest.mark.parametrize("where", ["host", "device"])
def test_reduced_model_matches_numpy(ctx, cplx, r, n, where):
    A = _with_diag(random_sparse(n, 5.0 / n, seed=41, complex_=cplx))
    M = ctx.matrix(A.indptr, A.indices, A.data)
    V = np.stack([vec(n, 100 + i, cplx) for i in range(r)])
    W = np.stack([vec(n, 200 + i, cplx) for i in range(r)])
    b, c = vec(n, 300, cplx), vec(n, 301, cplx)
    if where == "device":
        import torch
        args = [torch.from_numpy(a).cuda() for a in (V, W, b, c)]
    else:
        args = [V, W, b, c]
    Ar, Er, br, cr = ctx.reduced_model(M, *args)
    AV = (A @ V.T)
    ref = (W.conj() @ AV, W.conj() @ V.T, W.conj() @ b, V.conj() @ c)
    for got, exp in zip((Ar, Er, br, cr), ref):
        assert np.linalg.norm(got - exp) <= 1e-12 * np.linalg.norm(exp)
    M.free()
