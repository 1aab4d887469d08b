"""Thin Python API over the C ABI (names follow include/rbicg.h).

Host NumPy arrays are passed with on_device=0 (the library does the H2D/D2H
copies inside the call); torch CUDA tensors are passed with on_device=1.
No arithmetic of the method happens here.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import lib, check, Opts, Result, F64, C128


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        assert a.is_cuda and a.is_contiguous()
        return C.c_void_p(a.data_ptr())
    assert isinstance(a, np.ndarray) and a.flags.c_contiguous, type(a)
    return C.c_void_p(a.ctypes.data)


def _dtype_code(a):
    if _is_torch(a):
        import torch
        return C128 if a.dtype == torch.complex128 else F64
    return C128 if np.iscomplexobj(a) else F64


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 of a mode-0 group; broadcast it)."""
    buf = (C.c_uint8 * 128)()
    check(lib.rbicg_nccl_unique_id(buf))
    return bytes(buf)


class Context:
    """rbicg_ctx on one GPU; adopts torch's current stream when available.

    dist: None (one GPU) or dict(rank=q, nranks=P, mode=0|1, key=bytes[128])
    for the row-partitioned path (include/rbicg.h rbicg_dist): mode 0 = one
    process per GPU over NCCL (key = nccl_unique_id() of rank 0), mode 1 =
    virtual ranks (P contexts in P host threads of one process, any shared
    key)."""

    def __init__(self, device: int = 0, stream=None, dist=None):
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    torch.cuda.set_device(device)
                    stream = torch.cuda.current_stream(device).cuda_stream
            except ImportError:   # pragma: no cover
                stream = None
        self.device = device
        self._children = []          # weakrefs to matrices / recycle handles
        self._h = C.c_void_p()
        d = None
        self.rank, self.nranks = 0, 1
        if dist is not None:
            d = _lib.Dist()
            d.rank, d.nranks = int(dist["rank"]), int(dist["nranks"])
            d.mode = int(dist.get("mode", 0))
            d.force_partition = int(dist.get("force_partition", 0))
            key = bytes(dist["key"])[:128].ljust(128, b"\0")
            for i in range(128):
                d.nccl_id[i] = key[i]
            self.rank, self.nranks = d.rank, d.nranks
        check(lib.rbicg_init(C.byref(self._h), device,
                             C.c_void_p(stream) if stream else None,
                             C.byref(d) if d is not None else None))

    def close(self):
        if self._h:
            for ref in self._children:
                obj = ref()
                if obj is not None:
                    obj.free()
            self._children = []
            lib.rbicg_finalize(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ matrices
    def matrix(self, indptr, indices, data, shift=None):
        """Store of A; with shift=sigma the store of sigma I - A, formed on the
        device (rbicg_matrix_shifted_csr, IRKA's shifted systems)."""
        return Matrix(self, indptr, indices, data, shift=shift)

    def reduced_model(self, A, V, W, b, c):
        """(W^*AV, W^*V, W^*b, V^*c) of IRKA step 2d (rbicg_reduced_model):
        V, W of shape (r, n) (one solution per row, contiguous), b, c of
        length n, all numpy or all CUDA tensors of A's dtype.  Returns numpy
        arrays (r x r, r x r, r, r)."""
        r = int(V.shape[0])
        dev = _is_torch(V)
        if not dev:
            dt = np.complex128 if A.complex_ else np.float64
            V, W, b, c = (np.ascontiguousarray(a, dtype=dt) for a in (V, W, b, c))
        else:
            V, W, b, c = (a.contiguous() for a in (V, W, b, c))
        dt = np.complex128 if A.complex_ else np.float64
        Ar, Er = np.zeros((r, r), dt), np.zeros((r, r), dt)
        br, cr = np.zeros(r, dt), np.zeros(r, dt)
        check(lib.rbicg_reduced_model(self._h, A._h, r, _ptr(V), _ptr(W), _ptr(b), _ptr(c),
                                      1 if dev else 0, _ptr(Ar), _ptr(Er), _ptr(br), _ptr(cr)))
        return Ar, Er, br, cr

    def recycle(self, n, k_max, complex_=False):
        return Recycle(self, n, k_max, complex_)

    # ------------------------------------------------------------ solve
    def precond_ilut(self, indptr, indices, data, droptol=0.05):
        """Crout ILUT split preconditioner M = L U ≈ A (rbicg_prec_ilut,
        SURVEY §8(f) NEXT-4)."""
        return Precond(self, indptr, indices, data, droptol)

    def solve_dual(self, A, b, bt, x=None, xt=None, R=None, *, k=10, s=40,
                   tol=1e-8, max_itn=20000, trunc_tol=1e-6, update_recycle=True,
                   force_iters=0, xt_redraw=None, history=False, inplace=False,
                   pencil="plain", M=None):
        """inplace=True: x, xt (given, contiguous, b's dtype) are the in/out
        buffers themselves (e.g. page-locked host arrays); otherwise copies.
        pencil: "plain" (explicit Grams) or "fast" (§4.4 recurrences,
        rbicg_opts.pencil = 1).  M: a Precond -- split-preconditioned solve
        (rbicg_solve_dual_pc; the recycle space belongs to L^{-1}AU^{-1})."""
        if pencil not in ("plain", "fast"):
            raise ValueError(pencil)
        dev = _is_torch(b)
        if inplace:
            assert x is not None and xt is not None
        else:
            if x is None:
                x = b * 0
            if xt is None:
                xt = bt * 0
            if dev:
                x = x.clone()
                xt = xt.clone()
            else:
                x = np.array(x, dtype=b.dtype, copy=True)
                xt = np.array(xt, dtype=b.dtype, copy=True)
        o = Opts(k=k, s=s, max_itn=max_itn, tol=tol, trunc_tol=trunc_tol, seed=0,
                 update_recycle=1 if update_recycle else 0,
                 record_history=1 if history else 0, force_iters=force_iters,
                 pencil=1 if pencil == "fast" else 0)
        res = Result()
        hist = None
        if history:
            if dev:
                import torch
                hist = torch.zeros((max(max_itn, force_iters), 6),
                                   dtype=torch.float64, device=b.device)
            else:
                hist = np.zeros((max(max_itn, force_iters), 6))
        if M is not None:
            code = lib.rbicg_solve_dual_pc(self._h, A._h, M._h, _ptr(b), _ptr(bt), _ptr(x),
                                           _ptr(xt), _ptr(xt_redraw),
                                           R._h if R is not None else None,
                                           C.byref(o), 1 if dev else 0, C.byref(res),
                                           _ptr(hist))
        else:
            code = lib.rbicg_solve_dual(self._h, A._h, _ptr(b), _ptr(bt), _ptr(x),
                                        _ptr(xt), _ptr(xt_redraw),
                                        R._h if R is not None else None,
                                        C.byref(o), 1 if dev else 0, C.byref(res),
                                        _ptr(hist))
        check(code)
        r = res.as_dict()
        if hist is not None:
            hist = hist[:res.iterations]
        return x, xt, r, hist

    def bilinear(self, A, u, w, R=None, *, k=10, s=40, tol=1e-8, max_itn=20000,
                 trunc_tol=1e-6, update_recycle=True):
        dev = _is_torch(u)
        o = Opts(k=k, s=s, max_itn=max_itn, tol=tol, trunc_tol=trunc_tol,
                 update_recycle=1 if update_recycle else 0)
        res = Result()
        val = (C.c_double * 2)()
        check(lib.rbicg_bilinear(self._h, A._h, _ptr(u), _ptr(w),
                                 R._h if R is not None else None, C.byref(o),
                                 1 if dev else 0, val, C.byref(res)))
        v = complex(val[0], val[1]) if A.complex_ else val[0]
        return v, res.as_dict()

    # ------------------------------------------------------------ parity hooks
    def spmv_pair(self, A, p, pt):
        if _is_torch(p):
            z, zt = p.clone(), pt.clone()
        else:
            z, zt = np.empty_like(p), np.empty_like(pt)
        check(lib.rbicg_dbg_spmv_pair(self._h, A._h, _ptr(p), _ptr(pt), _ptr(z),
                                      _ptr(zt), 1 if _is_torch(p) else 0))
        return z, zt

    def project(self, A, R, z, zt, trunc_tol=1e-6):
        """Refreshed basis of R for A and ζ = D_c^{-1}C~^*z, ζ~ = D_c^{-1}C^*z~
        (host outputs; z, zt host arrays)."""
        n, kmax = A.n, R.k_max
        dt = np.complex128 if A.complex_ else np.float64
        zeta = np.zeros(max(kmax, 1), dt)
        zetat = np.zeros(max(kmax, 1), dt)
        kout = C.c_int32()
        mats = [np.zeros((max(kmax, 1), n), dt) for _ in range(4)]
        d = np.zeros(max(kmax, 1))
        check(lib.rbicg_dbg_project(self._h, A._h, R._h, trunc_tol, _ptr(z),
                                    _ptr(zt), _ptr(zeta), _ptr(zetat),
                                    C.byref(kout), *[_ptr(m) for m in mats],
                                    _ptr(d), 0))
        k = kout.value
        U, Ut, Cm, Ct = [m[:k].T.copy() for m in mats]
        return dict(k=k, zeta=zeta[:k], zetat=zetat[:k], U=U, Ut=Ut, C=Cm,
                    Ct=Ct, d=d[:k])

    def time_kernels(self, A, R=None, *, k=10, s=40, iters=20, trunc_tol=1e-6):
        o = Opts(k=k, s=s, max_itn=iters + 1, tol=0.0, trunc_tol=trunc_tol)
        ms = (C.c_double * 17)()
        check(lib.rbicg_dbg_time_kernels(self._h, A._h,
                                         R._h if R is not None else None,
                                         C.byref(o), iters, ms))
        return dict(pass1_ms=ms[0], pass2_ms=ms[1], done_flag=ms[2], k=int(ms[3]),
                    lazy_x=bool(ms[4]), tma_pass1=bool(ms[5]), graph_iter_ms=ms[6],
                    graph_done_flag=ms[7], loop_iter_ms=ms[8], loop_done_flag=ms[9],
                    pass1_graph_ms=ms[10], pass2_graph_ms=ms[11], graph_each_done_flag=ms[12],
                    shared_cols=bool(ms[13]), fused_ms=ms[14], fused_done_flag=ms[15],
                    dcols=bool(ms[16]))


class Matrix:
    """Device SELL-32 store of A and A^* (rbicg_matrix_csr)."""

    def __init__(self, ctx, indptr, indices, data, shift=None):
        self.ctx = ctx
        dev = _is_torch(data)
        if not dev:
            indptr = np.ascontiguousarray(indptr, dtype=np.int32)
            indices = np.ascontiguousarray(indices, dtype=np.int32)
            data = np.ascontiguousarray(data)
            if data.dtype not in (np.float64, np.complex128):
                data = data.astype(np.float64)
        self.n = int(len(indptr) - 1)
        self.nnz = int(len(indices))
        self.complex_ = _dtype_code(data) == C128
        self._h = C.c_void_p()
        ctx._children.append(weakref.ref(self))
        if shift is None:
            check(lib.rbicg_matrix_csr(ctx._h, self.n, self.nnz, _ptr(indptr),
                                       _ptr(indices), _ptr(data),
                                       C128 if self.complex_ else F64,
                                       1 if dev else 0, C.byref(self._h)))
        else:
            sg = complex(shift)
            check(lib.rbicg_matrix_shifted_csr(ctx._h, self.n, self.nnz, _ptr(indptr),
                                               _ptr(indices), _ptr(data),
                                               C128 if self.complex_ else F64,
                                               sg.real, sg.imag, 1 if dev else 0,
                                               C.byref(self._h)))

    def free(self):
        if self._h:
            lib.rbicg_matrix_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Precond:
    """Split preconditioner M = L U ≈ A by Crout ILUT (rbicg_prec_ilut)."""

    def __init__(self, ctx, indptr, indices, data, droptol):
        self.ctx = ctx
        dev = _is_torch(data)
        if not dev:
            indptr = np.ascontiguousarray(indptr, dtype=np.int32)
            indices = np.ascontiguousarray(indices, dtype=np.int32)
            data = np.ascontiguousarray(data)
            if data.dtype not in (np.float64, np.complex128):
                data = data.astype(np.float64)
        self.n = int(len(indptr) - 1)
        self.complex_ = _dtype_code(data) == C128
        self._h = C.c_void_p()
        ctx._children.append(weakref.ref(self))
        check(lib.rbicg_prec_ilut(ctx._h, self.n, int(len(indices)), _ptr(indptr), _ptr(indices),
                                  _ptr(data), C128 if self.complex_ else F64, float(droptol),
                                  1 if dev else 0, C.byref(self._h)))

    def factor(self, which):
        """scipy CSR of L (which="L", unit diagonal included) or U."""
        import scipy.sparse as sp
        w = 0 if which == "L" else 1
        nnz = C.c_int64()
        check(lib.rbicg_prec_export(self._h, w, None, None, None, C.byref(nnz)))
        rp = np.zeros(self.n + 1, np.int32)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        v = np.zeros(max(nnz.value, 1), np.complex128 if self.complex_ else np.float64)
        check(lib.rbicg_prec_export(self._h, w, _ptr(rp), _ptr(ci), _ptr(v), C.byref(nnz)))
        F = sp.csr_matrix((v[:nnz.value], ci[:nnz.value], rp), shape=(self.n, self.n))
        if which == "L":
            F = (F + sp.identity(self.n, dtype=v.dtype, format="csr")).tocsr()
        F.sort_indices()
        return F

    def free(self):
        if self._h:
            lib.rbicg_prec_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Recycle:
    """Recycle space handle (U, Ũ) carried between systems."""

    def __init__(self, ctx, n, k_max, complex_=False):
        self.ctx, self.n, self.k_max, self.complex_ = ctx, n, k_max, complex_
        self._h = C.c_void_p()
        ctx._children.append(weakref.ref(self))
        check(lib.rbicg_recycle_new(ctx._h, n, k_max, C128 if complex_ else F64,
                                    C.byref(self._h)))

    @property
    def k(self):
        k = C.c_int32()
        check(lib.rbicg_recycle_export(self._h, C.byref(k), None, None, 0))
        return k.value

    def export(self):
        dt = np.complex128 if self.complex_ else np.float64
        k = self.k
        U = np.zeros((max(k, 1), self.n), dt)
        Ut = np.zeros((max(k, 1), self.n), dt)
        kk = C.c_int32()
        check(lib.rbicg_recycle_export(self._h, C.byref(kk), _ptr(U), _ptr(Ut), 0))
        return U[:k].T.copy(), Ut[:k].T.copy()

    def import_(self, U, Ut):
        dt = np.complex128 if self.complex_ else np.float64
        k = U.shape[1]
        Uc = np.ascontiguousarray(np.asarray(U, dt).T)
        Utc = np.ascontiguousarray(np.asarray(Ut, dt).T)
        check(lib.rbicg_recycle_import(self._h, k, _ptr(Uc), _ptr(Utc), 0))

    def clear(self):
        """Empty the space (k = 0)."""
        check(lib.rbicg_recycle_import(self._h, 0, None, None, 0))

    def copy_from(self, other):
        """This handle's space := other's (device to device, through the C ABI
        export/import with on_device = 1)."""
        import torch
        k = other.k
        if k == 0:
            self.clear()
            return
        dt = torch.complex128 if other.complex_ else torch.float64
        dev = f"cuda:{self.ctx.device}"
        U = torch.empty((k, other.n), dtype=dt, device=dev)
        Ut = torch.empty((k, other.n), dtype=dt, device=dev)
        kk = C.c_int32()
        check(lib.rbicg_recycle_export(other._h, C.byref(kk), _ptr(U), _ptr(Ut), 1))
        check(lib.rbicg_recycle_import(self._h, k, _ptr(U), _ptr(Ut), 1))

    def free(self):
        if self._h:
            lib.rbicg_recycle_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def launch_count():
    return lib.rbicg_launch_count()
