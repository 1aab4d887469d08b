"""ctypes binding of librbicg.so (include/rbicg.h) -- argument marshalling only.

Every numerical step runs inside the library's sm_100a kernels; this module
only converts Python/NumPy/torch arguments to pointers.  Missing library =>
loud ImportError (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import glob
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librbicg.so")


def _lapack_path():
    """OpenBLAS shipped inside scipy (no system LAPACK in this image)."""
    try:
        import scipy
    except ImportError:      # pragma: no cover
        return None
    base = os.path.dirname(os.path.dirname(scipy.__file__))
    libs = sorted(glob.glob(os.path.join(base, "scipy.libs",
                                         "libscipy_openblas*.so")))
    return libs[0] if libs else None


def _nccl_path():
    """The NCCL that ships with torch (nvidia-nccl wheel), for the row-partitioned path."""
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except ImportError:      # pragma: no cover
        pass
    return None


if "RBICG_NCCL" not in os.environ:
    _p = _nccl_path()
    if _p:
        os.environ["RBICG_NCCL"] = _p

if "RBICG_LAPACK" not in os.environ:
    _p = _lapack_path()
    if _p:
        os.environ["RBICG_LAPACK"] = _p

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import "
        "__graft_entry__ as g; g.build()'` (there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

F64, C128 = 0, 1
STATUS = {0: "ok", 1: "maxiter", 2: "breakdown_serious", 3: "breakdown_second",
          4: "recycle_empty"}


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_id", C.c_uint8 * 128), ("row_begin", C.c_int64),
                ("row_end", C.c_int64), ("mode", C.c_int32),
                ("force_partition", C.c_int32)]


class Opts(C.Structure):
    _fields_ = [("k", C.c_int32), ("s", C.c_int32), ("max_itn", C.c_int32),
                ("tol", C.c_double), ("trunc_tol", C.c_double),
                ("seed", C.c_uint64), ("update_recycle", C.c_int32),
                ("record_history", C.c_int32), ("force_iters", C.c_int32),
                ("pencil", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int32),
                ("cycles", C.c_int32), ("k_in", C.c_int32), ("k_out", C.c_int32),
                ("relres_rec", C.c_double), ("relres_dual_rec", C.c_double),
                ("relres_true", C.c_double), ("relres_dual_true", C.c_double),
                ("t_loop_ms", C.c_double), ("t_cycle_dev_ms", C.c_double),
                ("t_host_eig_ms", C.c_double), ("t_refresh_ms", C.c_double),
                ("t_total_ms", C.c_double), ("alg_bytes", C.c_double),
                ("kernel_launches", C.c_int32), ("lookahead_cancellations", C.c_int32)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["status_name"] = STATUS.get(self.status, str(self.status))
        return d


vp = C.c_void_p
_sig = {
    "rbicg_init": (C.c_int, [C.POINTER(vp), C.c_int, vp, C.POINTER(Dist)]),
    "rbicg_finalize": (C.c_int, [vp]),
    "rbicg_matrix_csr": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, C.c_int,
                                   C.c_int, C.POINTER(vp)]),
    "rbicg_matrix_shifted_csr": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, C.c_int,
                                           C.c_double, C.c_double, C.c_int, C.POINTER(vp)]),
    "rbicg_reduced_model": (C.c_int, [vp, vp, C.c_int32, vp, vp, vp, vp, C.c_int,
                                      vp, vp, vp, vp]),
    "rbicg_matrix_free": (C.c_int, [vp]),
    "rbicg_recycle_new": (C.c_int, [vp, C.c_int64, C.c_int32, C.c_int,
                                    C.POINTER(vp)]),
    "rbicg_recycle_export": (C.c_int, [vp, C.POINTER(C.c_int32), vp, vp, C.c_int]),
    "rbicg_recycle_import": (C.c_int, [vp, C.c_int32, vp, vp, C.c_int]),
    "rbicg_recycle_free": (C.c_int, [vp]),
    "rbicg_solve_dual": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp,
                                   C.POINTER(Opts), C.c_int, C.POINTER(Result),
                                   vp]),
    "rbicg_prec_ilut": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, C.c_int, C.c_double,
                                  C.c_int, C.POINTER(vp)]),
    "rbicg_prec_free": (C.c_int, [vp]),
    "rbicg_prec_export": (C.c_int, [vp, C.c_int, vp, vp, vp, C.POINTER(C.c_int64)]),
    "rbicg_solve_dual_pc": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      C.POINTER(Opts), C.c_int, C.POINTER(Result), vp]),
    "rbicg_bilinear": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(Opts), C.c_int,
                                 vp, C.POINTER(Result)]),
    "rbicg_dbg_spmv_pair": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int]),
    "rbicg_dbg_project": (C.c_int, [vp, vp, vp, C.c_double, vp, vp, vp, vp,
                                    C.POINTER(C.c_int32), vp, vp, vp, vp, vp,
                                    C.c_int]),
    "rbicg_dbg_time_kernels": (C.c_int, [vp, vp, vp, C.POINTER(Opts), C.c_int,
                                         vp]),
    "rbicg_plan_partition": (C.c_int, [C.c_int64, vp, vp, C.c_int32, C.c_int32,
                                       vp, vp, vp, vp, vp, vp, vp]),
    "rbicg_nccl_unique_id": (C.c_int, [vp]),
    "rbicg_strerror": (C.c_char_p, [C.c_int]),
    "rbicg_launch_count": (C.c_int64, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


class RBiCGError(RuntimeError):
    pass


def check(code):
    if code < 0:
        raise RBiCGError(f"librbicg: {lib.rbicg_strerror(code).decode()} ({code})")
    return code
