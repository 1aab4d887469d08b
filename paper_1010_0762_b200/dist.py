"""Row-partition plan of the multi-GPU path (rbicg_plan_partition, host-only).

Marshalling only: the plan is computed by the library's host code
(csrc/dist.cpp) and is the same plan the device halo exchange uses.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib, check


def plan_partition(indptr, indices, nranks: int, rank: int) -> dict:
    indptr = np.ascontiguousarray(indptr, dtype=np.int32)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    n = len(indptr) - 1
    counts = np.zeros(6, dtype=np.int64)
    p = lambda a: C.c_void_p(a.ctypes.data) if a is not None else None
    check(lib.rbicg_plan_partition(n, p(indptr), p(indices), nranks, rank, p(counts),
                                   None, None, None, None, None, None))
    r0, r1, ng, nr, ns, nsi = (int(v) for v in counts)
    ghost = np.zeros(max(ng, 1), np.int64)
    recv_nbr = np.zeros(max(nr, 1), np.int32)
    recv_cnt = np.zeros(max(nr, 1), np.int64)
    send_nbr = np.zeros(max(ns, 1), np.int32)
    send_cnt = np.zeros(max(ns, 1), np.int64)
    send_idx = np.zeros(max(nsi, 1), np.int32)
    check(lib.rbicg_plan_partition(n, p(indptr), p(indices), nranks, rank, p(counts),
                                   p(ghost), p(recv_nbr), p(recv_cnt), p(send_nbr),
                                   p(send_cnt), p(send_idx)))
    return dict(row_begin=r0, row_end=r1, ghost=ghost[:ng], recv_nbr=recv_nbr[:nr],
                recv_cnt=recv_cnt[:nr], send_nbr=send_nbr[:ns], send_cnt=send_cnt[:ns],
                send_idx=send_idx[:nsi])
