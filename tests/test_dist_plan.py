"""Host logic of the multi-GPU row partition (CPU only, ``-m "not gpu"``).

* the partition plan of every rank is consistent with every other rank's
  (what q sends to q' is exactly q''s ghosts owned by q, in q''s order);
* a world-size-2 ``gloo`` job runs the row-partitioned BiCG exactly the way
  the device path does (halo of p, r and their duals before the SpMV pair,
  sum-allreduce of the scalar batches) using the library's plan, and
  reproduces the serial oracle's iterates.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from synth import CONFIGS, system_sequence
from synth.small import random_sparse, vec


def _plan(indptr, indices, P, q):
    from paper_1010_0762_b200.dist import plan_partition
    return plan_partition(indptr, indices, P, q)


def _local(pl, c):
    r0, r1 = pl["row_begin"], pl["row_end"]
    if r0 <= c < r1:
        return c - r0
    return (r1 - r0) + int(np.searchsorted(pl["ghost"], c))


@pytest.mark.parametrize("P", [2, 3, 5])
def test_plans_are_mutually_consistent(P):
    cfg = CONFIGS["C2"].scaled(12, systems=1)
    it = next(system_sequence(cfg))
    indptr, indices, n = it["indptr"], it["indices"], it["n"]
    plans = [_plan(indptr, indices, P, q) for q in range(P)]
    assert plans[0]["row_begin"] == 0 and plans[-1]["row_end"] == n
    for q in range(P - 1):
        assert plans[q]["row_end"] == plans[q + 1]["row_begin"]
    A = sp.csr_matrix((it["data"], indices, indptr), shape=(n, n))
    AH = A.conj().T.tocsr()
    for q, pl in enumerate(plans):
        r0, r1 = pl["row_begin"], pl["row_end"]
        # ghosts = off-block columns of local rows of A and A^*
        want = set()
        for M in (A, AH):
            sub = M[r0:r1]
            want |= {c for c in sub.indices if not (r0 <= c < r1)}
        assert sorted(want) == list(pl["ghost"])
        # receive ranges follow ownership
        off = 0
        for o, cnt in zip(pl["recv_nbr"], pl["recv_cnt"]):
            g = pl["ghost"][off:off + cnt]
            assert np.all((g >= plans[o]["row_begin"]) & (g < plans[o]["row_end"]))
            off += cnt
        assert off == len(pl["ghost"])
        # what each owner sends me, in my ghost order
        for o, cnt in zip(pl["recv_nbr"], pl["recv_cnt"]):
            po = plans[o]
            j = list(po["send_nbr"]).index(q)
            start = int(np.sum(po["send_cnt"][:j]))
            sent = po["send_idx"][start:start + po["send_cnt"][j]] + po["row_begin"]
            mine = [c for c in pl["ghost"] if po["row_begin"] <= c < po["row_end"]]
            assert list(sent) == mine


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_bicg_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = random_sparse(90, 0.06, seed=7)
        indptr, indices, data = t
        n = len(indptr) - 1
        A = sp.csr_matrix((data, indices, indptr), shape=(n, n))
        AH = A.T.tocsr()
        b, bt = vec(n, 8), vec(n, 9)
        pl = _plan(indptr, indices, world, rank)
        r0, r1 = pl["row_begin"], pl["row_end"]
        nloc, ng = r1 - r0, len(pl["ghost"])

        def local_mat(M):
            sub = M[r0:r1].tocoo()
            cols = np.array([_local(pl, c) for c in sub.col])
            return sp.csr_matrix((sub.data, (sub.row, cols)), shape=(nloc, nloc + ng))

        Al, AHl = local_mat(A), local_mat(AH)

        def halo(vecs):
            """send own boundary values, receive ghosts (grouped sends/recvs)"""
            ext = [np.concatenate([v, np.zeros(ng)]) for v in vecs]
            reqs = []
            off = 0
            for o, cnt in zip(pl["send_nbr"], pl["send_cnt"]):
                idx = pl["send_idx"][off:off + cnt]
                buf = torch.from_numpy(np.concatenate([v[idx] for v in vecs]).copy())
                reqs.append(dist.isend(buf, int(o)))
                off += cnt
            off = 0
            for o, cnt in zip(pl["recv_nbr"], pl["recv_cnt"]):
                buf = torch.zeros(len(vecs) * int(cnt), dtype=torch.float64)
                dist.recv(buf, int(o))
                for j, e in enumerate(ext):
                    e[nloc + off:nloc + off + cnt] = buf[j * cnt:(j + 1) * cnt].numpy()
                off += cnt
            for r in reqs:
                r.wait()
            return ext

        def allsum(vals):
            t = torch.tensor(vals, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        r, rt = b[r0:r1].copy(), bt[r0:r1].copy()
        x, xt = np.zeros(nloc), np.zeros(nloc)
        p, pt = np.zeros(nloc), np.zeros(nloc)
        rho = allsum([rt @ r])[0]
        beta = 0.0
        for i in range(q["iters"]):
            # the device path gathers r and p_old at ghost columns (fused
            # direction update): halo of r, p, r~, p~ before the SpMV pair
            re_, pe, rte, pte = halo([r, p, rt, pt])
            pext, ptext = re_ + beta * pe, rte + beta * pte
            p, pt = pext[:nloc], ptext[:nloc]
            z, zt = Al @ pext, AHl @ ptext
            sigma = allsum([pt @ z])[0]                # allreduce #1
            alpha = rho / sigma
            x += alpha * p
            xt += alpha * pt
            r = r - alpha * z
            rt = rt - alpha * zt
            rho_new = allsum([rt @ r])[0]              # allreduce #2
            beta = rho_new / rho
            rho = rho_new
        xs = [None] * world
        dist.all_gather_object(xs, (r0, x))
        if rank == 0:
            q["x"] = np.concatenate([v for _, v in sorted(xs)])
            np.save(q["out"], q["x"])
    finally:
        dist.destroy_process_group()


def test_gloo_world2_row_partitioned_bicg_matches_serial(tmp_path):
    import torch.multiprocessing as mp
    from oracle.bicg import bicg
    t = random_sparse(90, 0.06, seed=7)
    n = len(t[0]) - 1
    A = sp.csr_matrix((t[2], t[1], t[0]), shape=(n, n))
    b, bt = vec(n, 8), vec(n, 9)
    iters = 25
    ref = bicg(A, b, bt, np.zeros(n), np.zeros(n), 1e-30, iters, force_iters=iters)
    out = str(tmp_path / "x.npy")
    mp.spawn(_dist_bicg_worker, args=(2, _free_port(), {"iters": iters, "out": out}),
             nprocs=2, join=True)
    x = np.load(out)
    assert np.linalg.norm(x - ref["x"]) <= 1e-10 * np.linalg.norm(ref["x"])
