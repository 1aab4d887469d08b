#!/usr/bin/env python
"""RBiCG iterations/s on B200 (BASELINE.json metric) -- one JSON line.

Workload (N=1, default): BASELINE.json configs[2] = C3, the 3-D conv-diff
sequence on a 192^3 grid (n = 7,077,888, nnz = 49.3 M, fp64, k = 10, s = 40,
tol 1e-8, 8 dual pairs; synthetic, seeded per SURVEY.md §8(d)) -- a config of
the metric's 1/2/4/8-GPU set.  Under the recycle rule (Q13 at the
paper's 1e-6, Q32) a system starts with the recycle space the previous one
left after truncation: `config.k_in_per_system` records its width (C3 chain:
4, 0, 5, 0, 0 on the timed systems), systems with k_in > 0 run the augmented
iteration with its projections, the others plain BiCG steps plus the
cycle-end recycle updates (DESIGN §3 table).
--config C2|C4|C5 selects another config.

A *step* is one dual-pair solve of the sequence through the C ABI
(rbicg_matrix_csr from device CSR -> SELL-32 + conj-transpose build,
rbicg_solve_dual: refresh, init, the graph-replayed hot loop, cycle-end
recycle updates, step 7, true residuals), carrying the recycle space from
system to system.  value = iterations / device time of the K timed steps.

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize and
CUDA events; max over ranks.  Per-iteration traffic (C3: 1.7 GB with k = 1,
4.1 GB with k = 10; C2: 0.2 GB) is larger than the 126 MB L2 except C2's
(L2 hits of the vectors written by the previous launch are counted by ncu's
DRAM bytes in `roofline.traffic`), so no explicit flush is needed.

roofline: the dominant hot-loop kernel of the last timed system's matrix and
recycle space, each kernel timed alone as back-to-back launches in a CUDA
graph on the library stream; `traffic` = ncu DRAM bytes per launch of the
same kernel, captured in-run by a subprocess after the timed region
(scripts/kernel_traffic.py, same config and recycle width).

--impl reference runs the CPU oracle (the only other allowed use of oracle/)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
DEFAULT_CONFIG = "C3"
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's own start-up (driver queries) must not fall into the
            # timed region: wait for its first sample (it stalled the first
            # timed C4 solve by up to 40 ms otherwise)
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_systems(cfg, idx):
    from synth import system_sequence
    want = sorted(set(j % cfg.systems for j in idx))
    got = {it["j"]: it for it in system_sequence(cfg, systems=want)}
    return [got[j % cfg.systems] for j in idx]


def workload_name(cfg):
    if cfg.kind == "irka":
        op = (f"IRKA-like shifted systems (sigma I - K), K = -(3-D Laplacian {cfg.N}^3) + "
              f"0.1 N(0,1) off-diagonal perturbation, complex128, 10 sweeps x 6 shifts")
    else:
        op = f"{cfg.d}-D {cfg.scheme} conv-diff {cfg.N}^{cfg.d}"
    return (f"{cfg.name}: {op}, n={cfg.n}, nnz={cfg.nnz}, k={cfg.k}, s={cfg.s}, "
            f"tol={cfg.tol}, trunc_tol={cfg.trunc_tol}")


def alg_bytes(cfg_n, nnz, k, w=8, lazy_x=True, shared_cols=False):
    """Algorithmic HBM bytes per launch of the two hot kernels:
    pass 1 streams A and A^* (CSR-equivalent: values + int32 column indices +
    row pointers; one column array for both when A is structurally symmetric),
    C and C~ once, reads r, p, r~, p~ and writes p, p~, z, z~;
    pass 2 reads C, C~, z, z~, r, r~ and writes r, r~ (with lazy x; eager x
    adds reads of x, x~, p, p~ and writes of x, x~)."""
    mat = 2 * (nnz * (w + 4) + 4 * (cfg_n + 1)) - (4 * nnz if shared_cols else 0)
    p1 = mat + 2 * k * cfg_n * w + 8 * cfg_n * w
    p2 = 2 * k * cfg_n * w + (6 if lazy_x else 12) * cfg_n * w
    return p1, p2


def alg_bytes_fused(cfg_n, nnz, w=8, shared_cols=False, dcols=False):
    """Algorithmic HBM bytes per launch of the fused iteration kernel (k = 0,
    DESIGN.md §6): the A, A^* streams as in pass 1, reads r_{i-2}, z_{i-1},
    p_{i-1} and writes r_{i-1}, z_i, p_i on both sides (12 n-vectors); with
    int16 column deltas (banded A) the shared pattern costs 2 bytes per nonzero."""
    mat = 2 * (nnz * (w + 4) + 4 * (cfg_n + 1)) - (4 * nnz if shared_cols else 0)
    if shared_cols and dcols:
        mat -= 2 * nnz
    return mat + 12 * cfg_n * w


NCU_KERNELS = {"pass1": "k_pass1", "pass2": "k_pass2", "fused": "k_fused"}


def ncu_traffic(cfg, k, dom):
    """ncu DRAM bytes (read + write) per launch of the dominant kernel, from a
    subprocess run of scripts/kernel_traffic.py on the same config and
    recycle width (after the timed region; its times are never reported)."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    name = NCU_KERNELS[dom]
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum",
           "--kernel-name", f"regex:^{name}", "--launch-skip", "2", "--launch-count", "3",
           "--csv", "--clock-control", "none", sys.executable,
           os.path.join(ROOT, "scripts", "kernel_traffic.py"), cfg.name, str(k)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    except Exception as e:   # noqa: BLE001
        return None, f"ncu failed: {e}"
    rows = [r for r in csv.reader(io.StringIO(out.stdout)) if len(r) > 10]
    start = [i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r]
    if not start:
        return None, "ncu produced no rows (rc %d): %s" % (out.returncode, out.stderr[-200:])
    rows = rows[start[0]:]
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                       hdr.index("Metric Value"), hdr.index("ID"))
    per = {}
    for r in rows[1:]:
        if not re.search(rf"(^|[\s:]){name}s?<", r[ik]):
            continue
        v = float(r[iv].replace(",", ""))
        per.setdefault(r[iid], 0.0)
        per[r[iid]] += v
    if not per:
        return None, "no %s launches in the capture" % name
    unit = "byte"
    for r in rows[1:]:
        if re.search(rf"(^|[\s:]){name}s?<", r[ik]):
            unit = r[hdr.index("Metric Unit")]
            break
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    vals = [v * scale for v in per.values()]
    return sum(vals) / len(vals), (f"ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                   f"{name} (k = {k}), mean of {len(vals)} launches, "
                                   f"scripts/kernel_traffic.py {cfg.name} {k}")


def run_gpu(args, rank, world):
    import torch
    from paper_1010_0762_b200 import api
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    # N > 1: the row-partitioned path -- every rank holds a row
    # block, halo exchange + scalar allreduces over NCCL; --replicas runs N
    # independent copies instead.
    part = world > 1 and not args.replicas
    r0, r1 = 0, cfg.n
    if part:
        import torch.distributed as tdist
        obj = [api.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        ctx = api.Context(dev, dist=dict(rank=rank, nranks=world, mode=0, key=obj[0]))
        r0, r1 = (cfg.n * rank) // world, (cfg.n * (rank + 1)) // world
    else:
        ctx = api.Context(dev)
    steps = args.warmup + args.steps
    systems = build_systems(cfg, list(range(steps)))
    # inputs resident in HBM before the timed region (the matrix is passed
    # whole; vectors are this rank's rows)
    def local_csr(it):
        """This rank's rows of A: local rowptr, GLOBAL columns (§8(b))."""
        ip = it["indptr"]
        a, b = int(ip[r0]), int(ip[r1])
        return {"indptr": np.ascontiguousarray(ip[r0:r1 + 1] - ip[r0], dtype=np.int32),
                "indices": np.ascontiguousarray(it["indices"][a:b]),
                "data": np.ascontiguousarray(it["data"][a:b])}

    def upload(it):
        loc = local_csr(it)
        d = {k: torch.from_numpy(loc[k]).to(f"cuda:{dev}") for k in ("indptr", "indices", "data")}
        for k in ("b", "bt"):
            d[k] = torch.from_numpy(np.ascontiguousarray(it[k][r0:r1])).to(f"cuda:{dev}")
        return d
    # the timed systems are resident before the timed region; a warm-up
    # system is uploaded for its step and dropped after it (C5: ~6 GB each)
    dsys = [None] * args.warmup + [upload(it) for it in systems[args.warmup:]]
    torch.cuda.synchronize()
    R = ctx.recycle(r1 - r0, cfg.k, cfg.complex)
    stream = torch.cuda.current_stream()
    res_all, times = [], []

    build_ms = []
    host_ms = []   # (solve_dual call, free) wall ms per timed step

    prev = {}   # C4 (Q7): previous sweep's solution of the same shift slot

    # the roofline times the hot-loop kernels with the largest input space a
    # timed system started from (copied device to device before that step,
    # outside its events) -- the iteration the timed region mostly ran
    snap = {"R": None, "k": 0}
    # (not for spaces over 8 GB -- C5 with k = 20 on one GPU needs the memory;
    # the roofline then times the space the sequence ends with)
    snap_ok = 2 * cfg.n * cfg.k * (16 if cfg.complex else 8) <= 8 << 30

    def one(i, timed):
        d = dsys[i] if dsys[i] is not None else upload(systems[i])
        slot = systems[i].get("slot")
        if timed and not part and snap_ok:
            kin = R.k
            if kin > snap["k"]:
                if snap["R"] is None:
                    snap["R"] = ctx.recycle(r1 - r0, cfg.k, cfg.complex)
                snap["R"].copy_from(R)
                snap["k"] = kin
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        A = ctx.matrix(d["indptr"], d["indices"], d["data"])
        eb.record(stream)
        eb.synchronize()
        if timed:
            build_ms.append(e0.elapsed_time(eb))
        t0 = time.perf_counter()
        x0, xt0 = prev.get(slot, (None, None))
        x, xt, res, _ = ctx.solve_dual(A, d["b"], d["bt"], x0, xt0, R=R, k=cfg.k, s=cfg.s,
                                       tol=cfg.tol, max_itn=cfg.max_itn,
                                       trunc_tol=cfg.trunc_tol,
                                       update_recycle=not args.no_update)
        if slot is not None:
            prev[slot] = (x, xt)
        t1 = time.perf_counter()
        A.free()
        e1.record(stream)
        e1.synchronize()
        if timed:
            host_ms.append((round(1e3 * (t1 - t0), 2), round(1e3 * (time.perf_counter() - t1), 2)))
        return res, e0.elapsed_time(e1)

    for i in range(args.warmup):
        one(i, False)
    torch.cuda.empty_cache()   # the dropped warm-up inputs go back to the device
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    clk.start()
    l0 = api.launch_count()
    for i in range(args.warmup, steps):
        r, ms = one(i, True)
        res_all.append(r)
        times.append(ms)
    torch.cuda.synchronize()
    launches = api.launch_count() - l0
    clocks = clk.stop()
    if world > 1:
        torch.distributed.barrier()
    total_ms = float(sum(times))
    iters = int(sum(r["iterations"] for r in res_all))
    t = torch.tensor([total_ms, iters], dtype=torch.float64, device=f"cuda:{dev}")
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax[:1], op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum[1:], op=torch.distributed.ReduceOp.SUM)
        # partitioned: every rank did the same (replicated) iterations
        total_ms = float(tmax[0])
        iters = int(tsum[1]) // world if part else int(tsum[1])

    # ---- roofline of the dominant kernel: per-kernel CUDA events on the
    # library stream, resident state of the last system and the recycle space
    # the sequence carries (the timed systems' own k)
    last = dsys[-1]
    kctx, kR = ctx, (snap["R"] if snap["R"] is not None else R)
    if part:   # the partitioned context has no timing hook: the kernels on one GPU
        kctx = api.Context(dev)
        kR = kctx.recycle(cfg.n, cfg.k, cfg.complex)
    if part:
        g = systems[-1]
        A = kctx.matrix(g["indptr"], g["indices"], g["data"])
    else:
        A = kctx.matrix(last["indptr"], last["indices"], last["data"])
    kt = kctx.time_kernels(A, kR, k=cfg.k, s=cfg.s, iters=args.kernel_iters,
                           trunc_tol=cfg.trunc_tol)
    A.free()
    w = 16 if cfg.complex else 8
    p1, p2 = alg_bytes(cfg.n, cfg.nnz, kt["k"], w, kt["lazy_x"], kt["shared_cols"])
    peak, peak_kind = hbm_peak()
    # kernel durations: each kernel as back-to-back launches in one CUDA graph
    # (CUDA events around the graph on the library stream) -- its duration
    # inside the solver's loop graph; the event-bracketed single launches
    # (which add the host launch gap) are reported beside them
    ok = kt["graph_each_done_flag"] == 0 and kt["pass1_graph_ms"] > 0
    k1 = kt["pass1_graph_ms"] if ok else kt["pass1_ms"]
    k2 = kt["pass2_graph_ms"] if ok else kt["pass2_ms"]
    dom_bytes, dom_ms, dom = (p1, k1, "pass1") if k1 >= k2 else (p2, k2, "pass2")
    # without a recycle space the solver's loop runs the fused iteration
    # kernel: that kernel is then the dominant one
    fused = kt["k"] == 0 and kt["fused_ms"] > 0 and kt["fused_done_flag"] == 0
    pf = alg_bytes_fused(cfg.n, cfg.nnz, w, kt["shared_cols"], kt["dcols"])
    if fused:
        dom_bytes, dom_ms, dom = pf, kt["fused_ms"], "fused"
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic, traffic_info = None, "skipped (--no-traffic)"
    if not args.no_traffic and rank == 0:
        try:
            traffic, traffic_info = ncu_traffic(cfg, kt["k"], dom)
        except Exception as e:   # noqa: BLE001  (a profiler problem never fails the bench)
            traffic, traffic_info = None, f"ncu capture failed: {e!r}"

    # C2-type workloads end without a recycle space: probe the k = cfg.k
    # iteration on a seeded random space so its kernels are measured too
    probe = None
    if kt["k"] == 0 and cfg.k > 0 and not args.no_k_probe and cfg.n <= 16_000_000:
        g = systems[-1] if part else last
        A = kctx.matrix(g["indptr"], g["indices"], g["data"])
        rng = np.random.default_rng(cfg.seed + 777)
        shp = (cfg.n, cfg.k)
        if cfg.complex:
            Uq = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
            Utq = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
        else:
            Uq, Utq = rng.standard_normal(shp), rng.standard_normal(shp)
        Rq = kctx.recycle(cfg.n, cfg.k, cfg.complex)
        Rq.import_(Uq, Utq)
        del Uq, Utq
        kq = kctx.time_kernels(A, Rq, k=cfg.k, s=cfg.s, iters=args.kernel_iters,
                               trunc_tol=1e-300)
        q1, q2 = alg_bytes(cfg.n, cfg.nnz, kq["k"], w, kq["lazy_x"], kq["shared_cols"])
        okq = kq["graph_each_done_flag"] == 0 and kq["pass1_graph_ms"] > 0
        m1 = kq["pass1_graph_ms"] if okq else kq["pass1_ms"]
        m2 = kq["pass2_graph_ms"] if okq else kq["pass2_ms"]
        probe = {"k_active": kq["k"], "pass1_ms": m1, "pass2_ms": m2,
                 "pass1_GBps": q1 / (m1 * 1e-3) / 1e9, "pass2_GBps": q2 / (m2 * 1e-3) / 1e9,
                 "loop_graph_iter_ms": kq["graph_iter_ms"],
                 "iter_GBps": (q1 + q2) / (kq["graph_iter_ms"] * 1e-3) / 1e9,
                 "iter_frac": (q1 + q2) / (kq["graph_iter_ms"] * 1e-3) / 1e9 / peak,
                 "alg_bytes_per_iter": q1 + q2,
                 "space": "seeded N(0,1) U, U~ (%d columns), truncation off" % cfg.k}
        A.free()

    # ---- e2e through the public API with HOST buffers (H2D/D2H in the call)
    e2e = None
    if not args.no_e2e:
        R2 = ctx.recycle(r1 - r0, cfg.k, cfg.complex)

        def pinned(a):   # NumPy view of page-locked host memory holding a copy of a
            t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
            out = t.numpy()
            out[...] = a
            return out
        h_sys = []
        for it in systems[args.warmup:steps]:
            loc = local_csr(it)
            hs = {k: pinned(loc[k]) for k in ("indptr", "indices", "data")}
            for k in ("b", "bt"):
                hs[k] = pinned(np.ascontiguousarray(it[k][r0:r1]))
            hs["x"] = pinned(np.zeros_like(hs["b"]))
            hs["xt"] = pinned(np.zeros_like(hs["bt"]))
            h_sys.append(hs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ei, h2d, d2h = 0, 0, 0
        per = []
        for it in h_sys:
            ts = time.perf_counter()
            A = ctx.matrix(it["indptr"], it["indices"], it["data"])
            x, xt, res, _ = ctx.solve_dual(A, it["b"], it["bt"], it["x"], it["xt"], R=R2, k=cfg.k,
                                           s=cfg.s, tol=cfg.tol,
                                           max_itn=cfg.max_itn,
                                           trunc_tol=cfg.trunc_tol, inplace=True)
            A.free()
            ei += res["iterations"]
            h2d += it["indptr"].nbytes + it["indices"].nbytes + it["data"].nbytes \
                + it["b"].nbytes + it["bt"].nbytes + it["x"].nbytes + it["xt"].nbytes
            d2h += x.nbytes + xt.nbytes
            per.append(round(1e3 * (time.perf_counter() - ts), 2))
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:   # whole job: slowest rank; iterations replicated (partition) or summed
            tt = torch.tensor([el, ei], dtype=torch.float64, device=f"cuda:{dev}")
            tm = tt.clone()
            torch.distributed.all_reduce(tm[:1], op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(tt[1:], op=torch.distributed.ReduceOp.SUM)
            el, ei = float(tm[0]), float(tt[1]) / (world if part else 1)
        e2e = {"value": ei / el, "unit": "iterations/s",
               "h2d_bytes_per_step": h2d // max(1, len(h_sys)),
               "d2h_bytes_per_step": d2h // max(1, len(h_sys)),
               "ms_per_system": per}

    out = {
        "metric": "RBiCG iterations/sec (dual pair) and achieved HBM GB/s",
        "value": iters / (total_ms * 1e-3),
        "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / max(1, args.steps),
        "higher_is_better": True,
        "scaling": "strong" if part else "weak",
        "vs_baseline": None,
        "dtype": "c128" if cfg.complex else "f64",
        "data": f"synthetic (seeded {'IRKA-like shifted' if cfg.kind == 'irka' else 'conv-diff'} sequence, SURVEY §8(d))",
        "config": {"workload": workload_name(cfg),
                   "systems_timed": [int(j % cfg.systems) for j in range(args.warmup, steps)],
                   "iterations_per_system": [r["iterations"] for r in res_all],
                   "status_per_system": [r["status_name"] for r in res_all],
                   "k_in_per_system": [r["k_in"] for r in res_all],
                   "host_eig_ms": sum(r["t_host_eig_ms"] for r in res_all),
                   "cycle_end_ms": sum(r["t_cycle_dev_ms"] for r in res_all),
                   "loop_ms": sum(r["t_loop_ms"] for r in res_all),
                   "matrix_build_ms": sum(build_ms),
                   "solve_call_ms": [h[0] for h in host_ms],
                   "free_ms": [h[1] for h in host_ms],
                   "step_ms": [round(t, 2) for t in times],
                   "solve_total_ms": sum(r["t_total_ms"] for r in res_all),
                   "l2": "per-iteration traffic > 126 MB L2 (no flush needed)",
                   "parallelism": (f"row partition x{world} (NCCL halo + allreduce)" if part
                                   else ("replicas" if world > 1 else "single GPU"))},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": dom_bytes,
                     "timing": ("each kernel as %d back-to-back launches in one CUDA graph"
                                % args.kernel_iters) if ok else "event-bracketed single launches",
                     "pass1_ms": k1, "pass2_ms": k2,
                     "pass1_event_ms": kt["pass1_ms"], "pass2_event_ms": kt["pass2_ms"],
                     "loop_graph_iter_ms": kt["graph_iter_ms"],
                     "k_active": kt["k"], "lazy_x": kt["lazy_x"], "shared_cols": kt["shared_cols"],
                     "int16_col_deltas": kt["dcols"],
                     "tma_pass1": kt["tma_pass1"],
                     "traffic_source": traffic_info,
                     "pass1_alg_bytes": p1, "pass2_alg_bytes": p2,
                     "iter_GBps": (p1 + p2) / (kt["graph_iter_ms"] * 1e-3) / 1e9,
                     "iter_frac": (p1 + p2) / (kt["graph_iter_ms"] * 1e-3) / 1e9 / peak,
                     "fused_ms": kt["fused_ms"] if kt["fused_ms"] > 0 else None,
                     "fused_alg_bytes": pf,
                     "k_probe": probe},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    return out


def host_info():
    """CPU model, usable cores and a single-thread STREAM triad (a = b + s c,
    NumPy, 2^25 doubles per array, best of 5) measured in this run."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    nel = 1 << 25
    bb = np.random.default_rng(1).random(nel)
    cc = np.random.default_rng(2).random(nel)
    aa = np.empty(nel)
    best = float("inf")
    for _ in range(5):
        t0 = time.perf_counter()
        np.multiply(cc, 3.0, out=aa)
        np.add(aa, bb, out=aa)
        best = min(best, time.perf_counter() - t0)
    # the two NumPy passes move 5 arrays' worth (read c, write a; read a, b,
    # write a); STREAM's triad counts 3
    return {"cpu_model": model, "host_cores_available": len(os.sched_getaffinity(0)),
            "stream_triad_gbs_1thread": 3 * 8 * nel / best / 1e9,
            "stream_note": "NumPy a = 3c; a += b on 2^25 doubles, best of 5, counted as "
                           "STREAM triad bytes (3 arrays)"}


def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads", 1) for p in threadpool_info()] or [1])
    except Exception:   # noqa: BLE001
        return 1


def _seeded_space(cfg, k):
    """A seeded N(0,1) k-column input space (the oracle's timing sample needs
    the projections active without running the whole first system)."""
    rng = np.random.default_rng(cfg.seed + 777)
    shp = (cfg.n, k)
    if cfg.complex:
        return (rng.standard_normal(shp) + 1j * rng.standard_normal(shp),
                rng.standard_normal(shp) + 1j * rng.standard_normal(shp))
    return rng.standard_normal(shp), rng.standard_normal(shp)


def cpu_baseline(args, cfg, sample_iters, k_active):
    """The oracle as it stands, on a bounded sample: `sample_iters` forced
    iterations (stop test off, Q27) of system 1 of the sequence, from a
    seeded k_active-column input space when the timed systems ran with one
    (so the sample runs the same augmented iteration), host cores (the
    oracle's BLAS is limited to one thread, reading Q26; SciPy's SpMV is
    single-threaded)."""
    import scipy.sparse as sp
    from oracle import rbicg as R
    from synth import system_sequence
    it = next(system_sequence(cfg, systems=[1], **({"lam_r": 0.0} if cfg.kind == "irka" else {})))
    A = sp.csr_matrix((it["data"], it["indices"], it["indptr"]), shape=(cfg.n, cfg.n))
    U = Ut = None
    if k_active > 0:
        U, Ut = _seeded_space(cfg, k_active)
    t0 = time.perf_counter()
    res = R.solve_dual(A, it["b"], it["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s, tol=cfg.tol,
                       max_itn=sample_iters, trunc_tol=cfg.trunc_tol,
                       force_iters=sample_iters)
    el = time.perf_counter() - t0
    out = {"value": res.iterations / el, "unit": "iterations/s",
           "cores": int(_oracle_threads()), "kind": "oracle",
           "sample": f"{cfg.name} system 1, first {sample_iters} iterations (force_iters, incl. "
                     f"{sample_iters // cfg.s} cycle ends, refresh of a seeded "
                     f"{k_active}-column input space -> k_in = {res.basis_in.k}), {el:.1f} s"}
    out.update(host_info())
    return out


def run_reference(args):
    """--impl reference: the CPU oracle on the same config/metric, each step a
    bounded sample (one cycle of s iterations of system j)."""
    import scipy.sparse as sp
    from oracle import rbicg as R
    from synth import CONFIGS, system_sequence
    cfg = CONFIGS[args.config]
    steps = args.warmup + args.steps
    items = build_systems(cfg, list(range(steps)))
    tot_it, tot_t = 0, 0.0
    U = Ut = None
    for i, it in enumerate(items):
        A = sp.csr_matrix((it["data"], it["indices"], it["indptr"]), shape=(cfg.n, cfg.n))
        t0 = time.perf_counter()
        res = R.solve_dual(A, it["b"], it["bt"], U=U, Ut=Ut, k=cfg.k, s=cfg.s,
                           tol=cfg.tol, max_itn=cfg.s, trunc_tol=cfg.trunc_tol,
                           force_iters=cfg.s)
        el = time.perf_counter() - t0
        U, Ut = res.basis_out.U, res.basis_out.Ut
        if i >= args.warmup:
            tot_it += res.iterations
            tot_t += el
    blas_threads = _oracle_threads()
    v = tot_it / tot_t
    sample = f"{cfg.name}: per step one cycle ({cfg.s} iterations, stop test off) of system j"
    return {"impl": "reference", "metric": "RBiCG iterations/sec (dual pair) and achieved HBM GB/s",
            "value": v, "unit": "iterations/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if cfg.complex else "f64",
            "data": f"synthetic (seeded {'IRKA-like shifted' if cfg.kind == 'irka' else 'conv-diff'} sequence, SURVEY §8(d))",
            "config": {"workload": workload_name(cfg), "sample": sample,
                       "parallelism": "CPU oracle (host cores)"},
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": int(blas_threads),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--kernel-iters", type=int, default=20)
    ap.add_argument("--cpu-sample-iters", type=int, default=0,
                    help="oracle sample length (0: 80 iterations at n ~ 1M, scaled "
                         "down with n to keep the sample near 10-30 s, at least 8)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-k-probe", action="store_true",
                    help="skip the k = cfg.k kernel probe in the roofline block")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu capture of the dominant kernel's DRAM bytes")
    ap.add_argument("--no-update", action="store_true",
                    help="diagnostic only: no recycle-space updates (not the method's workload)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent copies instead of the row partition")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun
        port = os.environ.get("MASTER_PORT", "29517")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", port, os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        if rank == 0:   # the other ranks exit without work
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    out = run_gpu(args, rank, world)
    if rank == 0:
        if not args.no_cpu and world == 1:
            from synth import CONFIGS
            cfg = CONFIGS[args.config]
            m = args.cpu_sample_iters or max(8, min(80, int(80 * 3.2e6 / cfg.n)))
            out["cpu_baseline"] = cpu_baseline(args, cfg, m, out["roofline"]["k_active"])
        elif not args.no_cpu:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
