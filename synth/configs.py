"""The five BASELINE.json configurations and their seeded draw order.

Readings:
* Q8  -- system j (0-based) uses convection β^{(j)} = β (1 + δ j).
* Q9  -- discretisation, see ``synth.convdiff``.
* Q10 -- C4 operator K = -L + offdiag(0.1 ξ), A = σ I - K, shifts right of
  λ_R = max(0, max Re λ(K)) rounded up to a 1e-4 grid.
* Q21 -- max_itn.
* Q24 -- numpy Generator(PCG64(101007620 + c)); per system j the draw order is
  b_j ~ U(-1,1)^n then b~_j ~ U(-1,1)^n.
* Q4  -- the step-3 re-initialisation vector for system index j is drawn from
  Generator(PCG64(101007620 + c + 1_000_000 (1 + j))) as U(-1,1)^n.

Nothing here performs arithmetic of the RBiCG method.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .convdiff import convdiff_csr, laplacian_offdiag_positions, convdiff_nnz

SEED_BASE = 101007620


@dataclass(frozen=True)
class Config:
    name: str
    index: int             # c in 1..5 (seed offset)
    kind: str              # "convdiff" | "irka"
    N: int
    d: int
    beta: tuple = ()
    delta: float = 0.0
    scheme: str = "central"
    systems: int = 1
    k: int = 10
    s: int = 40
    tol: float = 1e-8
    max_itn: int = 20000
    trunc_tol: float = 1e-6   # PAPER.md:694, :1405 on unit-norm columns (Q13)
    complex: bool = False

    @property
    def n(self) -> int:
        return self.N ** self.d

    @property
    def nnz(self) -> int:
        return convdiff_nnz(self.N, self.d)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index

    def scaled(self, N: int, systems: int | None = None, **kw) -> "Config":
        """Same operator family at another grid size (parity-test analogue)."""
        d = dict(self.__dict__)
        d.update(N=N, name=f"{self.name}@{N}^{self.d}")
        if systems is not None:
            d["systems"] = systems
        d.update(kw)
        return Config(**d)


CONFIGS = {
    "C1": Config("C1", 1, "convdiff", 32, 2, (10.0, 10.0), 0.01, "central",
                 systems=4, k=6, s=20, tol=1e-10, max_itn=2000),
    "C2": Config("C2", 2, "convdiff", 1024, 2, (50.0, 50.0), 0.005, "upwind",
                 systems=10, k=10, s=40, tol=1e-8, max_itn=20000),
    "C3": Config("C3", 3, "convdiff", 192, 3, (20.0, -10.0, 5.0), 0.01,
                 "central", systems=8, k=10, s=40, tol=1e-8, max_itn=20000),
    "C4": Config("C4", 4, "irka", 100, 3, (), 0.0, "central", systems=60,
                 k=8, s=40, tol=1e-8, max_itn=20000, complex=True),
    "C5": Config("C5", 5, "convdiff", 384, 3, (30.0, 15.0, -10.0), 0.005,
                 "central", systems=6, k=20, s=50, tol=1e-8, max_itn=20000),
}


def redraw_vector(cfg: Config, system_index: int, n: int | None = None):
    """Step-3 re-initialisation vector x~_{-1} (reading Q4)."""
    n = cfg.n if n is None else n
    rng = np.random.Generator(
        np.random.PCG64(cfg.seed + 1_000_000 * (1 + system_index)))
    v = rng.uniform(-1.0, 1.0, n)
    return v.astype(np.complex128) if cfg.complex else v


def _convdiff_sequence(cfg: Config, systems):
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    n = cfg.n
    for j in range(cfg.systems):
        b = rng.uniform(-1.0, 1.0, n)
        bt = rng.uniform(-1.0, 1.0, n)
        if systems is not None and j not in systems:
            continue
        beta = tuple(float(x) * (1.0 + cfg.delta * j) for x in cfg.beta)
        indptr, indices, data, _ = convdiff_csr(cfg.N, cfg.d, beta, cfg.scheme)
        yield dict(j=j, n=n, indptr=indptr, indices=indices, data=data,
                   b=b, bt=bt, beta=beta)


def irka_operator(cfg: Config, lam_r: float | None = None):
    """K = -L + offdiag(0.1 ξ) on N^3 plus b, c and the shift schedule (Q10).

    ``lam_r`` overrides the ARPACK estimate of max Re λ(K) (tests at small N
    pass it to avoid the eigensolve; it is recorded in the metadata).
    """
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    indptr, indices, offmask, n = laplacian_offdiag_positions(cfg.N, cfg.d)
    xi = rng.standard_normal(int(offmask.sum()))
    b = rng.standard_normal(n)
    c = rng.standard_normal(n)
    kdata = np.where(offmask, 1.0, -2.0 * cfg.d)  # -L
    kdata = kdata.astype(np.float64)
    kdata[offmask] += 0.1 * xi
    if lam_r is None:
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        K = sp.csr_matrix((kdata, indices, indptr), shape=(n, n))
        vals = spla.eigs(K, k=4, which="LR", tol=1e-6, ncv=40,
                         v0=np.ones(n), return_eigenvectors=False)
        lam_r = max(0.0, float(np.max(vals.real)))
        lam_r = math.ceil(lam_r / 1e-4) * 1e-4
    a = 10.0 ** rng.uniform(-2.0, 0.0, 3)
    bi = a * rng.uniform(0.1, 1.0, 3)
    o = np.argsort(a)
    a, bi = a[o], bi[o]
    delta = np.array([a[0] + 1j * bi[0], a[0] - 1j * bi[0],
                      a[1] + 1j * bi[1], a[1] - 1j * bi[1],
                      a[2] + 1j * bi[2], a[2] - 1j * bi[2]])
    return dict(indptr=indptr, indices=indices, kdata=kdata, n=n, b=b, c=c,
                lam_r=lam_r, delta=delta)


def irka_shift(op, t: int, slot: int) -> complex:
    """σ^{(t)}_slot = λ_R + δ_slot (1 + 0.5^t)."""
    return complex(op["lam_r"] + op["delta"][slot] * (1.0 + 0.5 ** t))


def _irka_sequence(cfg: Config, systems, lam_r=None):
    op = irka_operator(cfg, lam_r)
    n = op["n"]
    rows = np.repeat(np.arange(n), np.diff(op["indptr"]))
    diagmask = op["indices"] == rows
    for j in range(cfg.systems):
        if systems is not None and j not in systems:
            continue
        t, slot = divmod(j, 6)
        sigma = irka_shift(op, t, slot)
        data = (-op["kdata"]).astype(np.complex128)
        data[diagmask] += sigma
        yield dict(j=j, n=n, indptr=op["indptr"], indices=op["indices"],
                   data=data, b=op["b"].astype(np.complex128),
                   bt=op["c"].astype(np.complex128), sigma=sigma, sweep=t,
                   slot=slot, lam_r=op["lam_r"])


def system_sequence(cfg: Config, systems=None, lam_r=None):
    """Yield the systems of ``cfg`` in order (optionally only the indices in
    ``systems``).  Each item holds CSR arrays (int32 indptr/indices, float64
    or complex128 data), b and b~ and metadata."""
    if cfg.kind == "convdiff":
        yield from _convdiff_sequence(cfg, systems)
    elif cfg.kind == "irka":
        yield from _irka_sequence(cfg, systems, lam_r)
    else:
        raise ValueError(cfg.kind)
