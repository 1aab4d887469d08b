"""CPU oracle for recycling BiCG (arXiv 1010.0762) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct fp64 / complex128
implementation of what the B200 hot path computes.  It is written from
PAPER.md alone and shares no code with ``paper_1010_0762_b200`` (the CUDA
path); neither imports the other.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may
import or execute anything under ``oracle/``.

Modules
* ``bicg``   -- Algorithm 1.
* ``rbicg``  -- Algorithm 2 with the recycle-space
  construction of §4.1-§4.3 assembled with plain explicit
  products (reading Q15), and the bilinear form u^*A^{-1}w (PAPER.md:63-67,
  reading Q19).
* ``sequence`` -- the system-to-system driver.

Q26 (fixed reduction order): importing this package limits the BLAS thread
pool to one thread (threadpoolctl), so every reduction (vdot, gemv^T, the
Grams) runs in one fixed order whatever the core count, and the oracle is
bitwise-reproducible on a given host.  SciPy's SpMV is single-threaded anyway.

Every reading of an ambiguous passage is listed in
DESIGN.md §3.  Pins: tests/test_oracle_*.py (all ``-m "not gpu"``).
Parity unpinned: nothing in this package is unpinned except the paper's
figure/table values that need unavailable data.
"""

# load every BLAS the oracle uses (NumPy's and SciPy's bundled OpenBLAS)
# before limiting them, so the limit reaches both
import numpy as _np  # noqa: E402
import scipy.linalg as _sla  # noqa: E402,F401
import scipy.sparse.linalg as _spla  # noqa: E402,F401
from threadpoolctl import threadpool_limits as _threadpool_limits  # noqa: E402

_np.dot(_np.ones(2), _np.ones(2))   # (OpenBLAS initialises its pool on first use)
_threadpool_limits(1)   # Q26: one fixed reduction order (see above)
