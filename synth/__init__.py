"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the RBiCG method.  It only builds the
operators and right-hand sides of the workloads (readings
Q8-Q10, Q24) so that both sides see bit-identical inputs:

* ``convdiff``  -- finite-difference convection-diffusion matrices in CSR
  (stand-ins for the paper's §6.1 problem).
* ``irka``      -- the IRKA-like shifted complex sequence (C4; stand-in for the
  rail model of PAPER.md:1380-1443).
* ``configs``   -- the five BASELINE.json configurations C1-C5 and the seeded
  draw order of every random vector.
* ``small``     -- tiny seeded matrices for the oracle pins and parity tests.

Random numbers the *method* draws (the step-3 re-initialisation of x~_{-1},
PAPER.md:450) are also produced here and passed to both sides as inputs.
"""
from .convdiff import convdiff_csr, convdiff_nnz
from .configs import CONFIGS, Config, system_sequence, redraw_vector

__all__ = ["convdiff_csr", "convdiff_nnz", "CONFIGS", "Config",
           "system_sequence", "redraw_vector"]
