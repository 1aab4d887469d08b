"""B200-native recycling BiCG (arXiv 1010.0762) hot path.

The product path is librbicg.so (include/rbicg.h): SELL-32 SpMV pair, fused
projection/update kernels, CUDA-graph loop, device Grams, host LAPACK pencil.
``api`` is argument marshalling only.  Importing ``api`` without the built
library raises ImportError -- there is no CPU fallback.
"""
__all__ = ["api"]


def __getattr__(name):
    if name == "api":
        from . import api
        return api
    raise AttributeError(name)
