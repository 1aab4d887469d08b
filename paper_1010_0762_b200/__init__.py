"""B200-native recycling BiCG (arXiv 1010.0762) hot path.

The product path is librbicg.so (include/rbicg.h): SELL-32 SpMV pair, fused
projection/update kernels, CUDA-graph loop, device Grams, host LAPACK pencil.
``paper_1010_0762_b200.api`` is argument marshalling only; importing it
without the built library raises ImportError -- there is no CPU fallback.
"""
