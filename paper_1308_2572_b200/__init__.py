"""B200-native aggregate risk analysis (arXiv 1308.2572): the YET -> YLT -> PML/TVaR hot path.

The method runs in ``libara.so`` (CUDA kernels for sm_100a behind the C ABI of
``include/ara.h``).  ``ara`` is the thin ctypes binding with the same call names; ``dist`` shards
trials over GPUs with ``torch.distributed``.  Importing the package does not load the library;
``paper_1308_2572_b200.ara.lib()`` does and raises if it is missing (no CPU fallback).
"""
__all__ = ["ara", "dist", "build"]
