"""B200-native (sm_100a) fast filtered back projection hot path of arXiv 2007.06289:
recursive (IIR) ramp filter + Fast Hough Transform back projection.

The compute lives in libfbp.so (C ABI, include/fbp.h); ``fbp.Plan`` is the thin
Python binding.  ``dist`` shards slice batches over one process per GPU.
"""
from .fbp import Plan, FbpError, lib  # noqa: F401

__all__ = ["Plan", "FbpError", "lib"]
