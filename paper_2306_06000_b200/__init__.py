"""B200-native S^3 (arXiv 2306.06000) length-aware KV-cache decode step.

The method runs in libs3.so (hand-written sm_100a CUDA + a C++ control
plane) behind the C ABI in include/s3.h; ``s3`` is its ctypes binding and
``engine.S3Engine`` allocates the caller-owned buffers with torch.
"""
from . import s3  # noqa: F401

__all__ = ["s3", "engine"]
