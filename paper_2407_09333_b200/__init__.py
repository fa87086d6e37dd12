"""B200-native batched-hash engine (SHA-1 / MD5 / SM3) with the *hyper*
staging and task-splitting semantics of arXiv 2407.09333's HETOCompiler.

Public surface mirrors the reference package ``hetoc``:
  * ``paper_2407_09333_b200.crypto``  <- ``hetoc.crypto``  (batch_digest, hash_batch, digest, ...)
  * ``paper_2407_09333_b200.passes``  <- ``hetoc.passes.partition`` (partition_range)
  * ``paper_2407_09333_b200.device``  kernel-only entry points over CUDA tensors
  * ``paper_2407_09333_b200.runtime`` <- ``hetoc.runtime`` for lowered *hyper*
    hash programs (executor, device table) on GPUs
The compute lives in ``libhetoc_b200.so`` (C ABI: include/hetoc_b200.h).
"""

from . import crypto, passes, runtime  # noqa: F401
from ._native import LIB_PATH, device_count, device_info, launch_count  # noqa: F401

__all__ = ["crypto", "passes", "runtime", "device_count", "device_info", "launch_count", "LIB_PATH"]
