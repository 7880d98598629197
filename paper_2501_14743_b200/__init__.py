"""paper_2501_14743_b200 -- B200-native paged-KV pull (KVDirect, arXiv 2501.14743).

* ``kvd``   -- ctypes binding of include/kvd.h (names = the C names).
* ``torch_cache`` -- helpers that allocate paged caches as torch tensors and
  register them (torch is only the device-memory / stream provider).
* ``build`` -- in-tree nvcc build of libkvd.so for sm_100a.

Importing this package does not load libkvd.so; ``from
paper_2501_14743_b200 import kvd`` does, and fails loudly if it is missing.
"""
__all__ = ["kvd", "torch_cache", "build"]
