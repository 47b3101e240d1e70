"""B200-native index-batched DCRNN training step of PGT-I (arXiv 2507.11683).

* ``csrc/``     CUDA (sm_100a) kernels + the C ABI of ``include/pgti.h`` -> ``libpgti.so``
* ``build``     in-tree nvcc build of libpgti.so
* ``pgti``      ctypes binding (same names as the C ABI; argument marshalling only)
* ``trainer``   host driver: halo-sharded distributed-index-batching over NCCL

Nothing here imports ``oracle/`` (test infrastructure); there is no CPU fallback.
"""
