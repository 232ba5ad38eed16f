"""B200-native (sm_100a) matricized least-squares polynomial fit (arXiv 1512.08017).

The hot path — power sums -> Hankel normal system -> Gaussian elimination — is
hand-written CUDA in ``lib/liblsqfit_cuda.so`` behind the C ABI of
``include/lsqfit_cuda.h``. ``lsqfit`` mirrors the reference's C++ API
(``proj/include/lsqfit``) in Python; ``lib/liblsqfit_b200.so`` is the C++
drop-in with the reference's own signatures; ``device`` exposes the
device-resident entry points used by the benchmark and multi-GPU sharding.
"""
from . import _capi  # noqa: F401

__all__ = ["lsqfit", "device", "sharded"]
