"""B200-native LightKernel (LK) persistent-worker runtime (arXiv 2310.01212).

Drop-in for the ``native`` executor of the reference package ``persistkern``:
``native.NativeSession`` boots one resident sm_100a CTA per SM and dispatches
work by mailbox words; ``protocol``, ``host``, ``device`` and ``errors``
mirror the reference modules of the same names.  All compute and all
spinning live in liblk.so (C ABI: include/lk.h).
"""
__version__ = "0.1.0"

from . import errors, host, protocol  # noqa: F401
