"""B200-native MPDP: exact join-order DP over connected relation subsets
(arXiv 2202.13511) as hand-written sm_100a CUDA behind a C ABI (include/mpdp.h).

`paper_2202_13511_b200.mpdp` is the ctypes binding; the compute lives in
libmpdp.so (built by paper_2202_13511_b200.build / __graft_entry__.build()).
"""
from . import mpdp  # noqa: F401
