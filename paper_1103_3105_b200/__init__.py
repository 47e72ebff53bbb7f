"""B200-native GPUTx: bulk execution of stored-procedure transactions (TPC-B, TM-1,
TPC-C NewOrder+Payment) under TPL / PART / K-SET (He & Yu, PVLDB 2011,
arXiv 1103.3105), behind the C ABI of include/gputx.h.

Every step of the hot path runs in libgputx.so (sm_100a CUDA); this package only
marshals arguments.  There is no CPU fallback: importing the binding without the
built library raises.
"""
from .gputx import (GPUTX_KSET, GPUTX_PART, GPUTX_TPL, KSET, PART, TPL, STRATEGIES, Database, GputxError,
                    library_path, load_library)

__all__ = ["Database", "GputxError", "KSET", "PART", "TPL", "STRATEGIES", "GPUTX_KSET", "GPUTX_PART",
           "GPUTX_TPL", "load_library", "library_path"]
