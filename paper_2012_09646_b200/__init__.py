"""paper_2012_09646_b200 -- B200-native run-time DAG scheduler for
multi-kernel GPU programs (arXiv 2012.09646), with the paper's six
task-parallel benchmarks as hand-written sm_100a kernels.

* ``dagrt``     -- ctypes binding of the C ABI (include/dagrt.h, libdagrt.so)
* ``programs``  -- the six benchmark host programs, written sequentially as the
                   paper's users would (L528-530), plus their hand-written CUDA
                   Graph schedules (baseline)

The CUDA library is required: nothing here falls back to a CPU path.
"""
from . import dagrt  # noqa: F401

__all__ = ["dagrt"]
