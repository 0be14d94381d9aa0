"""B200-native (sm_100a) CSR SpMM engine for the Sgap schedule space
(arXiv 2209.02882): a drop-in for the executor path of the reference package
``spmmlab`` (``run`` / ``build_kernel`` / ``verify_point`` and the point
grammar ``nnz:1,col:4,r:32``).

Modules mirror the reference's: ``matrices``, ``space``, ``templates``,
``lowering`` (integer geometry only), ``sim`` (the executor -- on the GPU),
``runner``.  B200-specific: ``device`` (HBM-resident operands, stream-ordered
calls), ``generators`` (the BASELINE workloads), ``selector`` (schedule
choice), ``partition`` / ``parallel`` (nnz-balanced multi-GPU row shards).
All arithmetic runs in ``libsgap.so`` (include/sgap.h); there is no CPU path.
"""

from .lowering import KernelConfig, LoweredKernel, compute_block_starts
from .matrices import CsrMatrix, DenseMatrix, random_csr, random_dense
from .space import SchedulePoint, enumerate_space, parse_point

__all__ = [
    "CsrMatrix", "DenseMatrix", "KernelConfig", "LoweredKernel", "SchedulePoint",
    "compute_block_starts", "enumerate_space", "parse_point", "random_csr", "random_dense",
]

__version__ = "0.1.0"
