"""B200-native solve phase of the composite / multi-vector aggregation AMG
(arXiv 1907.04417): drop-in device versions of the reference `mvamg` operator
API (MultigridOperator, pcg, apply_composite_symmetrized, test_phase) running
hand-written sm_100a CUDA kernels from libmvamg_b200.so through a ctypes C ABI.
"""

from ._lib import build, load
from .composite import (
    GpuComposite,
    GpuCompositePreconditioner,
    a_norm,
    apply_composite_symmetrized,
    gpu_composite_of,
    test_phase,
)
from .cycles import (
    GS_BACKWARD,
    GS_FORWARD,
    WEIGHTED_JACOBI,
    CycleSpec,
    GpuMultigridOperator,
    SmootherSpec,
)
from .device import DeviceCSR, GpuConfig, as_csr, gs_analyse
from .exceptions import AmgError, DeviceError, NotSpdError
from .krylov import SolveReport, pcg
from .estimator import MultiVectorAMG

MultigridOperator = GpuMultigridOperator

__all__ = [
    "build", "load", "GpuComposite", "GpuCompositePreconditioner", "a_norm",
    "apply_composite_symmetrized", "gpu_composite_of", "test_phase", "MultiVectorAMG", "GS_BACKWARD", "GS_FORWARD",
    "WEIGHTED_JACOBI", "CycleSpec", "GpuMultigridOperator", "MultigridOperator",
    "SmootherSpec", "DeviceCSR", "GpuConfig", "as_csr", "gs_analyse", "AmgError",
    "DeviceError", "NotSpdError", "SolveReport", "pcg",
]
