"""B200-native (sm_100a, FP64) YASPS Newton-step hot path: local evaluation,
deterministic block-sparse assembly and block-Jacobi PCG behind the C-ABI of
include/yasps_b200.h."""
from ._lib import (CudaError, DeclError, Error, InternalError, NumericalError, UserError,  # noqa: F401
                   ValidationError)
from .engine import BlockSystem, Engine  # noqa: F401
