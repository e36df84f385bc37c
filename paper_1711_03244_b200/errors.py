"""Exception taxonomy of the reference (proj/core/include/voxmc/errors.hpp:9-59),
restated for the Python host API. The C-ABI returns VMC_ERR_VALIDATION for the
ValidationError family and VMC_ERR_RUNTIME for CUDA/NCCL/allocation failures
(raised as RuntimeError, as the reference's std::runtime_error)."""


class ValidationError(RuntimeError):
    """Invalid user-supplied value (errors.hpp:9-13)."""


class ParseError(RuntimeError):
    """Malformed input (errors.hpp:15-19)."""


class IoError(RuntimeError):
    pass


class VoxelOutOfRange(IndexError):
    pass


class DimensionMismatch(ValueError):
    pass


class AlreadyNormalized(RuntimeError):
    pass


class SourceOutsideDomain(ValidationError):
    """Launch point outside the grid (transport.cpp:96-99)."""


class NonPositiveSlope(RuntimeError):
    """Pilot timings gave T2 <= T1 (scheduler.cpp:386-388)."""


class InstanceTooLarge(ValueError):
    pass


class NonPositiveRadius(ValueError):
    pass
