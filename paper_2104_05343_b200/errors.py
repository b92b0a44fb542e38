"""Error classes raised at the drop-in boundary.

The names and the inheritance tree are the public contract of the reference
(summagrid errors.py:4-29): code that catches ``ShapeError`` or
``ConfigError`` around the reference operators keeps working. Return codes of
the C ABI (include/sg.h) are translated into these in ``_lib.check``; CUDA and
NCCL failures surface as the base class.
"""


class SummaGridError(Exception):
    """Root of the hierarchy; also used for CUDA / NCCL runtime failures."""


class ShapeError(SummaGridError):
    """Raised for mismatched or non-divisible operand extents (SG_ERR_SHAPE)."""


class ConfigError(SummaGridError):
    """Raised when a mesh, model or argument value is invalid (SG_ERR_CONFIG)."""


class MeshMismatchError(SummaGridError):
    """Raised when the operands of one call belong to two different meshes."""


class BufferOverflowError(SummaGridError):
    """Raised when a planned workspace category would exceed its capacity."""


class CheckpointMissingError(SummaGridError):
    """Raised when a layer input needed by the recompute was not stored."""


class VerificationError(SummaGridError):
    """Raised by the verify harness when a parity check exceeds tolerance."""
