"""Exception types with the reference's names and bases.

ShapeError       linalg.py:28      (ValueError)
BoundsError      kv_cache.py:26    (IndexError)
DegenerateInputError   attention.py:52   (ValueError)
ReusePreconditionError attention.py:56   (RuntimeError)
StalenessError   sparse.py:43      (RuntimeError)
"""


class ShapeError(ValueError):
    """Operand dimensions do not line up."""


class BoundsError(IndexError):
    """A row range / boundary lies outside the key set."""


class DegenerateInputError(ValueError):
    """An attention result was requested over zero keys."""


class ReusePreconditionError(RuntimeError):
    """A cached external partial cannot be reused."""


class StalenessError(RuntimeError):
    """A cached residual does not belong to the given mask/block."""
