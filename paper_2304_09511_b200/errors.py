"""Exception types — same names and hierarchy as the reference (errors.py:1-53).

The C ABI returns integer status codes; `_lib.check` maps them onto these
classes, so callers see exactly the reference's error contract.
"""


class SparseError(Exception):
    """Base class for every error raised by this package (errors.py:4)."""


class DimensionMismatch(SparseError):
    """Operand dimensions do not agree (errors.py:8)."""


class UnsortedInput(SparseError):
    """Operation requires a sorted, duplicate-free COO matrix (errors.py:12)."""


class FillRatioExceeded(SparseError):
    """DIA storage would exceed the configured fill budget (errors.py:16)."""


class UnsupportedCombination(SparseError):
    """No kernel is registered for the requested (format, version) pair (errors.py:20)."""


class IndexOverflow(SparseError):
    """Requested problem size exceeds the 32-bit index range (errors.py:36)."""


class DeviceError(SparseError):
    """A CUDA call inside the engine failed (no reference counterpart)."""


class Diverged(SparseError):
    """Iterative solve produced a non-finite quantity (errors.py:40)."""


class AllCandidatesFailed(SparseError):
    """Every tuning candidate failed, so no choice can be made (errors.py:24)."""


class EmptyInput(SparseError):
    """Operation requires at least one input element (errors.py:52)."""


class ParseError(SparseError):
    """Malformed Matrix Market content (errors.py:28)."""


class UnsupportedField(SparseError):
    """Matrix Market field or symmetry this reader does not support (errors.py:32)."""


class MissingBaseline(SparseError):
    """Report input lacks the baseline pair for a matrix (errors.py:48-49)."""
