"""Exception taxonomy of the drop-in surface (lrqbench errors.py:8-26).

The class names and bases are part of the reference API: callers catch
``ValidationError`` as a ``ValueError`` and the CLI maps the three families
onto exit codes 2 (validation), 3 (capacity) and 4 (runtime).  The C ABI
(include/lrq.h) returns the same codes.
"""


class ValidationError(ValueError):
    """Bad input: sizes, indices, angles, circuit shape, files."""


class CapacityError(RuntimeError):
    """The request does not fit a resource limit (memory budget, HBM, n)."""


class StateError(RuntimeError):
    """Required state is missing (unsolved instance, no device result, no GPU)."""


class FitError(ValidationError):
    """A fit has no usable data points (kept for API compatibility)."""


class AbortedRunError(RuntimeError):
    """A multi-device run stopped because one rank failed."""


EXIT_CODES = ((ValidationError, 2), (CapacityError, 3), (StateError, 4), (AbortedRunError, 4))
