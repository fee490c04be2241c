"""Exception taxonomy of the array context: same class names and meaning as the reference's
(/root/reference/pkg/src/laze/errors.py:11-119), so that tests written against the reference
read the same.  C-ABI status codes (include/dgb200.h) are mapped onto these by `_cabi.check`."""


class LazeError(Exception):
    """Base class (errors.py:11)."""


class ShapeMismatch(LazeError):
    """Operand shapes are incompatible (errors.py:17)."""


class DTypeMismatch(LazeError):
    """Unsupported or incompatible element types (errors.py:20)."""


class BadSubscript(LazeError):
    """Malformed einsum or array subscript (errors.py:23)."""


class UnboundPlaceholder(LazeError):
    pass


class CommunicationInSingleProcessGraph(LazeError):
    pass


class TracingError(LazeError):
    pass


class SignatureUnsupported(LazeError):
    """A compiled-function argument is not an array, scalar or None (frontend.py:589-603)."""


class BindingMismatch(LazeError):
    """A bound value disagrees with what the callee expects (backend.py:42-56)."""


class MismatchedCommunication(LazeError):
    """A send or receive has no counterpart on the peer rank (errors.py:65-75)."""

    def __init__(self, message, keys=()):
        super().__init__(message)
        self.keys = tuple(keys)


class DeadlockDetected(LazeError):
    """Distributed execution cannot make progress (errors.py:86-97)."""

    def __init__(self, message, missing=()):
        super().__init__(message)
        self.missing = tuple(missing)


class OutOfBoundsIndex(LazeError):
    """A gather index fell outside the accessed extent (errors.py; backend.py:59-68)."""


class ExtensionMissing(LazeError):
    """The sm_100a shared library is not built / not loadable.  There is no CPU fallback."""
