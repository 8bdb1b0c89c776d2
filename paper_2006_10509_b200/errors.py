"""Exception classes raised on the hot path.

Same names and base class as the reference taxonomy
(``cghkit/errors.py:4-5,79-108``) so callers catching the reference's
exceptions by name keep working; plus two backend errors the CPU reference
cannot raise (missing device / unsupported shape).
"""


class CghError(Exception):
    """Base class (errors.py:4-5)."""


class NonFiniteError(CghError):
    """Field contains NaN or Inf (errors.py:79-80)."""


class InvalidSpecError(CghError):
    """Bad propagation spec (errors.py:91-92)."""


class ZeroFieldError(CghError):
    """Replay energy is zero (errors.py:95-96)."""


class EmptyMaskError(CghError):
    """Metric mask has no true pixel (errors.py:99-100)."""


class ZeroTargetError(CghError):
    """Target is zero inside the mask (errors.py:103-104)."""


class DimensionMismatchError(CghError):
    """Shapes disagree (errors.py:107-108)."""


class OutOfBoundsError(CghError):
    """Rectangle outside the plane (errors.py:87-88, raised by rect_mask)."""


class BackendUnavailableError(CghError, RuntimeError):
    """libcghb200.so or a CUDA device is missing; there is no CPU fallback."""


class UnsupportedShapeError(CghError, NotImplementedError):
    """Shape outside what the CUDA path implements (plan sides 2..4096, slab planes)."""


class DeviceError(CghError, RuntimeError):
    """CUDA runtime failure reported by the library."""


# .hgi containers (cghkit/errors.py:44-76; raised by serialio.py)
class MalformedJsonError(CghError):
    pass


class ChecksumMismatchError(CghError):
    pass


class TruncatedPayloadError(CghError):
    pass


class EmptyImageError(CghError):
    pass
