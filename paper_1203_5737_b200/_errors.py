"""Exception classes of the argcsr API (proj/include/argcsr/errors.hpp:9-66).

The reference module registers one Python exception, ``argcsr.Error``
(proj/python/bindings.cpp:15); here every C++ class maps to a subclass of
``Error``, so ``except Error`` keeps working and callers can be more specific.
"""


class Error(RuntimeError):
    """Base class for all errors raised by this library."""


class BoundsError(Error):
    """An index refers to a position outside the valid range."""


class DimensionError(Error):
    """Matrix/vector shapes do not agree, or a dimension is zero."""


class ParameterError(Error):
    """A tuning or configuration parameter has an invalid value."""


class InternalError(Error):
    """Internal consistency violation or a device failure."""


class CudaError(InternalError):
    """A CUDA runtime call failed (including: no CUDA device)."""


class NcclError(InternalError):
    """A collective failed."""


class OutOfMemoryError(InternalError):
    """A device or pinned-host allocation failed."""


class ParseError(Error):
    """Input text or byte stream is malformed or truncated."""


class UnsupportedError(Error):
    """Well-formed input that this library does not handle."""


class FormatError(Error):
    """A binary container's magic, version, or tag does not match."""


class IoError(Error):
    """Writing to a sink failed."""


class CorrectnessError(Error):
    """A product disagrees with the reference beyond tolerance."""
