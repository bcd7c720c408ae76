"""Exception hierarchy mirroring /root/reference/proj/include/ktruss/errors.hpp:9-48.

The C ABI (include/ktg.h) returns status codes; the host layer maps them back
to these types with the reference's messages, so callers catch the same things
they caught with the reference library.
"""


class Error(RuntimeError):
    """ktruss::Error (errors.hpp:9-11)."""


class ParseError(Error):
    """ktruss::ParseError (errors.hpp:14-18)."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


class EmptyInputError(Error):
    """ktruss::EmptyInputError (errors.hpp:21)."""


class EmptyGraphError(Error):
    """ktruss::EmptyGraphError (errors.hpp:26)."""


class InvalidInputError(Error):
    """ktruss::InvalidInputError (errors.hpp:31)."""


class CorruptCacheError(Error):
    """ktruss::CorruptCacheError (errors.hpp:35)."""


class InvalidParameterError(Error):
    """ktruss::InvalidParameterError (errors.hpp:39)."""


class SupportOverflowError(Error):
    """ktruss::SupportOverflowError{slot} (errors.hpp:44-48)."""

    def __init__(self, slot: int, what: str):
        super().__init__(what)
        self.slot = slot


class DeviceError(Error):
    """CUDA / NCCL failure inside the engine (no reference counterpart)."""
