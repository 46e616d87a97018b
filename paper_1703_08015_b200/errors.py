"""Exception hierarchy of the reference (proj/include/splbm/errors.hpp:9-53)."""
from __future__ import annotations


class Error(RuntimeError):
    """Base class for all errors raised by the library (errors.hpp:9-13)."""


class ParseError(Error):
    """Malformed input data (errors.hpp:15-27)."""

    def __init__(self, what: str, line: int = 0, column: int = 0):
        super().__init__(what)
        self.line = line
        self.column = column


class ConfigError(Error):
    """Invalid configuration or parameters (errors.hpp:29-33)."""


class DomainError(Error):
    """Mathematical domain violation (errors.hpp:35-39)."""


class NumericalError(Error):
    """Non-finite values detected during time stepping (errors.hpp:41-48)."""

    def __init__(self, what: str, step: int):
        super().__init__(f"{what} at step {step}")
        self.step = step


class IoError(Error):
    """File system / stream failures (errors.hpp:50-54)."""


class CudaError(Error):
    """Device or driver failure (no reference counterpart: the reference is CPU-only)."""


def from_status(code: int, msg: str, step: int | None = None) -> Error:
    if code == 1:
        return ConfigError(msg)
    if code == 2:
        return DomainError(msg)
    if code == 3:
        return NumericalError(msg, step or 0)
    if code == 4:
        return IoError(msg)
    if code == 5:
        return ParseError(msg)
    return CudaError(msg)
