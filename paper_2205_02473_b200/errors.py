"""Exception hierarchy of proj/include/dpro/errors.hpp:26-125 (the subset the
replay path raises; same names, same base class, same messages)."""
from __future__ import annotations


class Error(RuntimeError):
    """dpro::Error (errors.hpp:26-29)."""


class LookupError_(Error):
    """dpro::LookupError (errors.hpp:72-75)."""


# Export under the reference name as well; Python's builtin LookupError is
# shadowed only inside this module's namespace.
LookupError = LookupError_  # noqa: A001


class CycleError(Error):
    """dpro::CycleError (errors.hpp:77-82): `cycle` lists stuck op ids."""

    def __init__(self, what: str, cycle: list[str]):
        super().__init__(what)
        self.cycle = cycle


class MissingProfileError(Error):
    """dpro::MissingProfileError (errors.hpp:93-96)."""


class TransformError(Error):
    """dpro::TransformError (errors.hpp:104-107)."""


class TopologyError(Error):
    """dpro::TopologyError (errors.hpp:53-56)."""


class EngineError(Error):
    """CUDA / engine failure (no reference counterpart: the reference is CPU)."""


class MissingMetaError(Error):
    """dpro::MissingMetaError (errors.hpp:99-102)."""


class ParseError(Error):
    """dpro::ParseError (errors.hpp:32-38)."""

    def __init__(self, what: str, byte_offset: int):
        super().__init__(f"{what} (byte offset {byte_offset})")
        self.byte_offset = byte_offset


class IoError(Error):
    """dpro::IoError (errors.hpp:117-120)."""


class SchemaError(Error):
    """dpro::SchemaError (errors.hpp:41-46)."""

    def __init__(self, what: str, field: str):
        super().__init__(f"{what}: field '{field}'")
        self.field = field


class SpliceError(Error):
    """dpro::SpliceError (errors.hpp:62-65)."""


class UnknownSymbolError(Error):
    """dpro::UnknownSymbolError (errors.hpp:48-53)."""

    def __init__(self, symbol: str):
        super().__init__(f"unknown symbol '{symbol}'")
        self.symbol = symbol
