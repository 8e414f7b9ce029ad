"""Error types at the drop-in boundary.

When the reference package is importable its own classes are reused, so a
caller's ``except halopart.DomainError`` keeps working (errors.py:4-13 of the
reference); otherwise same-named local classes with the same hierarchy.
"""

try:  # pragma: no cover - depends on the environment
    from halopart.errors import DomainError, HalopartError, ParseError  # type: ignore
except Exception:  # noqa: BLE001
    class HalopartError(Exception):
        """Base class for errors raised at the hot-path boundary."""

    class ParseError(HalopartError, ValueError):
        """Malformed input text."""

    class DomainError(HalopartError, ValueError):
        """Structurally valid input that violates an operation's preconditions."""

__all__ = ["DomainError", "HalopartError", "ParseError"]
