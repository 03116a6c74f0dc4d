"""Exception classes of the reference operator API, same names and bases.

Callers written against ``tripleid`` catch these by base class (ValueError,
RuntimeError, ...), so defining identically named subclasses of the same bases
keeps their error handling working unchanged.

- TooManySubqueries(ValueError)         kernel.py:48
- StoreError / BadMagic / BadVersion /
  TruncatedFile                          store.py:41-54
- InvariantViolation(ValueError)        store.py:57-58
- DisconnectedPatterns(ValueError)      query_ops.py:40-41
- ResourceLimit(RuntimeError)           query_ops.py:44-45
- ParseError(ValueError)                 nt.py:26-33
"""


class TooManySubqueries(ValueError):
    """More keys than the fixed mark-set width supports."""


class StoreError(Exception):
    pass


class BadMagic(StoreError):
    pass


class BadVersion(StoreError):
    pass


class TruncatedFile(StoreError):
    """Declared triple count exceeds the bytes actually present."""


class InvariantViolation(ValueError):
    """A zero ID was passed where only stored (nonzero) IDs are legal."""


class DisconnectedPatterns(ValueError):
    """A pattern shares no variable with any earlier pattern."""


class ResourceLimit(RuntimeError):
    """A join intermediate exceeded the configured row cap."""


class ParseError(ValueError):
    """Malformed statement; carries the line number and byte offset (nt.py:26-33)."""

    def __init__(self, message: str, line_number: int, offset: int):
        super().__init__(f"line {line_number}, byte {offset}: {message}")
        self.message = message
        self.line_number = line_number
        self.offset = offset

    @classmethod
    def from_message(cls, text: str) -> "ParseError":
        """From libtidq's "line N, byte B: message"."""
        head, _, message = text.partition(": ")
        try:
            ln, off = head.split(", byte ")
            return cls(message, int(ln.split("line ")[1]), int(off))
        except (ValueError, IndexError):
            return cls(text, 0, 0)
