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
