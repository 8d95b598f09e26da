"""Exception types of the reference API (cache.py:29-39, attention.py:30-31)."""


class Tier2UnavailableError(RuntimeError):
    """Full-precision originals are required but missing (cache.py:29-34)."""


class PagingError(RuntimeError):
    """A block required by the attend pass was never paged in (cache.py:37-39)."""


class EmptyCacheError(ValueError):
    """Attention over an empty cache is undefined (attention.py:30-31)."""
