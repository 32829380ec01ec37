"""Exception taxonomy of the drop-in, mirroring ``rrann.errors`` (pkg/src/rrann/errors.py:8-39).

Same class names and ``category`` values (usage -> exit 2, data -> 3,
internal -> 4; cli.py:20).  When the reference package is importable the
classes also subclass the reference's own, so ``except rrann.ParameterError``
catches errors raised by the B200 path -- the drop-in contract of SURVEY.md §8(b).
"""

from __future__ import annotations

try:  # the reference, when installed next to us
    from rrann import errors as _ref
except Exception:  # noqa: BLE001 - GPU box / standalone: no reference available
    _ref = None


def _bases(name: str):
    return (getattr(_ref, name),) if _ref is not None else ()


class RrannError(*(_bases("RrannError") or (Exception,))):
    category = "internal"


class ShapeError(RrannError, *_bases("ShapeError")):
    """Operands have incompatible dimensions."""

    category = "usage"


class ParameterError(RrannError, *_bases("ParameterError")):
    """A parameter is out of its documented range."""

    category = "usage"


class DataError(RrannError, *_bases("DataError")):
    """Input data violates a precondition (non-finite values, empty corpus)."""

    category = "data"


class FormatError(RrannError, *_bases("FormatError")):
    """A serialized artifact is malformed. Message names the section and offset."""

    category = "data"


class BuildError(RrannError, *_bases("BuildError")):
    category = "internal"


BY_NAME = {c.__name__: c for c in (RrannError, ShapeError, ParameterError, DataError, FormatError, BuildError)}
