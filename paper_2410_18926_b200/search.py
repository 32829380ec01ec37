"""Drop-in ``query`` / ``query_batch`` with the reference's signature and contract.

Reference: ``query`` (pkg/src/rrann/index.py:286-335), ``query_batch``
(index.py:338-340), ``QueryParams`` (index.py:85-100), ``QueryResult``
(index.py:103-107).  Contract:

1. same signature and return type -- ``list[QueryResult]`` with int64 ids
   best-first, float32 scores, ``truncated = len(ids) < k``;
2. same validation order and exception types: batch ``DataError`` (non-2-D /
   non-finite, index.py:339 -> 144-150) first, then ``ParameterError`` from
   ``QueryParams.validate``, ``ShapeError`` for a dimension mismatch, and
   ``ParameterError`` when re-ranking an index without a corpus; an empty batch
   returns ``[]`` without validating parameters;
3. the reference ``RrrIndex`` stays the owner of host data; its device copy is
   derived once and cached per index object;
4. concurrent calls are legal (per-thread workspace, per-call outputs).

All arithmetic runs in librrg.so (sm_100a); nothing here computes scores.
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np

from .device_index import DeviceIndex
from .errors import DataError, ShapeError

F32 = np.float32

try:  # return the reference's own result/param types when it is installed
    from rrann.index import QueryParams as _RefQueryParams
    from rrann.index import QueryResult as _RefQueryResult
except Exception:  # noqa: BLE001
    _RefQueryParams = None
    _RefQueryResult = None


@dataclass(frozen=True)
class QueryParams:
    """Mirror of rrann.index.QueryParams (index.py:85-100)."""

    k: int = 10
    w: int = 1
    t: int = 100
    rerank: bool = True

    def validate(self, L: int) -> None:
        from .errors import ParameterError

        if self.k < 1:
            raise ParameterError("k must be >= 1")
        if not 1 <= self.w <= L:
            raise ParameterError(f"w={self.w} out of range [1, {L}]")
        if self.t < 1:
            raise ParameterError("t must be >= 1")
        if self.rerank and self.k > self.t:
            raise ParameterError(f"k={self.k} must be <= t={self.t} when re-ranking")


@dataclass(frozen=True)
class _QueryResult:
    ids: np.ndarray
    scores: np.ndarray
    truncated: bool = False


QueryResult = _RefQueryResult if _RefQueryResult is not None else _QueryResult

_cache_lock = threading.Lock()
_device_cache: dict[int, tuple[weakref.ref, DeviceIndex]] = {}


def device_index_for(index, device: int = 0) -> DeviceIndex:
    """DeviceIndex for a DeviceIndex (identity) or an rrann.RrrIndex (cached upload)."""
    if isinstance(index, DeviceIndex):
        return index
    key = id(index)
    with _cache_lock:
        hit = _device_cache.get(key)
        if hit is not None and hit[0]() is index:
            return hit[1]
    dev = DeviceIndex.from_rrr(index, device=device)

    def _evict(_ref, key=key):
        with _cache_lock:
            _device_cache.pop(key, None)

    with _cache_lock:
        _device_cache[key] = (weakref.ref(index, _evict), dev)
    return dev


def _check_finite(a) -> np.ndarray:
    """_check_finite(queries, "queries"), index.py:144-150."""
    m = np.ascontiguousarray(a, dtype=F32)
    if m.ndim != 2:
        raise DataError("queries: expected 2-D array")
    if not np.all(np.isfinite(m)):
        raise DataError("queries: contains non-finite values")
    return m


def _params(params):
    return int(params.k), int(params.w), int(params.t), bool(params.rerank)


class QueryResults(list):
    """``list[QueryResult]`` that builds each ``QueryResult`` on first access.

    The search returns three dense arrays (ids [Q, k], scores [Q, k], count [Q]);
    packaging one frozen dataclass per query costs ~1-2 us in Python (SURVEY.md §7
    hard part 9), more than the whole device search per query at 10k-query batches.
    Items are created when indexed or iterated and cached in the list itself; every
    ``QueryResult`` owns its arrays (``ids[i, :c].copy()``, as the reference's fresh
    per-query arrays).  It is a real ``list`` (isinstance, len, ==, iteration, slicing,
    pickling all behave like the reference's return value); code that reads the raw
    list storage from C without going through the sequence protocol sees ``None`` for
    items never accessed -- ``materialize()`` fills them all.
    """

    __slots__ = ("_ids", "_scores", "_count", "_k", "_pending")

    def __init__(self, ids: np.ndarray, scores: np.ndarray, count: np.ndarray, k: int):
        n = int(ids.shape[0])
        super().__init__([None] * n)
        self._ids, self._scores, self._count, self._k = ids, scores, count, k
        self._pending = n

    def _make(self, i: int):
        c = int(self._count[i])
        r = QueryResult(ids=self._ids[i, :c].copy(), scores=self._scores[i, :c].copy(),
                        truncated=c < self._k)
        list.__setitem__(self, i, r)
        self._pending -= 1
        if self._pending == 0:  # every item built: the arrays are no longer needed
            self._ids = self._scores = self._count = None
        return r

    def _get(self, i: int):
        v = list.__getitem__(self, i)
        if v is None and self._pending:
            v = self._make(i if i >= 0 else i + len(self))
        return v

    def materialize(self) -> "QueryResults":
        if self._pending:
            for i in range(len(self)):
                self._get(i)
        return self

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._get(j) for j in range(*i.indices(len(self)))]
        return self._get(i)

    def __iter__(self):
        for i in range(len(self)):
            yield self._get(i)

    def __reversed__(self):
        for i in range(len(self) - 1, -1, -1):
            yield self._get(i)

    def __contains__(self, x):
        return any(x == v for v in self)

    def __eq__(self, other):
        self.materialize()
        if isinstance(other, QueryResults):
            other.materialize()
        return list.__eq__(self, other)

    def __ne__(self, other):
        return not self.__eq__(other)

    __hash__ = None

    def __repr__(self):
        return list.__repr__(self.materialize())

    def __reduce_ex__(self, protocol):
        return (list, (list(self),))

    def __copy__(self):
        return list(self)

    def copy(self):
        return list(self)

    def index(self, x, *args):
        return list.index(self.materialize(), x, *args)

    def count(self, x):
        return list.count(self.materialize(), x)

    def __add__(self, other):
        return list(self) + list(other)


def _package(ids: np.ndarray, scores: np.ndarray, count: np.ndarray, k: int) -> list:
    return QueryResults(ids, scores, count, k)


def query_batch(index, queries, params) -> list:
    """Drop-in for rrann.query_batch (index.py:338-340), computed on the B200."""
    dev = device_index_for(index)
    try:
        import torch
        is_cuda = isinstance(queries, torch.Tensor) and queries.is_cuda
    except ImportError:  # pragma: no cover
        is_cuda = False
    k, w, t, rerank = _params(params)
    if is_cuda:
        if queries.dim() != 2:
            raise DataError("queries: expected 2-D array")
        q = queries.to(torch.float32).contiguous()
        if not bool(torch.isfinite(q).all()):
            raise DataError("queries: contains non-finite values")
        if q.shape[0] == 0:
            return []
        ids, scores, count = dev.search_device(q, k, w, t, rerank)
        return _package(ids.cpu().numpy(), scores.cpu().numpy(), count.cpu().numpy(), k)
    q = np.ascontiguousarray(queries, dtype=F32)
    if q.ndim != 2:
        raise DataError("queries: expected 2-D array")
    if q.shape[0] == 0:
        return []
    # non-finite values are detected on the GPU by rrg_search_host (DataError,
    # raised ahead of parameter errors like index.py:339)
    ids, scores, count = dev.search_host(q, k, w, t, rerank)
    return _package(ids, scores, count, k)


def query(index, x, params):
    """Drop-in for rrann.query (index.py:286-335): one query through the batched path."""
    dev = device_index_for(index)
    k, w, t, rerank = _params(params)
    # validation order of query(): params, then shape, then finiteness (index.py:288-293)
    (params if hasattr(params, "validate") else QueryParams(k, w, t, rerank)).validate(dev.n_clusters)
    xv = np.ascontiguousarray(x, dtype=F32).ravel()
    if xv.size != dev.dim:
        raise ShapeError(f"query dimension {xv.size} != index dimension {dev.dim}")
    if not np.all(np.isfinite(xv)):
        raise DataError("query contains non-finite values")
    ids, scores, count = dev.search_host(xv[None, :], k, w, t, rerank)
    return _package(ids, scores, count, k)[0]


def install() -> None:
    """Opt-in: route rrann.query_batch / RrrIndex.query_batch through the B200 path."""
    import rrann
    import rrann.index as ri

    ri.query_batch = query_batch
    ri.query = query
    rrann.query_batch = query_batch
    rrann.query = query
