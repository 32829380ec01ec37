"""CPU ORACLE for the LoRANN query path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped path (``paper_2410_18926_b200``)
must never route through it.

It is a NumPy restatement of the reference ``rrann`` query path
(``/root/reference/pkg/src/rrann``), stage by stage, exposing every
intermediate so the CUDA path can be checked stage by stage:

=====================  ===============================================
stage                  reference (file:line)
=====================  ===============================================
file parsing           index.py:405-507 (``_Cursor``, ``_read_quantized``, ``deserialize``)
validation             index.py:92-100 (``QueryParams.validate``), 144-150, 288-295
projection (K1)        index.py:298
routing (K2)           cluster.py:46-58 (``_sq_distances``/``_dissimilarities``), 254-264 (``route``)
query quantize (K3)    quantize.py:28-29, 61-77 (``quantize_vector``)
int8 scoring (K4)      rrr.py:97-100, 181-203; quantize.py:109-156
top-t (K5)             index.py:303-316
rerank + top-k (K6)    index.py:278-283, 318-335
=====================  ===============================================

Parity pinning: this restatement is checked bit-for-bit against the
reference itself (imported from /root/reference in this container) by
``tests/test_oracle.py`` and against the committed golden vectors in
``tests/golden/`` (made by ``tests/golden/make_golden.py`` from the reference).
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
F64 = np.float64

MAGIC = b"RRRANN01"                      # index.py:40
_HEADER = struct.Struct("<BIIIIQI")      # index.py:41
FLAG_QUANTIZED = 1 << 0                  # index.py:43-46
FLAG_CORPUS = 1 << 1
FLAG_BALANCED = 1 << 2
FLAG_EXACT_IVF = 1 << 3
METRICS = {0: "euclidean", 1: "ip", 2: "cosine"}   # index.py:48-49


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # "ShapeError" | "ParameterError" | "DataError" | "FormatError"


# --------------------------------------------------------------------------- file


@dataclass
class OQuant:
    head_row: np.ndarray    # f32[cols]
    col_scales: np.ndarray  # f32[cols]
    values: np.ndarray      # int8[rows-1, cols] (zero pad row dropped, index.py:430)
    rows: int
    cols: int


@dataclass
class OCluster:
    ids: np.ndarray              # int64[m_l]
    a: object                    # OQuant | f32[s, cols]
    b: object                    # OQuant | f32[r, m_l] | None
    norms: np.ndarray | None     # f32[m_l] (euclidean)
    exact: bool


@dataclass
class OIndex:
    metric: str
    d: int
    s: int
    r: int
    L: int
    m: int
    flags: int
    projection: np.ndarray   # f32[d, s]
    centroids: np.ndarray    # f32[L, s]
    clusters: list = field(default_factory=list)
    corpus: np.ndarray | None = None

    @property
    def quantized(self) -> bool:
        return bool(self.flags & FLAG_QUANTIZED)


def read_index(data: bytes) -> OIndex:
    """Restates ``deserialize`` (index.py:443-507) including its error checks."""
    off = 0

    def take(n, section):
        nonlocal off
        if off + n > len(data):
            raise OracleError("FormatError", f"truncated file: {section} at offset {off}")
        chunk = data[off:off + n]
        off += n
        return chunk

    def arr(dtype, count, section):
        dt = np.dtype(dtype)
        return np.frombuffer(take(dt.itemsize * count, section), dtype=dt).copy()

    magic = take(len(MAGIC), "magic")
    if magic != MAGIC:
        raise OracleError("FormatError", f"bad magic {magic!r}; expected {MAGIC!r}")
    mc, d, s, r, L, m, flags = _HEADER.unpack(take(_HEADER.size, "header"))
    if mc not in METRICS:
        raise OracleError("FormatError", f"unknown metric code {mc}")
    metric = METRICS[mc]
    quantized = bool(flags & FLAG_QUANTIZED)
    exact_ivf = bool(flags & FLAG_EXACT_IVF)
    proj = arr("<f4", d * s, "projection").reshape(d, s)
    cents = arr("<f4", L * s, "centroids").reshape(L, s)

    def factor(rows, cols, section):
        if quantized:
            head = arr("<f4", cols, f"{section} head row")
            sc = arr("<f4", cols, f"{section} scales")
            vals = arr(np.int8, rows * cols, f"{section} values").reshape(rows, cols)
            return OQuant(head, sc, np.ascontiguousarray(vals[1:]), rows, cols)
        return arr("<f4", rows * cols, section).reshape(rows, cols)

    clusters = []
    total = 0
    for l in range(L):
        sec = f"cluster {l}"
        (ml,) = struct.unpack("<I", take(4, f"{sec} size"))
        ids = arr("<u8", ml, f"{sec} ids").astype(np.int64)
        exact = exact_ivf or ml < r
        a = factor(s, ml if exact else r, f"{sec} factor A")
        b = None if exact else factor(r, ml, f"{sec} factor B")
        norms = arr("<f4", ml, f"{sec} norms") if metric == "euclidean" else None
        clusters.append(OCluster(ids, a, b, norms, exact))
        total += ml
    if total != m:
        raise OracleError("FormatError", f"cluster records cover {total} points, header says {m}")
    corpus = None
    if flags & FLAG_CORPUS:
        corpus = arr("<f4", m * d, "corpus").reshape(m, d)
    crc_off = off
    (stored,) = struct.unpack("<I", take(4, "crc32"))
    actual = zlib.crc32(data[:crc_off]) & 0xFFFFFFFF
    if stored != actual:
        raise OracleError("FormatError", f"crc mismatch at offset {crc_off}: {stored:#x} != {actual:#x}")
    if off != len(data):
        raise OracleError("FormatError",
                          f"unknown trailing section at offset {off}: {len(data) - off} extra bytes")
    return OIndex(metric, d, s, r, L, m, flags, proj, cents, clusters, corpus)


# ---------------------------------------------------------------------- arithmetic


def q8(v: np.ndarray):
    """quantize_vector(v, mixed_precision=True), quantize.py:61-77 -> (head, scale, codes int8[n-1])."""
    v = np.ascontiguousarray(v, dtype=F32).ravel()
    head = F32(v[0])
    tail = v[1:]
    absmax = float(np.max(np.abs(tail))) if tail.size else 0.0
    if absmax == 0.0:
        return head, F32(1.0), np.zeros(tail.size, dtype=np.int8)
    scale = F32(127.0 / absmax)                         # f64 quotient, one f32 rounding
    p = tail.astype(F64) * F64(scale)                   # exact product
    codes = np.sign(p) * np.floor(np.abs(p) + 0.5)      # _round_half_away, quantize.py:28-29
    return head, scale, np.clip(codes, -127, 127).astype(np.int8)


def int8_dot(codes: np.ndarray, values: np.ndarray) -> np.ndarray:
    """int8_gemv (quantize.py:109-126): exact int32 product (int64 accumulate, then int32)."""
    if values.shape[0] == 0:
        return np.zeros(values.shape[1], dtype=np.int32)
    return (codes.astype(np.int64) @ values.astype(np.int64)).astype(np.int32)


def deq(raw, scale, col_scales, head, head_row):
    """dequantize_product + head term (quantize.py:129-136,152-155), IEEE f32, unfused."""
    den = (F32(scale) * col_scales).astype(F32)
    hc = (F32(head) * head_row).astype(F32)
    return ((raw.astype(F32) / den).astype(F32) + hc).astype(F32)


def project(queries: np.ndarray, W: np.ndarray) -> np.ndarray:
    """index.py:298, batched: f32(f64(x) @ f64(W))."""
    return (np.ascontiguousarray(queries, dtype=F32).astype(F64) @ W.astype(F64)).astype(F32)


def centroid_sqnorms(centroids: np.ndarray) -> np.ndarray:
    c = centroids.astype(F64)
    return (c * c).sum(axis=1)


def route_dissimilarities(xp: np.ndarray, centroids: np.ndarray, metric: str) -> np.ndarray:
    """_dissimilarities for one projected query (cluster.py:46-58); metric = index metric."""
    p = xp.astype(F64).reshape(1, -1)
    c = centroids.astype(F64)
    if metric == "euclidean":
        d2 = (p * p).sum(axis=1)[:, None] - 2.0 * (p @ c.T) + (c * c).sum(axis=1)[None, :]
        return np.maximum(d2, 0.0)[0]
    return -(p @ c.T)[0]


def route(xp: np.ndarray, centroids: np.ndarray, w: int, metric: str) -> np.ndarray:
    """cluster.py:254-264: stable argsort, first w ids (ties -> lower id)."""
    return np.argsort(route_dissimilarities(xp, centroids, metric), kind="stable")[:w].astype(np.int64)


def score_cluster(xp, qx, cl: OCluster, metric: str, trace: dict | None = None) -> np.ndarray:
    """rrr.py:181-203 for a quantized model, with the query quantized once (index.py:302)."""
    head, scale, codes = qx
    a = cl.a
    raw1 = int8_dot(codes, a.values)
    inter = deq(raw1, scale, a.col_scales, head, a.head_row)
    if cl.b is None:
        yhat = inter
        if trace is not None:
            trace.update(raw1=raw1)
    else:
        b = cl.b
        h2, s2, c2 = q8(inter)
        raw2 = int8_dot(c2, b.values)
        yhat = deq(raw2, s2, b.col_scales, h2, b.head_row)
        if trace is not None:
            trace.update(raw1=raw1, inter=inter, qr=(h2, s2, c2), raw2=raw2)
    if metric == "euclidean":
        return (F32(-2.0) * yhat + cl.norms).astype(F32)
    return yhat


def score_cluster_f32(xp, cl: OCluster, metric: str) -> np.ndarray:
    """Unquantized model: x @ A (@ B) in f32 (rrr.py:97-100) -- tolerance-level only."""
    x = np.ascontiguousarray(xp, dtype=F32)
    inter = x @ cl.a
    yhat = (inter if cl.b is None else inter.astype(F32) @ cl.b).astype(F32)
    if metric == "euclidean":
        return (-2.0 * yhat + cl.norms).astype(F32)
    return yhat


# ------------------------------------------------------------------------- query


@dataclass
class OResult:
    ids: np.ndarray
    scores: np.ndarray
    truncated: bool


def validate_params(k, w, t, rerank, L):
    """QueryParams.validate, index.py:92-100."""
    if k < 1:
        raise OracleError("ParameterError", "k must be >= 1")
    if not 1 <= w <= L:
        raise OracleError("ParameterError", f"w={w} out of range [1, {L}]")
    if t < 1:
        raise OracleError("ParameterError", "t must be >= 1")
    if rerank and k > t:
        raise OracleError("ParameterError", f"k={k} must be <= t={t} when re-ranking")


def exact_dissimilarity(index: OIndex, x: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """index.py:278-283 (NumPy pairwise f32 row sums for euclidean)."""
    block = index.corpus[ids]
    if index.metric == "euclidean":
        diff = block - x[None, :]
        return (diff * diff).sum(axis=1).astype(F32)
    return (-(block @ x)).astype(F32)


def query(index: OIndex, x, k: int, w: int, t: int, rerank: bool = True,
          trace: dict | None = None, xp: np.ndarray | None = None) -> OResult:
    """index.py:286-335 restated; ``trace`` collects every intermediate."""
    validate_params(k, w, t, rerank, index.L)
    x = np.ascontiguousarray(x, dtype=F32).ravel()
    if x.size != index.d:
        raise OracleError("ShapeError", f"query dimension {x.size} != index dimension {index.d}")
    if not np.all(np.isfinite(x)):
        raise OracleError("DataError", "query contains non-finite values")
    if rerank and index.corpus is None:
        raise OracleError("ParameterError", "index was built without the corpus; re-ranking unavailable")
    metric = index.metric
    if xp is None:
        xp = (x.astype(F64) @ index.projection.astype(F64)).astype(F32)
    sel = route(xp, index.centroids, w, metric)
    qx = q8(xp) if index.quantized else None
    ids_chunks, key_chunks = [], []
    cl_traces = []
    for l in sel:
        cl = index.clusters[int(l)]
        ct = {} if trace is not None else None
        sc = score_cluster(xp, qx, cl, metric, ct) if index.quantized else score_cluster_f32(xp, cl, metric)
        if ct is not None:
            ct.update(cluster=int(l), scores=sc)
            cl_traces.append(ct)
        ids_chunks.append(cl.ids)
        key_chunks.append(sc if metric == "euclidean" else -sc)
    cand_ids = np.concatenate(ids_chunks)
    cand_keys = np.concatenate(key_chunks)
    take = min(t if rerank else k, cand_ids.shape[0])
    order = np.lexsort((cand_ids, cand_keys))[:take]
    top_ids = cand_ids[order]
    if rerank:
        diss = exact_dissimilarity(index, x, top_ids)
        keep = np.lexsort((top_ids, diss))[: min(k, top_ids.shape[0])]
        ids = top_ids[keep]
        scores = diss[keep] if metric == "euclidean" else -diss[keep]
    else:
        diss = None
        ids = top_ids
        scores = cand_keys[order]
        scores = (scores + F32(x @ x)).astype(F32) if metric == "euclidean" else (-scores).astype(F32)
    if trace is not None:
        trace.update(xp=xp, selected=sel, qx=qx, clusters=cl_traces, cand_ids=cand_ids,
                     cand_keys=cand_keys, top_ids=top_ids, diss=diss)
    return OResult(ids.astype(np.int64), scores.astype(F32), ids.shape[0] < k)


def check_queries(queries) -> np.ndarray:
    """_check_finite(queries), index.py:144-150."""
    q = np.ascontiguousarray(queries, dtype=F32)
    if q.ndim != 2:
        raise OracleError("DataError", "queries: expected 2-D array")
    if not np.all(np.isfinite(q)):
        raise OracleError("DataError", "queries: contains non-finite values")
    return q


def query_batch(index: OIndex, queries, k: int, w: int, t: int, rerank: bool = True) -> list:
    """index.py:338-340."""
    q = check_queries(queries)
    return [query(index, q[i], k, w, t, rerank) for i in range(q.shape[0])]


def pairwise_sum_f32(a: np.ndarray) -> F32:
    """NumPy's float32 pairwise summation (the tree ``sum(axis=1)`` uses), restated."""
    n = a.size
    if n < 8:
        res = F32(0.0)
        for v in a:
            res = F32(res + v)
        return res
    if n <= 128:
        r = [F32(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = F32(r[j] + a[i + j])
            i += 8
        res = F32(F32(F32(r[0] + r[1]) + F32(r[2] + r[3])) + F32(F32(r[4] + r[5]) + F32(r[6] + r[7])))
        while i < n:
            res = F32(res + a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return F32(pairwise_sum_f32(a[:n2]) + pairwise_sum_f32(a[n2:]))


def brute_force_knn(corpus, queries, k: int, metric: str = "euclidean") -> np.ndarray:
    """rrann.bench.brute_force_knn (bench.py:85-124) restated: f64 distances, stable argsort."""
    c = np.asarray(corpus, dtype=F32).astype(F64)
    m = c.shape[0]
    if k < 1 or k > m:
        raise OracleError("ParameterError", f"k={k} out of range [1, {m}]")
    if metric == "cosine":
        n = np.linalg.norm(c, axis=1, keepdims=True)
        n[n == 0] = 1.0
        c = c / n
    q = np.asarray(queries, dtype=F32).astype(F64)
    if metric == "euclidean":
        diss = (q * q).sum(1)[:, None] - 2.0 * (q @ c.T) + (c * c).sum(1)[None, :]
    else:
        diss = -(q @ c.T)
    return np.argsort(diss, axis=1, kind="stable")[:, :k]
