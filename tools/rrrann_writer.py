"""Streaming RRRANN01 writer (index construction side, off the query path).

The reference serializes an index into ONE in-memory ``bytearray`` and copies it once
more for the CRC (``serialize``, pkg/src/rrann/index.py:365-402): ~2x the file size in
host memory, 3.1 GB for C2 and ~80 GB for a 10M x 960 corpus.  ``RrrWriter`` emits the
identical byte stream section by section -- header (index.py:40-41,379-388), projection,
centroids, one record per cluster (n_points, ids, factor A, factor B, norm terms,
index.py:389-397; quantized factors as head_row, col_scales, the zero pad row and the
codes, index.py:346-353), the corpus in original id order, and the CRC32 trailer
(index.py:401) accumulated incrementally -- so a file of any size is written with one
cluster (or one corpus chunk) in memory at a time.

``write_index(index, path)`` streams an ``rrann.RrrIndex``; tests/test_writer.py checks
that the bytes equal ``rrann.serialize`` for every metric / mode of the golden cases.
tools/c4.py uses the writer for the GPU-built C4 index (``--write``).
"""

from __future__ import annotations

import os
import struct
import zlib

import numpy as np

MAGIC = b"RRRANN01"
HEADER = struct.Struct("<BIIIIQI")  # metric, dim, reduced_dim, rank, n_clusters, n_points, flags
METRIC_CODES = {"euclidean": 0, "ip": 1, "cosine": 2}
FLAG_QUANTIZED, FLAG_CORPUS, FLAG_BALANCED, FLAG_EXACT_IVF = 1, 2, 4, 8


class RrrWriter:
    """Write an RRRANN01 file section by section (call order = file order)."""

    def __init__(self, path, *, metric: str, dim: int, reduced_dim: int, rank: int, n_clusters: int,
                 n_points: int, flags: int):
        self.path = os.fspath(path)
        self.tmp = self.path + ".tmp"
        self.f = open(self.tmp, "wb")
        self.crc = 0
        self.bytes = 0
        self.dim, self.s, self.r, self.L, self.m, self.flags = dim, reduced_dim, rank, n_clusters, n_points, flags
        self.metric = metric
        self.quantized = bool(flags & FLAG_QUANTIZED)
        self.clusters = 0
        self.corpus_rows = 0
        self._put(MAGIC)
        self._put(HEADER.pack(METRIC_CODES[metric], dim, reduced_dim, rank, n_clusters, n_points, flags))

    def _put(self, b) -> None:
        mv = memoryview(b).cast("B")
        self.crc = zlib.crc32(mv, self.crc)
        self.f.write(mv)
        self.bytes += mv.nbytes

    def _f32(self, a) -> None:
        self._put(np.ascontiguousarray(a, dtype="<f4"))

    def projection(self, w) -> None:  # dim x reduced_dim
        self._f32(w)

    def centroids(self, c) -> None:  # n_clusters x reduced_dim
        self._f32(c)

    def _factor(self, fac) -> None:
        """Quantized: (head_row, col_scales, codes) with the codes as the file stores them -- the
        zero pad row first for mixed-precision factors (index.py:346-353); else f32 rows x cols."""
        if not self.quantized:
            self._f32(fac)
            return
        head, scales, codes = fac
        self._f32(head)
        self._f32(scales)
        self._put(np.ascontiguousarray(codes, dtype=np.int8))

    def cluster(self, point_ids, a, b=None, norm_terms=None) -> None:
        """One cluster record: ids (u64), factor A, factor B (non-exact models), norm terms
        (euclidean)."""
        ids = np.ascontiguousarray(point_ids, dtype="<u8")
        self._put(struct.pack("<I", ids.shape[0]))
        self._put(ids)
        self._factor(a)
        if b is not None:
            self._factor(b)
        if self.metric == "euclidean":
            self._f32(norm_terms)
        self.clusters += 1

    def corpus(self, rows) -> None:
        """A chunk of corpus rows in original id order."""
        rows = np.ascontiguousarray(rows, dtype="<f4")
        self._f32(rows)
        self.corpus_rows += rows.shape[0]

    def close(self) -> int:
        if self.clusters != self.L:
            raise ValueError(f"wrote {self.clusters} cluster records, header says {self.L}")
        if (self.flags & FLAG_CORPUS) and self.corpus_rows != self.m:
            raise ValueError(f"wrote {self.corpus_rows} corpus rows, header says {self.m}")
        crc = self.crc & 0xFFFFFFFF
        self.f.write(struct.pack("<I", crc))
        self.f.close()
        os.replace(self.tmp, self.path)
        return crc


def _quant(qm):
    """rrann QuantizedMatrix -> (head_row, col_scales, codes with the pad row)."""
    vals = np.asarray(qm.values, dtype=np.int8)
    if qm.mixed:
        vals = np.concatenate([np.zeros((1, qm.cols), np.int8), vals])
    return qm.head_row, qm.col_scales, vals


def write_index(index, path, corpus_chunk_rows: int = 1 << 16) -> int:
    """Stream an ``rrann.RrrIndex`` to ``path``; returns the CRC32 trailer."""
    cfg = index.config
    quant = bool(cfg.rrr.quantize)
    flags = ((FLAG_QUANTIZED if quant else 0) | (FLAG_CORPUS if index.corpus is not None else 0)
             | (FLAG_BALANCED if cfg.balanced else 0) | (FLAG_EXACT_IVF if cfg.scoring_mode == "exact_ivf" else 0))
    w = RrrWriter(path, metric=cfg.metric, dim=index.dim, reduced_dim=index.reduced_dim, rank=cfg.rrr.rank,
                  n_clusters=index.n_clusters, n_points=index.n_points, flags=flags)
    w.projection(index.projection)
    w.centroids(index.centroids)
    for mdl in index.models:
        a = _quant(mdl.a) if quant else mdl.a
        b = None if mdl.b is None else (_quant(mdl.b) if quant else mdl.b)
        w.cluster(mdl.point_ids, a, b, mdl.norm_terms if cfg.metric == "euclidean" else None)
    if index.corpus is not None:
        for i in range(0, index.corpus.shape[0], corpus_chunk_rows):
            w.corpus(index.corpus[i:i + corpus_chunk_rows])
    return w.close()
