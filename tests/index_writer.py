"""Test-only writer of random but well-formed RRRANN01 index files (format: index.py:365-402).

Lets the parity tests sweep shapes the reference build would be slow to
produce (any d, s, r, L, tiny/empty clusters, exact fallback models, duplicate
corpus rows) while the oracle -- which parses the same bytes -- supplies the
expected results.
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

F32 = np.float32


def _quant(rng, rows, cols):
    head = rng.standard_normal(cols).astype("<f4")
    scale = rng.uniform(0.5, 40.0, cols).astype("<f4")
    vals = rng.integers(-127, 128, size=(rows, cols), dtype=np.int8)
    vals[0] = 0  # the file's zero pad row (index.py:349-352)
    return head.tobytes() + scale.tobytes() + vals.tobytes()


def _f32(rng, rows, cols):
    return (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype("<f4").tobytes()


def _const(rng, rows, cols):
    """Zero codes and a constant head row: every column scores the same."""
    head = np.full(cols, 0.5, dtype="<f4")
    scale = np.full(cols, 3.0, dtype="<f4")
    return head.tobytes() + scale.tobytes() + np.zeros((rows, cols), np.int8).tobytes()


def random_index(d, s, r, L, m, metric="euclidean", seed=0, exact_ivf=False, with_corpus=True,
                 sizes=None, dup_rows=0, corpus_scale=1.0, quantize=True, all_ties=False):
    """all_ties: every point gets the same score and the same corpus row (tie-breaking by id)."""
    rng = np.random.default_rng(seed)
    mc = {"euclidean": 0, "ip": 1, "cosine": 2}[metric]
    flags = (1 if quantize else 0) | (2 if with_corpus else 0) | (8 if exact_ivf else 0)
    factor = _const if all_ties else (_quant if quantize else _f32)
    out = bytearray(b"RRRANN01")
    out += struct.pack("<BIIIIQI", mc, d, s, r, L, m, flags)
    W = (rng.standard_normal((d, s)) / np.sqrt(d)).astype("<f4")
    cent = rng.standard_normal((L, s)).astype("<f4")
    out += W.tobytes() + cent.tobytes()
    if sizes is None:
        cuts = np.sort(rng.integers(0, m + 1, size=L - 1))
        sizes = np.diff(np.concatenate([[0], cuts, [m]]))
    perm = rng.permutation(m)
    corpus = (rng.standard_normal((m, d)) * corpus_scale).astype("<f4")
    if all_ties:
        corpus[:] = corpus[0]
    for i in range(dup_rows):
        corpus[perm[2 * i]] = corpus[perm[2 * i + 1]]
    pos = 0
    for l in range(L):
        ml = int(sizes[l])
        ids = perm[pos:pos + ml].astype("<u8")
        pos += ml
        out += struct.pack("<I", ml) + ids.tobytes()
        exact = exact_ivf or ml < r
        out += factor(rng, s, ml if exact else r)
        if not exact:
            out += factor(rng, r, ml)
        if metric == "euclidean":
            c64 = corpus[ids.astype(np.int64)].astype(np.float64)
            out += (c64 * c64).sum(axis=1).astype("<f4").tobytes()
    if with_corpus:
        out += corpus.tobytes()
    out += struct.pack("<I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)
