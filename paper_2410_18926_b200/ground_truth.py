"""Exact k-NN ground truth on the GPU: drop-in for ``rrann.bench.brute_force_knn``.

``brute_force_knn(corpus, queries, k, metric, threads)`` keeps the reference's
signature, validation and result (pkg/src/rrann/bench.py:85-124): f64
distances, ids ordered by (distance, id) like ``argsort(kind="stable")``.  The
work runs in ``rrg_ground_truth`` (librrg.so): FP64 tensor-core distance blocks
and a per-query radix select (paper_2410_18926_b200/csrc/rrg_ground_truth.cu).
Recall@k of the 1M / 10M workloads is computed with it.
"""

from __future__ import annotations

import numpy as np

from ._native import check, lib
from .errors import ParameterError, ShapeError

_METRIC_CODES = {"euclidean": 0, "ip": 1, "cosine": 2}


def ground_truth_device(corpus, queries, k: int, metric: str = "euclidean", stream=None):
    """Device entry: CUDA f32 tensors corpus [m, d], queries [nq, d] -> int64 ids [nq, k]."""
    import torch

    if metric not in _METRIC_CODES:
        raise ParameterError(f"unknown metric: {metric!r}")
    if corpus.dim() != 2 or queries.dim() != 2:
        raise ShapeError("corpus and queries must be 2-D")
    m, d = corpus.shape
    if queries.shape[1] != d:
        raise ShapeError(f"query dimension {queries.shape[1]} != corpus dimension {d}")
    if not 1 <= k <= m:
        raise ParameterError(f"k={k} out of range [1, {m}]")
    corpus = corpus.contiguous()
    queries = queries.contiguous()
    assert corpus.dtype == torch.float32 and queries.dtype == torch.float32
    out = torch.empty((queries.shape[0], k), dtype=torch.int64, device=corpus.device)
    st = stream if stream is not None else torch.cuda.current_stream(corpus.device)
    with torch.cuda.device(corpus.device):
        check(lib.rrg_ground_truth(corpus.data_ptr(), m, d, queries.data_ptr(), queries.shape[0], k,
                                   _METRIC_CODES[metric], out.data_ptr(), st.cuda_stream))
    return out


def brute_force_knn(corpus, queries, k: int, metric: str = "euclidean", threads: int = 1,
                    device: int = 0) -> np.ndarray:
    """rrann.bench.brute_force_knn on the GPU (``threads`` is accepted and ignored)."""
    import torch

    del threads
    c = np.asarray(corpus, dtype=np.float32)
    q = np.asarray(queries, dtype=np.float32)
    if c.ndim != 2 or q.ndim != 2:
        raise ShapeError("corpus and queries must be 2-D")
    m = c.shape[0]
    if k < 1 or k > m:
        raise ParameterError(f"k={k} out of range [1, {m}]")
    if metric not in _METRIC_CODES:
        raise ParameterError(f"unknown metric: {metric!r}")
    dev = torch.device(f"cuda:{device}")
    ids = ground_truth_device(torch.from_numpy(np.ascontiguousarray(c)).to(dev),
                              torch.from_numpy(np.ascontiguousarray(q)).to(dev), k, metric)
    return ids.cpu().numpy()
