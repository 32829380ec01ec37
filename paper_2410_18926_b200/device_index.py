"""DeviceIndex: a read-only HBM copy of an ``RRRANN01`` index, owned by librrg.so.

Two ways in, mirroring the reference's two ways to hold an index:

* ``DeviceIndex.from_file(path)``   <- ``RrrIndex.load`` / ``deserialize``
  (index.py:138-141, 443-507): the native loader streams the file, checks the
  CRC32 trailer and raises ``FormatError`` with the reference's section/offset
  messages; the corpus block is scattered into cluster order on the device
  without ever holding the whole file in host memory.
* ``DeviceIndex.from_rrr(index)``   <- an in-memory ``rrann.RrrIndex``
  (index.py:110-118): its arrays are handed over as an ``RrgIndexDesc``.

HBM layout (all owned by the library): projection W [d,s] f32,
centroids [L,s] f32 + f64 squared norms, per-cluster A^T int8 codes
[n_rrr][r][s_pad] + head/scale, per-point B^T codes [P][r_pad] (32 B/point at
r=32), per-point head/scale/norm/id SoA, and the corpus reordered by cluster
[P][d_stride] f32.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native
from ._native import RrgIndexDesc, RrgIndexInfo, check, lib
from .errors import ParameterError

_METRIC_CODES = {"euclidean": 0, "ip": 1, "cosine": 2}
_METRIC_NAMES = {v: k for k, v in _METRIC_CODES.items()}
FLAG_QUANTIZED, FLAG_CORPUS, FLAG_BALANCED, FLAG_EXACT_IVF = 1, 2, 4, 8


class DeviceIndex:
    """Handle to a device-resident index.  Immutable; safe for concurrent searches (each
    thread and stream gets its own workspace; outputs are per call)."""

    def __init__(self, handle: int, device: int, source: str):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        self.source = source
        info = RrgIndexInfo()
        check(lib.rrg_index_info(self._h, ctypes.byref(info)))
        self.metric = _METRIC_NAMES[info.metric]
        self.dim = info.dim
        self.reduced_dim = info.reduced_dim
        self.rank = info.rank
        self.n_clusters = info.n_clusters
        self.n_points = info.n_points
        self.flags = info.flags
        self.n_exact_clusters = info.n_exact_clusters
        self.max_cluster_size = info.max_cluster_size
        self.device_bytes = info.device_bytes
        self._tls = threading.local()

    @property
    def has_corpus(self) -> bool:
        return bool(self.flags & FLAG_CORPUS)

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.rrg_index_destroy(h)
            self._h = ctypes.c_void_p(0)

    def __repr__(self) -> str:
        return (f"DeviceIndex(metric={self.metric!r}, m={self.n_points}, d={self.dim}, "
                f"s={self.reduced_dim}, r={self.rank}, L={self.n_clusters}, cuda:{self.device}, "
                f"{self.device_bytes / 2**20:.1f} MiB)")

    # ------------------------------------------------------------------ build

    @classmethod
    def from_file(cls, path, device: int = 0, shard: tuple[int, int] | None = None) -> "DeviceIndex":
        h = ctypes.c_void_p()
        p = os.fsencode(os.fspath(path))
        if shard is None:
            check(lib.rrg_index_open(p, device, ctypes.byref(h)))
        else:
            check(lib.rrg_index_open_shard(p, device, int(shard[0]), int(shard[1]), ctypes.byref(h)))
        return cls(h.value, device, f"file:{os.fspath(path)}")

    @classmethod
    def from_rrr(cls, index, device: int = 0) -> "DeviceIndex":
        """Upload an in-memory ``rrann.RrrIndex`` (int8 or f32 factors, index.py:110-118)."""
        cfg = index.config
        quant = bool(cfg.rrr.quantize)
        models = index.models
        L = len(models)
        s = index.projection.shape[1]
        r = cfg.rrr.rank

        def full_values(qm):
            # file layout (index.py:349-353): zero pad row + tail rows
            return np.concatenate([np.zeros((1, qm.cols), np.int8), np.asarray(qm.values, np.int8)], axis=0)

        sizes = np.array([mdl.n_points for mdl in models], dtype=np.uint32)
        ids = np.ascontiguousarray(np.concatenate([mdl.point_ids for mdl in models]).astype(np.int64))
        bm = [mdl for mdl in models if mdl.b is not None]
        f32 = np.float32
        a_head = a_scale = a_vals = b_head = b_scale = b_vals = a_f32 = b_f32 = None
        if quant:
            a_head = np.concatenate([mdl.a.head_row for mdl in models]).astype(f32)
            a_scale = np.concatenate([mdl.a.col_scales for mdl in models]).astype(f32)
            a_vals = np.concatenate([full_values(mdl.a).ravel() for mdl in models]).astype(np.int8)
            b_head = np.concatenate([mdl.b.head_row for mdl in bm]).astype(f32) if bm else np.zeros(1, f32)
            b_scale = np.concatenate([mdl.b.col_scales for mdl in bm]).astype(f32) if bm else np.zeros(1, f32)
            b_vals = (np.concatenate([full_values(mdl.b).ravel() for mdl in bm]).astype(np.int8)
                      if bm else np.zeros(1, np.int8))
        else:  # f32 factors, file layout (index.py:355-356)
            a_f32 = np.ascontiguousarray(np.concatenate([np.asarray(mdl.a, f32).ravel() for mdl in models]))
            b_f32 = (np.ascontiguousarray(np.concatenate([np.asarray(mdl.b, f32).ravel() for mdl in bm]))
                     if bm else np.zeros(1, f32))
        norms = None
        if cfg.metric == "euclidean":
            norms = np.concatenate([mdl.norm_terms for mdl in models])
        extra = (FLAG_BALANCED if cfg.balanced else 0) | (FLAG_EXACT_IVF if cfg.scoring_mode == "exact_ivf" else 0)
        return cls.from_arrays(
            metric=cfg.metric, rank=r, projection=index.projection, centroids=index.centroids,
            cluster_sizes=sizes, point_ids=ids, a_head=a_head, a_scale=a_scale, a_values=a_vals,
            b_head=b_head, b_scale=b_scale, b_values=b_vals, norms=norms, corpus=index.corpus,
            a_values_f32=a_f32, b_values_f32=b_f32, n_points=index.n_points, extra_flags=extra,
            device=device, source="rrr")

    @classmethod
    def from_arrays(cls, *, metric: str, rank: int, projection, centroids, cluster_sizes, point_ids,
                    a_head=None, a_scale=None, a_values=None, b_head=None, b_scale=None, b_values=None,
                    norms=None, corpus=None, a_values_f32=None, b_values_f32=None, n_points=None,
                    extra_flags: int = 0, device: int = 0, source: str = "arrays",
                    shard: tuple[int, int] | None = None) -> "DeviceIndex":
        """Upload host arrays laid out as ``RrgIndexDesc`` documents (include/rrg.h): the
        fields of an in-memory index (index.py:110-118), per-cluster payloads concatenated
        in cluster order, quantized factors with their zero pad row (index.py:346-353).
        Quantized iff ``a_values`` is given; ``shard=(begin, end)`` keeps only that
        cluster range's payloads (``rrg_index_create_shard``, the layout of
        ``from_file(..., shard=...)``)."""
        f32 = np.float32

        def arr(a, dt):
            return None if a is None else np.ascontiguousarray(a, dtype=dt)

        proj, cent = arr(projection, f32), arr(centroids, f32)
        sizes, ids = arr(cluster_sizes, np.uint32), arr(point_ids, np.int64)
        a_head, a_scale, a_vals = arr(a_head, f32), arr(a_scale, f32), arr(a_values, np.int8)
        b_head, b_scale, b_vals = arr(b_head, f32), arr(b_scale, f32), arr(b_values, np.int8)
        norms = arr(norms, f32)
        corpus_dev = corpus is not None and getattr(corpus, "is_cuda", False)  # torch CUDA f32 [m, d]
        if corpus_dev:
            corpus = corpus.float().contiguous()
        else:
            corpus = arr(corpus, f32)
        a_f32, b_f32 = arr(a_values_f32, f32), arr(b_values_f32, f32)
        quant = a_vals is not None
        flags = (FLAG_QUANTIZED if quant else 0) | (FLAG_CORPUS if corpus is not None else 0) | extra_flags
        d, s = proj.shape
        L = cent.shape[0]
        m = int(sizes.sum()) if n_points is None else int(n_points)
        keep = [proj, cent, sizes, ids, a_head, a_scale, a_vals, b_head, b_scale, b_vals, norms, corpus,
                a_f32, b_f32]

        def ptr(a):
            if a is None:
                return None
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

        desc = RrgIndexDesc(
            metric=_METRIC_CODES[metric], dim=d, reduced_dim=s, rank=rank, n_clusters=L,
            n_points=m, flags=flags, projection=ptr(proj), centroids=ptr(cent),
            cluster_sizes=ptr(sizes), point_ids=ptr(ids), a_head=ptr(a_head), a_scale=ptr(a_scale),
            a_values=ptr(a_vals), b_head=ptr(b_head), b_scale=ptr(b_scale), b_values=ptr(b_vals),
            norms=ptr(norms), corpus=ptr(corpus), a_values_f32=ptr(a_f32), b_values_f32=ptr(b_f32))
        h = ctypes.c_void_p()
        if shard is None:
            check(lib.rrg_index_create(ctypes.byref(desc), device, ctypes.byref(h)))
        else:
            check(lib.rrg_index_create_shard(ctypes.byref(desc), device, int(shard[0]), int(shard[1]),
                                             ctypes.byref(h)))
            source = f"{source}[{shard[0]}:{shard[1]}]"
        del keep
        return cls(h.value, device, source)

    # ----------------------------------------------------------------- search

    def cluster_sizes(self) -> np.ndarray:
        out = np.zeros(self.n_clusters, dtype=np.uint32)
        check(lib.rrg_index_cluster_sizes(self._h, out.ctypes.data))
        return out

    def workspace_bytes(self, nq: int, k: int, w: int, t: int, rerank: bool) -> int:
        return int(lib.rrg_search_workspace_bytes(self._h, nq, k, w, t, int(rerank)))

    def _workspace(self, nbytes: int, st):
        """Scratch for one search, cached per (thread, stream).  It is allocated while
        ``st`` is current, so torch's caching allocator ties the block to the stream
        the search runs on: a grown buffer's old block is only reused by later work on
        that same stream, and two streams never share one workspace."""
        import torch

        cache = getattr(self._tls, "ws", None)
        if cache is None:
            cache = self._tls.ws = {}
        ws = cache.get(st.cuda_stream)
        if ws is None or ws.numel() < nbytes:
            with torch.cuda.stream(st):
                ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            cache[st.cuda_stream] = ws
        return ws

    def search_device(self, queries, k: int, w: int, t: int, rerank: bool = True, out=None,
                      stream=None):
        """Device-level entry (no host sync): queries = CUDA f32 tensor [nq, d].

        Returns (ids int64 [nq,k], scores f32 [nq,k], count int32 [nq]) CUDA tensors.
        Finiteness of ``queries`` is the caller's responsibility (the drop-in
        ``query_batch`` checks it first, like index.py:339).
        """
        import torch

        if queries.dim() != 2:
            from .errors import DataError
            raise DataError("queries: expected 2-D array")
        nq, dim = queries.shape
        q = queries
        if q.dtype != torch.float32 or not q.is_contiguous():
            q = q.to(torch.float32).contiguous()
        dev = torch.device(f"cuda:{self.device}")
        if out is None:
            ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
            scores = torch.empty((nq, k), dtype=torch.float32, device=dev)
            count = torch.empty((nq,), dtype=torch.int32, device=dev)
        else:
            ids, scores, count = out
        nbytes = self.workspace_bytes(nq, k, w, t, rerank) if nq else 0
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        ws = self._workspace(nbytes, st)
        check(lib.rrg_search(self._h, q.data_ptr(), nq, dim, k, w, t, int(rerank), ids.data_ptr(),
                             scores.data_ptr(), count.data_ptr(), ws.data_ptr(), ws.numel(),
                             st.cuda_stream))
        return ids, scores, count

    def search_host(self, queries: np.ndarray, k: int, w: int, t: int, rerank: bool = True,
                    out=None):
        """Host-buffer entry through the C ABI (``rrg_search_host``)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        if q.ndim != 2:
            from .errors import DataError
            raise DataError("queries: expected 2-D array")
        nq, dim = q.shape
        if out is None:
            ids = np.empty((nq, k), dtype=np.int64)
            scores = np.empty((nq, k), dtype=np.float32)
            count = np.empty((nq,), dtype=np.int32)
        else:
            ids, scores, count = out
        check(lib.rrg_search_host(self._h, q.ctypes.data, nq, dim, k, w, t, int(rerank),
                                  ids.ctypes.data, scores.ctypes.data, count.ctypes.data))
        return ids, scores, count

    def search_host_many(self, batches, k: int, w: int, t: int, rerank: bool = True, outs=None):
        """Several host batches through ``rrg_search_host_many`` (H2D / search / D2H of
        consecutive batches overlapped); returns [(ids, scores, count)] per batch."""
        qs = [np.ascontiguousarray(b, dtype=np.float32) for b in batches]
        for q in qs:
            if q.ndim != 2:
                from .errors import DataError
                raise DataError("queries: expected 2-D array")
        dim = qs[0].shape[1] if qs else 0
        if any(q.shape[1] != dim for q in qs):
            from .errors import ShapeError
            raise ShapeError("batches have different dimensions")
        if outs is None:
            outs = [(np.empty((q.shape[0], k), np.int64), np.empty((q.shape[0], k), np.float32),
                     np.empty((q.shape[0],), np.int32)) for q in qs]
        nb = len(qs)
        P = ctypes.c_void_p * max(nb, 1)
        qp = P(*[q.ctypes.data for q in qs])
        ip = P(*[o[0].ctypes.data for o in outs])
        sp = P(*[o[1].ctypes.data for o in outs])
        cp = P(*[o[2].ctypes.data for o in outs])
        nqa = (ctypes.c_int64 * max(nb, 1))(*[q.shape[0] for q in qs])
        check(lib.rrg_search_host_many(self._h, nb, qp, nqa, dim, k, w, t, int(rerank), ip, sp, cp))
        return outs

    # ------------------------------------------------------------- stage APIs

    def stage_project(self, queries):
        import torch

        nq = queries.shape[0]
        dev = queries.device
        xp = torch.empty((nq, self.reduced_dim), dtype=torch.float32, device=dev)
        s_pad = (self.reduced_dim + 15) // 16 * 16
        qc = torch.empty((nq, s_pad), dtype=torch.int8, device=dev)
        qs = torch.empty((nq,), dtype=torch.float32, device=dev)
        qh = torch.empty((nq,), dtype=torch.float32, device=dev)
        st = torch.cuda.current_stream(dev)
        check(lib.rrg_stage_project(self._h, queries.data_ptr(), nq, xp.data_ptr(), qc.data_ptr(),
                                    qs.data_ptr(), qh.data_ptr(), st.cuda_stream))
        return xp, qc, qs, qh

    def stage_score(self, queries, sel):
        """K4 stage outputs for probes ``sel`` [nq, w] (``rrg_stage_score``): returns
        (raw1 int32 [nq, w, rank], raw2 int32 [N], scores f32 [N], cand_off int32 [nq+1])
        with the candidates of query q at cand_off[q]:cand_off[q+1], probes in sel order."""
        import torch

        nq, w = sel.shape
        dev = queries.device
        sel = sel.to(device=dev, dtype=torch.int32).contiguous()
        sizes = torch.from_numpy(self.cluster_sizes().astype(np.int64)).to(dev)
        total = int(sizes[sel.long()].sum()) if nq else 0
        raw1 = torch.zeros((nq, w, self.rank), dtype=torch.int32, device=dev)
        raw2 = torch.zeros((max(total, 1),), dtype=torch.int32, device=dev)
        sc = torch.zeros((max(total, 1),), dtype=torch.float32, device=dev)
        off = torch.zeros((nq + 1,), dtype=torch.int32, device=dev)
        nb = int(lib.rrg_stage_score_workspace_bytes(self._h, nq, w))
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream(dev)
        check(lib.rrg_stage_score(self._h, queries.data_ptr(), nq, w, sel.data_ptr(), raw1.data_ptr(),
                                  raw2.data_ptr(), sc.data_ptr(), off.data_ptr(), ws.data_ptr(),
                                  ws.numel(), st.cuda_stream))
        return raw1, raw2[:total], sc[:total], off

    def reload_options(self) -> None:
        """Re-read the RRG_* variant switches from the environment (``rrg_index_reload_options``);
        they are otherwise resolved once, when the index is created."""
        check(lib.rrg_index_reload_options(self._h))

    def stage_route(self, xp, w: int):
        import torch

        nq = xp.shape[0]
        s_pad = (self.reduced_dim + 15) // 16 * 16
        nbytes = nq * self.n_clusters * 8 + nq * 8 + nq * s_pad + 4096
        ws = torch.empty(nbytes, dtype=torch.uint8, device=xp.device)
        sel = torch.empty((nq, w), dtype=torch.int32, device=xp.device)
        st = torch.cuda.current_stream(xp.device)
        check(lib.rrg_stage_route(self._h, xp.data_ptr(), nq, w, sel.data_ptr(), ws.data_ptr(),
                                  nbytes, st.cuda_stream))
        return sel


def last_launch_count() -> int:
    return int(lib.rrg_last_launch_count())


def version() -> str:
    return lib.rrg_version().decode()


__all__ = ["DeviceIndex", "last_launch_count", "version", "_native"]
