"""Cluster-sharded search across GPUs with exact reference semantics.

Each rank holds a contiguous range of clusters (balanced by points) with their
factors and corpus rows (``rrg_index_open_shard``); projection and centroids are
replicated, so every rank routes every query identically.  Because the
reference re-ranks the GLOBAL top-t (index.py:314-322), one exchange after a
per-rank re-rank would not be equivalent; two are needed:

1. phase 1: each rank scores the probed clusters it holds and keeps its local
   top-t by (key, corpus id); all-gather; every rank merges the identical global
   top-t (``rrg_merge_candidates``);
2. phase 2: each rank re-ranks the global candidates it holds (exact distances)
   and keeps its local top-k; all-gather; merge -> the final top-k
   (``rrg_merge_results``), id-for-id equal to the single-GPU and CPU results.

The orchestration here is engine-agnostic: ``CudaShardEngine`` drives librrg.so
(NCCL all-gathers over NVLink through ``TorchExchange``); the CPU tests plug
in an oracle-backed engine and a gloo exchange with the same control flow.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from ._native import check, lib
from .errors import ParameterError


# ------------------------------------------------------------------ partitioning


def scan_cluster_sizes(path) -> np.ndarray:
    """m_l of every cluster record, walking the RRRANN01 layout (index.py:365-402)
    without reading payloads."""
    with open(path, "rb") as f:
        head = f.read(8 + 29)
        mc, d, s, r, L, m, flags = struct.unpack("<BIIIIQI", head[8:])
        quant = bool(flags & 1)
        exact_ivf = bool(flags & 8)
        off = 8 + 29 + 4 * d * s + 4 * L * s
        sizes = np.empty(L, dtype=np.int64)

        def factor_bytes(rows, cols):
            return (8 * cols + rows * cols) if quant else 4 * rows * cols

        for l in range(L):
            f.seek(off)
            (ml,) = struct.unpack("<I", f.read(4))
            sizes[l] = ml
            off += 4 + 8 * ml
            exact = exact_ivf or ml < r
            off += factor_bytes(s, ml if exact else r)
            if not exact:
                off += factor_bytes(r, ml)
            if mc == 0:
                off += 4 * ml
    return sizes


def partition_clusters(sizes, world: int) -> list[tuple[int, int]]:
    """Contiguous cluster ranges with near-equal point counts (one per rank)."""
    sizes = np.asarray(sizes, dtype=np.int64)
    L = sizes.shape[0]
    if world < 1 or world > L:
        raise ParameterError(f"cannot split {L} clusters over {world} ranks")
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = cum[-1]
    cuts = [0]
    for g in range(1, world):
        target = total * g / world
        c = int(np.searchsorted(cum, target, side="left"))
        if c > 0 and abs(cum[c - 1] - target) <= abs(cum[min(c, L)] - target):
            c -= 1  # nearest prefix boundary
        c = min(max(c, cuts[-1] + 1), L - (world - g))
        cuts.append(c)
    cuts.append(L)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


# -------------------------------------------------------------------- exchanges


class TorchExchange:
    """all-gather over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def max_scalar(self, t) -> int:
        """max over ranks of a one-element int tensor (all-reduce MAX)."""
        t = t.clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def all_gather(self, t):
        import torch

        t = t.contiguous()
        if t.is_cuda:  # NCCL: one fused all-gather into the [G, ...] layout
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]  # gloo (CPU tests)
        self.dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts)


    def all_to_all(self, t):
        """[G, S, ...] -> [G, S, ...]: block g goes to rank g; block r of the result came
        from rank r (equal splits, no host sync)."""
        import torch

        t = t.contiguous()
        out = torch.empty_like(t)
        self.dist.all_to_all_single(out, t, group=self.group)
        return out


class LocalExchange:
    """In-process stand-in: the G shards live in one process (tests, 1-GPU emulation)."""

    def __init__(self, world: int):
        self.world = world


# ---------------------------------------------------------------------- engines


@dataclass
class Front:
    """Per-query outputs of the front stages (projection index.py:298, query quantization
    quantize.py:61-77, routing cluster.py:254-264), rows in batch order (RrgFront)."""

    xp: object      # [n, s] f32
    qcodes: object  # [n, s_pad] int8
    qscale: object  # [n] f32
    qhead: object   # [n] f32
    pp: object      # [n] f64
    xx: object      # [n] f32
    sel: object     # [n, w] int32
    prim: object    # [n] int32

    FIELDS = ("xp", "qcodes", "qscale", "qhead", "pp", "xx", "sel", "prim")


@dataclass
class Candidates:
    keys: object   # [nq, t] uint32 (as int32 tensors / uint32 arrays)
    ids: object    # [nq, t] uint32
    count: object  # [nq] int32


class CudaShardEngine:
    """librrg.so shard of a DeviceIndex; tensors are torch CUDA tensors."""

    def __init__(self, dev):
        self.dev = dev

    @property
    def metric_code(self) -> int:
        return {"euclidean": 0, "ip": 1, "cosine": 2}[self.dev.metric]

    def _ws(self, nbytes):
        import torch

        ws = getattr(self, "_wsbuf", None)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.dev.device}")
            self._wsbuf = ws
        return ws

    def phase1(self, q, k, w, t):
        import torch

        nq, dim = q.shape
        dev = q.device
        keys = torch.empty((nq, t), dtype=torch.int32, device=dev)
        ids = torch.empty((nq, t), dtype=torch.int32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        nb = int(lib.rrg_shard_workspace_bytes(self.dev.handle, nq, k, w, t))
        ws = self._ws(nb)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_shard_phase1(self.dev.handle, q.data_ptr(), nq, dim, k, w, t, keys.data_ptr(),
                                   ids.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(), st))
        return Candidates(keys, ids, cnt)

    def front(self, q, w):
        """Front stages of a query slice (``rrg_search_front``)."""
        import torch

        n = q.shape[0]
        dev, s, sp = q.device, self.dev.reduced_dim, (self.dev.reduced_dim + 15) // 16 * 16
        f = Front(xp=torch.empty((n, s), dtype=torch.float32, device=dev),
                  qcodes=torch.empty((n, sp), dtype=torch.int8, device=dev),
                  qscale=torch.empty((n,), dtype=torch.float32, device=dev),
                  qhead=torch.empty((n,), dtype=torch.float32, device=dev),
                  pp=torch.empty((n,), dtype=torch.float64, device=dev),
                  xx=torch.empty((n,), dtype=torch.float32, device=dev),
                  sel=torch.empty((n, w), dtype=torch.int32, device=dev),
                  prim=torch.empty((n,), dtype=torch.int32, device=dev))
        if n:
            nb = int(lib.rrg_front_workspace_bytes(self.dev.handle, n, w))
            ws = self._ws(nb)
            st = torch.cuda.current_stream(dev).cuda_stream
            check(lib.rrg_search_front(self.dev.handle, q.data_ptr(), n, q.shape[1], w,
                                       ctypes.byref(_rrg_front(f)), ws.data_ptr(), ws.numel(), st))
        return f

    def search_from_front(self, q, front, k, w, t):
        """Full search of the queries whose probes this shard holds (others: count 0)."""
        import torch

        nq, dim = q.shape
        dev = q.device
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        sc = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        nb = self.dev.workspace_bytes(nq, k, w, t, True)
        ws = self._ws(nb)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_search_from_front(self.dev.handle, q.data_ptr(), nq, dim, k, w, t, 1,
                                        ctypes.byref(_rrg_front(front)), ids.data_ptr(), sc.data_ptr(),
                                        cnt.data_ptr(), ws.data_ptr(), ws.numel(), st))
        return ids, sc, cnt

    def phase1_from_front(self, q, front, k, w, t):
        import torch

        nq, dim = q.shape
        dev = q.device
        keys = torch.empty((nq, t), dtype=torch.int32, device=dev)
        ids = torch.empty((nq, t), dtype=torch.int32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        nb = int(lib.rrg_shard_workspace_bytes(self.dev.handle, nq, k, w, t))
        ws = self._ws(nb)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_shard_phase1_from_front(self.dev.handle, q.data_ptr(), nq, dim, k, w, t,
                                              ctypes.byref(_rrg_front(front)), keys.data_ptr(),
                                              ids.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(), st))
        return Candidates(keys, ids, cnt)

    def merge_candidates(self, gk, gi, gc, take):
        import torch

        G, nq, cap = gk.shape
        dev = gk.device
        keys = torch.empty((nq, take), dtype=torch.int32, device=dev)
        ids = torch.empty((nq, take), dtype=torch.int32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_merge_candidates(nq, G, cap, gk.data_ptr(), gi.data_ptr(), gc.data_ptr(), take,
                                       keys.data_ptr(), ids.data_ptr(), cnt.data_ptr(), st))
        return Candidates(keys, ids, cnt)

    def pack_candidates(self, c: Candidates):
        """Local lists packed back to back: (keys [nq*cap], ids [nq*cap], offsets [nq+1])."""
        import torch

        nq, cap = c.keys.shape
        dev = c.keys.device
        pk = torch.empty((max(nq * cap, 1),), dtype=torch.int32, device=dev)
        pi = torch.empty_like(pk)
        off = torch.empty((nq + 1,), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_pack_candidates(nq, cap, c.keys.data_ptr(), c.ids.data_ptr(), c.count.data_ptr(),
                                      pk.data_ptr(), pi.data_ptr(), off.data_ptr(), st))
        return pk, pi, off

    def unpack_candidates(self, gk, gi, goff, cap):
        """G gathered packed lists -> the [G, nq, cap] layout of merge_candidates."""
        import torch

        G, stride = gk.shape
        nq = goff.shape[1] - 1
        dev = gk.device
        keys = torch.empty((G, nq, cap), dtype=torch.int32, device=dev)
        ids = torch.empty_like(keys)
        cnt = torch.empty((G, nq), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_unpack_candidates(nq, G, stride, cap, gk.data_ptr(), gi.data_ptr(), goff.data_ptr(),
                                        keys.data_ptr(), ids.data_ptr(), cnt.data_ptr(), st))
        return keys, ids, cnt

    def phase2(self, q, cand: Candidates, k):
        import torch

        nq, dim = q.shape
        cap = cand.ids.shape[1]
        dev = q.device
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        sc = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        nb = 2 * (nq * cap * 4 + nq * 4) + 1024
        ws = self._ws(nb)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_shard_phase2(self.dev.handle, q.data_ptr(), nq, dim, cand.ids.data_ptr(),
                                   cand.count.data_ptr(), cap, k, ids.data_ptr(), sc.data_ptr(),
                                   cnt.data_ptr(), ws.data_ptr(), ws.numel(), st))
        return ids, sc, cnt

    def merge_results(self, gi, gs, gc, k):
        import torch

        G, nq, _ = gi.shape
        dev = gi.device
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        sc = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        check(lib.rrg_merge_results(nq, G, k, self.metric_code, gs.data_ptr(), gi.data_ptr(),
                                    gc.data_ptr(), sc.data_ptr(), ids.data_ptr(), cnt.data_ptr(), st))
        return ids, sc, cnt


# --------------------------------------------------------------- orchestration


def exchange_candidates(engine, exchange, c1: Candidates, sparse: bool = True):
    """Phase-1 all-gather.  Sparse: each rank's lists travel packed (offsets + the
    max-over-ranks total of entries, padded to it) and are unpacked to the [G, nq, t]
    layout on arrival -- about G-fold fewer bytes when a query's probes sit on one
    rank (w = 1); dense: the padded [nq, t] lists as they are."""
    if not sparse:
        return exchange.all_gather(c1.keys), exchange.all_gather(c1.ids), exchange.all_gather(c1.count)
    pk, pi, off = engine.pack_candidates(c1)
    tot = max(exchange.max_scalar(off[-1:]), 1)
    gk = exchange.all_gather(pk[:tot])
    gi = exchange.all_gather(pi[:tot])
    goff = exchange.all_gather(off)
    return engine.unpack_candidates(gk, gi, goff, c1.keys.shape[1])


def gathered_front(engine, exchange, queries, w: int) -> Front:
    """Data-parallel front stages: rank r projects, quantizes and routes rows
    [r*S, (r+1)*S) of the batch (S = ceil(nq / G)); one all-gather per field gives every
    rank the whole batch's rows, so projection and routing are not replicated."""
    nq, G, r = queries.shape[0], exchange.world, exchange.rank
    S = -(-nq // G)
    a, b = min(nq, r * S), min(nq, (r + 1) * S)
    loc = engine.front(queries[a:b], w)
    out = {}
    for name in Front.FIELDS:
        v = getattr(loc, name)
        if v.shape[0] < S:  # pad the last slices to the common size
            pad = v.new_zeros((S - v.shape[0],) + tuple(v.shape[1:]))
            v = _cat(v, pad)
        g = exchange.all_gather(v)
        out[name] = g.reshape((G * S,) + tuple(g.shape[2:]))[:nq].contiguous()
    return Front(**out)


def _cat(a, b):
    import torch

    return torch.cat([a, b])


def sharded_search(engine, exchange, queries, k: int, w: int, t: int, sparse: bool = True,
                   data_parallel_front: bool = True, results: str = "all"):
    """Exact sharded search for one rank (all ranks call it collectively).

    Front stages are data-parallel (``gathered_front``).  With w = 1 every query's
    candidates live on the one rank that holds its cluster, so that rank's local search
    (top-t over its clusters, exact re-rank, top-k) is already the global answer: one
    all-gather of the results and a merge finish the batch, with no candidate exchange
    and no host synchronisation.  With w > 1 a query's probes may span ranks and the
    reference re-ranks the GLOBAL top-t (index.py:314-322), so two exchanges are
    needed: local top-t -> all-gather -> global top-t -> owner re-rank -> all-gather
    -> final top-k.

    ``results="all"``: every rank returns the whole batch's results (all-gather + merge);
    ``"slice"``: rank r returns rows [r*S, (r+1)*S) (S = ceil(Q/G), its front slice) via
    one all-to-all (``slice_results``) -- data-parallel serving, each rank answering the
    queries it was given."""
    if k > t:
        raise ParameterError(f"k={k} must be <= t={t} when re-ranking")
    if results not in ("all", "slice"):
        raise ParameterError(f"results must be 'all' or 'slice', got {results!r}")
    front = gathered_front(engine, exchange, queries, w) if data_parallel_front else None
    if front is not None and w == 1:
        ids, sc, cnt = engine.search_from_front(queries, front, k, w, t)
    else:
        c1 = (engine.phase1_from_front(queries, front, k, w, t) if front is not None
              else engine.phase1(queries, k, w, t))
        gk, gi, gc = exchange_candidates(engine, exchange, c1, sparse)
        cand = engine.merge_candidates(gk, gi, gc, t)
        ids, sc, cnt = engine.phase2(queries, cand, k)
    if results == "slice":
        return slice_results(engine, exchange, ids, sc, cnt, k)
    return engine.merge_results(exchange.all_gather(ids), exchange.all_gather(sc),
                                exchange.all_gather(cnt), k)


def _slices(x, G: int, S: int):
    """[nq, ...] -> [G, S, ...], the last slice padded (count 0 rows for results)."""
    nq = x.shape[0]
    if nq < G * S:
        x = _cat(x, x.new_zeros((G * S - nq,) + tuple(x.shape[1:])))
    return x.reshape((G, S) + tuple(x.shape[1:]))


def slice_results(engine, exchange, ids, sc, cnt, k: int):
    """Each rank keeps the results of its own query slice (rows [r*S, (r+1)*S), the
    slice whose front stages it ran): one all-to-all of the [Q, k] result rows by
    slice, then a merge over the G candidates of each row.  Per rank it receives
    (G-1)*S rows instead of the (G-1)*Q of the all-gather (C4 at G = 8: 10.5 MB vs
    84 MB) and merges S rows instead of Q."""
    G, r, nq = exchange.world, exchange.rank, ids.shape[0]
    S = -(-nq // G)
    gi = exchange.all_to_all(_slices(ids, G, S))
    gs = exchange.all_to_all(_slices(sc, G, S))
    gc = exchange.all_to_all(_slices(cnt, G, S))
    a, b = min(nq, r * S), min(nq, (r + 1) * S)
    return tuple(x[:b - a] for x in engine.merge_results(gi, gs, gc, k))


def _rrg_front(f: Front):
    from ._native import RrgFront

    return RrgFront(*(getattr(f, n).data_ptr() for n in Front.FIELDS))


def sharded_search_local(engines, queries, k: int, w: int, t: int, sparse: bool = False,
                         data_parallel_front: bool = True):
    """All G shards in one process (tests, the 1-GPU emulation): the same flow as
    ``sharded_search`` -- the front stages computed slice by slice on the G shards and
    concatenated (the all-gather), w = 1 answered by each query's owner shard, w > 1
    through the two merges (sparse: the packed phase-1 exchange)."""
    import torch

    G, nq = len(engines), queries.shape[0]
    front = None
    if data_parallel_front:
        S = -(-nq // G)
        parts = [e.front(queries[min(nq, g * S):min(nq, (g + 1) * S)], w) for g, e in enumerate(engines)]
        front = Front(**{n: torch.cat([getattr(p, n) for p in parts]) for n in Front.FIELDS})
    if front is not None and w == 1:
        res = [e.search_from_front(queries, front, k, w, t) for e in engines]
    else:
        c1 = [e.phase1_from_front(queries, front, k, w, t) if front is not None else e.phase1(queries, k, w, t)
              for e in engines]
        if sparse:
            packed = [e.pack_candidates(c) for e, c in zip(engines, c1)]
            tot = max(max(int(p[2][-1]) for p in packed), 1)
            gk, gi, gc = engines[0].unpack_candidates(torch.stack([p[0][:tot] for p in packed]),
                                                      torch.stack([p[1][:tot] for p in packed]),
                                                      torch.stack([p[2] for p in packed]), t)
        else:
            gk = torch.stack([c.keys for c in c1])
            gi = torch.stack([c.ids for c in c1])
            gc = torch.stack([c.count for c in c1])
        cand = engines[0].merge_candidates(gk, gi, gc, t)
        res = [e.phase2(queries, cand, k) for e in engines]
    return engines[0].merge_results(torch.stack([r[0] for r in res]), torch.stack([r[1] for r in res]),
                                    torch.stack([r[2] for r in res]), k)
