"""CPU (oracle-backed) shard engine with the same interface as ``sharded.CudaShardEngine``.

Test infrastructure only: lets the multi-process (gloo) tests exercise the
two-phase sharded orchestration of ``paper_2410_18926_b200.sharded`` on CPU.
Arithmetic per stage is the oracle's (oracle/rrann_oracle.py); ordering is by
(key, corpus id) with -0.0 == +0.0, as in the kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import rrann_oracle as O
from paper_2410_18926_b200.sharded import Candidates, Front

F32 = np.float32


def mono32(f: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(f, dtype=F32).view(np.uint32).astype(np.uint64)
    u = np.where(u == 0x80000000, 0, u)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000).astype(np.uint32)


def _as_i32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32).copy())


class OracleShardEngine:
    def __init__(self, index: O.OIndex, c0: int, c1: int):
        self.ix = index
        self.c0, self.c1 = c0, c1
        self.owner = np.full(index.m, False)
        for l in range(c0, c1):
            self.owner[index.clusters[l].ids] = True

    def front(self, q, w):
        """Front stages of a query slice (the oracle's projection, q8, route)."""
        qn = q.numpy()
        n, s = qn.shape[0], self.ix.projection.shape[1]
        sp = (s + 15) // 16 * 16
        xp = O.project(qn, self.ix.projection) if n else np.zeros((0, s), F32)
        codes = np.zeros((n, sp), np.int8)
        scale = np.zeros(n, F32)
        head = np.zeros(n, F32)
        sel = np.zeros((n, w), np.int32)
        for i in range(n):
            h, sc, c = O.q8(xp[i])
            head[i], scale[i], codes[i, 1:s] = h, sc, c
            sel[i] = O.route(xp[i], self.ix.centroids, w, self.ix.metric)
        t = torch.from_numpy
        return Front(xp=t(np.ascontiguousarray(xp, F32)), qcodes=t(codes), qscale=t(scale), qhead=t(head),
                     pp=t(np.zeros(n)), xx=t(np.zeros(n, F32)), sel=t(sel), prim=t(sel[:, 0].copy()))

    def _front_row(self, front, i):
        xp = front.xp[i].numpy()
        s = xp.shape[0]
        qx = (F32(front.qhead[i].item()), F32(front.qscale[i].item()), front.qcodes[i, 1:s].numpy())
        return xp, front.sel[i].numpy(), qx

    def search_from_front(self, q, front, k, w, t):
        """Full search of the queries whose probes this shard holds (others: count 0)."""
        c1 = self.phase1_from_front(q, front, k, w, t)
        return self.phase2(q, c1, k)

    def phase1_from_front(self, q, front, k, w, t):
        return self.phase1(q, k, w, t, front=front)

    def phase1(self, q, k, w, t, front=None):
        qn = q.numpy()
        nq = qn.shape[0]
        keys = np.full((nq, t), 0xFFFFFFFF, np.uint32)
        ids = np.full((nq, t), 0xFFFFFFFF, np.uint32)
        cnt = np.zeros(nq, np.int32)
        for i in range(nq):
            if front is not None:
                xp, sel, qx = self._front_row(front, i)
            else:
                xp = O.project(qn[i][None, :], self.ix.projection)[0]
                sel = O.route(xp, self.ix.centroids, w, self.ix.metric)
                qx = O.q8(xp)
            kk, ii = [], []
            for l in sel:
                if not self.c0 <= int(l) < self.c1:
                    continue
                cl = self.ix.clusters[int(l)]
                sc = O.score_cluster(xp, qx, cl, self.ix.metric)
                kk.append(sc if self.ix.metric == "euclidean" else -sc)
                ii.append(cl.ids)
            if not kk:
                continue
            kv = mono32(np.concatenate(kk))
            iv = np.concatenate(ii).astype(np.uint32)
            order = np.lexsort((iv, kv))[:t]
            keys[i, :len(order)] = kv[order]
            ids[i, :len(order)] = iv[order]
            cnt[i] = len(order)
        return Candidates(_as_i32(keys), _as_i32(ids), torch.from_numpy(cnt))

    @staticmethod
    def pack_candidates(c: Candidates):
        keys, ids, cnt = c.keys.numpy(), c.ids.numpy(), c.count.numpy()
        nq, cap = keys.shape
        off = np.zeros(nq + 1, np.int32)
        off[1:] = np.cumsum(cnt)
        pk = np.zeros(max(nq * cap, 1), np.int32)
        pi = np.zeros_like(pk)
        for i in range(nq):
            pk[off[i]:off[i + 1]] = keys[i, :cnt[i]]
            pi[off[i]:off[i + 1]] = ids[i, :cnt[i]]
        return torch.from_numpy(pk), torch.from_numpy(pi), torch.from_numpy(off)

    @staticmethod
    def unpack_candidates(gk, gi, goff, cap):
        gk, gi, goff = gk.numpy(), gi.numpy(), goff.numpy()
        G, nq = gk.shape[0], goff.shape[1] - 1
        keys = np.full((G, nq, cap), -1, np.int32)
        ids = np.full((G, nq, cap), -1, np.int32)
        cnt = np.zeros((G, nq), np.int32)
        for g in range(G):
            for i in range(nq):
                n = goff[g, i + 1] - goff[g, i]
                keys[g, i, :n] = gk[g, goff[g, i]:goff[g, i + 1]]
                ids[g, i, :n] = gi[g, goff[g, i]:goff[g, i + 1]]
                cnt[g, i] = n
        return torch.from_numpy(keys), torch.from_numpy(ids), torch.from_numpy(cnt)

    @staticmethod
    def _gather(gk, gi, gc):
        gk = gk.numpy().view(np.uint32)
        gi = gi.numpy().view(np.uint32)
        gc = gc.numpy()
        return gk, gi, gc

    def merge_candidates(self, gk, gi, gc, take):
        gk, gi, gc = self._gather(gk, gi, gc)
        G, nq, _ = gk.shape
        keys = np.full((nq, take), 0xFFFFFFFF, np.uint32)
        ids = np.full((nq, take), 0xFFFFFFFF, np.uint32)
        cnt = np.zeros(nq, np.int32)
        for i in range(nq):
            kv = np.concatenate([gk[g, i, :gc[g, i]] for g in range(G)])
            iv = np.concatenate([gi[g, i, :gc[g, i]] for g in range(G)])
            order = np.lexsort((iv, kv))[:take]
            keys[i, :len(order)] = kv[order]
            ids[i, :len(order)] = iv[order]
            cnt[i] = len(order)
        return Candidates(_as_i32(keys), _as_i32(ids), torch.from_numpy(cnt))

    def phase2(self, q, cand, k):
        qn = q.numpy()
        nq = qn.shape[0]
        cids = cand.ids.numpy().view(np.uint32)
        ccnt = cand.count.numpy()
        out_ids = np.full((nq, k), -1, np.int64)
        out_sc = np.full((nq, k), np.nan, F32)
        out_cnt = np.zeros(nq, np.int32)
        for i in range(nq):
            ids = cids[i, :ccnt[i]].astype(np.int64)
            ids = ids[self.owner[ids]]
            if ids.size == 0:
                continue
            diss = O.exact_dissimilarity(self.ix, qn[i], ids)
            keep = np.lexsort((ids, mono32(diss)))[:k]
            out_ids[i, :len(keep)] = ids[keep]
            out_sc[i, :len(keep)] = diss[keep] if self.ix.metric == "euclidean" else -diss[keep]
            out_cnt[i] = len(keep)
        return torch.from_numpy(out_ids), torch.from_numpy(out_sc), torch.from_numpy(out_cnt)

    def merge_results(self, gi, gs, gc, k):
        gi, gs, gc = gi.numpy(), gs.numpy(), gc.numpy()
        G, nq, _ = gi.shape
        out_ids = np.full((nq, k), -1, np.int64)
        out_sc = np.full((nq, k), np.nan, F32)
        out_cnt = np.zeros(nq, np.int32)
        for i in range(nq):
            iv = np.concatenate([gi[g, i, :gc[g, i]] for g in range(G)])
            sv = np.concatenate([gs[g, i, :gc[g, i]] for g in range(G)]).astype(F32)
            diss = sv if self.ix.metric == "euclidean" else -sv
            keep = np.lexsort((iv, mono32(diss)))[:k]
            out_ids[i, :len(keep)] = iv[keep]
            out_sc[i, :len(keep)] = sv[keep]
            out_cnt[i] = len(keep)
        return torch.from_numpy(out_ids), torch.from_numpy(out_sc), torch.from_numpy(out_cnt)
