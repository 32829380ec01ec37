"""Pin the CPU oracle: against the reference's golden vectors and (here) the live reference."""

import struct

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import rrann_oracle as O

F32 = np.float32


def _results_to_arrays(res, k):
    ids = np.full((len(res), k), -1, dtype=np.int64)
    sc = np.full((len(res), k), np.nan, dtype=F32)
    cnt = np.zeros(len(res), dtype=np.int32)
    for i, r in enumerate(res):
        ids[i, :len(r.ids)] = r.ids
        sc[i, :len(r.ids)] = r.scores
        cnt[i] = len(r.ids)
    return ids, sc, cnt


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_matches_golden(case):
    g = load_golden(case)
    idx = O.read_index(g["index_bytes"].tobytes())
    for pi, (k, w, t, rr) in enumerate(g["params"]):
        if f"p{pi}_ids" not in g:
            continue
        w = min(int(w), idx.L)
        res = O.query_batch(idx, g["queries"], int(k), w, int(t), bool(rr))
        ids, sc, cnt = _results_to_arrays(res, int(k))
        np.testing.assert_array_equal(cnt, g[f"p{pi}_count"])
        np.testing.assert_array_equal(ids, g[f"p{pi}_ids"])
        exact_scores = idx.metric == "euclidean" and bool(rr)
        if exact_scores:
            np.testing.assert_array_equal(sc.view(np.int32), g[f"p{pi}_scores"].view(np.int32))
        else:  # BLAS sgemv / sdot order: tolerance per north_star (1e-5 relative)
            np.testing.assert_allclose(sc, g[f"p{pi}_scores"], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_stage_traces(case):
    g = load_golden(case)
    idx = O.read_index(g["index_bytes"].tobytes())
    for qi in range(3):
        x = g["queries"][qi]
        xp = O.project(x[None, :], idx.projection)[0]
        np.testing.assert_array_equal(xp.view(np.int32), g[f"trace{qi}_xp"].view(np.int32))
        sel = O.route(xp, idx.centroids, min(4, idx.L), idx.metric)
        np.testing.assert_array_equal(sel, g[f"trace{qi}_selected"])
        if not idx.quantized:
            continue
        head, scale, codes = O.q8(xp)
        assert head == g[f"trace{qi}_qhead"] and scale == g[f"trace{qi}_qscale"]
        np.testing.assert_array_equal(codes, g[f"trace{qi}_qcodes"])
        raws, raws2, scores = [], [], []
        for l in sel:
            cl = idx.clusters[int(l)]
            raws.append(O.int8_dot(codes, cl.a.values))
            tr = {}
            scores.append(O.score_cluster(xp, (head, scale, codes), cl, idx.metric, trace=tr))
            if "raw2" in tr:
                raws2.append(tr["raw2"])
        np.testing.assert_array_equal(np.concatenate(raws), g[f"trace{qi}_raw1"])
        np.testing.assert_array_equal(np.concatenate(raws2) if raws2 else np.zeros(0, np.int32),
                                      g[f"trace{qi}_raw2"])
        np.testing.assert_array_equal(np.concatenate(scores).view(np.int32),
                                      g[f"trace{qi}_scores"].view(np.int32))


@pytest.mark.parametrize("d", [1, 2, 7, 8, 9, 17, 64, 100, 127, 128, 129, 200, 300, 513, 768, 960, 1536, 2049])
def test_pairwise_restatement_matches_numpy(d):
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((20, d)) * rng.uniform(0.1, 10, (20, d))).astype(F32)
    sq = x * x
    ref = sq.sum(axis=1)
    emu = np.array([O.pairwise_sum_f32(r) for r in sq], dtype=F32)
    np.testing.assert_array_equal(ref.view(np.int32), emu.view(np.int32))


def test_read_index_errors():
    g = load_golden("euclid_q")
    blob = g["index_bytes"].tobytes()
    with pytest.raises(O.OracleError, match="bad magic"):
        O.read_index(b"XXXXXXXX" + blob[8:])
    with pytest.raises(O.OracleError, match="truncated file"):
        O.read_index(blob[:100])
    bad = bytearray(blob)
    bad[200] ^= 0xFF
    with pytest.raises(O.OracleError, match="crc mismatch"):
        O.read_index(bytes(bad))
    with pytest.raises(O.OracleError, match="trailing"):
        O.read_index(blob + b"\0\0\0\0")
    hdr = bytearray(blob)
    struct.pack_into("<B", hdr, 8, 7)
    with pytest.raises(O.OracleError, match="unknown metric"):
        O.read_index(bytes(hdr))


def test_validation_order():
    g = load_golden("euclid_q")
    idx = O.read_index(g["index_bytes"].tobytes())
    with pytest.raises(O.OracleError, match="k must be"):
        O.query(idx, g["queries"][0], 0, 1, 10)
    with pytest.raises(O.OracleError, match="out of range"):
        O.query(idx, g["queries"][0], 5, idx.L + 1, 10)
    with pytest.raises(O.OracleError, match="when re-ranking"):
        O.query(idx, g["queries"][0], 11, 1, 10)
    with pytest.raises(O.OracleError, match="query dimension"):
        O.query(idx, g["queries"][0][:3], 5, 1, 10)


# ----------------------------------------------------------- live reference (dev container)


@pytest.mark.parametrize("case", ["euclid_q", "ip_q", "euclid_exact_ivf", "euclid_d100"])
def test_oracle_matches_live_reference(rrann_ref, case):
    g = load_golden(case)
    blob = g["index_bytes"].tobytes()
    ref_idx = rrann_ref.deserialize(blob)
    idx = O.read_index(blob)
    rng = np.random.default_rng(5)
    q = (g["queries"][:32] + rng.standard_normal(g["queries"][:32].shape).astype(F32) * 0.3).astype(F32)
    for k, w, t in [(3, 2, 9), (10, idx.L, 10_000)]:
        ref = rrann_ref.query_batch(ref_idx, q, rrann_ref.QueryParams(k=k, w=w, t=t))
        mine = O.query_batch(idx, q, k, w, t)
        for a, b in zip(ref, mine):
            np.testing.assert_array_equal(a.ids, b.ids)
            if idx.metric == "euclidean":
                np.testing.assert_array_equal(a.scores.view(np.int32), b.scores.view(np.int32))
            assert a.truncated == b.truncated


def test_batched_projection_equals_per_query_gemv(rrann_ref):
    """the batched dgemm projection equals the reference's per-query dgemv."""
    rng = np.random.default_rng(0)
    for d, s in [(128, 64), (768, 256), (24, 12)]:
        W = rng.standard_normal((d, s)).astype(F32)
        X = (rng.standard_normal((64, d)) * 3).astype(F32)
        batched = O.project(X, W)
        per = np.stack([(x.astype(np.float64) @ W.astype(np.float64)).astype(F32) for x in X])
        np.testing.assert_array_equal(batched.view(np.int32), per.view(np.int32))
