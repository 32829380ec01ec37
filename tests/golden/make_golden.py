"""Generate golden vectors from the UNMODIFIED reference ``rrann`` (run in the dev container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For each case: build a small index with ``rrann.build`` (index.py:167-275),
serialize it (index.py:365-402), run ``rrann.query_batch`` (index.py:338-340)
for several ``QueryParams`` and store the file bytes, the queries and the
reference outputs (ids, scores, truncated) plus per-stage intermediates of a
few queries (projection, routing, query codes, per-cluster int32 products and
scores) in ``tests/golden/<case>.npz``.  Nothing here runs on the GPU box; the
.npz files are what travel.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import rrann  # noqa: E402
from rrann.bench import synth_dataset  # noqa: E402
from rrann.cluster import route  # noqa: E402
from rrann.index import IndexConfig, QueryParams, build, serialize  # noqa: E402
from rrann.quantize import QuantizedMatrix, int8_gemv, quantize_vector, quantized_vecmat  # noqa: E402
from rrann.rrr import RrrConfig, cluster_metric, score_cluster  # noqa: E402

F32 = np.float32
OUT = Path(__file__).resolve().parent

PARAMS = [
    # (k, w, t, rerank)
    (5, 1, 20, True),
    (10, 3, 50, True),
    (10, 4, 200, True),
    (7, 2, 7, True),
    (10, 3, 1, False),
    (12, 5, 100, False),
]


def corpus_with_outliers(m, d, seed, n_blobs):
    ds = synth_dataset(m, 64, d, kind="clustered", seed=seed, n_blobs=n_blobs)
    rng = np.random.default_rng(seed + 100)
    # a few far-away singletons force clusters smaller than the rank (exact models)
    out = rng.standard_normal((6, d)).astype(F32) * 40.0
    vecs = np.vstack([ds.vectors, out]).astype(F32)
    # an exact duplicate pair exercises the (key, id) tie rule
    vecs[5] = vecs[17]
    q = ds.queries.copy()
    q[3] = vecs[17]          # query sitting on a duplicated corpus point
    q[4] = 0.0               # zero query
    return vecs, q


CASES = {
    "euclid_q": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="euclidean", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12), seed=0)),
    "euclid_q_s_eq_d": dict(m=1200, d=16, n_blobs=12, cfg=IndexConfig(
        metric="euclidean", n_clusters=10, rrr=RrrConfig(rank=5, reduced_dim=None), seed=1)),
    "euclid_exact_ivf": dict(m=900, d=20, n_blobs=9, cfg=IndexConfig(
        metric="euclidean", n_clusters=9, rrr=RrrConfig(rank=4, reduced_dim=10),
        scoring_mode="exact_ivf", seed=2)),
    "ip_q": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="ip", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12), seed=3)),
    "cosine_q": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="cosine", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12), seed=4)),
    "euclid_norerank": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="euclidean", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12), rerank=False, seed=5)),
    "euclid_d100": dict(m=2000, d=100, n_blobs=20, cfg=IndexConfig(
        metric="euclidean", n_clusters=16, rrr=RrrConfig(rank=8, reduced_dim=20), seed=6)),
    "euclid_f32": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="euclidean", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12, quantize=False), seed=7)),
    # unquantized (f32 factor) scoring across metrics / modes
    "ip_f32": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="ip", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12, quantize=False), seed=8)),
    "cosine_f32_s_eq_d": dict(m=1200, d=16, n_blobs=12, cfg=IndexConfig(
        metric="cosine", n_clusters=10, rrr=RrrConfig(rank=5, reduced_dim=None, quantize=False), seed=9)),
    "euclid_exact_ivf_f32": dict(m=900, d=20, n_blobs=9, cfg=IndexConfig(
        metric="euclidean", n_clusters=9, rrr=RrrConfig(rank=4, reduced_dim=10, quantize=False),
        scoring_mode="exact_ivf", seed=10)),
    "euclid_f32_norerank": dict(m=1500, d=24, n_blobs=15, cfg=IndexConfig(
        metric="euclidean", n_clusters=14, rrr=RrrConfig(rank=6, reduced_dim=12, quantize=False),
        rerank=False, seed=11)),
}


def stage_trace(index, x):
    metric = index.config.metric
    xp = (x.astype(np.float64) @ index.projection.astype(np.float64)).astype(F32)
    w = min(4, index.n_clusters)
    sel = route(xp, index.centroids, w, cluster_metric(metric))
    out = dict(xp=xp, selected=sel)
    if not index.config.rrr.quantize:
        out["scores"] = np.concatenate([score_cluster(xp, index.models[int(l)], metric) for l in sel])
        return out
    qx = quantize_vector(xp, mixed_precision=True)
    out.update(qhead=F32(qx.head), qscale=F32(qx.scale), qcodes=qx.values)
    raws, raws2, scores = [], [], []
    for l in sel:
        model = index.models[int(l)]
        raws.append(int8_gemv(qx, model.a))
        if model.b is not None:  # stage B: the re-quantized intermediate (rrr.py:196-197)
            inter = quantized_vecmat(xp, model.a, qx=qx)
            raws2.append(int8_gemv(quantize_vector(inter.astype(F32), mixed_precision=model.b.mixed),
                                   model.b))
        scores.append(score_cluster(xp, model, metric, query_quantized=qx))
    out["raw1"] = np.concatenate(raws)
    out["raw2"] = np.concatenate(raws2) if raws2 else np.zeros(0, np.int32)
    out["scores"] = np.concatenate(scores)
    return out


def main(only=None):
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        vecs, queries = corpus_with_outliers(spec["m"], spec["d"], seed=11, n_blobs=spec["n_blobs"])
        index = build(vecs, spec["cfg"], workers=4)
        blob = serialize(index)
        rec = dict(index_bytes=np.frombuffer(blob, dtype=np.uint8), queries=queries,
                   n_exact=np.int64(sum(m.exact for m in index.models)),
                   params=np.array([[k, w, t, int(rr)] for k, w, t, rr in PARAMS], dtype=np.int64))
        for pi, (k, w, t, rr) in enumerate(PARAMS):
            if rr and index.corpus is None:
                continue
            w = min(w, index.n_clusters)
            res = rrann.query_batch(index, queries, QueryParams(k=k, w=w, t=t, rerank=rr))
            kk = max(len(r.ids) for r in res)
            ids = np.full((len(res), k), -1, dtype=np.int64)
            sc = np.full((len(res), k), np.nan, dtype=F32)
            cnt = np.zeros(len(res), dtype=np.int32)
            for i, r in enumerate(res):
                ids[i, :len(r.ids)] = r.ids
                sc[i, :len(r.ids)] = r.scores
                cnt[i] = len(r.ids)
            rec[f"p{pi}_ids"] = ids
            rec[f"p{pi}_scores"] = sc
            rec[f"p{pi}_count"] = cnt
            assert kk <= k
        for qi in range(3):
            for key, val in stage_trace(index, queries[qi]).items():
                rec[f"trace{qi}_{key}"] = np.asarray(val)
        np.savez_compressed(OUT / f"{name}.npz", **rec)
        print(name, len(blob), "bytes", "exact clusters:", int(rec["n_exact"]))


def ground_truth_case():
    """rrann.bench.brute_force_knn outputs for the GPU ground truth (bench.py:85-124)."""
    from rrann.bench import brute_force_knn

    rng = np.random.default_rng(21)
    corpus = (rng.standard_normal((3000, 40)) * 2.0).astype(F32)
    corpus[7] = corpus[2900]        # duplicate rows: equal distances, lower id first
    corpus[11] = 0.0                # zero row (cosine norm 0 -> 1)
    queries = rng.standard_normal((48, 40)).astype(F32)
    queries[0] = corpus[2900]
    rec = dict(corpus=corpus, queries=queries)
    for metric in ("euclidean", "ip", "cosine"):
        rec[f"{metric}_k10"] = brute_force_knn(corpus, queries, 10, metric)
        rec[f"{metric}_k100"] = brute_force_knn(corpus, queries, 100, metric)
    np.savez_compressed(OUT / "ground_truth.npz", **rec)
    print("ground_truth", corpus.shape)


if __name__ == "__main__":
    if sys.argv[1:] == ["ground_truth"]:
        ground_truth_case()
        sys.exit(0)
    main(sys.argv[1:] or None)
