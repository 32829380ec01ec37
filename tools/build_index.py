"""Build a workload's index with the UNMODIFIED reference ``rrann`` (this container only).

Index construction is out of scope for the B200 path (BASELINE.json
north_star: "Index construction ... stays in the reference's Python, so both paths
search the identical index file").  This tool:

1. generates the corpus with ``rrann.bench.synth_dataset`` (clustered) and checks it
   equals ``paper_2410_18926_b200.workloads.synth_clustered`` bit for bit;
2. calls ``rrann.build`` + ``RrrIndex.save`` (``index.py:167-275,134-136``);
3. writes the model sidecar (file bytes before the corpus block) and a manifest with
   the file's CRC32 so the GPU box can re-materialise the identical file;
4. computes exact ground truth with ``brute_force_knn`` semantics
   (``bench.py:85-124``: f64 distances, ties to the lower id) -- chunked and with
   precomputed norms, same arithmetic expression;
5. optionally runs the reference ``query_batch`` over a (w, t) grid on a query
   sample to locate the recall@k >= 0.90 operating point.

Usage: python tools/build_index.py c2 [--workers 8] [--grid]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import workloads as W  # noqa: E402


def exact_gt(corpus: np.ndarray, queries: np.ndarray, k: int, chunk: int = 256) -> np.ndarray:
    """brute_force_knn (euclidean) with the reference's expression and stable ties."""
    c = corpus.astype(np.float64)
    cc = (c * c).sum(1)
    out = np.empty((queries.shape[0], k), dtype=np.int64)
    for s in range(0, queries.shape[0], chunk):
        q = queries[s:s + chunk].astype(np.float64)
        diss = (q * q).sum(1)[:, None] - 2.0 * (q @ c.T) + cc[None, :]
        part = np.argpartition(diss, k - 1, axis=1)[:, :k]
        for i in range(q.shape[0]):
            row = diss[i]
            kth = row[part[i]].max()
            cand = np.nonzero(row <= kth)[0]  # ascending ids -> stable ties
            order = cand[np.argsort(row[cand], kind="stable")][:k]
            out[s + i] = order
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--grid", action="store_true")
    ap.add_argument("--grid-queries", type=int, default=200)
    args = ap.parse_args()

    from rrann.bench import synth_dataset
    from rrann.index import IndexConfig, QueryParams, build
    from rrann.rrr import RrrConfig

    cfg = W.WORKLOADS[args.name]
    paths = W.workload_paths(args.name)
    W.DATA_DIR.mkdir(parents=True, exist_ok=True)
    t0 = time.perf_counter()
    ds = synth_dataset(cfg["m"], cfg["n_queries"], cfg["d"], kind="clustered",
                       seed=cfg["seed"], n_blobs=cfg["n_blobs"])
    corpus, queries = ds.vectors, ds.queries
    del ds
    mine_c, mine_q = W.synth_clustered(cfg["m"], cfg["n_queries"], cfg["d"], cfg["seed"], cfg["n_blobs"])
    assert np.array_equal(mine_c, corpus) and np.array_equal(mine_q, queries), "generator restatement drifted"
    del mine_c, mine_q
    print(f"synth {time.perf_counter() - t0:.1f}s", flush=True)

    train = None
    if cfg.get("ood"):  # out-of-distribution queries + the RRR training sample (C5)
        train, queries = W.ood_queries(cfg["d"], cfg["ood"]["n_train"], cfg["n_queries"],
                                       cfg["ood"]["seed"])
        np.save(paths["queries"], queries)
    t0 = time.perf_counter()
    icfg = IndexConfig(metric="euclidean", n_clusters=cfg["L"],
                       rrr=RrrConfig(rank=cfg["r"], reduced_dim=cfg["s"],
                                     train_source="query_sample" if train is not None else "corpus"),
                       seed=0)
    idx = build(corpus, icfg, train=train, workers=args.workers)
    del train
    build_s = time.perf_counter() - t0
    sizes = np.array([mdl.n_points for mdl in idx.models])
    print(f"build {build_s:.1f}s sizes min/med/max {sizes.min()}/{int(np.median(sizes))}/{sizes.max()} "
          f"exact {sum(mdl.exact for mdl in idx.models)}", flush=True)

    idx.save(paths["full"])
    data = paths["full"].read_bytes()
    corpus_bytes = corpus.nbytes
    corpus_off = len(data) - 4 - corpus_bytes
    assert data[corpus_off:corpus_off + corpus_bytes] == corpus.tobytes()
    paths["sidecar"].write_bytes(data[:corpus_off])
    crc = int.from_bytes(data[-4:], "little")
    assert crc == zlib.crc32(data[:-4]) & 0xFFFFFFFF
    man = dict(name=args.name, generator=dict(m=cfg["m"], d=cfg["d"], n_queries=cfg["n_queries"],
                                              seed=cfg["seed"], n_blobs=cfg["n_blobs"]),
               index=dict(L=cfg["L"], s=cfg["s"], r=cfg["r"], metric="euclidean", seed=0,
                          train_source="query_sample" if cfg.get("ood") else "corpus"),
               **({"ood": cfg["ood"]} if cfg.get("ood") else {}),
               k=cfg["k"], file_size=len(data), corpus_offset=corpus_off, crc32=crc,
               build_seconds=round(build_s, 1), built_by="rrann (reference, unmodified) via tools/build_index.py")
    del data

    t0 = time.perf_counter()
    gt = exact_gt(corpus, queries, max(100, cfg["k"]))
    np.save(paths["gt"], gt)
    print(f"gt {time.perf_counter() - t0:.1f}s", flush=True)

    if args.grid:
        from rrann.bench import mean_recall
        nq = args.grid_queries
        grid = []
        ws = (8, 16, 24, 32, 48, 64, 128, 256) if cfg.get("ood") else (1, 2, 4, 8, 16)
        ts = (800, 1600) if cfg.get("ood") else (100, 200, 400, 800, 1600)
        for w in ws:
            for t in ts:
                if t < cfg["k"]:
                    continue
                t1 = time.perf_counter()
                res = idx.query_batch(queries[:nq], QueryParams(k=cfg["k"], w=w, t=t))
                el = time.perf_counter() - t1
                rec = mean_recall(res, gt[:nq], cfg["k"])
                grid.append(dict(w=w, t=t, recall=round(rec, 5), qps_1core=round(nq / el, 1)))
                print(grid[-1], flush=True)
        man["grid"] = dict(queries=nq, points=grid)
    with open(paths["manifest"], "w") as f:
        json.dump(man, f, indent=1)
    print("done", flush=True)


if __name__ == "__main__":
    main()
