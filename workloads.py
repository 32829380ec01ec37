"""Synthetic workloads and index materialisation (off the hot path).

``synth_clustered`` restates the reference generator ``rrann.bench.synth_dataset``
(kind="clustered", ``pkg/src/rrann/bench.py:140-170``) call for call on the same
``numpy.random.Generator`` stream, so corpus and queries are bit-identical to the
reference's for the same seed.  It generates the corpus noise in row chunks (the
PCG64 normal stream is sequential, so chunked draws equal one big draw) to keep
peak host memory near the f32 output size instead of 3x the f64 size.

Index files are built once, off the GPU box, by the unmodified reference
(``tools/build_index.py``).  The corpus block of an ``RRRANN01`` file is the raw
f32 corpus, which is deterministic from the generator seed, so what travels to
the GPU box is the file *minus* its corpus block (a "model sidecar") plus a small
JSON manifest; ``materialize_index`` regenerates the corpus, splices it back and
checks the result against the original file's own CRC32 trailer
(``pkg/src/rrann/index.py:401``), proving byte identity with the reference's file.
"""

from __future__ import annotations

import json
import os
import struct
import zlib
from pathlib import Path

import numpy as np

F32 = np.float32

REPO_ROOT = Path(__file__).resolve().parent
DATA_DIR = REPO_ROOT / "data"

# Workload registry: name -> generator / index parameters.  C1 and C2 follow
# BASELINE.json configs[0] and configs[1]; n_blobs = m/1000 per SURVEY.md §8(d).
WORKLOADS = {
    "c1": dict(m=100_000, d=128, n_queries=10_000, seed=1, n_blobs=100,
               L=256, s=64, r=32, k=10),
    "c2": dict(m=1_000_000, d=768, n_queries=10_000, seed=1, n_blobs=1000,
               L=1024, s=256, r=32, k=100),
    # C3 (BASELINE.json configs[2]): OpenAI-embedding shape, s = 64 (the reference default)
    "c3": dict(m=1_000_000, d=1536, n_queries=10_000, seed=1, n_blobs=1000,
               L=2048, s=64, r=32, k=100),
    # C5 (configs[4]): C2's corpus, out-of-distribution queries (test_acceptance.py:321-329
    # scaled up), RRR fitted on a held-out query sample (RrrConfig(train_source="query_sample"))
    "c5": dict(m=1_000_000, d=768, n_queries=10_000, seed=1, n_blobs=1000,
               L=1024, s=256, r=32, k=100, ood=dict(n_train=100_000, seed=5)),
    # tiny workload for smoke tests / golden fixtures
    "tiny": dict(m=4_000, d=32, n_queries=256, seed=7, n_blobs=40,
                 L=32, s=16, r=8, k=10),
}

_CHUNK_ROWS = 65_536


def synth_clustered(m: int, n_queries: int, d: int, seed: int, n_blobs: int,
                    with_corpus: bool = True):
    """(corpus f32 m x d | None, queries f32 n_queries x d), reference bit-exact.

    Call order mirrors bench.py:156-165: centers, labels, corpus noise,
    query labels, query noise.
    """
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((n_blobs, d)) * 6.0
    labels = rng.integers(n_blobs, size=m)
    corpus = np.empty((m, d), dtype=F32) if with_corpus else None
    for start in range(0, m, _CHUNK_ROWS):
        stop = min(m, start + _CHUNK_ROWS)
        noise = rng.standard_normal((stop - start, d))
        if corpus is not None:
            corpus[start:stop] = (centers[labels[start:stop]] + noise).astype(F32)
    qlabels = rng.integers(n_blobs, size=n_queries)
    queries = (centers[qlabels] + rng.standard_normal((n_queries, d))).astype(F32)
    return corpus, queries


def ood_queries(d: int, n_train: int, n_queries: int, seed: int):
    """(train, queries) f32 drawn like test_acceptance.py:_ood_trial (lines 321-333):
    (z * 2*0.85^i + shift) @ R^T with shift ~ 1.5 N(0, I) and R = random_rotation(d, seed+1000)
    (linalg.py:109-117).  Run in the dev container; the queries are stored in data/
    (the QR's last bits depend on the host's LAPACK kernels)."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from rrann.linalg import random_rotation

    rng = np.random.default_rng(seed)
    rot = random_rotation(d, seed=seed + 1000).astype(np.float64)
    scales = 2.0 * (0.85 ** np.arange(d))
    shift = rng.standard_normal(d) * 1.5

    def draw(n):
        z = rng.standard_normal((n, d)) * scales
        return ((z + shift) @ rot.T).astype(F32)

    train = draw(n_train)
    return train, draw(n_queries)


def workload_paths(name: str):
    return dict(
        full=DATA_DIR / f"{name}.rrr",
        sidecar=DATA_DIR / f"{name}.rrrm",
        manifest=DATA_DIR / f"{name}.json",
        gt=DATA_DIR / f"{name}.gt.npy",
        queries=DATA_DIR / f"{name}.queries.npy",
    )


def load_manifest(name: str) -> dict:
    with open(workload_paths(name)["manifest"]) as f:
        return json.load(f)


def materialize_index(name: str, out_path: str | os.PathLike | None = None) -> Path:
    """Return a path to the full RRRANN01 file for ``name``.

    Uses ``data/<name>.rrr`` when present and intact; otherwise rebuilds it from
    the sidecar + regenerated corpus and verifies the CRC32 stored in the
    manifest (== the reference file's trailer).
    """
    paths = workload_paths(name)
    man = load_manifest(name)
    full = Path(out_path) if out_path is not None else paths["full"]
    if full.exists() and full.stat().st_size == man["file_size"]:
        return full
    if not paths["sidecar"].exists():
        raise FileNotFoundError(f"{paths['sidecar']} missing; run tools/build_index.py {name}")
    head = paths["sidecar"].read_bytes()
    if len(head) != man["corpus_offset"]:
        raise ValueError("sidecar size does not match manifest corpus_offset")
    g = man["generator"]
    corpus, _ = synth_clustered(g["m"], 1, g["d"], g["seed"], g["n_blobs"])
    crc = zlib.crc32(head)
    crc = zlib.crc32(memoryview(corpus).cast("B"), crc) & 0xFFFFFFFF
    if crc != man["crc32"]:
        raise ValueError(f"regenerated {name} index CRC {crc:#x} != reference {man['crc32']:#x}")
    full.parent.mkdir(parents=True, exist_ok=True)
    tmp = full.with_suffix(".tmp")
    with open(tmp, "wb") as f:
        f.write(head)
        f.write(memoryview(corpus).cast("B"))
        f.write(struct.pack("<I", crc))
    os.replace(tmp, full)
    return full


def load_queries(name: str, n: int | None = None) -> np.ndarray:
    man = load_manifest(name)
    g = man["generator"]
    nq = g["n_queries"] if n is None else n
    qp = workload_paths(name)["queries"]
    if qp.exists():  # stored query set (out-of-distribution workloads)
        return np.load(qp)[:nq]
    # queries come after the corpus in the rng stream; skip corpus materialisation
    _, q = synth_clustered(g["m"], g["n_queries"], g["d"], g["seed"], g["n_blobs"],
                           with_corpus=False)
    return q[:nq]


def load_ground_truth(name: str) -> np.ndarray | None:
    p = workload_paths(name)["gt"]
    return np.load(p) if p.exists() else None
