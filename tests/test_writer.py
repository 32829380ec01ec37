"""The streaming RRRANN01 writer (tools/rrrann_writer.py) emits rrann.serialize's exact bytes."""

import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import golden_cases, load_golden

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))


@pytest.mark.parametrize("case", golden_cases())
def test_streamed_file_equals_reference_serialize(rrann_ref, tmp_path, case):
    from rrann.index import deserialize, serialize

    import rrrann_writer as RW

    blob = load_golden(case)["index_bytes"].tobytes()
    idx = deserialize(blob)
    assert serialize(idx) == blob
    p = tmp_path / f"{case}.rrr"
    crc = RW.write_index(idx, p, corpus_chunk_rows=97)  # ragged corpus chunks
    assert p.read_bytes() == blob
    assert crc == int.from_bytes(blob[-4:], "little")


def test_streamed_build_roundtrip(rrann_ref, tmp_path):
    """A fresh reference build streamed to disk loads back (deserialize, the CRC check) and
    answers queries exactly like the in-memory index."""
    from rrann.bench import synth_dataset
    from rrann.index import IndexConfig, QueryParams, RrrIndex, build
    from rrann.rrr import RrrConfig

    import rrrann_writer as RW

    ds = synth_dataset(3000, 40, 32, kind="clustered", seed=3, n_blobs=30)
    idx = build(ds.vectors, IndexConfig(metric="euclidean", n_clusters=20,
                                        rrr=RrrConfig(rank=8, reduced_dim=16), seed=0), workers=4)
    p = tmp_path / "b.rrr"
    RW.write_index(idx, p, corpus_chunk_rows=1000)
    back = RrrIndex.load(str(p))
    qp = QueryParams(k=10, w=3, t=50)
    for a, b in zip(idx.query_batch(ds.queries, qp), back.query_batch(ds.queries, qp)):
        np.testing.assert_array_equal(a.ids, b.ids)
        np.testing.assert_array_equal(a.scores, b.scores)


def test_writer_rejects_short_files(tmp_path):
    import rrrann_writer as RW

    w = RW.RrrWriter(tmp_path / "x.rrr", metric="euclidean", dim=4, reduced_dim=2, rank=2, n_clusters=2,
                     n_points=3, flags=RW.FLAG_QUANTIZED)
    w.projection(np.zeros((4, 2)))
    w.centroids(np.zeros((2, 2)))
    w.cluster(np.arange(3), (np.zeros(3), np.ones(3), np.zeros((2, 3), np.int8)), None, np.zeros(3))
    with pytest.raises(ValueError):
        w.close()
