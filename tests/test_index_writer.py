"""The test-only random index writer produces files the oracle (deserialize restated) accepts."""

import numpy as np

from index_writer import random_index
from oracle import rrann_oracle as O


def test_random_index_parses_and_queries():
    blob = random_index(20, 8, 4, 5, 200, seed=1, dup_rows=2)
    idx = O.read_index(blob)
    assert idx.m == 200 and idx.L == 5 and idx.corpus.shape == (200, 20)
    res = O.query_batch(idx, np.random.default_rng(0).standard_normal((3, 20)).astype(np.float32), 5, 2, 30)
    assert all(len(r.ids) <= 5 for r in res)


def test_random_index_matches_reference_loader(rrann_ref):
    blob = random_index(33, 10, 5, 6, 150, metric="ip", seed=2)
    ref = rrann_ref.deserialize(blob)
    idx = O.read_index(blob)
    q = np.random.default_rng(1).standard_normal((8, 33)).astype(np.float32)
    a = rrann_ref.query_batch(ref, q, rrann_ref.QueryParams(k=4, w=3, t=20))
    b = O.query_batch(idx, q, 4, 3, 20)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.ids, y.ids)
