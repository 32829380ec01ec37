"""Host logic of the drop-in's lazily materialising result list (no GPU needed)."""

import pickle

import numpy as np


def _results(n=5, k=4):
    from paper_2410_18926_b200.search import QueryResults

    rng = np.random.default_rng(0)
    ids = rng.integers(0, 1000, size=(n, k)).astype(np.int64)
    sc = rng.standard_normal((n, k)).astype(np.float32)
    cnt = np.array([k, k - 1, 0, k, 2][:n], dtype=np.int32)
    return QueryResults(ids, sc, cnt, k), ids, sc, cnt


def test_items_match_dense_arrays():
    res, ids, sc, cnt = _results()
    assert isinstance(res, list) and len(res) == 5
    for i, r in enumerate(res):
        c = int(cnt[i])
        np.testing.assert_array_equal(r.ids, ids[i, :c])
        np.testing.assert_array_equal(r.scores, sc[i, :c])
        assert r.ids.dtype == np.int64 and r.scores.dtype == np.float32
        assert r.truncated == (c < 4)
    assert res[-1].ids.shape == (2,)
    assert [r.ids.shape[0] for r in res[1:3]] == [3, 0]
    assert [r.ids.shape[0] for r in reversed(res)] == [2, 4, 0, 3, 4]


def test_items_own_their_arrays_and_are_cached():
    res, ids, _, _ = _results()
    a = res[0]
    assert res[0] is a                     # built once
    a.ids[0] = -5                          # independent of the dense buffer and of others
    assert ids[0, 0] != -5
    assert None not in list.__iter__(res.materialize())


def test_pickle_and_list_conversion():
    res, ids, _, _ = _results()
    back = pickle.loads(pickle.dumps(res))
    assert type(back) is list and len(back) == 5
    np.testing.assert_array_equal(back[3].ids, ids[3])
    plain = list(res)
    assert len(plain) == 5 and all(p is q for p, q in zip(plain, res))
