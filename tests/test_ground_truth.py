"""Exact k-NN ground truth (rrann.bench.brute_force_knn, bench.py:85-124) on the GPU.

CPU tests pin the oracle restatement to the reference's own outputs
(tests/golden/ground_truth.npz, made by make_golden.py from the unmodified
reference); GPU tests compare rrg_ground_truth with both.  Ids are compared
exactly: the f64 distances of the device (tensor-core summation order) and of
NumPy/OpenBLAS differ only at the 1e-16 level, far below the gaps of these
inputs, and exact ties (duplicate rows) resolve to the lower id on both.
"""

import numpy as np
import pytest

from conftest import load_golden

METRICS = ["euclidean", "ip", "cosine"]


@pytest.mark.parametrize("metric", METRICS)
def test_oracle_matches_reference_golden(metric):
    from oracle import rrann_oracle as O

    g = load_golden("ground_truth")
    for k in (10, 100):
        np.testing.assert_array_equal(O.brute_force_knn(g["corpus"], g["queries"], k, metric),
                                      g[f"{metric}_k{k}"])


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_18926_b200 as p
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("metric", METRICS)
@pytest.mark.parametrize("chunk", [None, "700"])
def test_gpu_matches_reference_golden(pkg, metric, chunk, monkeypatch):
    if chunk:  # several corpus chunks: exercises the running top-k merge
        monkeypatch.setenv("RRG_GT_CHUNK", chunk)
    g = load_golden("ground_truth")
    for k in (10, 100):
        ids = pkg.brute_force_knn(g["corpus"], g["queries"], k, metric)
        np.testing.assert_array_equal(ids, g[f"{metric}_k{k}"], err_msg=f"{metric} k={k}")


@pytest.mark.gpu
@pytest.mark.parametrize("m,d,nq,k,metric,chunk", [
    (5000, 3, 64, 10, "euclidean", None),       # d=3: many near-equal distances
    (20000, 128, 200, 100, "euclidean", "3000"),
    (8000, 768, 40, 100, "euclidean", None),
    (6000, 100, 50, 1000, "ip", "2500"),
    (300, 16, 30, 300, "cosine", None),          # k == m: everything selected
    (4000, 64, 33, 1, "euclidean", "999"),
    (50000, 32, 100, 2048, "euclidean", None),   # k at the device maximum
])
def test_gpu_matches_oracle_random(pkg, m, d, nq, k, metric, chunk, monkeypatch):
    from oracle import rrann_oracle as O

    if chunk:
        monkeypatch.setenv("RRG_GT_CHUNK", chunk)
    rng = np.random.default_rng(m + d)
    c = rng.standard_normal((m, d)).astype(np.float32)
    c[10:20] = c[0]  # a block of exact duplicates
    q = rng.standard_normal((nq, d)).astype(np.float32)
    q[1] = c[0]
    ids = pkg.brute_force_knn(c, q, k, metric)
    ref = O.brute_force_knn(c, q, k, metric)
    np.testing.assert_array_equal(ids, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("n_tie,k", [(4000, 2000), (6000, 100), (9000, 2048)])
def test_gpu_heavy_ties(pkg, n_tie, k):
    """More exact ties at the k-th distance than fit on-chip: resolved on the id digits."""
    c = np.ones((n_tie + 3000, 8), np.float32)
    c[1500:1500 + n_tie] = 0.0  # n_tie rows at distance 0 from the zero query
    q = np.zeros((3, 8), np.float32)
    ids = pkg.brute_force_knn(c, q, k)
    np.testing.assert_array_equal(ids, np.tile(np.arange(1500, 1500 + k), (3, 1)))


@pytest.mark.gpu
def test_gpu_errors(pkg):
    c = np.zeros((50, 8), np.float32)
    q = np.zeros((4, 8), np.float32)
    with pytest.raises(pkg.ParameterError, match="out of range"):
        pkg.brute_force_knn(c, q, 0)
    with pytest.raises(pkg.ParameterError, match="out of range"):
        pkg.brute_force_knn(c, q, 51)
    with pytest.raises(pkg.ParameterError, match="unknown metric"):
        pkg.brute_force_knn(c, q, 5, "l1")
    with pytest.raises(pkg.ShapeError):
        pkg.brute_force_knn(c, q[:, :3], 5)


@pytest.mark.gpu
def test_c2_ground_truth_matches_cpu(pkg):
    """Full C2 (1M x 768, 10k queries, k=100) vs the CPU exact ground truth of tools/build_index.py."""
    import torch

    import workloads as W

    gt = W.load_ground_truth("c2")
    if gt is None:
        pytest.skip("workload c2 not built")
    man = W.load_manifest("c2")
    g = man["generator"]
    corpus, q = W.synth_clustered(g["m"], g["n_queries"], g["d"], g["seed"], g["n_blobs"])
    c_dev = torch.from_numpy(corpus).cuda()
    ids = pkg.ground_truth_device(c_dev, torch.from_numpy(q).cuda(), gt.shape[1]).cpu().numpy()
    bad = np.nonzero((ids != gt).any(axis=1))[0]
    for i in bad:  # only f64 rounding-level near-ties may reorder
        x = q[i].astype(np.float64)
        cand = np.union1d(ids[i], gt[i])
        dd = ((corpus[cand].astype(np.float64) - x) ** 2).sum(1)
        kth = np.sort(dd)[gt.shape[1] - 1]
        diff = np.setxor1d(ids[i], gt[i])
        dmap = dict(zip(cand.tolist(), dd.tolist()))
        assert all(abs(dmap[int(v)] - kth) <= 1e-9 * kth for v in diff), i
    assert len(bad) <= 5, len(bad)
