import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_cases():
    """Index fixtures (an RRRANN01 file + reference query results); ground_truth.npz is separate."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "ground_truth")


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@pytest.fixture(scope="session")
def rrann_ref():
    """The unmodified reference, importable only in the dev container."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import rrann
    return rrann


def assert_topk_equivalent(ids, sc, ref_ids, ref_sc, rtol=1e-5, scale=None, what=""):
    """ids/scores equal up to documented ties for BLAS-order-dependent floats.

    Scores must agree within ``rtol`` (relative to ``scale`` when given -- e.g. the
    x.x term a no-rerank euclidean score is shifted by -- else to the score).  Ids
    may differ only at positions whose reference score is tied, within that
    tolerance, with the score of a position holding the other id (a swap inside a
    near-tie group) or with the k-th (boundary) score.
    """
    ids = np.asarray(ids)
    ref_ids = np.asarray(ref_ids)
    sc = np.asarray(sc, dtype=np.float64)
    ref_sc = np.asarray(ref_sc, dtype=np.float64)
    assert ids.shape == ref_ids.shape, what
    mag = np.abs(ref_sc) if scale is None else np.maximum(np.abs(ref_sc), abs(scale))
    tol = rtol * mag + 1e-30
    assert np.all(np.abs(sc - ref_sc) <= tol), (what, sc, ref_sc)
    if np.array_equal(ids, ref_ids):
        return
    ref_pos = {int(v): j for j, v in enumerate(ref_ids)}
    for i in np.nonzero(ids != ref_ids)[0]:
        j = ref_pos.get(int(ids[i]))
        if j is not None:
            assert abs(ref_sc[j] - ref_sc[i]) <= tol[i] + tol[j], (what, i, j)
        else:  # id not in the reference top-k: must tie with the boundary
            assert abs(sc[i] - ref_sc[-1]) <= tol[i] + tol[-1], (what, i)
