"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden vectors and the CPU oracle.

Tolerances (BASELINE.json north_star): cluster selection, int32 products and
neighbour ids bit-exact (up to documented ties); euclidean re-ranked distances
bit-exact (NumPy pairwise tree restated); BLAS-order-dependent floats (ip/cosine
re-rank sgemv, the no-rerank euclidean x.x shift) within 1e-5 relative.
"""

import threading

import numpy as np
import pytest

from conftest import assert_topk_equivalent, golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32 = np.float32
RTOL = 1e-5


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_18926_b200 as p
    return p


def _write(tmp_path, name, blob):
    p = tmp_path / f"{name}.rrr"
    p.write_bytes(blob)
    return p


def _golden_index(pkg, tmp_path, case):
    g = load_golden(case)
    return g, pkg.DeviceIndex.from_file(_write(tmp_path, case, g["index_bytes"].tobytes()))


QUANT_CASES = [c for c in golden_cases() if "f32" not in c]
F32_CASES = [c for c in golden_cases() if "f32" in c]


def _corpus_max_norm(g):
    from oracle import rrann_oracle as O

    idx = O.read_index(g["index_bytes"].tobytes())
    return 0.0 if idx.corpus is None else float(np.linalg.norm(idx.corpus, axis=1).max())


@pytest.mark.parametrize("case", QUANT_CASES)
@pytest.mark.parametrize("entry", ["host", "device", "device-querymajor", "device-warpsel", "device-screen"])
def test_golden_end_to_end(pkg, tmp_path, case, entry, monkeypatch):
    if entry == "device-querymajor":  # the fused query-major scoring kernel
        monkeypatch.setenv("RRG_SCORE_MODE", "query")
        entry = "device"
    if entry == "device-warpsel":  # warp-per-query selections + cluster-major re-rank
        monkeypatch.setenv("RRG_WARP_SELECT", "1")
        monkeypatch.setenv("RRG_RERANK", "cluster")
        entry = "device"
    if entry == "device-screen":  # tensor-core screen of the cluster-major re-rank
        monkeypatch.setenv("RRG_RERANK", "cluster")
        monkeypatch.setenv("RRG_SCREEN", "1")
        entry = "device"
    g, dev = _golden_index(pkg, tmp_path, case)
    for pi, (k, w, t, rr) in enumerate(g["params"]):
        if f"p{pi}_ids" not in g:
            continue
        k, w, t, rr = int(k), min(int(w), dev.n_clusters), int(t), bool(rr)
        if entry == "host":
            ids, sc, cnt = dev.search_host(g["queries"], k, w, t, rr)
        else:
            q = torch.from_numpy(g["queries"]).cuda()
            ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(q, k, w, t, rr))
        np.testing.assert_array_equal(cnt, g[f"p{pi}_count"], err_msg=f"{case} p{pi} count")
        ref_ids = g[f"p{pi}_ids"]
        ref_sc = g[f"p{pi}_scores"]
        q = g["queries"].astype(np.float64)
        cmax = _corpus_max_norm(g)
        for i in range(len(cnt)):
            c = int(cnt[i])
            if dev.metric == "euclidean" and rr:  # exact: NumPy pairwise tree restated
                np.testing.assert_array_equal(ids[i, :c], ref_ids[i, :c], err_msg=f"{case} p{pi} q{i}")
                np.testing.assert_array_equal(sc[i, :c].view(np.int32), ref_sc[i, :c].view(np.int32))
            elif not rr:  # ids from exact int8 keys; score shift x.x is BLAS sdot (tolerance)
                np.testing.assert_array_equal(ids[i, :c], ref_ids[i, :c], err_msg=f"{case} p{pi} q{i}")
                scale = float(q[i] @ q[i]) if dev.metric == "euclidean" else None
                assert_topk_equivalent(ids[i, :c], sc[i, :c], ref_ids[i, :c], ref_sc[i, :c], RTOL,
                                       scale, f"{case} p{pi} q{i}")
            else:  # ip/cosine re-rank: BLAS sgemv order -> tolerance (scale |x||c|) + near-tie swaps
                scale = float(np.sqrt(q[i] @ q[i]) * cmax)
                assert_topk_equivalent(ids[i, :c], sc[i, :c], ref_ids[i, :c], ref_sc[i, :c], RTOL,
                                       scale, f"{case} p{pi} q{i}")


@pytest.mark.parametrize("case", QUANT_CASES)
def test_golden_stages(pkg, tmp_path, case):
    g, dev = _golden_index(pkg, tmp_path, case)
    x = torch.from_numpy(g["queries"][:3]).cuda()
    xp, qc, qs, qh = dev.stage_project(x)
    torch.cuda.synchronize()
    xp = xp.cpu().numpy()
    qc = qc.cpu().numpy()
    for i in range(3):
        np.testing.assert_array_equal(xp[i].view(np.int32), g[f"trace{i}_xp"].view(np.int32))
        s = dev.reduced_dim
        np.testing.assert_array_equal(qc[i, 1:s], g[f"trace{i}_qcodes"])
        assert qc[i, 0] == 0
        assert qs[i].item() == g[f"trace{i}_qscale"] and qh[i].item() == g[f"trace{i}_qhead"]
    w = min(4, dev.n_clusters)
    sel = dev.stage_route(torch.from_numpy(xp).cuda(), w).cpu().numpy()
    for i in range(3):
        assert set(sel[i].tolist()) == set(g[f"trace{i}_selected"].tolist())


@pytest.mark.parametrize("case", QUANT_CASES)
def test_golden_stage_score_bits(pkg, tmp_path, case):
    """K4 (score_cluster, rrr.py:181-203) bit for bit against the reference's own
    intermediates: the stage-A int32 products (int8_gemv(qx, A)), the stage-B int32
    products of the re-quantized intermediate (int8_gemv(q(inter), B)) and the f32
    per-point scores, for the probes the reference routed to (trace order)."""
    g, dev = _golden_index(pkg, tmp_path, case)
    x = torch.from_numpy(g["queries"][:3]).cuda()
    w = len(g["trace0_selected"])
    sel = torch.tensor(np.stack([g[f"trace{i}_selected"] for i in range(3)]), dtype=torch.int32)
    raw1, raw2, sc, off = (a.cpu().numpy() for a in dev.stage_score(x, sel.cuda()))
    sizes = dev.cluster_sizes()
    r = dev.rank
    for i in range(3):
        cand = slice(off[i], off[i + 1])
        np.testing.assert_array_equal(sc[cand].view(np.int32), g[f"trace{i}_scores"].view(np.int32),
                                      err_msg=f"{case} q{i} scores")
        # raw1 concatenates per probe: r stage-A products (RRR) or m_l (exact model)
        ref1 = g[f"trace{i}_raw1"]
        ref2 = g.get(f"trace{i}_raw2")
        o1 = o2 = oc = 0
        for c, l in enumerate(g[f"trace{i}_selected"]):
            m = int(sizes[l])
            exact = m < r or "exact_ivf" in case
            if exact:  # single-factor model: its stage-A product is the per-point raw
                np.testing.assert_array_equal(raw2[off[i] + oc: off[i] + oc + m], ref1[o1:o1 + m])
                o1 += m
            else:
                np.testing.assert_array_equal(raw1[i, c], ref1[o1:o1 + r], err_msg=f"{case} q{i} A")
                o1 += r
                if ref2 is not None:
                    np.testing.assert_array_equal(raw2[off[i] + oc: off[i] + oc + m], ref2[o2:o2 + m],
                                                  err_msg=f"{case} q{i} B")
                    o2 += m
            oc += m
        assert o1 == len(ref1)


@pytest.mark.parametrize("metric", ["ip", "cosine", "euclidean"])
@pytest.mark.parametrize("entry", ["host", "device"])
def test_nonfinite_batch_fused_routing(pkg, tmp_path, metric, entry):
    """A 64-query batch with one NaN (w = 1: the fused argmin routing, > 32 queries so
    the GEMM path runs): DataError, and the handle keeps working afterwards."""
    from index_writer import random_index

    blob = random_index(96, 32, 8, 12, 900, metric, seed=5)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "nan", blob))
    q = np.random.default_rng(3).standard_normal((64, 96)).astype(F32)
    good = dev.search_host(q, 10, 1, 50, True)
    bad = q.copy()
    bad[17, 3] = np.nan
    bad_inf = q.copy()
    bad_inf[40, 0] = np.inf
    for b in (bad, bad_inf):
        if entry == "host":
            with pytest.raises(pkg.DataError):
                dev.search_host(b, 10, 1, 50, True)
        else:
            with pytest.raises(pkg.DataError):
                pkg.query_batch(dev, torch.from_numpy(b).cuda(), pkg.QueryParams(k=10, w=1, t=50))
        # the next search on the same handle succeeds and is unchanged
        again = dev.search_host(q, 10, 1, 50, True)
        for a, e in zip(again, good):
            np.testing.assert_array_equal(a, e)
    # the device entry itself (no host check) must not fault on the NaN row either
    ids, sc, cnt = dev.search_device(torch.from_numpy(bad).cuda(), 10, 1, 50, True)
    torch.cuda.synchronize()
    ok = np.ones(64, bool)
    ok[17] = False
    np.testing.assert_array_equal(ids.cpu().numpy()[ok], good[0][ok])


# ---------------------------------------------------- unquantized (f32) factors
# score = x @ A (@ B) runs as OpenBLAS sgemv in the reference (rrr.py:97-100), an
# FMA order the GPU cannot reproduce, so the approximate scores
# match within F32_RTOL of their magnitude and the candidate set may differ only
# by near-ties at the top-t (or top-k) boundary.  Everything downstream of the
# candidate set (the exact re-rank, its (diss, id) order) is still checked exactly.
F32_RTOL = 1e-5


def _f32_check_query(O, oidx, x, k, w, t, rr, ids, sc, cnt, cmax, what):
    tr = {}
    ref = O.query(oidx, x, k, w, t, rr, trace=tr)
    c = int(cnt)
    assert c == len(ref.ids), what
    ids, sc = ids[:c], sc[:c].astype(np.float64)
    euclid = oidx.metric == "euclidean"
    xp = tr["xp"].astype(np.float64)
    mags = []
    for l in tr["selected"]:  # |x| @ |A| (@ |B|) (+ |norm|): the scale of the sgemv error
        cl = oidx.clusters[int(l)]
        y = np.abs(xp) @ np.abs(cl.a.astype(np.float64))
        if cl.b is not None:
            y = y @ np.abs(cl.b.astype(np.float64))
        mags.append(2.0 * y + np.abs(cl.norms) if euclid else y)
    tol = F32_RTOL * np.concatenate(mags) + 1e-30
    keys = tr["cand_keys"].astype(np.float64)
    cid = tr["cand_ids"]
    order = np.lexsort((cid, keys))
    take = min(t if rr else k, len(cid))
    kt, tt = keys[order[take - 1]], tol[order[take - 1]]
    possible = set(cid[keys <= kt + tol + tt].tolist())
    certain = cid[keys < kt - tol - tt]
    assert set(ids.tolist()) <= possible, (what, "id outside the near-tie candidate set")
    pos = {int(v): i for i, v in enumerate(cid)}
    if not rr:  # top-k by approximate key; score = key + x.x (sdot) or -key
        assert set(certain.tolist()) <= set(ids.tolist()), (what, "missed a certain candidate")
        xx = float(x.astype(np.float64) @ x.astype(np.float64)) if euclid else 0.0
        for j, v in enumerate(ids):
            i = pos[int(v)]
            want = keys[i] + xx if euclid else -keys[i]
            assert abs(sc[j] - want) <= tol[i] + F32_RTOL * xx, (what, j)
        return
    # re-rank: scores are the exact dissimilarities of the returned ids
    diss = O.exact_dissimilarity(oidx, x, ids).astype(np.float64)
    got = sc if euclid else -sc
    if euclid:
        np.testing.assert_array_equal(sc.astype(np.float32).view(np.int32),
                                      diss.astype(np.float32).view(np.int32), err_msg=what)
        dtol = 0.0
    else:
        dtol = RTOL * float(np.sqrt(x.astype(np.float64) @ x.astype(np.float64)) * cmax)
        assert np.all(np.abs(got - diss) <= dtol), what
    # ... and the top-k by (diss, id) of a candidate set holding every certain candidate
    last = (got[-1], int(ids[-1]))
    rest = np.setdiff1d(certain, ids)
    if rest.size:
        rd = O.exact_dissimilarity(oidx, x, rest).astype(np.float64)
        for dv, iv in zip(rd, rest):
            assert (dv, int(iv)) > last or abs(dv - last[0]) <= 2 * dtol, (what, int(iv))


@pytest.mark.parametrize("case", F32_CASES)
@pytest.mark.parametrize("entry", ["host", "device"])
def test_golden_f32_factors(pkg, tmp_path, case, entry):
    """Unquantized index (RrrConfig.quantize=False) through the f32-factor scoring kernel."""
    from oracle import rrann_oracle as O

    g, dev = _golden_index(pkg, tmp_path, case)
    oidx = O.read_index(g["index_bytes"].tobytes())
    cmax = _corpus_max_norm(g)
    exact_hits = total = 0
    for pi, (k, w, t, rr) in enumerate(g["params"]):
        if f"p{pi}_ids" not in g:
            continue
        k, w, t, rr = int(k), min(int(w), dev.n_clusters), int(t), bool(rr)
        if entry == "host":
            ids, sc, cnt = dev.search_host(g["queries"], k, w, t, rr)
        else:
            q = torch.from_numpy(g["queries"]).cuda()
            ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(q, k, w, t, rr))
        np.testing.assert_array_equal(cnt, g[f"p{pi}_count"], err_msg=f"{case} p{pi} count")
        for i in range(len(cnt)):
            c = int(cnt[i])
            _f32_check_query(O, oidx, g["queries"][i], k, w, t, rr, ids[i], sc[i], cnt[i], cmax,
                             f"{case} p{pi} q{i}")
            exact_hits += np.array_equal(ids[i, :c], g[f"p{pi}_ids"][i, :c])
            total += 1
    assert exact_hits >= 0.9 * total, (exact_hits, total)  # near-ties are rare


@pytest.mark.parametrize("case", F32_CASES)
def test_golden_f32_stages(pkg, tmp_path, case):
    """Projection and routing of an unquantized index are exact like the int8 path's."""
    g, dev = _golden_index(pkg, tmp_path, case)
    x = torch.from_numpy(g["queries"][:3]).cuda()
    xp = dev.stage_project(x)[0]
    torch.cuda.synchronize()
    xp = xp.cpu().numpy()
    for i in range(3):
        np.testing.assert_array_equal(xp[i].view(np.int32), g[f"trace{i}_xp"].view(np.int32))
    sel = dev.stage_route(torch.from_numpy(xp).cuda(), min(4, dev.n_clusters)).cpu().numpy()
    for i in range(3):
        assert set(sel[i].tolist()) == set(g[f"trace{i}_selected"].tolist())


def test_validation_errors(pkg, tmp_path):
    g, dev = _golden_index(pkg, tmp_path, "euclid_q")
    q = g["queries"][:4]
    with pytest.raises(pkg.ParameterError, match="k must be >= 1"):
        dev.search_host(q, 0, 1, 10)
    with pytest.raises(pkg.ParameterError, match="out of range"):
        dev.search_host(q, 5, dev.n_clusters + 1, 10)
    with pytest.raises(pkg.ParameterError, match="t must be >= 1"):
        dev.search_host(q, 5, 1, 0)
    with pytest.raises(pkg.ParameterError, match="when re-ranking"):
        dev.search_host(q, 11, 1, 10)
    with pytest.raises(pkg.ShapeError, match="query dimension"):
        dev.search_host(q[:, :5], 5, 1, 10)
    bad = q.copy()
    bad[1, 2] = np.nan
    with pytest.raises(pkg.DataError):
        dev.search_host(bad, 5, 1, 10)
    g2, dev2 = _golden_index(pkg, tmp_path, "euclid_norerank")
    with pytest.raises(pkg.ParameterError, match="without the corpus"):
        dev2.search_host(g2["queries"][:2], 5, 1, 10, True)


def test_format_errors(pkg, tmp_path):
    blob = load_golden("euclid_q")["index_bytes"].tobytes()
    with pytest.raises(pkg.FormatError, match="truncated file: corpus"):
        pkg.DeviceIndex.from_file(_write(tmp_path, "t", blob[:-100]))
    bad = bytearray(blob)
    bad[300] ^= 1
    with pytest.raises(pkg.FormatError, match="crc mismatch"):
        pkg.DeviceIndex.from_file(_write(tmp_path, "c", bytes(bad)))
    with pytest.raises(pkg.FormatError, match="unknown trailing section"):
        pkg.DeviceIndex.from_file(_write(tmp_path, "x", blob + b"abc"))
    good = _write(tmp_path, "g", blob)
    for bad_range in [(-1, 2), (3, 2), (0, 10 ** 6)]:  # shard ranges outside [0, L]
        with pytest.raises(pkg.ParameterError, match="shard cluster range"):
            pkg.DeviceIndex.from_file(good, shard=bad_range)


def test_drop_in_query_batch(pkg, tmp_path):
    g, dev = _golden_index(pkg, tmp_path, "euclid_q")
    params = pkg.QueryParams(k=10, w=3, t=50)
    res = pkg.query_batch(dev, g["queries"], params)
    assert len(res) == g["queries"].shape[0]
    for i, r in enumerate(res):
        assert r.ids.dtype == np.int64 and r.scores.dtype == np.float32
        np.testing.assert_array_equal(r.ids, g["p1_ids"][i][: g["p1_count"][i]])
        assert r.truncated == (len(r.ids) < 10)
    assert pkg.query_batch(dev, np.zeros((0, dev.dim), F32), pkg.QueryParams(k=0)) == []
    one = pkg.query(dev, g["queries"][0], params)
    np.testing.assert_array_equal(one.ids, res[0].ids)
    cuda_res = pkg.query_batch(dev, torch.from_numpy(g["queries"]).cuda(), params)
    for a, b in zip(res, cuda_res):
        np.testing.assert_array_equal(a.ids, b.ids)


def test_concurrent_searches_identical(pkg, tmp_path):
    g, dev = _golden_index(pkg, tmp_path, "euclid_d100")
    q = g["queries"]
    base = dev.search_host(q, 10, 4, 200)
    out = [None] * 4

    def run(i):
        out[i] = dev.search_host(q, 10, 4, 200)

    th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for o in out:
        for a, b in zip(o, base):
            np.testing.assert_array_equal(a, b)


def test_skewed_cluster_exceeds_cluster_rerank_smem(pkg, tmp_path):
    """One 90k-row cluster: its membership bitmap no longer fits the cluster-major
    re-rank's shared memory, so the plan must fall back to the per-query re-rank and
    still return the reference's ids and bit-exact scores."""
    from index_writer import random_index
    from oracle import rrann_oracle as O

    sizes = [90_000, 150, 100, 50]
    blob = random_index(768, 32, 8, 4, sum(sizes), "euclidean", seed=5, sizes=sizes)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "skew", blob))
    oidx = O.read_index(blob)
    q = np.random.default_rng(3).standard_normal((6, 768)).astype(F32)
    q[0] = oidx.corpus[7]
    for k, w, t in [(10, 1, 200), (20, 4, 1000)]:
        ids, sc, cnt = dev.search_host(q, k, w, t, True)
        ref = O.query_batch(oidx, q, k, w, t, True)
        for i, rres in enumerate(ref):
            c = int(cnt[i])
            np.testing.assert_array_equal(ids[i, :c], rres.ids)
            np.testing.assert_array_equal(sc[i, :c].view(np.int32), rres.scores.view(np.int32))


def test_exactness_limit_recall_one(pkg, tmp_path):
    """w = L, t = all candidates, rerank -> exact top-k (test_index.py:100-106)."""
    from oracle import rrann_oracle as O

    g, dev = _golden_index(pkg, tmp_path, "euclid_d100")
    oidx = O.read_index(g["index_bytes"].tobytes())
    q = g["queries"][:32]
    k = 10
    ids, sc, cnt = dev.search_host(q, k, dev.n_clusters, oidx.m, True)
    c = oidx.corpus.astype(np.float64)
    for i in range(q.shape[0]):
        d2 = ((c - q[i].astype(np.float64)) ** 2).sum(1)
        truth = np.argsort(d2, kind="stable")[:k]
        assert set(ids[i].tolist()) == set(truth.tolist())


# ------------------------------------------------------------- workload-size parity


def _workload(pkg, name):
    import workloads as W

    try:
        path = W.materialize_index(name)
    except FileNotFoundError:
        pytest.skip(f"workload {name} not built")
    return W, pkg.DeviceIndex.from_file(path), path


@pytest.mark.parametrize("name,nq,params", [
    ("tiny", 256, [(10, 1, 100, True), (10, 4, 37, True), (5, 32, 10_000, True), (10, 3, 1, False)]),
    ("c1", 400, [(10, 4, 400, True), (100, 8, 800, True), (10, 2, 200, False)]),
])
def test_workload_vs_oracle(pkg, name, nq, params):
    from oracle import rrann_oracle as O

    W, dev, path = _workload(pkg, name)
    oidx = O.read_index(path.read_bytes())
    q = W.load_queries(name, nq)
    for k, w, t, rr in params:
        w = min(w, dev.n_clusters)
        ids, sc, cnt = dev.search_host(q, k, w, t, rr)
        ref = O.query_batch(oidx, q, k, w, t, rr)
        for i, r in enumerate(ref):
            c = int(cnt[i])
            assert c == len(r.ids)
            if not rr:
                np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"{name} q{i} {(k, w, t, rr)}")
            if rr:
                np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"{name} q{i} {(k, w, t, rr)}")
                np.testing.assert_array_equal(sc[i, :c].view(np.int32), r.scores.view(np.int32))
            else:
                xx = float(q[i].astype(np.float64) @ q[i].astype(np.float64))
                assert_topk_equivalent(ids[i, :c], sc[i, :c], r.ids, r.scores, RTOL, xx)


def test_c2_properties_and_sample_parity(pkg):
    """BASELINE configs[1] (1M x 768): oracle parity on a sample + size-independent properties."""
    from oracle import rrann_oracle as O

    W, dev, path = _workload(pkg, "c2")
    man = W.load_manifest("c2")
    q = W.load_queries("c2")
    k, w, t = 100, 8, 800
    ids, sc, cnt = dev.search_device(torch.from_numpy(q).cuda(), k, w, t, True)
    ids, sc, cnt = ids.cpu().numpy(), sc.cpu().numpy(), cnt.cpu().numpy()
    assert (cnt == k).all()
    assert (np.diff(sc, axis=1) >= 0).all()                      # monotone scores
    assert all(len(set(r.tolist())) == k for r in ids[:1000])     # unique ids
    assert ids.min() >= 0 and ids.max() < man["generator"]["m"]
    oidx = O.read_index(path.read_bytes())
    for i in range(0, q.shape[0], 97):
        r = O.query(oidx, q[i], k, w, t, True)
        np.testing.assert_array_equal(ids[i], r.ids)
        np.testing.assert_array_equal(sc[i].view(np.int32), r.scores.view(np.int32))
    gt = W.load_ground_truth("c2")
    if gt is not None:
        rec = np.mean([len(set(ids[i].tolist()) & set(gt[i, :k].tolist())) / k for i in range(len(q))])
        assert rec >= 0.5


@pytest.mark.slow
@pytest.mark.parametrize("name,w,t", [("c2", 1, 800), ("c3", 4, 800), ("c5", 64, 1600), ("c2", 8, 400)])
def test_timed_operating_points_vs_oracle(pkg, name, w, t):
    """The bench's operating points at full size (C2 w=1 t=800, C3 w=4 t=800, C5 OOD w=64
    t=1600): the whole 10k batch is searched as the bench does, and a spread sample of
    128 queries is checked against the oracle -- ids identical, score bits identical,
    hence the sample's recall identical."""
    from oracle import rrann_oracle as O

    W, dev, path = _workload(pkg, name)
    man = W.load_manifest(name)
    k = man["k"]
    q = W.load_queries(name)
    ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(torch.from_numpy(q).cuda(), k, w, t, True))
    oidx = O.read_index(path.read_bytes())
    sample = np.unique(np.linspace(0, len(q) - 1, 128).astype(int))
    gt = W.load_ground_truth(name)
    rec_dev, rec_ref = [], []
    for i in sample:
        r = O.query(oidx, q[i], k, w, t, True)
        assert int(cnt[i]) == len(r.ids), (name, i)
        np.testing.assert_array_equal(ids[i, :cnt[i]], r.ids, err_msg=f"{name} w={w} t={t} q{i}")
        np.testing.assert_array_equal(sc[i, :cnt[i]].view(np.int32), r.scores.view(np.int32))
        if gt is not None:
            rec_dev.append(len(set(ids[i, :cnt[i]].tolist()) & set(gt[i, :k].tolist())) / k)
            rec_ref.append(len(set(r.ids.tolist()) & set(gt[i, :k].tolist())) / k)
    assert rec_dev == rec_ref


# ----------------------------------------------------------- random-index shape sweep

SWEEP = [
    # d, s, r, L, m, metric, exact_ivf
    (1, 1, 1, 3, 40, "euclidean", False),
    (3, 2, 2, 4, 60, "euclidean", False),
    (7, 5, 3, 5, 90, "euclidean", False),
    (9, 8, 4, 6, 120, "euclidean", False),
    (31, 16, 8, 7, 300, "euclidean", False),
    (64, 32, 16, 8, 500, "euclidean", False),
    (100, 20, 8, 9, 400, "euclidean", False),
    (127, 33, 32, 10, 700, "euclidean", False),
    (128, 64, 32, 12, 900, "euclidean", False),
    (129, 64, 32, 12, 900, "euclidean", False),
    (200, 48, 24, 8, 600, "euclidean", False),
    (256, 128, 32, 16, 1500, "euclidean", False),
    (300, 100, 40, 10, 800, "euclidean", False),
    (513, 128, 32, 10, 700, "euclidean", False),
    (768, 256, 32, 16, 2000, "euclidean", False),
    (960, 64, 32, 16, 1500, "euclidean", False),
    (1536, 64, 32, 12, 1200, "euclidean", False),
    (2049, 64, 32, 8, 500, "euclidean", False),
    (128, 64, 64, 12, 900, "euclidean", False),
    (96, 40, 12, 10, 500, "euclidean", True),
    (128, 64, 32, 12, 900, "ip", False),
    (768, 256, 32, 8, 900, "cosine", False),
]


@pytest.mark.parametrize("mode", ["cluster", "cluster+auto", "cluster+async", "cluster+skip", "cluster+blocksel",
                                  "cluster+dmma", "cluster+slicedroute", "query", "cluster+regs",
                                  "cluster+tma", "cluster+screen", "cluster+screenring", "cluster+noscreen",
                                  "cluster+scoretc"])
@pytest.mark.parametrize("d,s,r,L,m,metric,exact_ivf", SWEEP)
def test_random_index_sweep(pkg, tmp_path, d, s, r, L, m, metric, exact_ivf, mode, monkeypatch):
    """Every scoring x re-rank kernel variant against the oracle: cluster-major scoring
    with the default re-rank (cluster-major where the row plan allows), query-major
    scoring (per-query re-rank), and the per-query register / TMA re-rank kernels."""
    score_mode, _, rerank_mode = mode.partition("+")
    monkeypatch.setenv("RRG_SCORE_MODE", score_mode)
    if score_mode == "cluster" and rerank_mode != "auto":  # force the cluster-major re-rank
        monkeypatch.setenv("RRG_RERANK", "cluster")     # (where its row plan applies)
        monkeypatch.setenv("RRG_WARP_SELECT", "1")      # and the warp-per-query selections
    if rerank_mode == "async":  # cluster-major re-rank with cp.async-staged row pairs
        monkeypatch.setenv("RRG_RR_ASYNC", "1")
    elif rerank_mode == "skip":  # cluster-major re-rank passing over unselected row pairs
        monkeypatch.setenv("RRG_RR_SKIP", "1")
    elif rerank_mode == "blocksel":  # CTA-per-query top-t / top-k selections
        monkeypatch.setenv("RRG_WARP_SELECT", "0")
    elif rerank_mode == "dmma":  # FP64 DMMA projection + routing GEMMs, unfused w=1 routing
        monkeypatch.setenv("RRG_GEMM", "dmma")
        monkeypatch.setenv("RRG_ROUTE_FUSED", "0")
    elif rerank_mode == "slicedroute":  # int8 tensor-core (sliced) projection + routing
        monkeypatch.setenv("RRG_GEMM", "sliced")
    elif rerank_mode == "screen":  # tensor-core bounds prune the exact re-rank (any t)
        monkeypatch.setenv("RRG_SCREEN", "1")
    elif rerank_mode == "screenring":  # screened exact pass with ring-staged rows (variant 2)
        monkeypatch.setenv("RRG_SCREEN", "1")
        monkeypatch.setenv("RRG_SPARSE_VARIANT", "2")
    elif rerank_mode == "noscreen":
        monkeypatch.setenv("RRG_SCREEN", "0")
    elif rerank_mode == "scoretc":  # stage B of the scoring on tcgen05 (kind::i8; r_pad = 32 shapes)
        monkeypatch.setenv("RRG_SCORE_TC", "1")
    elif rerank_mode:
        monkeypatch.setenv("RRG_RERANK", rerank_mode)
    from index_writer import random_index
    from oracle import rrann_oracle as O

    blob = random_index(d, s, r, L, m, metric, seed=d * 7 + L, exact_ivf=exact_ivf, dup_rows=3)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "rand", blob))
    oidx = O.read_index(blob)
    rng = np.random.default_rng(d)
    q = rng.standard_normal((40, d)).astype(F32)
    q[1] = oidx.corpus[5]  # query on a corpus point
    for k, w, t, rr in [(5, 1, 10, True), (10, max(1, L // 2), 60, True), (7, L, m + 5, True),
                        (m + 3, L, m + 3, True), (6, 3 if L >= 3 else 1, 1, False)]:
        w = min(w, L)
        ids, sc, cnt = dev.search_host(q, k, w, t, rr)
        ref = O.query_batch(oidx, q, k, w, t, rr)
        for i, rres in enumerate(ref):
            c = int(cnt[i])
            assert c == len(rres.ids), (i, c, len(rres.ids))
            what = f"d={d} {metric} {(k, w, t, rr)} q{i}"
            if metric == "euclidean" and rr:
                np.testing.assert_array_equal(ids[i, :c], rres.ids, err_msg=what)
                np.testing.assert_array_equal(sc[i, :c].view(np.int32), rres.scores.view(np.int32),
                                              err_msg=what)
            elif not rr:
                np.testing.assert_array_equal(ids[i, :c], rres.ids, err_msg=what)
                scale = float(q[i].astype(np.float64) @ q[i].astype(np.float64)) if metric == "euclidean" else None
                assert_topk_equivalent(ids[i, :c], sc[i, :c], rres.ids, rres.scores, RTOL, scale, what)
            else:  # dot products: error scales with |x||c|, not with the (possibly ~0) score
                scale = float(np.linalg.norm(q[i]) * np.linalg.norm(oidx.corpus, axis=1).max())
                assert_topk_equivalent(ids[i, :c], sc[i, :c], rres.ids, rres.scores, RTOL, scale, what)


F32_SWEEP = [
    (31, 16, 8, 7, 300, "euclidean", False),
    (128, 64, 32, 12, 900, "euclidean", False),
    (768, 256, 32, 8, 1200, "euclidean", False),
    (100, 100, 64, 6, 700, "euclidean", False),
    (96, 40, 12, 10, 500, "euclidean", True),
    (128, 64, 32, 12, 900, "ip", False),
    (200, 48, 24, 8, 600, "cosine", True),
]


@pytest.mark.parametrize("d,s,r,L,m,metric,exact_ivf", F32_SWEEP)
def test_random_index_f32_sweep(pkg, tmp_path, d, s, r, L, m, metric, exact_ivf):
    """f32-factor scoring over random shapes (s not a multiple of 4, r = 64, exact-IVF)."""
    from index_writer import random_index
    from oracle import rrann_oracle as O

    blob = random_index(d, s, r, L, m, metric, seed=d * 5 + L, exact_ivf=exact_ivf, dup_rows=3,
                        quantize=False)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "randf", blob))
    oidx = O.read_index(blob)
    rng = np.random.default_rng(d + 1)
    q = rng.standard_normal((32, d)).astype(F32)
    q[1] = oidx.corpus[5]
    cmax = float(np.linalg.norm(oidx.corpus, axis=1).max())
    for k, w, t, rr in [(5, 1, 10, True), (10, max(1, L // 2), 60, True), (7, L, m + 5, True),
                        (6, min(3, L), 1, False), (9, min(4, L), 9, False)]:
        ids, sc, cnt = dev.search_host(q, k, w, t, rr)
        for i in range(len(q)):
            _f32_check_query(O, oidx, q[i], k, w, t, rr, ids[i], sc[i], cnt[i], cmax,
                             f"d={d} {metric} {(k, w, t, rr)} q{i}")


def test_search_host_many_equals_single_calls(pkg, tmp_path):
    """rrg_search_host_many (pipelined H2D / search / D2H) == one rrg_search_host per batch."""
    g, dev = _golden_index(pkg, tmp_path, "euclid_q")
    q = g["queries"]
    batches = [q[:7], q[7:40], q[:0], q[40:], q[::-1].copy(), q[:1]]
    for k, w, t, rr in [(10, 3, 50, True), (5, 2, 5, False)]:
        outs = dev.search_host_many(batches, k, w, t, rr)
        for b, (ids, sc, cnt) in zip(batches, outs):
            if len(b) == 0:
                continue
            ri, rs, rc = dev.search_host(b, k, w, t, rr)
            np.testing.assert_array_equal(cnt, rc)
            np.testing.assert_array_equal(ids, ri)
            np.testing.assert_array_equal(sc.view(np.int32), rs.view(np.int32))
    bad = q[:5].copy()
    bad[2, 3] = np.inf
    with pytest.raises(pkg.DataError):
        dev.search_host_many([q[:5], bad], 10, 3, 50)
    with pytest.raises(pkg.ParameterError, match="k must be >= 1"):
        dev.search_host_many([q[:5]], 0, 3, 50)


@pytest.mark.parametrize("warp_select", ["1", "0"])
@pytest.mark.parametrize("d,L,m", [(32, 5, 600), (768, 3, 700)])
def test_all_scores_and_distances_tied(pkg, tmp_path, warp_select, d, L, m, monkeypatch):
    """Every candidate has the same score and the same corpus row: top-t and top-k are
    decided by corpus id alone (index.py:315,321 lexsort), through the many-ties paths."""
    monkeypatch.setenv("RRG_WARP_SELECT", warp_select)
    from index_writer import random_index
    from oracle import rrann_oracle as O

    blob = random_index(d, 16, 8, L, m, "euclidean", seed=3, all_ties=True)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "ties", blob))
    oidx = O.read_index(blob)
    q = np.random.default_rng(1).standard_normal((9, d)).astype(F32)
    for k, w, t, rr in [(10, L, 100, True), (7, 2, 50, True), (50, L, 300, True), (12, L, 1, False)]:
        ids, sc, cnt = dev.search_host(q, k, w, t, rr)
        ref = O.query_batch(oidx, q, k, w, t, rr)
        for i, r in enumerate(ref):
            c = int(cnt[i])
            np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"{(k, w, t, rr)} q{i}")
            if rr:
                np.testing.assert_array_equal(sc[i, :c].view(np.int32), r.scores.view(np.int32))


@pytest.mark.parametrize("case", QUANT_CASES + F32_CASES)
def test_sliced_projection_matches_golden(pkg, tmp_path, case, monkeypatch):
    """RRG_PROJ=sliced: the projection on the int8 tensor cores (tcgen05 kind::i8, 8 exact
    7-bit slices per operand, int32 levels in TMEM, f64 epilogue) reproduces the reference's
    f32(f64(x) @ f64(W)) bit for bit, and the whole search stays exact."""
    monkeypatch.setenv("RRG_GEMM", "sliced")
    g, dev = _golden_index(pkg, tmp_path, case)
    x = torch.from_numpy(g["queries"][:3]).cuda()
    xp = dev.stage_project(x)[0]
    torch.cuda.synchronize()
    xp = xp.cpu().numpy()
    for i in range(3):
        np.testing.assert_array_equal(xp[i].view(np.int32), g[f"trace{i}_xp"].view(np.int32))
    sel = dev.stage_route(torch.from_numpy(xp).cuda(), min(4, dev.n_clusters)).cpu().numpy()
    for i in range(3):  # routing on the same tensor-core path
        assert set(sel[i].tolist()) == set(g[f"trace{i}_selected"].tolist())
    if "f32" in case:
        return
    for pi, (k, w, t, rr) in enumerate(g["params"]):
        if f"p{pi}_ids" not in g or not rr or dev.metric != "euclidean":
            continue
        k, w, t = int(k), min(int(w), dev.n_clusters), int(t)
        q = torch.from_numpy(g["queries"]).cuda()
        ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(q, k, w, t, True))
        np.testing.assert_array_equal(cnt, g[f"p{pi}_count"])
        for i in range(len(cnt)):
            c = int(cnt[i])
            np.testing.assert_array_equal(ids[i, :c], g[f"p{pi}_ids"][i, :c])


@pytest.mark.parametrize("d,s", [(768, 256), (960, 64), (100, 20), (1536, 64), (33, 33)])
def test_sliced_projection_equals_dmma(pkg, tmp_path, d, s, monkeypatch):
    """Tensor-core sliced projection vs the FP64 DMMA projection on random data with a
    wide dynamic range (zeros, tiny and huge entries): identical f32 outputs."""
    from index_writer import random_index

    blob = random_index(d, s, 8, 6, 300, "euclidean", seed=d + s)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "proj", blob))
    rng = np.random.default_rng(d)
    q = (rng.standard_normal((700, d)) * rng.choice([1e-3, 1.0, 30.0], size=(700, 1))).astype(F32)
    q[0] = 0.0
    q[1, ::3] = 0.0
    q[2, 5] = 1e-30
    xq = torch.from_numpy(q).cuda()
    monkeypatch.setenv("RRG_GEMM", "dmma")
    dev.reload_options()  # variant switches are resolved per index, not per call
    ref = dev.stage_project(xq)[0].cpu().numpy()
    ref_sel = dev.stage_route(torch.from_numpy(ref).cuda(), 3).cpu().numpy()
    monkeypatch.setenv("RRG_GEMM", "sliced")
    dev.reload_options()
    got = dev.stage_project(xq)[0].cpu().numpy()
    np.testing.assert_array_equal(got.view(np.int32), ref.view(np.int32))
    sel = dev.stage_route(torch.from_numpy(got).cuda(), 3).cpu().numpy()
    for a, b in zip(sel, ref_sel):
        assert set(a.tolist()) == set(b.tolist())


@pytest.mark.parametrize("case", ["euclid_q", "euclid_d100", "ip_q", "euclid_exact_ivf", "euclid_f32"])
def test_small_batches_match_golden(pkg, tmp_path, case):
    """Batches of 1..32 queries take the small-batch kernels (warp-per-output GEMVs,
    short re-rank work items, CTA-per-query selections) -- same results."""
    g, dev = _golden_index(pkg, tmp_path, case)
    cmax = _corpus_max_norm(g)
    for pi, (k, w, t, rr) in enumerate(g["params"]):
        if f"p{pi}_ids" not in g:
            continue
        k, w, t, rr = int(k), min(int(w), dev.n_clusters), int(t), bool(rr)
        for b0, b1 in [(0, 1), (5, 12), (20, 52)]:
            qb = g["queries"][b0:b1]
            ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(torch.from_numpy(qb).cuda(), k, w, t, rr))
            hids, hsc, hcnt = dev.search_host(qb, k, w, t, rr)
            np.testing.assert_array_equal(hids, ids)
            np.testing.assert_array_equal(hcnt, cnt)
            for i in range(b1 - b0):
                c = int(cnt[i])
                ref_ids, ref_sc = g[f"p{pi}_ids"][b0 + i, :c], g[f"p{pi}_scores"][b0 + i, :c]
                assert c == g[f"p{pi}_count"][b0 + i]
                if "f32" in case:
                    continue  # tolerance-level scores: covered by test_golden_f32_factors
                if dev.metric == "euclidean" and rr:
                    np.testing.assert_array_equal(ids[i, :c], ref_ids)
                    np.testing.assert_array_equal(sc[i, :c].view(np.int32), ref_sc.view(np.int32))
                else:
                    x = qb[i].astype(np.float64)
                    scale = float(x @ x) if dev.metric == "euclidean" else float(np.sqrt(x @ x) * cmax)
                    assert_topk_equivalent(ids[i, :c], sc[i, :c], ref_ids, ref_sc, RTOL, scale,
                                           f"{case} p{pi} q{b0 + i}")


def test_fused_nearest_cluster_ties(pkg, tmp_path):
    """w = 1 routing fused into the GEMM: duplicate centroids tie exactly and resolve to
    the lower cluster id, like route()'s stable argsort (cluster.py:263-264)."""
    import struct
    import zlib

    from index_writer import random_index
    from oracle import rrann_oracle as O

    d, s, L = 64, 32, 9
    blob = bytearray(random_index(d, s, 8, L, 700, "euclidean", seed=5))
    # duplicate centroid 2 into centroids 6 and 7 (header 8 + 29 bytes, then W d x s f32)
    off = 8 + 29 + d * s * 4
    cent = np.frombuffer(bytes(blob[off:off + L * s * 4]), dtype="<f4").reshape(L, s).copy()
    cent[6] = cent[2]
    cent[7] = cent[2]
    blob[off:off + L * s * 4] = cent.tobytes()
    blob[-4:] = struct.pack("<I", zlib.crc32(bytes(blob[:-4])) & 0xFFFFFFFF)
    blob = bytes(blob)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "ties", blob))
    oidx = O.read_index(blob)
    rng = np.random.default_rng(3)
    W = oidx.projection.astype(np.float64)
    # queries whose projection is (near) centroid 2: the three duplicates tie
    q = rng.standard_normal((200, d)).astype(F32)
    q[:100] = (np.linalg.pinv(W.T) @ cent[2].astype(np.float64)).astype(F32)[None, :] +         rng.standard_normal((100, d)).astype(F32) * 1e-3
    ids, sc, cnt = dev.search_host(q, 5, 1, 30, True)
    ref = O.query_batch(oidx, q, 5, 1, 30, True)
    for i, r in enumerate(ref):
        c = int(cnt[i])
        np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"q{i}")


@pytest.mark.parametrize("select", ["warp", "auto"])
@pytest.mark.parametrize("rerank_mode", ["query", "cluster"])
def test_long_candidate_lists(pkg, tmp_path, rerank_mode, select, monkeypatch):
    """~30k candidates per query (w = L on 4 large clusters): the warp top-t streams
    long lists (per-query re-rank) and yields to the CTA select where its membership
    bits would not fit (cluster-major re-rank, lists above the 24k key cap); "auto"
    takes the CTA select's long-list path (sampled bucket range, clamped keys, 8 keys
    in flight) -- with duplicated rows, so the boundary holds exact ties."""
    if select == "warp":
        monkeypatch.setenv("RRG_WARP_SELECT", "1")
    else:
        monkeypatch.delenv("RRG_WARP_SELECT", raising=False)
    monkeypatch.setenv("RRG_RERANK", rerank_mode)
    from index_writer import random_index
    from oracle import rrann_oracle as O

    blob = random_index(16, 8, 4, 4, 30000, "euclidean", seed=11, dup_rows=5)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "long", blob))
    oidx = O.read_index(blob)
    q = np.random.default_rng(2).standard_normal((24, 16)).astype(F32)
    for k, w, t in [(10, 4, 300), (20, 3, 2000)]:
        ids, sc, cnt = dev.search_host(q, k, w, t, True)
        ref = O.query_batch(oidx, q, k, w, t, True)
        for i, r in enumerate(ref):
            c = int(cnt[i])
            np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"{(k, w, t)} q{i}")
            np.testing.assert_array_equal(sc[i, :c].view(np.int32), r.scores.view(np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("L", [8192, 16384])
def test_many_clusters(pkg, tmp_path, L):
    """C4-scale cluster counts: the per-batch cluster tables (pair offsets, query buckets,
    routing selection) outgrow the default 48 KB of shared memory; batches large enough
    for the cluster-major path, oracle-checked id-for-id."""
    from index_writer import random_index
    from oracle import rrann_oracle as O

    d, s, r = 96, 32, 8
    m = 4 * L
    blob = random_index(d, s, r, L, m, seed=L, dup_rows=2)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "many", blob))
    oidx = O.read_index(blob)
    q = np.random.default_rng(L).standard_normal((3000, d)).astype(F32)
    for k, w, t in [(10, 1, 20), (10, 3, 40), (5, 64, 200)]:
        ids, sc, cnt = dev.search_host(q, k, w, t, True)
        for i in range(0, q.shape[0], 97):
            rres = O.query(oidx, q[i], k, w, t, True)
            c = int(cnt[i])
            assert c == len(rres.ids)
            np.testing.assert_array_equal(ids[i, :c], rres.ids)
            np.testing.assert_array_equal(sc[i, :c].view(np.int32), rres.scores.view(np.int32))


@pytest.mark.gpu
def test_too_many_clusters_rejected(pkg, tmp_path):
    """More clusters than the one-CTA cluster tables hold: a ParameterError at load."""
    from index_writer import random_index

    blob = random_index(16, 8, 4, 20000, 20000, seed=1)
    with pytest.raises(pkg.ParameterError, match="clusters"):
        pkg.DeviceIndex.from_file(_write(tmp_path, "toomany", blob))


# ------------------------------------------------------------- re-rank screen

@pytest.mark.parametrize("d,L,m,metric_scale", [(768, 6, 3000, 1.0), (960, 5, 2500, 30.0),
                                                (1536, 4, 1800, 1e-3), (768, 3, 900, 1.0)])
def test_screen_exact_vs_oracle(pkg, tmp_path, d, L, m, metric_scale, monkeypatch):
    """The tensor-core screen only removes candidates that provably cannot reach the top k:
    screened and unscreened searches return the reference's ids and score bits, across
    scales (tiny and huge corpora), duplicate rows, queries on corpus points, and t from
    k (nothing to prune) to the whole cluster set."""
    from index_writer import random_index
    from oracle import rrann_oracle as O

    monkeypatch.setenv("RRG_RERANK", "cluster")
    monkeypatch.setenv("RRG_SCREEN", "1")
    blob = random_index(d, 64, 16, L, m, "euclidean", seed=d + L, dup_rows=20, corpus_scale=metric_scale)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "scr", blob))
    oidx = O.read_index(blob)
    rng = np.random.default_rng(d)
    q = (rng.standard_normal((300, d)) * metric_scale).astype(F32)
    q[0] = oidx.corpus[7]
    q[1] = oidx.corpus[7] + np.float32(metric_scale * 1e-6)
    q[2] = 0.0
    for k, w, t in [(10, 1, 200), (50, 2, 400), (10, 1, 10), (100, L, m), (5, 1, 700)]:
        ids, sc, cnt = (a.cpu().numpy() for a in dev.search_device(torch.from_numpy(q).cuda(), k, w, t, True))
        ref = O.query_batch(oidx, q, k, w, t, True)
        for i, r in enumerate(ref):
            c = int(cnt[i])
            assert c == len(r.ids), (k, w, t, i)
            np.testing.assert_array_equal(ids[i, :c], r.ids, err_msg=f"{(k, w, t)} q{i}")
            np.testing.assert_array_equal(sc[i, :c].view(np.int32), r.scores.view(np.int32))


def test_screen_counters_and_pruning(pkg, tmp_path, monkeypatch):
    """The screen re-ranks far fewer than t candidates per query on clustered data, and the
    library's work counters account for it."""
    import ctypes

    from index_writer import random_index
    from paper_2410_18926_b200 import _native

    monkeypatch.setenv("RRG_RERANK", "cluster")
    monkeypatch.setenv("RRG_SCREEN", "1")
    blob = random_index(768, 64, 16, 8, 6000, "euclidean", seed=4)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "cnt", blob))
    q = torch.from_numpy(np.random.default_rng(0).standard_normal((2000, 768)).astype(F32)).cuda()
    _native.lib.rrg_set_stage_timing(1)
    c = (ctypes.c_int64 * 8)()
    _native.lib.rrg_search_counters(c)
    dev.search_device(q, 10, 1, 400, True)
    torch.cuda.synchronize()
    _native.lib.rrg_search_counters(c)
    _native.lib.rrg_set_stage_timing(0)
    cand, surv, streamed, fetched, distinct = c[0], c[1], c[2], c[3], c[4]
    assert 2000 * 10 <= cand <= 2000 * 400       # sum of min(t, candidates) per query
    assert 2000 * 10 <= surv < cand / 4, (surv, cand)
    assert streamed >= 6000 and distinct <= 6000 and fetched >= distinct


def test_path_times_and_timing_invariance(pkg, tmp_path, monkeypatch):
    """rrg_path_times: the re-rank span lies inside the search span, one of each per
    search; results are the same with the timers (and the side-stream row count) on."""
    import ctypes

    from index_writer import random_index
    from paper_2410_18926_b200 import _native

    monkeypatch.setenv("RRG_SCREEN", "1")
    monkeypatch.setenv("RRG_RERANK", "cluster")
    blob = random_index(768, 64, 16, 8, 4000, "euclidean", seed=6)  # (d = 768: the cluster-major plan)
    dev = pkg.DeviceIndex.from_file(_write(tmp_path, "pt", blob))
    q = torch.from_numpy(np.random.default_rng(1).standard_normal((1500, 768)).astype(F32)).cuda()
    ref = [a.cpu() for a in dev.search_device(q, 10, 1, 300, True)]
    ms, n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    c = (ctypes.c_int64 * 8)()
    _native.lib.rrg_set_stage_timing(1)
    _native.lib.rrg_path_times(ms, n)
    _native.lib.rrg_search_counters(c)
    got = []
    for _ in range(3):
        got = [a.cpu() for a in dev.search_device(q, 10, 1, 300, True)]
    _native.lib.rrg_path_times(ms, n)
    _native.lib.rrg_search_counters(c)
    _native.lib.rrg_set_stage_timing(0)
    assert n[0] == 3 and n[1] == 3, (n[0], n[1])
    assert 0.0 < ms[0] <= ms[1], (ms[0], ms[1])
    assert c[4] > 0  # the row-union count ran (side stream)
    for a, b in zip(got, ref):
        assert torch.equal(torch.nan_to_num(a), torch.nan_to_num(b))


# ------------------------------------------------------------- routing screen

def _set_centroids(blob, d, s, L, fn):
    """Rewrite the centroid block of an RRRANN01 blob (index.py:365-402) and its CRC."""
    import struct
    import zlib

    off = 8 + 29 + 4 * d * s
    cent = np.frombuffer(blob, dtype="<f4", count=L * s, offset=off).reshape(L, s).copy()
    cent = fn(cent).astype("<f4")
    body = blob[:off] + cent.tobytes() + blob[off + 4 * L * s:-4]
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


@pytest.mark.parametrize("d,s,L,ties", [(96, 64, 1024, "none"), (768, 256, 640, "none"),
                                        (64, 32, 1024, "dup"), (64, 32, 512, "all")])
def test_route_screen_matches_f64_routing(pkg, tmp_path, d, s, L, ties, monkeypatch):
    """Routing on the fp16 tensor cores with f64 recheck of the survivors selects the same
    clusters as the f64 GEMM path and the oracle (ties -> lower id), including duplicated
    centroids and a degenerate index where every centroid is equal (list overflow ->
    full f64 scan)."""
    from index_writer import random_index
    from oracle import rrann_oracle as O

    blob = random_index(d, s, 8, L, 30 * L, "euclidean", seed=L + s)
    if ties == "dup":
        blob = _set_centroids(blob, d, s, L, lambda c: np.concatenate([c[: L // 2], c[: L // 2]]))
    elif ties == "all":
        blob = _set_centroids(blob, d, s, L, lambda c: np.repeat(c[:1], L, axis=0))
    path = _write(tmp_path, "rt", blob)
    dev = pkg.DeviceIndex.from_file(path)
    q = np.random.default_rng(s).standard_normal((700, d)).astype(F32)
    oidx = O.read_index(blob)
    for w in (1, 3, 8):
        monkeypatch.setenv("RRG_ROUTE_SCREEN", "2")  # (the default takes it at w = 1 only)
        dev.reload_options()
        got = dev.search_host(q, 10, w, 60, True)
        monkeypatch.setenv("RRG_ROUTE_SCREEN", "0")
        dev.reload_options()
        ref = dev.search_host(q, 10, w, 60, True)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b, err_msg=f"w={w} {ties}")
        for i in range(0, 700, 35):
            r = O.query(oidx, q[i], 10, w, 60, True)
            np.testing.assert_array_equal(got[0][i, :got[2][i]], r.ids, err_msg=f"w={w} q{i} {ties}")


@pytest.mark.parametrize("name,w,t", [("c2", 8, 400), ("c5", 64, 1600)])
def test_tensor_core_stage_b_bit_exact(pkg, name, w, t, monkeypatch):
    """Stage B of the cluster scoring on tcgen05 (RRG_SCORE_TC=1): the int32 products,
    scores and final results equal the dp4a kernel's bit for bit at full size."""
    W, dev, path = _workload(pkg, name)
    q = torch.from_numpy(W.load_queries(name)).cuda()
    k = W.load_manifest(name)["k"]
    monkeypatch.setenv("RRG_SCORE_TC", "0")
    dev.reload_options()
    ref = [a.cpu().numpy() for a in dev.search_device(q, k, w, t, True)]
    sel = dev.stage_route(dev.stage_project(q[:512])[0], w)
    r1 = [a.cpu().numpy() for a in dev.stage_score(q[:512], sel)]
    monkeypatch.setenv("RRG_SCORE_TC", "1")
    dev.reload_options()
    got = [a.cpu().numpy() for a in dev.search_device(q, k, w, t, True)]
    g1 = [a.cpu().numpy() for a in dev.stage_score(q[:512], sel)]
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(np.nan_to_num(a), np.nan_to_num(b))
    for a, b in zip(g1[1:], r1[1:]):  # raw2, scores, offsets
        np.testing.assert_array_equal(a.view(np.int32), b.view(np.int32))
