"""Cluster-sharded two-phase search: partitioning, orchestration (gloo, 2 ranks) and GPU shards."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import load_golden
from index_writer import random_index
from oracle import rrann_oracle as O
from paper_2410_18926_b200.sharded import (partition_clusters, scan_cluster_sizes,
                                           sharded_search_local)


def test_partition_clusters_balanced():
    sizes = np.array([5, 1, 1, 1, 10, 2, 2, 8])
    parts = partition_clusters(sizes, 3)
    assert parts[0][0] == 0 and parts[-1][1] == len(sizes)
    assert all(a < b for a, b in parts)
    assert all(parts[i][1] == parts[i + 1][0] for i in range(len(parts) - 1))
    loads = [sizes[a:b].sum() for a, b in parts]
    assert max(loads) <= 12
    assert partition_clusters(sizes, 8) == [(i, i + 1) for i in range(8)]


def test_scan_cluster_sizes(tmp_path):
    for case in ["euclid_q", "ip_q", "euclid_exact_ivf", "euclid_norerank"]:
        blob = load_golden(case)["index_bytes"].tobytes()
        p = tmp_path / f"{case}.rrr"
        p.write_bytes(blob)
        idx = O.read_index(blob)
        np.testing.assert_array_equal(scan_cluster_sizes(p), [c.ids.size for c in idx.clusters])


def _engines(blob, G):
    from oracle_shard_engine import OracleShardEngine

    idx = O.read_index(blob)
    parts = partition_clusters([c.ids.size for c in idx.clusters], G)
    return idx, [OracleShardEngine(idx, a, b) for a, b in parts]


@pytest.mark.parametrize("G", [1, 2, 3])
def test_local_shards_equal_unsharded(G):
    blob = random_index(40, 16, 8, 9, 700, seed=3, dup_rows=4)
    idx, engines = _engines(blob, G)
    q = np.random.default_rng(1).standard_normal((24, 40)).astype(np.float32)
    for k, w, t in [(5, 2, 20), (10, 9, 800), (7, 4, 7)]:
        ids, sc, cnt = sharded_search_local(engines, torch.from_numpy(q), k, w, t)
        ref = O.query_batch(idx, q, k, w, t, True)
        for i, r in enumerate(ref):
            c = int(cnt[i])
            assert c == len(r.ids)
            np.testing.assert_array_equal(ids[i, :c].numpy(), r.ids)
            np.testing.assert_array_equal(sc[i, :c].numpy().view(np.int32), r.scores.view(np.int32))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, blob, q, params, out_dir):
    import torch.distributed as dist

    from paper_2410_18926_b200.sharded import TorchExchange, sharded_search

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx, engines = _engines(blob, world)
        ex = TorchExchange()
        for j, (k, w, t) in enumerate(params):
            # alternate the packed (sparse) and padded phase-1 exchanges
            ids, sc, cnt = sharded_search(engines[rank], ex, torch.from_numpy(q), k, w, t,
                                          sparse=j % 2 == 0)
            np.savez(os.path.join(out_dir, f"r{rank}_p{j}.npz"), ids=ids.numpy(), sc=sc.numpy(),
                     cnt=cnt.numpy())
    finally:
        dist.destroy_process_group()


def _gloo_worker_dp(rank, world, port, blob, q, params, out_dir):
    """Data-parallel front stages + the w = 1 owner-local path / two-phase exchange."""
    import torch.distributed as dist

    from paper_2410_18926_b200.sharded import TorchExchange, sharded_search

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx, engines = _engines(blob, world)
        ex = TorchExchange()
        for j, (k, w, t) in enumerate(params):
            ids, sc, cnt = sharded_search(engines[rank], ex, torch.from_numpy(q), k, w, t,
                                          data_parallel_front=True)
            np.savez(os.path.join(out_dir, f"r{rank}_p{j}.npz"), ids=ids.numpy(), sc=sc.numpy(),
                     cnt=cnt.numpy())
            # each rank keeps its own slice's rows (one all-to-all instead of the all-gather)
            ids, sc, cnt = sharded_search(engines[rank], ex, torch.from_numpy(q), k, w, t,
                                          data_parallel_front=True, results="slice")
            np.savez(os.path.join(out_dir, f"r{rank}_p{j}_slice.npz"), ids=ids.numpy(), sc=sc.numpy(),
                     cnt=cnt.numpy())
    finally:
        dist.destroy_process_group()


def test_three_rank_gloo_data_parallel_front(tmp_path):
    """world_size 3: each rank projects/routes a third of the batch (17 queries: ragged
    slices), the rows are all-gathered; w = 1 needs no candidate exchange, w > 1 runs the
    two exchanges; every rank returns the unsharded result."""
    import sys

    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.dirname(__file__))
    blob = random_index(24, 12, 6, 10, 600, seed=9, dup_rows=3)
    q = np.random.default_rng(4).standard_normal((17, 24)).astype(np.float32)
    params = [(5, 1, 40), (10, 1, 600), (6, 3, 30)]
    world = 3
    mp.spawn(_gloo_worker_dp, args=(world, _free_port(), blob, q, params, str(tmp_path)), nprocs=world,
             join=True)
    idx = O.read_index(blob)
    S = -(-q.shape[0] // world)
    for j, (k, w, t) in enumerate(params):
        ref = O.query_batch(idx, q, k, w, t, True)
        for r in range(world):
            got = np.load(tmp_path / f"r{r}_p{j}.npz")
            sl = np.load(tmp_path / f"r{r}_p{j}_slice.npz")
            assert sl["cnt"].shape[0] == min(q.shape[0], (r + 1) * S) - r * S
            for i, rr in enumerate(ref):
                c = int(got["cnt"][i])
                assert c == len(rr.ids), (r, j, i)
                np.testing.assert_array_equal(got["ids"][i, :c], rr.ids)
                np.testing.assert_array_equal(got["sc"][i, :c].view(np.int32), rr.scores.view(np.int32))
                if r * S <= i < (r + 1) * S:
                    ii = i - r * S
                    assert int(sl["cnt"][ii]) == c
                    np.testing.assert_array_equal(sl["ids"][ii, :c], rr.ids)
                    np.testing.assert_array_equal(sl["sc"][ii, :c].view(np.int32), rr.scores.view(np.int32))


def test_two_rank_gloo_matches_unsharded(tmp_path):
    import sys

    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.dirname(__file__))
    blob = random_index(24, 12, 6, 10, 600, seed=5, dup_rows=3)
    q = np.random.default_rng(2).standard_normal((16, 24)).astype(np.float32)
    params = [(5, 3, 30), (10, 10, 600)]
    world = 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), blob, q, params, str(tmp_path)), nprocs=world,
             join=True)
    idx = O.read_index(blob)
    for j, (k, w, t) in enumerate(params):
        ref = O.query_batch(idx, q, k, w, t, True)
        outs = [np.load(tmp_path / f"r{r}_p{j}.npz") for r in range(world)]
        for o in outs[1:]:  # every rank holds the identical final result
            np.testing.assert_array_equal(o["ids"], outs[0]["ids"])
        for i, r in enumerate(ref):
            c = int(outs[0]["cnt"][i])
            assert c == len(r.ids)
            np.testing.assert_array_equal(outs[0]["ids"][i, :c], r.ids)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3])
def test_gpu_shards_equal_unsharded(tmp_path, G):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_18926_b200 import DeviceIndex
    from paper_2410_18926_b200.sharded import CudaShardEngine

    blob = random_index(128, 64, 32, 12, 3000, seed=G, dup_rows=5)
    p = tmp_path / "s.rrr"
    p.write_bytes(blob)
    full = DeviceIndex.from_file(p)
    parts = partition_clusters(scan_cluster_sizes(p), G)
    engines = [CudaShardEngine(DeviceIndex.from_file(p, shard=ab)) for ab in parts]
    q = torch.from_numpy(np.random.default_rng(G).standard_normal((64, 128)).astype(np.float32)).cuda()
    for k, w, t in [(10, 3, 100), (5, 12, 3000), (20, 6, 20)]:
        ids, sc, cnt = (x.cpu().numpy() for x in sharded_search_local(engines, q, k, w, t))
        rid, rsc, rcnt = (x.cpu().numpy() for x in full.search_device(q, k, w, t, True))
        np.testing.assert_array_equal(cnt, rcnt)
        np.testing.assert_array_equal(ids, rid)
        np.testing.assert_array_equal(np.nan_to_num(sc).view(np.int32), np.nan_to_num(rsc).view(np.int32))


def oindex_arrays(o):
    """An oracle-parsed index as the plain arrays of RrgIndexDesc (include/rrg.h): per-cluster
    payloads concatenated in cluster order, quantized factors with their zero pad row."""
    def full(q):
        return np.concatenate([np.zeros((1, q.cols), np.int8), q.values]).ravel()

    cl = o.clusters
    bm = [c for c in cl if c.b is not None]
    return dict(metric=o.metric, rank=o.r, projection=o.projection, centroids=o.centroids,
                cluster_sizes=np.array([c.ids.shape[0] for c in cl], np.uint32),
                point_ids=np.concatenate([c.ids for c in cl]),
                a_head=np.concatenate([c.a.head_row for c in cl]),
                a_scale=np.concatenate([c.a.col_scales for c in cl]),
                a_values=np.concatenate([full(c.a) for c in cl]),
                b_head=np.concatenate([c.b.head_row for c in bm]),
                b_scale=np.concatenate([c.b.col_scales for c in bm]),
                b_values=np.concatenate([full(c.b) for c in bm]),
                norms=np.concatenate([c.norms for c in cl]), corpus=o.corpus)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 3])
def test_gpu_array_shards_equal_unsharded(G):
    """rrg_index_create_shard (shards of an in-memory index, used by tools/c4.py) gives the
    unsharded result id-for-id, like the file shards above."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_18926_b200 import DeviceIndex
    from paper_2410_18926_b200.sharded import CudaShardEngine

    blob = random_index(128, 64, 32, 12, 3000, seed=10 + G, dup_rows=5)
    arrs = oindex_arrays(O.read_index(blob))
    full = DeviceIndex.from_arrays(**arrs)
    parts = partition_clusters(arrs["cluster_sizes"].astype(np.int64), G)
    engines = [CudaShardEngine(DeviceIndex.from_arrays(shard=ab, **arrs)) for ab in parts]
    q = torch.from_numpy(np.random.default_rng(G).standard_normal((64, 128)).astype(np.float32)).cuda()
    for (k, w, t), sparse in [((10, 3, 100), True), ((5, 12, 3000), False), ((10, 1, 200), True)]:
        ids, sc, cnt = (x.cpu().numpy() for x in sharded_search_local(engines, q, k, w, t, sparse))
        rid, rsc, rcnt = (x.cpu().numpy() for x in full.search_device(q, k, w, t, True))
        np.testing.assert_array_equal(cnt, rcnt)
        np.testing.assert_array_equal(ids, rid)
        np.testing.assert_array_equal(np.nan_to_num(sc).view(np.int32), np.nan_to_num(rsc).view(np.int32))
