"""Benchmark: batched LoRANN search QPS on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A *step* is one batched search of the workload's full query batch (C2: 10k
queries, 1M x 768 corpus, L=1024, s=256, r=32, k=100) through the device entry
``rrg_search`` with queries already resident in HBM (``value``), and through the
host-buffer C-ABI entry ``rrg_search_host`` with pinned host queries and results
copied inside the timed region (``e2e``).

Multi-GPU (torchrun, N>1), default ``--mode replica``: the C2 index (3.1 GB) fits
one GPU, so each rank searches its own 10k-query batch on a full index copy with no
collective on the data path ("weak"; value = all ranks' queries / max-over-ranks
time).  ``--mode sharded`` (the north star's layout for indexes larger than one
GPU): clusters with their factors and corpus rows are split over the ranks, the
query batch is replicated, and the two exact merges (global top-t, then top-k) are
NCCL all-gathers over NVLink ("strong").

``--impl reference`` times the reference's CPU algorithm (the oracle port of
rrann.query_batch, oracle/rrann_oracle.py) on the host cores, on a bounded
query sample, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "QPS at recall@100 >=0.90 (batched), 1/2/4/8 B200, vs CPU ref QPS"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("RRG_WORKLOAD", "c2"))
    ap.add_argument("--w", type=int, default=None)
    ap.add_argument("--t", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--parity-queries", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default=os.environ.get("RRG_BENCH_MODE"),
                    choices=["sharded", "replica"],
                    help="N>1: full-index replicas, each rank its own query batch (default for "
                         "C1-C3, C5: the index fits one GPU, no collective on the data path) or "
                         "the cluster-sharded index (default for C4): data-parallel front stages, "
                         "owner-local search at w=1, NCCL all-gathers (DESIGN.md §5)")
    return ap.parse_args()


def operating_point(man: dict, args):
    """(w, t) for the metric "QPS at recall@k >= 0.90": the cheapest point of the
    reference's own (w, t) grid (tools/build_index.py: recall measured by rrann on the
    workload's queries) that reaches recall@k >= 0.90 -- the smallest t, then the
    smallest w.  Both arms (--impl ours|reference) run this same point, so the
    driver's ratio compares equal work; the device run re-measures its recall on the
    whole batch (config.recall_at_k) and checks its ids against the reference
    (``parity``).  C2 -> (w=1, t=800), also the reference's best-QPS grid point."""
    if args.w and args.t:
        return args.w, args.t
    pts = [p for p in man.get("grid", {}).get("points", []) if p["recall"] >= 0.90]
    if not pts:
        return 8, 800
    best = min(pts, key=lambda p: (p["t"], p["w"]))
    return args.w or best["w"], args.t or best["t"]


# ------------------------------------------------------- reference CPU path (rrann)

_CPU = {}


def load_reference():
    """The unmodified reference package: ``baseline/_ref`` (pip-installed from
    /root/reference, travels to the GPU box) or the source tree in the dev container.
    None when neither exists (the oracle port stands in, kind "port")."""
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "rrann" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import rrann
            return rrann
    return None


class CpuReference:
    """rrann.query_batch on the host cores, loaded once (``RrrIndex.load``) from the same
    index file the device searches; timed with ``_timed_run`` semantics (wall time of
    query_batch over a query set, best of the repeats; rrann/bench.py:205-216) on one
    core and on every core (a fork pool made once after the load, 1 BLAS thread per
    worker, contiguous query chunks).  Without the reference package the oracle port
    (oracle/rrann_oracle.py, the same NumPy calls) is timed instead."""

    @classmethod
    def from_oracle(cls, oidx, k, w, t):
        """The oracle port over an index held in memory (C4: built on the GPU, no file)."""
        from oracle import rrann_oracle as O

        self = cls.__new__(cls)
        self.kind = "port"
        self.run = lambda q: O.query_batch(oidx, q, k, w, t, True)
        self.cores = os.cpu_count() or 1
        self.pool = None
        return self

    def __init__(self, path, k, w, t):
        rr = load_reference()
        if rr is not None:
            self.kind = "reference"
            index = rr.RrrIndex.load(str(path))
            params = rr.QueryParams(k=k, w=w, t=t, rerank=True)
            self.run = lambda q: index.query_batch(q, params)
        else:
            from oracle import rrann_oracle as O

            self.kind = "port"
            index = O.read_index(Path(path).read_bytes())
            self.run = lambda q: O.query_batch(index, q, k, w, t, True)
        self.cores = os.cpu_count() or 1
        self.pool = None

    def __enter__(self):
        import multiprocessing as mp

        _CPU["run"] = self.run
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_init)
        return self

    def __exit__(self, *exc):
        if self.pool is not None:
            self.pool.terminate()
            self.pool.join()

    def one_core(self, q, seconds: float, repeats: int = 3):
        """(QPS, sample size): best of `repeats` query_batch calls on one core."""
        from threadpoolctl import threadpool_limits

        with threadpool_limits(1):
            t0 = time.perf_counter()
            self.run(q[:8])
            per_q = max((time.perf_counter() - t0) / 8, 1e-5)
            n = int(min(len(q), max(16, seconds / repeats / per_q)))
            best = float("inf")
            for _ in range(repeats):
                t0 = time.perf_counter()
                self.run(q[:n])
                best = min(best, time.perf_counter() - t0)
        return n / best, n

    def all_cores(self, q):
        """Wall time of one query_batch over q split across the pool's workers."""
        bounds = np.linspace(0, len(q), self.cores + 1).astype(int)
        chunks = [q[a:b] for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        t0 = time.perf_counter()
        self.pool.map(_cpu_time_chunk, chunks)
        return time.perf_counter() - t0

    def results(self, q):
        """(ids [n, k] -1 padded, scores [n, k] NaN padded, count [n]) of the reference."""
        bounds = np.linspace(0, len(q), self.cores + 1).astype(int)
        parts = self.pool.map(_cpu_results_chunk, [q[a:b] for a, b in zip(bounds[:-1], bounds[1:]) if b > a])
        res = [r for p in parts for r in p]
        k = max([len(r[0]) for r in res] + [1])
        ids = np.full((len(res), k), -1, np.int64)
        sc = np.full((len(res), k), np.nan, np.float32)
        cnt = np.zeros(len(res), np.int32)
        for i, (a, b) in enumerate(res):
            ids[i, :len(a)], sc[i, :len(b)], cnt[i] = a, b, len(a)
        return ids, sc, cnt


def _cpu_init():
    from threadpoolctl import threadpool_limits

    _CPU["limit"] = threadpool_limits(1)


def _cpu_time_chunk(q):
    _CPU["run"](q)
    return 0


def _cpu_results_chunk(q):
    return [(r.ids, r.scores) for r in _CPU["run"](q)]


def cpu_reference_qps(cpu: CpuReference, q, seconds: float, repeats: int = 3):
    """All-core QPS of the reference (best of `repeats` over a bounded query sample)."""
    t0 = time.perf_counter()
    cpu.all_cores(q[:cpu.cores * 4])
    per_q = max((time.perf_counter() - t0) / (cpu.cores * 4), 1e-6)  # wall time per query, all cores
    n = int(min(len(q), max(cpu.cores * 8, seconds / repeats / per_q)))
    best = min(cpu.all_cores(q[:n]) for _ in range(repeats))
    return n / best, n


# ------------------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let nvidia-smi attach before the timed region starts
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------- main


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def run_reference(args):
    """--impl reference: the reference's own CPU query path (rrann.query_batch on the
    workload's index file, all host cores), same workload, metric and (w, t) as the
    device arm.  Each step is one query_batch over a bounded sample of the workload's
    queries split across a persistent fork pool; value = the best step (_timed_run)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.workload == "c4":
        print(json.dumps({"impl": "reference", "metric": METRIC, "unavailable":
                          "C4 (10M x 960) cannot be built by the reference's NumPy build() (k-means++ "
                          "is 8192 sequential passes over 10M rows), so no reference index exists; "
                          "the device run's cpu_baseline times the oracle port on the GPU-built arrays"}),
              flush=True)
        return
    import workloads as W

    man = W.load_manifest(args.workload)
    w, t = operating_point(man, args)
    k = man["k"]
    path = W.materialize_index(args.workload)
    q = W.load_queries(args.workload)
    cpu = CpuReference(path, k, w, t)
    with cpu:
        one_qps, n1 = cpu.one_core(q, min(10.0, args.cpu_seconds))
        t0 = time.perf_counter()
        cpu.all_cores(q[:cpu.cores * 4])
        per_q = max((time.perf_counter() - t0) / (cpu.cores * 4), 1e-6)
        n = int(min(len(q), max(cpu.cores * 8, 1.5 / per_q)))  # ~1.5 s per step
        for _ in range(args.warmup):
            cpu.all_cores(q[:n])
        steps = [cpu.all_cores(q[:n]) for _ in range(max(1, args.steps))]
    best = min(steps)
    v = n / best
    # the reference arm runs none of this repo's kernels: librrg.so is never loaded
    assert "paper_2410_18926_b200" not in sys.modules
    with open("/proc/self/maps") as f:
        assert "librrg" not in f.read()
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": best * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32/f64/int8", "data": "synthetic (rrann.bench.synth_dataset clustered)",
            "config": {"workload": args.workload, "queries": n, "k": k, "w": w, "t": t,
                       **{kk: man["generator"][kk] for kk in ("m", "d", "n_blobs")}, **man["index"]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu.cores, "kind": cpu.kind,
                             "one_core": {"value": one_qps, "sample": n1},
                             "median_step_value": n / float(np.median(steps)),
                             "sample": f"{n} of the workload's queries per step (~1.5 s), "
                                       f"{'rrann.RrrIndex.query_batch (unmodified reference)' if cpu.kind == 'reference' else 'oracle port'}"
                                       f", {cpu.cores}-process fork pool made once after RrrIndex.load, "
                                       "1 BLAS thread each; value = best step (bench._timed_run)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class C4Workload:
    """BASELINE.json configs[3]: 10M x 960 (GIST shape), L=8192, s=64, r=32, k=100.

    The reference's build cannot run at this size (k-means++ is 8192 sequential passes
    over 10M rows in NumPy), so the index is built on the GPU by tools/c4.py's restatement
    of build() -- rank 0 builds, the arrays are broadcast (NCCL), every rank regenerates
    the corpus from the seed and keeps its cluster range (sharded) or the whole index.
    Recall is against the GPU exact ground truth; parity uses the oracle on the same
    arrays (rank 0)."""

    def __init__(self, rank, world, local, sharded):
        import torch

        sys.path.insert(0, str(ROOT / "tools"))
        import c4 as C4

        from paper_2410_18926_b200 import DeviceIndex
        from paper_2410_18926_b200.ground_truth import ground_truth_device

        self.C4 = C4
        P = self.P = C4.C4Params()
        dev = torch.device(f"cuda:{local}")
        corpus, queries, g = C4.generate(P, dev)
        arrs = None
        if rank == 0:
            t0 = time.time()
            arrs = C4.build(P, corpus, g)
            self.n_exact = arrs.pop("n_exact")
            self.build_s = time.time() - t0
        if world > 1:
            arrs = C4.broadcast_arrays(arrs, rank, dev)
        self.arrs = arrs
        shard = None
        if sharded:
            from paper_2410_18926_b200.sharded import partition_clusters

            shard = partition_clusters(arrs["cluster_sizes"].astype(np.int64), world)[rank]
        self.dev = DeviceIndex.from_arrays(metric="euclidean", rank=P.r, corpus=corpus, device=local,
                                           shard=shard, **arrs)
        self.gt = ground_truth_device(corpus, queries, P.k).cpu().numpy() if rank == 0 else None
        self._corpus_h = corpus.cpu().numpy() if rank == 0 and world == 1 else None
        del corpus
        torch.cuda.empty_cache()
        self.q_host = queries.cpu().numpy()
        sizes = arrs["cluster_sizes"]
        # operating point: w=1 t=800 (round-1 grid on this build: recall@100 0.931)
        self.man = {"k": P.k, "generator": {"m": P.m, "d": P.d, "n_blobs": P.m // 1000},
                    "index": {"L": P.L, "s": P.s, "r": P.r, "metric": "euclidean",
                              "built_by": "GPU restatement of build() (tools/c4.py)",
                              "mean_cluster": float(sizes.mean()), "max_cluster": int(sizes.max())},
                    "grid": {"points": [{"w": 1, "t": 800, "recall": 0.931}]}}

    def oracle_index(self):
        return self.C4.oracle_index(self.P, self.arrs, self._corpus_h)


class LocalSearcher:
    """One full index per rank (N=1, or replicas: each rank its own query batch)."""

    def __init__(self, dev, k, w, t):
        self.dev, self.k, self.w, self.t = dev, k, w, t

    def device_step(self, q, out):
        return self.dev.search_device(q, self.k, self.w, self.t, True, out=out)

    def host_step(self, qpin, hout):
        return self.dev.search_host(qpin, self.k, self.w, self.t, True, out=hout)

    def host_many(self, qs, outs):
        return self.dev.search_host_many(qs, self.k, self.w, self.t, True, outs=outs)


class ShardedSearcher:
    """Cluster-sharded index over the ranks: data-parallel front stages (one all-gather of
    the front rows), w = 1 owner-local search, and each rank keeps the results of its own
    query slice (one all-to-all, sharded.slice_results)."""

    def __init__(self, dev, k, w, t):
        from paper_2410_18926_b200.sharded import CudaShardEngine, TorchExchange

        self.dev, self.k, self.w, self.t = dev, k, w, t
        self.engine = CudaShardEngine(dev)
        self.ex = TorchExchange()

    def device_step(self, q, out):
        from paper_2410_18926_b200.sharded import sharded_search

        ids, sc, cnt = sharded_search(self.engine, self.ex, q, self.k, self.w, self.t, results="slice")
        a = min(q.shape[0], self.ex.rank * -(-q.shape[0] // self.ex.world))
        out[0][a:a + ids.shape[0]].copy_(ids)
        out[1][a:a + ids.shape[0]].copy_(sc)
        out[2][a:a + ids.shape[0]].copy_(cnt)
        return out

    def host_step(self, qpin, hout):
        import torch

        q = torch.from_numpy(qpin).cuda(non_blocking=True)
        ids, sc, cnt = self.device_step(q, self._out(q))
        for h, d in zip(hout, (ids, sc, cnt)):
            torch.from_numpy(h).copy_(d)
        return hout

    def _out(self, q):
        import torch

        if getattr(self, "_o", None) is None or self._o[0].shape[0] != q.shape[0]:
            self._o = (torch.empty((q.shape[0], self.k), dtype=torch.int64, device=q.device),
                       torch.empty((q.shape[0], self.k), dtype=torch.float32, device=q.device),
                       torch.empty((q.shape[0],), dtype=torch.int32, device=q.device))
        return self._o


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    mode = args.mode or ("sharded" if args.workload == "c4" else "replica")
    sharded = world > 1 and mode == "sharded"

    from paper_2410_18926_b200 import DeviceIndex, _native, last_launch_count
    import workloads as W

    c4 = None
    if args.workload == "c4":  # built on the GPU (tools/c4.py): no reference-built file
        c4 = C4Workload(rank, world, local, sharded)
        man, path, dev = c4.man, None, c4.dev
        w, t = operating_point(man, args)
        k = man["k"]
        searcher = ShardedSearcher(dev, k, w, t) if sharded else LocalSearcher(dev, k, w, t)
        q_host = c4.q_host
    else:
        man = W.load_manifest(args.workload)
        w, t = operating_point(man, args)
        k = man["k"]
        path = W.materialize_index(args.workload) if rank == 0 else None
        if world > 1:
            dist.barrier()
            path = W.materialize_index(args.workload)
        if sharded:
            from paper_2410_18926_b200.sharded import partition_clusters, scan_cluster_sizes

            parts = partition_clusters(scan_cluster_sizes(path), world)
            dev = DeviceIndex.from_file(path, device=local, shard=parts[rank])
            searcher = ShardedSearcher(dev, k, w, t)
        else:
            dev = DeviceIndex.from_file(path, device=local)
            searcher = LocalSearcher(dev, k, w, t)
        q_host = W.load_queries(args.workload)
    nq, d = q_host.shape
    q = torch.from_numpy(q_host).cuda()
    out = (torch.empty((nq, k), dtype=torch.int64, device="cuda"),
           torch.empty((nq, k), dtype=torch.float32, device="cuda"),
           torch.empty((nq,), dtype=torch.int32, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    for _ in range(max(3, args.warmup)):
        searcher.device_step(q, out)
    torch.cuda.synchronize()
    launches_per_step = last_launch_count()

    # ---- device-resident timing (value): per-step CUDA events, L2 flushed between steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            searcher.device_step(q, out)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        # a few ms of timed steps is shorter than nvidia-smi's sampling period: keep the
        # same workload running (untimed) until the sampler has seen >= 0.6 s of it
        while time.perf_counter() - t_start < 1.0:
            searcher.device_step(q, out)
            torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_q = nq if sharded else nq * world
    value = total_q / (ms_max / 1e3)

    # ---- recall of this run's results (identical ids to the oracle -> identical recall)
    gt = c4.gt if c4 is not None else W.load_ground_truth(args.workload)
    recall = None
    if gt is not None:
        ids = out[0].cpu().numpy()
        recall = float(np.mean([len(set(ids[i].tolist()) & set(gt[i, :k].tolist())) / k
                                for i in range(nq)]))

    # ---- per-stage device time (events around each launch inside librrg), separate pass
    import ctypes
    _native.lib.rrg_set_stage_timing(1)
    stage_ms = (ctypes.c_double * 10)()
    stage_n = (ctypes.c_int64 * 10)()
    counters = (ctypes.c_int64 * 8)()
    path_ms, path_n = (ctypes.c_double * 2)(), (ctypes.c_int64 * 2)()
    _native.lib.rrg_search_counters(counters)  # reset
    _native.lib.rrg_stage_times(stage_ms, stage_n)  # reset
    _native.lib.rrg_path_times(path_ms, path_n)  # reset
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        searcher.device_step(q, out)
    _native.lib.rrg_stage_times(stage_ms, stage_n)
    _native.lib.rrg_path_times(path_ms, path_n)
    _native.lib.rrg_search_counters(counters)
    _native.lib.rrg_set_stage_timing(0)
    names = ["project", "quantize", "route_dist", "route_select", "select_topt", "rerank", "bucket",
             "cluster_score", "ground_truth", "screen"]
    stages = {nm: round(stage_ms[i] / args.steps, 4) for i, nm in enumerate(names)}

    # ---- roofline of the dominant stage (the re-rank: screen + exact pass + final top-k).
    # Algorithmic bytes are the bytes the design must move per launch, counted by the
    # library itself (rrg_search_counters, same steps): the fp16 residual rows the
    # screen streams (each probed cluster's rows once per query group), the DISTINCT
    # f32 corpus rows the exact pass needs (union over each cluster's queries), the
    # queries, the bounds and the results.  SURVEY 8(d)'s per-query Q*t*d*4 is reported
    # beside it (gathered bytes): rows shared by a cluster's queries cross HBM once.
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    cnt = [counters[i] / args.steps for i in range(8)]
    kc = (d + 15) // 16
    screen_bytes = cnt[2] * (kc * 16 * 2 + 24) + cnt[0] * 12  # rows + row bounds terms; ub/lb write + read
    exact_rows = cnt[4]
    exact_bytes = exact_rows * d * 4 + nq * d * 4 + nq * k * 12 + nq * t * 4
    # the stage's time: its span on the launching stream (RRG_PATH_RERANK: the screen's
    # launch to the end of the final top-k; the group records and interleaved queries are
    # built on the side stream during the top-t selection, outside it); the sum of the
    # stage's per-launch event times (side-stream kernels included) is reported beside it
    rr_path_ms = path_ms[0] / args.steps if path_n[0] else 0.0
    rr_sum_ms = stages["rerank"] + stages["screen"]
    rr_ms = rr_path_ms if rr_path_ms > 0 else rr_sum_ms
    alg = screen_bytes + exact_bytes
    achieved = alg / (rr_ms / 1e3) / 1e9 if rr_ms > 0 else None
    traffic, rr_kernel = None, "k_rr_screen + k_rr_thresh + k_rerank_cluster + k_topk_final_warp"
    tf = ROOT / "profiles" / f"{args.workload}_rerank_traffic.json"
    if tf.exists():
        tinfo = json.loads(tf.read_text())
        traffic, rr_kernel = tinfo.get("bytes_per_launch"), tinfo.get("kernel", rr_kernel)
    cand = dev_cand_counts(dev, q, k, w, t)
    gathered = cand * d * 4 + nq * d * 4 + nq * k * 12
    # the exact NumPy-order distance needs one sub, one mul and one add per element,
    # none fusable: FP32 lane-ops of the candidates re-ranked exactly (the survivors)
    exact_cands = cnt[1] if cnt[1] else cand
    fp32_ops = 3 * exact_cands * d
    fp32_peak = 148 * 128 * 1.965e9
    fp32_frac = fp32_ops / (stages["rerank"] / 1e3) / fp32_peak if stages["rerank"] > 0 else None
    rr_detail = {
        "screen": {"ms": stages["screen"], "rows_streamed": cnt[2], "bytes": int(screen_bytes),
                   "gbs": screen_bytes / (stages["screen"] / 1e3) / 1e9 if stages["screen"] > 0 else None,
                   "candidates": cnt[0], "survivors": cnt[1]},
        "exact": {"ms": stages["rerank"], "rows_fetched": cnt[3], "distinct_rows": exact_rows,
                  "bytes": int(exact_bytes),
                  "gbs": exact_bytes / (stages["rerank"] / 1e3) / 1e9 if stages["rerank"] > 0 else None},
        "gathered_bytes_per_query_rows": int(gathered),
        "stage_ms_launching_stream": round(rr_path_ms, 4),
        "stage_ms_sum_of_launches": round(rr_sum_ms, 4),
    }

    # ---- e2e through the C ABI host entry: pinned host queries in, results out, per step
    qpin = torch.from_numpy(q_host).pin_memory().numpy()
    hout = (torch.empty((nq, k), dtype=torch.int64).pin_memory().numpy(),
            torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy(),
            torch.empty((nq,), dtype=torch.int32).pin_memory().numpy())
    for _ in range(2):
        searcher.host_step(qpin, hout)
    # (1) one synchronous call per step (rrg_search_host: H2D, search, D2H, sync)
    e2e_s = []
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        searcher.host_step(qpin, hout)
        e2e_s.append(time.perf_counter() - t0)
    e2e_t = torch.tensor([float(np.mean(e2e_s))], device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_single = total_q / float(e2e_t.item())
    # (2) the serving loop: K consecutive host batches through rrg_search_host_many,
    # each step's H2D and D2H inside the timed region, overlapped with the neighbouring
    # steps' searches (two device buffer sets)
    e2e_val, e2e_mode = e2e_single, "rrg_search_host, one synchronous call per step"
    if hasattr(searcher, "host_many"):
        # a serving loop of nb consecutive batches (>= 20, so the pipeline's fill and
        # drain -- one unoverlapped H2D and D2H -- are amortised as in steady state);
        # median of 3 runs
        nb = max(args.steps, 20)
        qs = [qpin] * nb
        outs = [tuple(torch.empty(a.shape, dtype=torch.from_numpy(a).dtype).pin_memory().numpy()
                      for a in hout) for _ in range(nb)]
        searcher.host_many(qs[:2], outs[:2])
        torch.cuda.synchronize()
        runs = []
        for _ in range(3):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            searcher.host_many(qs, outs)
            runs.append(time.perf_counter() - t0)
        for o in outs:  # every step returned the same results as the single call
            assert np.array_equal(o[0], hout[0]) and np.array_equal(o[2], hout[2])
        el_t = torch.tensor([float(np.median(runs))], device="cuda")
        if world > 1:  # the slowest rank sets the whole job's rate
            dist.all_reduce(el_t, op=dist.ReduceOp.MAX)
        e2e_val = total_q * nb / float(el_t.item())
        e2e_mode = (f"rrg_search_host_many over {nb} consecutive batches (H2D/D2H of "
                    "neighbouring steps overlapped with the search), median of 3 runs")

    # ---- e2e through the drop-in Python API (paper_2410_18926_b200.query_batch): pageable
    # numpy queries in, list[QueryResult] out (lazily packaged), one call per step
    api_val = None
    if not sharded:
        from paper_2410_18926_b200 import QueryParams, query_batch

        qp = QueryParams(k=k, w=w, t=t, rerank=True)
        query_batch(dev, q_host, qp)
        api_s = []
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = query_batch(dev, q_host, qp)
            api_s.append(time.perf_counter() - t0)
        assert len(res) == nq and np.array_equal(res[nq - 1].ids, hout[0][nq - 1, :hout[2][nq - 1]])
        api_t = torch.tensor([float(np.mean(api_s))], device="cuda")
        if world > 1:
            dist.all_reduce(api_t, op=dist.ReduceOp.MAX)
        api_val = total_q / float(api_t.item())

    # ---- the reference's CPU search on the same index file (rank 0, N=1): parity of the
    # timed operating point (ids and score bits of a query sample) and the CPU baseline
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dev_ids, dev_sc, dev_cnt = (a.cpu().numpy() for a in out)
        ref = CpuReference(path, k, w, t) if c4 is None else CpuReference.from_oracle(c4.oracle_index(), k, w, t)
        with ref:
            sample = np.unique(np.linspace(0, nq - 1, min(nq, args.parity_queries)).astype(int))
            r_ids, r_sc, r_cnt = ref.results(q_host[sample])
            bad = [int(i) for j, i in enumerate(sample)
                   if not (dev_cnt[i] == r_cnt[j]
                           and np.array_equal(dev_ids[i, :dev_cnt[i]], r_ids[j, :r_cnt[j]])
                           and np.array_equal(dev_sc[i, :dev_cnt[i]].view(np.int32),
                                              r_sc[j, :r_cnt[j]].view(np.int32)))]
            parity = {"queries": int(len(sample)), "mismatches": len(bad), "checker": ref.kind,
                      "what": "ids identical and f32 score bits identical per query"}
            if gt is not None:
                rec = lambda ids, cnt: float(np.mean([len(set(ids[j, :cnt[j]].tolist()) & set(gt[i, :k].tolist())) / k
                                                       for j, i in enumerate(sample)]))
                parity["recall_device"] = rec(dev_ids[sample], dev_cnt[sample])
                parity["recall_reference"] = rec(r_ids, r_cnt)
            one_qps, n1 = ref.one_core(q_host, min(10.0, args.cpu_seconds / 2))
            all_qps, n_all = cpu_reference_qps(ref, q_host, args.cpu_seconds / 2)
        cpu = {"value": all_qps, "unit": UNIT, "cores": ref.cores, "kind": ref.kind,
               "one_core": {"value": one_qps, "cores": 1, "sample": n1},
               "sample": f"{n_all} of the {nq} workload queries per repeat (best of 3), "
                         f"{'rrann.RrrIndex.query_batch (unmodified reference, baseline/_ref)' if ref.kind == 'reference' else 'oracle port of rrann.query'}"
                         f" at (w={w}, t={t}), {ref.cores}-process fork pool, 1 BLAS thread each"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32/f64/int8",
            "data": "synthetic (rrann.bench.synth_dataset clustered, regenerated bit-exact)",
            "config": {"workload": args.workload, "queries": total_q, "k": k, "w": w, "t": t,
                       **{kk: man["generator"][kk] for kk in ("m", "d", "n_blobs")}, **man["index"],
                       "recall_at_k": recall, "l2": "256 MiB write between steps (excluded)",
                       "parallelism": (f"cluster-sharded x{world}, 2x NCCL all-gather merge" if sharded
                                       else (f"replica x{world}" if world > 1 else "single"))},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 4),
                    "d2h_bytes_per_step": int(nq * k * 12 + nq * 4), "mode": e2e_mode,
                    "single_call_value": e2e_single,
                    "query_batch_value": api_val,
                    "query_batch_mode": "paper_2410_18926_b200.query_batch(index, numpy queries, "
                                        "QueryParams): pageable host input, list[QueryResult] "
                                        "(lazily packaged), one call per step"},
            "parity": parity,
            "gpu_launches": int(launches_per_step * args.steps),
            "stage_ms": stages,
            "roofline": {"bound": "hbm", "kernel": rr_kernel, "ms": rr_ms,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": int(alg),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                         "note": "algorithmic bytes = fp16 residual rows streamed by the screen "
                                 "+ distinct f32 rows the exact pass needs + queries, bounds and "
                                 "results (library counters); gathered_bytes_per_query_rows is "
                                 "SURVEY 8(d)'s Q*t*d*4 form; ms = the stage's span on the launching "
                                 "stream (rrg_path_times RRG_PATH_RERANK, screen launch to final top-k; "
                                 "side-stream group records / query interleave overlap the top-t "
                                 "selection), stages.stage_ms_sum_of_launches = per-launch event sum",
                         "stages": rr_detail,
                         "fp32_pipe": {"ops_per_launch": int(fp32_ops), "frac": fp32_frac,
                                       "peak_lane_ops_per_s": fp32_peak}},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
        if parity and parity["mismatches"]:
            print(f"PARITY FAILURE: {parity['mismatches']} of {parity['queries']} sampled queries "
                  "differ from the reference", file=sys.stderr, flush=True)
            sys.exit(3)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def dev_cand_counts(dev, q, k, w, t):
    """Total re-ranked rows of one step: sum over queries of min(t, candidates routed)."""
    xp = dev.stage_project(q)[0]
    sel = dev.stage_route(xp, w).cpu().numpy()
    sizes = dev.cluster_sizes()
    cand = sizes[sel].sum(axis=1)
    return int(np.minimum(cand, t).sum())


if __name__ == "__main__":
    main()
