"""Latency/throughput and recall sweeps of the device query path (BASELINE.json configs[2], [4]).

    python tools/sweep.py batch --workload c3 [--batches 1,100,10000]
    python tools/sweep.py w     --workload c5 [--ws 8,16,...] [--t 800]

``batch``: for each batch size B, the mean device time of one ``rrg_search``
call over B resident queries (CUDA events on the launching stream, L2 flushed
between calls), its QPS, and the end-to-end time of ``rrg_search_host`` (host
buffers, copies included).  ``w``: recall@k against the workload's exact ground
truth and device QPS of the full query batch for each probe count w (the
recall-QPS curve).  One JSON object is printed; the committed copies live under
profiles/.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def recall(ids, gt, k):
    return float(np.mean([len(set(ids[i].tolist()) & set(gt[i, :k].tolist())) / k
                          for i in range(ids.shape[0])]))


def device_ms(dev, q, k, w, t, reps, flush):
    import torch

    st = torch.cuda.current_stream()
    out = None
    for _ in range(3):
        out = dev.search_device(q, k, w, t, True, out=out)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        out = dev.search_device(q, k, w, t, True, out=out)
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ts])), out


STAGES = ["project", "quantize", "route_dist", "route_select", "select_topt", "rerank", "bucket",
          "cluster_score", "ground_truth", "screen"]


def stage_ms(dev, q, k, w, t, reps, flush):
    """Per-stage device ms of one search (rrg_stage_times: events around every launch)."""
    import ctypes

    from paper_2410_18926_b200 import _native

    ms, n = (ctypes.c_double * 10)(), (ctypes.c_int64 * 10)()
    _native.lib.rrg_set_stage_timing(1)
    _native.lib.rrg_stage_times(ms, n)
    for i in range(reps):
        flush.fill_(i & 0xFF)
        dev.search_device(q, k, w, t, True)
    _native.lib.rrg_stage_times(ms, n)
    _native.lib.rrg_set_stage_timing(0)
    return {nm: round(ms[i] / reps, 4) for i, nm in enumerate(STAGES) if ms[i] > 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["batch", "w"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--batches", default="1,10,100,1000,10000")
    ap.add_argument("--ws", default="8,16,24,32,48,64,128,256")
    ap.add_argument("--w", type=int, default=None)
    ap.add_argument("--t", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()

    import torch

    from paper_2410_18926_b200 import DeviceIndex
    import workloads as W

    man = W.load_manifest(args.workload)
    k = man["k"]
    pts = [p for p in man.get("grid", {}).get("points", []) if p["recall"] >= 0.90]
    # the device path's operating point (bench.py operating_point): smallest t, then w
    best = min(pts, key=lambda p: (p["t"], p["w"])) if pts else {"w": 8, "t": 800}
    w0 = args.w or best["w"]
    t0 = args.t or best["t"]
    path = W.materialize_index(args.workload)
    dev = DeviceIndex.from_file(path, device=0)
    qh = W.load_queries(args.workload)
    gt = W.load_ground_truth(args.workload)
    q = torch.from_numpy(qh).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"workload": args.workload, "k": k, "index": man["index"], "generator": man["generator"],
           "device": torch.cuda.get_device_name(0), "points": []}
    if args.mode == "batch":
        res.update(w=w0, t=t0)
        for B in [int(x) for x in args.batches.split(",")]:
            B = min(B, q.shape[0])
            ms, _ = device_ms(dev, q[:B], k, w0, t0, args.reps, flush)
            hq = torch.from_numpy(qh[:B].copy()).pin_memory().numpy()  # pinned, as a server would
            dev.search_host(hq, k, w0, t0)
            e2e = []
            for _ in range(args.reps):
                t_0 = time.perf_counter()
                dev.search_host(hq, k, w0, t0)
                e2e.append(time.perf_counter() - t_0)
            e2e_ms = 1e3 * float(np.median(e2e))
            res["points"].append({"batch": B, "device_ms": ms, "device_qps": B / ms * 1e3,
                                  "e2e_ms": e2e_ms, "e2e_qps": B / e2e_ms * 1e3})
            print(res["points"][-1], file=sys.stderr, flush=True)
    else:
        res.update(t=t0)
        for w in [int(x) for x in args.ws.split(",")]:
            w = min(w, dev.n_clusters)
            ms, out = device_ms(dev, q, k, w, t0, max(3, args.reps // 4), flush)
            ids = out[0].cpu().numpy()
            pt = {"w": w, "t": t0, "device_ms": ms, "device_qps": q.shape[0] / ms * 1e3,
                  "recall_at_k": recall(ids, gt, k) if gt is not None else None,
                  "stage_ms": stage_ms(dev, q, k, w, t0, 3, flush)}
            res["points"].append(pt)
            print(pt, file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
