"""Time the re-rank screen variants (RRG_SCREEN_DIAG probes): stage ms per batch.

    python tools/probes/screen_diag.py [workload] [w]      (default c2 1)
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as W  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex, _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = int(sys.argv[2]) if len(sys.argv) > 2 else 1
path = W.materialize_index(name)
dev = DeviceIndex.from_file(path)
q = torch.from_numpy(W.load_queries(name)).cuda()
for diag in ("0", "1", "2", "0"):
    os.environ["RRG_SCREEN_DIAG"] = diag
    dev.reload_options()
    for _ in range(3):
        dev.search_device(q, 100, w, 800, True)
    torch.cuda.synchronize()
    _native.lib.rrg_set_stage_timing(1)
    ms = (ctypes.c_double * 10)()
    n = (ctypes.c_int64 * 10)()
    _native.lib.rrg_stage_times(ms, n)
    for _ in range(5):
        dev.search_device(q, 100, w, 800, True)
    _native.lib.rrg_stage_times(ms, n)
    _native.lib.rrg_set_stage_timing(0)
    print(f"diag={diag} screen stage {ms[9] / 5:.4f} ms  rerank {ms[5] / 5:.4f} ms", flush=True)
