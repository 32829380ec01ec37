"""C5 / C2 stage times with the dp4a and the tcgen05 stage-B scoring."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as W  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex, _native  # noqa: E402

for name, w, t in (("c5", 64, 1600), ("c5", 16, 1600), ("c2", 1, 800)):
    dev = DeviceIndex.from_file(W.materialize_index(name))
    q = torch.from_numpy(W.load_queries(name)).cuda()
    for tc in ("0", "1", "0", "1"):
        os.environ["RRG_SCORE_TC"] = tc
        dev.reload_options()
        for _ in range(2):
            dev.search_device(q, 100, w, t, True)
        torch.cuda.synchronize()
        _native.lib.rrg_set_stage_timing(1)
        ms, n = (ctypes.c_double * 10)(), (ctypes.c_int64 * 10)()
        _native.lib.rrg_stage_times(ms, n)
        for _ in range(3):
            dev.search_device(q, 100, w, t, True)
        _native.lib.rrg_stage_times(ms, n)
        _native.lib.rrg_set_stage_timing(0)
        print(f"{name} w={w} t={t} tc={tc}: cluster_score {ms[7] / 3:.4f} ms, total "
              f"{sum(ms[i] for i in range(10)) / 3:.4f} ms", flush=True)
    del dev
