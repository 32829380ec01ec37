"""Stage times of an index under RRG_* variants: python tools/probes/variant_probe.py c2 1 800 VAR=a,b ..."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as W  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex, _native  # noqa: E402

name, w, t = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
var, vals = sys.argv[4].split("=")
dev = DeviceIndex.from_file(W.materialize_index(name))
q = torch.from_numpy(W.load_queries(name)).cuda()
k = W.load_manifest(name)["k"]
ref = None
for v in vals.split(",") * 2:
    os.environ[var] = v
    dev.reload_options()
    out = [a.cpu() for a in dev.search_device(q, k, w, t, True)]
    if ref is None:
        ref = out
    same = all(torch.equal(torch.nan_to_num(a), torch.nan_to_num(b)) for a, b in zip(out, ref))
    torch.cuda.synchronize()
    _native.lib.rrg_set_stage_timing(1)
    ms, n = (ctypes.c_double * 10)(), (ctypes.c_int64 * 10)()
    _native.lib.rrg_stage_times(ms, n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        dev.search_device(q, k, w, t, True)
    _native.lib.rrg_stage_times(ms, n)
    _native.lib.rrg_set_stage_timing(0)
    e0.record()
    for _ in range(5):
        dev.search_device(q, k, w, t, True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} w={w} t={t} {var}={v}: step {e0.elapsed_time(e1) / 5:.4f} ms  rerank {ms[5] / 5:.4f}  "
          f"screen {ms[9] / 5:.4f}  same={same}", flush=True)
