"""One C5 search at (w, t) for ncu captures: python tools/probes/c5_probe.py 64 1600"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as W  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex  # noqa: E402

w, t = int(sys.argv[1]), int(sys.argv[2])
dev = DeviceIndex.from_file(W.materialize_index("c5"))
q = torch.from_numpy(W.load_queries("c5")).cuda()
for _ in range(2):
    dev.search_device(q, 100, w, t, True)
torch.cuda.synchronize()
