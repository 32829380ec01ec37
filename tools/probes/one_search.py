"""One search of a file workload at (w, t) for ncu captures: python tools/probes/one_search.py c3 4 800"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import workloads as W  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex  # noqa: E402

name, w, t = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dev = DeviceIndex.from_file(W.materialize_index(name))
q = torch.from_numpy(W.load_queries(name)).cuda()
k = W.load_manifest(name)["k"]
for _ in range(2):
    dev.search_device(q, k, w, t, True)
torch.cuda.synchronize()
