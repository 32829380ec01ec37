"""Probe where the host-buffer (e2e) time goes on the GPU box: PCIe copies vs chunked search."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2410_18926_b200 import DeviceIndex
import workloads as W

path = W.materialize_index("c2")
dev = DeviceIndex.from_file(path)
q = W.load_queries("c2")
qp = torch.from_numpy(q).pin_memory()
qd = torch.empty_like(qp, device="cuda")
for _ in range(3):
    qd.copy_(qp, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter(); qd.copy_(qp, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t0
print(f"H2D {qp.numel()*4/1e6:.1f} MB: {h2d*1e3:.3f} ms = {qp.numel()*4/h2d/1e9:.1f} GB/s")
res = torch.empty((10000, 100), dtype=torch.int64).pin_memory()
rd = torch.empty((10000, 100), dtype=torch.int64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); res.copy_(rd, non_blocking=True); torch.cuda.synchronize()
d2h = time.perf_counter() - t0
print(f"D2H 8 MB: {d2h*1e3:.3f} ms = {8e6/d2h/1e9:.1f} GB/s")
for n in (10000, 5000, 2500):
    for _ in range(3):
        dev.search_device(qd[:n], 100, 1, 800, True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dev.search_device(qd[:n], 100, 1, 800, True)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / 5
    print(f"device search n={n}: {el*1e3:.3f} ms ({n/el/1e6:.2f} M QPS)")
qpn = qp.numpy()
ids = torch.empty((10000, 100), dtype=torch.int64).pin_memory().numpy()
sc = torch.empty((10000, 100), dtype=torch.float32).pin_memory().numpy()
ct = torch.empty((10000,), dtype=torch.int32).pin_memory().numpy()
import os
for c in ("1", "2", "4", "8"):
    os.environ["RRG_HOST_PIECES"] = c
    for _ in range(2):
        dev.search_host(qpn, 100, 1, 800, True, out=(ids, sc, ct))
    t0 = time.perf_counter()
    for _ in range(5):
        dev.search_host(qpn, 100, 1, 800, True, out=(ids, sc, ct))
    el = (time.perf_counter() - t0) / 5
    print(f"host search pieces={c}: {el*1e3:.3f} ms ({10000/el/1e6:.2f} M QPS)")
