import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2410_18926_b200 import DeviceIndex
import workloads as W
path = W.materialize_index('c2'); dev = DeviceIndex.from_file(path)
q = W.load_queries('c2'); k, w, t = 100, 1, 800
qp = torch.from_numpy(q).pin_memory().numpy()
def outs(n): return [tuple(torch.empty(s, dtype=dt).pin_memory().numpy() for s, dt in (((10000, k), torch.int64), ((10000, k), torch.float32), ((10000,), torch.int32))) for _ in range(n)]
for nb in (2, 10, 20, 40):
    o = outs(nb); dev.search_host_many([qp] * 2, k, w, t, True, outs=o[:2]); torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter(); dev.search_host_many([qp] * nb, k, w, t, True, outs=o); el = time.perf_counter() - t0
        best = min(best, el)
    print(nb, 'batches:', round(nb * 10000 / best / 1e6, 3), 'M QPS', round(best / nb * 1e3, 3), 'ms/batch')
