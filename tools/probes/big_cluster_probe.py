"""Probe: d=960 indexes with one very large cluster (k-means on blob data can leave
clusters 10x the mean), searched at batch sizes that fill the GPU; oracle-checked."""
import sys
import traceback

import numpy as np
import torch

sys.path[:0] = ["tests", "."]
from index_writer import random_index  # noqa: E402
from oracle import rrann_oracle as O  # noqa: E402
from paper_2410_18926_b200 import DeviceIndex  # noqa: E402

for big, d in [(3000, 960), (8000, 960), (14120, 960), (14120, 768), (30000, 128)]:
    sizes = np.array([big, 1] + [1220] * 30)
    m = int(sizes.sum())
    blob = random_index(d, 64, 32, len(sizes), m, seed=3, sizes=sizes)
    open("/tmp/big.rrr", "wb").write(blob)
    dev = DeviceIndex.from_file("/tmp/big.rrr")
    oi = O.read_index(blob)
    q = np.random.default_rng(0).standard_normal((4000, d)).astype(np.float32)
    qd = torch.from_numpy(q).cuda()
    for k, w, t in [(100, 1, 200), (100, 1, 800), (100, 2, 800), (10, 4, 100)]:
        try:
            ids, sc, cnt = (x.cpu().numpy() for x in dev.search_device(qd, k, w, t, True))
            bad = 0
            for i in range(0, 4000, 250):
                r = O.query(oi, q[i], k, w, t, True)
                c = int(cnt[i])
                bad += not (c == len(r.ids) and np.array_equal(ids[i, :c], r.ids)
                            and np.array_equal(sc[i, :c].view(np.int32), r.scores.view(np.int32)))
            print(f"big={big} d={d} k={k} w={w} t={t}: ok, {bad} oracle mismatches / 16", flush=True)
        except Exception:
            print(f"big={big} d={d} k={k} w={w} t={t}: FAIL", traceback.format_exc().splitlines()[-1], flush=True)
