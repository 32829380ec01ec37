import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2410_18926_b200 as pkg
import workloads as W
man = W.load_manifest('c2'); g = man['generator']
c, q = W.synth_clustered(g['m'], g['n_queries'], g['d'], g['seed'], g['n_blobs'])
cd = torch.from_numpy(c).cuda(); qd = torch.from_numpy(q).cuda()
pkg.ground_truth_device(cd, qd[:64], 100); torch.cuda.synchronize()
t0 = time.perf_counter(); ids = pkg.ground_truth_device(cd, qd, 100); torch.cuda.synchronize()
print('gt seconds', time.perf_counter() - t0)
np.save('gpurun_out/c2_gt_gpu.npy', ids.cpu().numpy())
