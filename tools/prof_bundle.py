import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd())
import torch
from paper_1504_02687_b200 import bundler as B
from paper_1504_02687_b200.workloads import workload
w = workload(4)
for _ in range(2):
    r = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix); del r
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
r = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(28); print(s.getvalue()[:6000])
