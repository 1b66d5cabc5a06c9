import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np, cProfile, pstats
from paper_1504_02687_b200 import binning as PB
from paper_1504_02687_b200.workloads import workload
w = workload(2); f = PB.edge_features(w.graph, "od")
PB.select_bins(f[:5000], restarts=2, seed=0)
pr = cProfile.Profile(); t=time.perf_counter(); pr.enable(); PB.select_bins(f, restarts=100, seed=0); torch.cuda.synchronize(); pr.disable(); print("total", time.perf_counter()-t)
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
