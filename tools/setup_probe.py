import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1504_02687_b200 import bundler as B
from paper_1504_02687_b200.workloads import workload
import cProfile, pstats
w = workload(4)
B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
def go():
    c, bins_arr, matrix = B._resolve(w.graph, w.config, w.bins, w.matrix)
    eng, tr, lo, hi = B._setup(w.graph, c, bins_arr, matrix, False, None, 2.0)
    torch.cuda.synchronize()
    return eng
go(); torch.cuda.synchronize()
pr = cProfile.Profile(); t=time.perf_counter(); pr.enable(); go(); pr.disable(); print("total", time.perf_counter()-t)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
