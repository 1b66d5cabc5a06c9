"""Per-kernel times of a run with the graph's edges in their own order or
stably sorted by group (so each layer's points are contiguous and the advect
gathers one layer's quad field at a time).  Diagnostic only.

    python tools/order_probe.py [--config 5] [--iters 4] [--order none|group]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.model import Graph  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--order", default="none", choices=["none", "group"])
a = ap.parse_args()
w = workload(a.config)
w.config.iterations = a.iters
g = w.graph
if a.order == "group":
    order = np.argsort(np.asarray(w.bins), kind="stable")
    w = type(w)(**{**w.__dict__, "graph": Graph(g.positions, g.sources[order], g.targets[order]),
                   "bins": np.asarray(w.bins)[order]})
eng, tr, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix)
eng.run()  # warm
torch.cuda.synchronize()
eng.reset()
eng.trace = {}
t0 = time.perf_counter()
eng.run()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
out = {"config": w.name, "order": a.order, "iters": a.iters, "wall_ms": round(wall * 1e3, 1)}
for name, ev in eng.trace.items():
    ts = [x.elapsed_time(y) for x, y, _ in ev]
    out[name] = round(sum(ts) / len(ts), 3)
print(json.dumps(out))
