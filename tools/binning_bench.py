"""Time the device binning (select_bins: K-means over k in [4, 16] x restarts,
Davies-Bouldin pick) against the CPU oracle restatement on the same features.

    python tools/binning_bench.py [--config 2] [--criterion od] [--restarts 100]
                                  [--cpu-restarts 2]

The CPU leg (oracle/binning_oracle.py, numpy, one thread) runs a bounded
sample -- every k with --cpu-restarts restarts -- and is scaled per restart.
Prints one JSON object.  Diagnostic tool (the product path is
paper_1504_02687_b200.binning).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--criterion", default="od")
    ap.add_argument("--restarts", type=int, default=100)
    ap.add_argument("--cpu-restarts", type=int, default=2, help="0: skip the CPU leg")
    a = ap.parse_args()
    import torch

    import binning_oracle as BO
    from paper_1504_02687_b200 import binning as PB
    from paper_1504_02687_b200.workloads import workload

    w = workload(a.config)
    f = PB.edge_features(w.graph, a.criterion)
    PB.select_bins(f[:5000], restarts=2, seed=0)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    lab, k = PB.select_bins(f, restarts=a.restarts, seed=0)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t
    cpu_s = cpu_full = None
    if a.cpu_restarts > 0:
        t = time.perf_counter()
        BO.select_bins(f, a.cpu_restarts, 0)
        cpu_s = time.perf_counter() - t
        cpu_full = cpu_s * a.restarts / a.cpu_restarts
    print(json.dumps({
        "workload": w.name, "criterion": a.criterion, "edges": int(f.shape[0]),
        "features": int(f.shape[1]), "k_range": [4, 16], "restarts": a.restarts,
        "chosen_k": int(k), "gpu_select_bins_s": round(gpu_s, 3),
        "cpu_oracle_s_sample": cpu_s and round(cpu_s, 3), "cpu_sample_restarts": a.cpu_restarts,
        "cpu_oracle_s_scaled": cpu_full and round(cpu_full, 1),
        "speedup_vs_cpu_oracle": cpu_full and round(cpu_full / gpu_s, 1),
        "note": "CPU leg: oracle/binning_oracle.py (numpy, 1 thread), every k with "
                f"{a.cpu_restarts} restarts, scaled linearly to {a.restarts}",
    }))


if __name__ == "__main__":
    main()
