"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): config 1 (cfg1 grid, 2k edges) for 3 iterations through the
public bundle(), config 3 at 2 % scale (8 groups, repulsive matrix path),
and the standalone Laplacian+count / emit entry points.  Diagnostic only.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""

from __future__ import annotations

import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def main():
    for k, scale, iters in ((1, 1.0, 3), (3, 0.02, 2), (2, 0.05, 2)):
        w = workload(k, scale=scale)
        cfg = dataclasses.replace(w.config, iterations=iters)
        res = B.bundle(w.graph, cfg, bins=w.bins, matrix=w.matrix)
        torch.cuda.synchronize()
        print(w.name, int(res.sampled_edges.starts[-1]), "points", flush=True)


if __name__ == "__main__":
    main()
