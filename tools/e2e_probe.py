"""Phase breakdown of the public bundle() call (host in, host out).

    python tools/e2e_probe.py [--config 4]

Diagnostic tool; prints one JSON object with wall-clock seconds per phase.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200 import engine as EN  # noqa: E402
from paper_1504_02687_b200.model import make_transform  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    args = ap.parse_args()
    w = workload(args.config)
    g, cfg = w.graph, w.config
    B.bundle(g, cfg, bins=w.bins, matrix=w.matrix)  # warm
    torch.cuda.synchronize()
    out = {}
    t = time.perf_counter()

    def lap(name):
        nonlocal t
        torch.cuda.synchronize()
        now = time.perf_counter()
        out[name] = round(now - t, 4)
        t = now

    tr = make_transform(g.positions, cfg.grid_size, cfg.padding_cells)
    src = tr.world_to_grid(g.positions[g.sources])
    dst = tr.world_to_grid(g.positions[g.targets])
    lap("transform+world_to_grid")
    counts = EN.sample_counts(src, dst, cfg.delta)
    lap("sample_counts")
    eng, tr2, lo, hi = B.prepare_engine(g, cfg, bins=w.bins, matrix=w.matrix)
    lap("prepare_engine(total, incl. the two above again)")
    eng.run()
    lap("run")
    wd = eng.world_points(tr.origin, tr.cell_size, g.positions[g.sources],
                          g.positions[g.targets])
    lap("world_points")
    host = EN.download(wd)
    lap("download_world_pageable")
    pinned = torch.empty(wd.shape, dtype=wd.dtype, pin_memory=True)
    lap("alloc_pinned")
    pinned.copy_(wd)
    lap("d2h_pinned")
    arr = np.empty(wd.shape, dtype=np.float64)
    lap("np_empty")
    arr[...] = pinned.numpy()
    lap("memcpy_pinned_to_numpy")
    t0 = time.perf_counter()
    res = B.bundle(g, cfg, bins=w.bins, matrix=w.matrix)
    out["bundle_total"] = round(time.perf_counter() - t0, 4)
    out["n_points"] = int(res.sampled_edges.world.shape[0])
    del host
    print(json.dumps(out))


if __name__ == "__main__":
    main()
