"""The paper's Table 1 "random" row through the drop-in (cli.py:142-192).

    python tools/table1_bench.py [--bins 1,4,16] [--edges 200000] [--cpu]

For each B: cli.random_graph(edges) (24 samples per edge, grid 800, default
BundleConfig, bins = arange % B, interaction_matrix(B, 0.25)) bundled by
paper_1504_02687_b200.bundle() on one B200, like cli.bench does with the
reference.  Prints one JSON object: per B the bundling seconds (the
reference's timer: the iteration loop), the wall seconds of the whole
bundle() call (host arrays in, polylines out), the final sample count, the
histogram path, and -- for B = 1 and 4 -- whether the result equals the
committed reference golden (tests/golden/table1_b*.json).  --cpu adds the
oracle port of the reference CPU path on this host's cores for comparison.
Published (Java, 4-thread 1.3 GHz laptop): 6.1 / 19.9 / 72.2 s.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]

PAPER_SECONDS = {1: 6.1, 4: 19.9, 16: 72.2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bins", default="1,4,16")
    ap.add_argument("--edges", type=int, default=200_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    a = ap.parse_args()
    import torch

    from hb_hash import digest
    from paper_1504_02687_b200 import bundler as B
    from paper_1504_02687_b200.workloads import table1_workload

    out = {"edges": a.edges, "device": torch.cuda.get_device_name(0), "rows": []}
    for nb in [int(x) for x in a.bins.split(",")]:
        w = table1_workload(a.edges, nb)
        B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)  # warm
        torch.cuda.synchronize()
        walls, bund = [], []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            res = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix, workers=1)
            walls.append(time.perf_counter() - t0)
            bund.append(res.bundling_seconds)
        eng, _, _, _ = B.prepare_engine(w.graph, w.config, bins=w.bins, matrix=w.matrix)
        row = {"bins": nb, "bundling_seconds": min(bund), "wall_seconds": min(walls),
               "final_samples": int(res.sampled_edges.world.shape[0]),
               "histogram_path": eng.wkind, "paper_seconds": PAPER_SECONDS.get(nb)}
        del eng
        gpath = os.path.join(ROOT, "tests", "golden", f"table1_b{nb}{'_w1' if nb > 1 else ''}.json")
        if os.path.exists(gpath):
            g = json.load(open(gpath))
            row["equals_reference_golden"] = (
                digest(res.sampled_edges.world)["sha256"] == g["final_world"]["sha256"])
            row["reference_package_seconds_here"] = g.get("bundling_seconds_reference")
        if a.cpu:
            import oracle as O
            cores = len(os.sched_getaffinity(0))
            g = w.graph
            t0 = time.perf_counter()
            run = O.bundle_packed(g.positions, g.sources, g.targets, g.weights, w.bins, w.config,
                                  w.matrix, workers=cores)
            row["cpu_port_seconds"] = run.bundling_seconds
            row["cpu_port_cores"] = cores
            row["cpu_port_wall"] = time.perf_counter() - t0
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
