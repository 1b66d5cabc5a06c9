"""Binning fixtures made by running the REFERENCE (binning.py) in this container.

    python tests/golden/make_binning_golden.py

Imports /root/reference/pkg/src/histobundle/binning.py and records, on the
config-1 graph (2,000 edges, seed 0) and a duplicate-heavy feature set:
  * kmeans(features, k, restarts, seed) -> assignment, centroids, inertia
    for the od (d=4), origin (d=2) and length (d=1) criteria;
  * davies_bouldin of each of those clusterings;
  * select_bins (Davies-Bouldin over k in [4, 16]) on od and origin features;
  * assign_bins(graph, "length", "auto") (ordinal relabelling);
  * _update_centroids on assignments with emptied clusters (the reseed path,
    binning.py:145-154).
Writes tests/golden/binning.npz.  Versions are stored next to the arrays.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from histobundle import binning as RBIN  # noqa: E402
from histobundle import model as RM  # noqa: E402

from paper_1504_02687_b200.workloads import workload  # noqa: E402


def main():
    w = workload(1)
    g = w.graph
    rg = RM.Graph.from_arrays(g.positions, g.sources, g.targets, g.weights, g.bins)
    out = {"numpy": np.array(np.__version__)}
    cases = [("od", 5, 100, 3), ("origin", 7, 100, 11), ("length", 4, 100, 5),
             ("od", 12, 40, 7)]
    for i, (crit, k, restarts, seed) in enumerate(cases):
        f = RBIN.edge_features(rg, crit)
        c = RBIN.kmeans(f, k, restarts=restarts, seed=seed)
        out[f"km{i}_meta"] = np.array([k, restarts, seed])
        out[f"km{i}_crit"] = np.array(crit)
        out[f"km{i}_assign"] = c.assignment
        out[f"km{i}_cent"] = c.centroids
        out[f"km{i}_inertia"] = np.array(c.inertia)
        out[f"km{i}_db"] = np.array(RBIN.davies_bouldin(f, c))
    for crit, restarts, seed in [("od", 20, 0), ("origin", 20, 4)]:
        f = RBIN.edge_features(rg, crit)
        a, k = RBIN.select_bins(f, restarts=restarts, seed=seed)
        out[f"sel_{crit}_assign"] = a
        out[f"sel_{crit}_k"] = np.array(k)
        out[f"sel_{crit}_meta"] = np.array([restarts, seed])
    a, k, kind = RBIN.assign_bins(rg, "length", "auto", restarts=20, seed=2)
    out["ab_length_assign"], out["ab_length_k"] = a, np.array(k)
    # reseed path: a clustering whose assignment left clusters empty
    rng = np.random.default_rng(5)
    f = np.vstack([rng.normal(0.0, 1.0, (300, 2)), rng.normal(8.0, 0.5, (40, 2)),
                   np.repeat([[3.0, 3.0]], 25, axis=0)])
    cent = rng.normal(2.0, 3.0, (6, 2))
    assign = rng.integers(0, 3, f.shape[0]) * 2  # clusters 1, 3, 5 empty
    out["rs_features"], out["rs_cent"], out["rs_assign"] = f, cent, assign
    out["rs_out"] = RBIN._update_centroids(f, assign, cent)
    c = RBIN.kmeans(f, 6, restarts=50, seed=9)
    out["rs_km_assign"], out["rs_km_cent"] = c.assignment, c.centroids
    out["rs_km_inertia"] = np.array(c.inertia)
    np.savez_compressed(os.path.join(HERE, "binning.npz"), **out)
    print("wrote binning.npz", sorted(out))


if __name__ == "__main__":
    main()
