"""Golden fixture for the polyline export: runs the REFERENCE's
``histobundle.io.export_polylines`` (io.py:136-145) on a small synthetic
result and stores its exact text.  Run in the container that has
/root/reference (the fixture travels; the reference does not):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
"""

import io
import os
import sys
from types import SimpleNamespace

import numpy as np

from histobundle import io as ref_io  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def fixture():
    rng = np.random.default_rng(11)
    n_edges = 40
    lens = rng.integers(2, 30, size=n_edges)
    starts = np.zeros(n_edges + 1, dtype=np.int64)
    np.cumsum(lens, out=starts[1:])
    world = rng.normal(0.5, 0.3, size=(int(starts[-1]), 2))
    # awkward magnitudes and exact values for %.9g
    world[0] = [0.0, -0.0]
    world[1] = [1e-7, -3.25e-5]
    world[2] = [123456789.5, 1e22]
    world[3] = [0.5, 2.0]
    world[4] = [1.0000000005, 0.9999999995]
    weights = rng.uniform(0.1, 5.0, size=n_edges)
    weights[0] = 1.0
    bins = rng.integers(0, 7, size=n_edges)
    return world, starts, weights, bins


class _Edge:
    def __init__(self, edge_index, points):
        self.edge_index, self.points = edge_index, points

    def __len__(self):
        return len(self.points)


def main():
    world, starts, weights, bins = fixture()
    edges = [_Edge(e, world[starts[e]:starts[e + 1]]) for e in range(len(starts) - 1)]
    result = SimpleNamespace(graph=SimpleNamespace(bins=bins, weights=weights),
                             sampled_edges=edges)
    buf = io.StringIO()
    ref_io.export_polylines(result, buf)
    np.savez(os.path.join(HERE, "io_input.npz"), world=world, starts=starts, weights=weights,
             bins=bins)
    with open(os.path.join(HERE, "io_export.txt"), "w") as f:
        f.write(buf.getvalue())
    print("wrote", len(buf.getvalue()), "bytes")


if __name__ == "__main__":
    sys.exit(main())
