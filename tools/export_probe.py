"""Throughput of the bulk polyline export/import vs the reference's Python
formatting (io.py:136-145 expression) on a sample.  Diagnostic only.

    python tools/export_probe.py [--config 4] [--sample-edges 20000]
"""

from __future__ import annotations

import argparse
import io
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import bundler as B  # noqa: E402
from paper_1504_02687_b200 import io as hio  # noqa: E402
from paper_1504_02687_b200.workloads import workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--sample-edges", type=int, default=20000)
    a = ap.parse_args()
    w = workload(a.config)
    res = B.bundle(w.graph, w.config, bins=w.bins, matrix=w.matrix)
    se = res.sampled_edges
    n_pts = int(se.starts[-1])
    out = {"edges": len(se), "points": n_pts}
    t0 = time.perf_counter()
    with open("/dev/null", "w") as f:
        hio.export_polylines(res, f)
    t = time.perf_counter() - t0
    out["native_export_s"] = round(t, 3)
    out["native_export_Mpts_per_s"] = round(n_pts / t / 1e6, 1)
    # reference formatting expression on a sample of edges
    k = min(a.sample_edges, len(se))
    t0 = time.perf_counter()
    buf = io.StringIO()
    g = res.graph
    for e in range(k):
        s = se[e]
        coords = " ".join(f"{c:.9g}" for p in s.points for c in p)
        buf.write(f"{e} {g.bins[e]} {g.weights[e]:.9g} {len(s)} {coords}\n")
    t = time.perf_counter() - t0
    k_pts = int(se.starts[k])
    out["python_format_Mpts_per_s"] = round(k_pts / t / 1e6, 3)
    out["python_export_estimate_s"] = round(n_pts / (k_pts / t), 1)
    # import: native parser on the sample's text
    text = buf.getvalue()
    t0 = time.perf_counter()
    recs = hio.read_polylines(io.StringIO(text))
    out["native_read_sample_Mpts_per_s"] = round(k_pts / (time.perf_counter() - t0) / 1e6, 1)
    t0 = time.perf_counter()
    hio._read_python(text.split("\n"))
    out["python_read_sample_Mpts_per_s"] = round(k_pts / (time.perf_counter() - t0) / 1e6, 2)
    assert len(recs) == k
    out["cores"] = os.cpu_count()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
