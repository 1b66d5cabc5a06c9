"""Time hb_smooth (and its kernels) on a config-sized synthetic histogram.

    python tools/smooth_probe.py [--nbins 4 --nv 2047 --nu 2048 --sigma 51.2]

Prints one JSON object with ms per hb_smooth call and the algorithmic
GB/s (4 B/cell int32 read + 8 B/cell per pass).  Diagnostic only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1504_02687_b200 import _native as N  # noqa: E402
from paper_1504_02687_b200.engine import box_widths, ptr, stream_ptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nbins", type=int, default=4)
    ap.add_argument("--nv", type=int, default=2047)
    ap.add_argument("--nu", type=int, default=2048)
    ap.add_argument("--sigma", type=float, default=51.2)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    B, V, U = a.nbins, a.nv, a.nu
    g = torch.Generator(device="cuda").manual_seed(0)
    # bundled-looking counts: mostly zero, heavy tail
    hist = (torch.rand((B, V, U), generator=g, device="cuda") ** 8 * 3000).to(torch.int32)
    radii = torch.tensor([(w - 1) // 2 for w in box_widths(a.sigma, 3)], dtype=torch.int32)
    out = torch.empty((B, V, U), dtype=torch.float32, device="cuda")
    ws = torch.empty(int(N.lib().hb_smooth_workspace_bytes(B, V, U)), dtype=torch.uint8,
                     device="cuda")
    peak = torch.zeros(B, dtype=torch.float32, device="cuda")
    s = stream_ptr()

    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out2 = torch.empty_like(out)

    def run_float():
        N.call("hb_smooth", ptr(hist), None, None, B, V, U, radii.data_ptr(), int(radii.numel()),
               ptr(out), ptr(ws), ws.numel(), ptr(peak), s)

    def run_counts():
        N.call("hb_smooth_counts", ptr(hist), None, 1.0, float(2 ** 24), B, V, U,
               radii.data_ptr(), int(radii.numel()), ptr(out2), ptr(ws), ws.numel(), ptr(peak),
               ptr(status), s)

    G = B * V * U
    alg = 4 * G + 8 * G * int(radii.numel())
    res = {"shape": [B, V, U], "radii": radii.tolist(), "alg_bytes": alg,
           "peak_hbm_GBps": 6551.7}
    for name, fn in (("hb_smooth", run_float), ("hb_smooth_counts", run_counts)):
        fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res[name] = {"ms": round(ms, 4), "alg_GBps": round(alg / ms / 1e6, 1),
                     "frac": round(alg / ms / 1e6 / 6551.7, 4)}
    res["bit_identical"] = bool(torch.equal(out, out2))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
