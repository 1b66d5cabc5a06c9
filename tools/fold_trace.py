"""Per (strip, row block) event times of fold_kernel on layer 0 (diagnostic).

    python tools/build_variant.py trace -D HB_FOLD_TRACE=1
    HB_B200_LIB=paper_1504_02687_b200/_lib/var_trace/libhb_b200.so \\
        python tools/fold_trace.py [--nbins 1 --nv 1024 --nu 1024]

Events: 0 = C tile published, 1 = carry received, 2 = carry sent,
3 = T tile stored.  Prints, per strip, the times (us from the first event) of
block 0 and the last block, and the carry lag between neighbouring strips.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_02687_b200 import _native as N  # noqa: E402
from paper_1504_02687_b200.engine import ptr, stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nbins", type=int, default=1)
ap.add_argument("--nv", type=int, default=1024)
ap.add_argument("--nu", type=int, default=1024)
a = ap.parse_args()
B, V, U = a.nbins, a.nv, a.nu
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.rand((B, V, U), generator=g, device="cuda") ** 8 * 300).float()
radii = torch.tensor([5], dtype=torch.int32)
out = torch.empty_like(x)
ws = torch.empty(int(N.lib().hb_smooth_workspace_bytes(B, V, U)), dtype=torch.uint8, device="cuda")
for _ in range(3):
    N.call("hb_smooth", None, ptr(x), None, B, V, U, radii.data_ptr(), 1, ptr(out), ptr(ws),
           ws.numel(), None, stream_ptr())
torch.cuda.synchronize()
buf = np.zeros((64, 128, 4), dtype=np.uint64)
f = N.lib().hb_debug_fold_trace
f.argtypes = [ctypes.c_void_p]
assert f(buf.ctypes.data) == 0
S = 64 if B * ((U + 63) // 64) <= 148 else 128
ns, nb = (U + S - 1) // S, (V + 31) // 32
t = buf[:ns, :nb].astype(np.int64)
t0 = t[t > 0].min()
t = (t - t0) / 1000.0
print("S", S, "strips", ns, "blocks", nb, "kernel span us", t.max())
for k in range(ns):
    print(k, "blk0 C %.2f got %.2f sent %.2f done %.2f | last C %.2f got %.2f sent %.2f done %.2f" %
          (*t[k, 0], *t[k, nb - 1]))
lag = t[1:, :, 1] - t[:-1, :, 2]
print("carry transit (got[k] - sent[k-1]) us: mean %.3f min %.3f max %.3f" % (lag.mean(), lag.min(), lag.max()))
chain = t[:, :, 2] - t[:, :, 1]
print("chain (sent - got) us: mean %.3f" % chain.mean())
store = t[:, :, 3] - t[:, :, 2]
print("store (done - sent) us: mean %.3f" % store.mean())
colrate = np.diff(t[:, :, 0], axis=1)
print("column fold per block us: mean %.3f" % colrate.mean())
if "--detail" in sys.argv[1:] or True:
    for k in (0, 1, ns - 1):
        print("strip", k)
        for b in range(min(nb, 20)):
            print("  b%2d C %7.2f got %7.2f sent %7.2f done %7.2f" % (b, *t[k, b]))
