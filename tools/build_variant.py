"""Build an A/B variant of the native library for tools/kernel_probe.py.

    python tools/build_variant.py NAME [--rev REV --files a.cu,b.cuh] [-D X=1 ...]

Copies csrc/ to a scratch dir, replaces --files with their content at git
revision --rev, and builds paper_1504_02687_b200/_lib/var_NAME/libhb_b200.so
with extra -D defines.  Run the probe on it with HB_B200_LIB=<that path>.
Diagnostic tool; not part of the product path.
"""

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1504_02687_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--rev", default=None)
    ap.add_argument("--files", default="")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    tmp = tempfile.mkdtemp(prefix="hbvar_")
    src = os.path.join(tmp, "pkg", "csrc")  # keeps csrc's ../../include path valid
    shutil.copytree(N.CSRC, src)
    os.symlink(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    for f in filter(None, a.files.split(",")):
        rel = os.path.relpath(os.path.join(N.CSRC, f), ROOT)
        txt = subprocess.run(["git", "-C", ROOT, "show", f"{a.rev}:{rel}"], check=True,
                             capture_output=True, text=True).stdout
        with open(os.path.join(src, f), "w") as fh:
            fh.write(txt)
    old = N.CSRC
    N.CSRC = src
    try:
        out = N.build(out=os.path.join(N.LIB_DIR, "var_" + a.name, "libhb_b200.so"),
                      defines=tuple("-D" + d for d in a.D))
    finally:
        N.CSRC = old
        shutil.rmtree(tmp, ignore_errors=True)
    print(out)


if __name__ == "__main__":
    main()
