"""Loader for the sm_100a C-ABI library ``libhb_b200.so`` (csrc/*.cu).

The library is built in-tree (``build()`` below, called by
``__graft_entry__.build()``) with nvcc for ``sm_100a`` only, and loaded with
ctypes. There is no fallback: if the library is missing or no CUDA device is
present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_PKG, "csrc")
LIB_DIR = os.path.join(_PKG, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libhb_b200.so")
INCLUDE = os.path.join(os.path.dirname(_PKG), "include")

SOURCES = ["hb_api.cu", "hb_polyline.cu", "hb_field.cu", "hb_advect.cu", "hb_advect_flat.cu", "hb_lapcount.cu", "hb_splat.cu", "hb_binning.cu", "hb_render.cu", "hb_ordered.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit-exact float64: never contract a*b+c into FMA
    "--fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
]


class NativeError(RuntimeError):
    pass


def build(verbose: bool = False, out: str = LIB_PATH, defines: tuple = ()) -> str:
    """Compile csrc/*.cu into _lib/libhb_b200.so (cross-compiles without a GPU).
    ``out``/``defines`` build tuning variants for tools/ (``-DNAME=V``)."""
    lib_dir = os.path.dirname(out)
    os.makedirs(lib_dir, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objs = []
    for src in SOURCES:
        obj = os.path.join(lib_dir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *defines, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = out + ".tmp"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "--cudart=static", "-o", tmp, *objs], check=True)
    os.replace(tmp, out)
    return out


HOST_IO_SRC = os.path.join(_PKG, "csrc_host", "hb_io.cpp")
HOST_IO_LIB = os.path.join(LIB_DIR, "libhb_io.so")


def build_host_io(verbose: bool = False) -> str:
    """Compile the host polyline I/O library (g++, no GPU code)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    cxx = os.environ.get("CXX", "g++")
    tmp = HOST_IO_LIB + ".tmp"
    cmd = [cxx, "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread", "-fvisibility=hidden",
           HOST_IO_SRC, "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, HOST_IO_LIB)
    return HOST_IO_LIB


_P, _I64, _I, _D, _SZ = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                         ctypes.c_double, ctypes.c_size_t)

# name -> (restype, argtypes); mirrors include/histobundle_b200.h
SIGNATURES = {
    "hb_abi_version": (_I, []),
    "hb_last_error": (ctypes.c_char_p, []),
    "hb_device_sm_count": (_I, []),
    "hb_segment_widths": (_I, [_P, _P, _I64, _P, _P, _I, _I, _I, _P, _D, _D, _I, _P, _P]),
    "hb_advect_laplacian_count": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _I, _I, _I, _D, _D, _D,
                                       _I, _D, _I, _D, _P, _P, _P, _P, _P]),
    "hb_kmeans_assign": (_I, [_P, _I64, _I, _I, _P, _P, _I, _P, _P, _P]),
    "hb_kmeans_update": (_I, [_P, _I64, _I, _I, _P, _P, _I, _P, _P, _P]),
    "hb_kmeans_reseed_workspace_bytes": (_SZ, [_I64, _I]),
    "hb_kmeans_reseed": (_I, [_P, _I64, _I, _I, _P, _P, _I, _P, _P, _SZ, _P]),
    "hb_kmeans_lloyd": (_I, [_P, _I64, _I, _I, _P, _I, _P, _P, _I, _P, _SZ, _P]),
    "hb_kmeans_inertia_blocks": (_I, []),
    "hb_kmeans_inertia": (_I, [_P, _I64, _I, _I, _P, _I, _P, _P, _P]),
    "hb_kmeans_scatter": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P, _P]),
    "hb_launch_count": (ctypes.c_longlong, []),
    "hb_edge_prepare": (_I, [_P, _P, _P, _I64, _D, _D, _D, _D, _P, _P, _P, _P]),
    "hb_to_world_nodes": (_I, [_P, _P, _I64, _D, _D, _D, _P, _P, _P, _P, _P]),
    "hb_sample_fill": (_I, [_P, _P, _P, _I64, _P, _P]),
    "hb_offset": (_I, [_P, _P, _I64, _P, _P]),
    "hb_to_world": (_I, [_P, _P, _I64, _D, _D, _D, _P, _P, _P, _P]),
    "hb_tiles_geometry": (_I, [_I, _I, _I, _D, _P]),
    "hb_tiles_plan": (_I, [_P, _P, _P]),
    "hb_tiles_flush": (_I, [_P, _P, _I, _I, _P]),
    "hb_segtab_geometry": (_I, [_I, _I, _I, _D, _P, _P]),
    "hb_segtab_expand": (_I, [_P, _P, _I, _I, _P, _P]),
    "hb_splat": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _I, _I, _I, _P, _P, _P]),
    "hb_smooth_workspace_bytes": (_SZ, [_I, _I, _I]),
    "hb_smooth": (_I, [_P, _P, _P, _I, _I, _I, _P, _I, _P, _P, _SZ, _P, _P]),
    "hb_smooth_counts": (_I, [_P, _P, _D, _D, _I, _I, _I, _P, _I, _P, _P, _SZ, _P, _P, _P]),
    "hb_mix_layers": (_I, [_P, _P, _P, _I, _I, _I, _P, _P]),
    "hb_integral_image": (_I, [_P, _I, _I, _I, _P, _P]),
    "hb_used_cells": (_I, [_P, _P, _I, _I, _I, _D, _P, _P]),
    "hb_advect_partials": (_I64, []),
    "hb_grad_field_bytes": (_I64, [_I, _I, _I]),
    "hb_grad_field": (_I, [_P, _I, _I, _I, _P, _P]),
    "hb_advect_laplacian": (_I, [_P, _P, _P, _I64, _I64, _P, _P, _P, _I, _I, _I, _D, _D,
                                 _D, _I, _D, _I, _D, _P, _P, _P, _P, _P]),
    "hb_advect_points": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _I, _I, _I, _D, _D, _D, _I,
                              _P, _P, _P]),
    "hb_laplacian_count": (_I, [_P, _P, _P, _I64, _I64, _D, _I, _D, _P, _P, _P]),
    "hb_reduce_f64": (_I, [_P, _I64, _P, _P]),
    "hb_resample_count": (_I, [_P, _P, _I64, _D, _P, _P, _P]),
    "hb_scan_workspace_bytes": (_SZ, [_I64]),
    "hb_scan_counts": (_I, [_P, _I64, _P, _P, _SZ, _P]),
    "hb_resample_emit": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _I, _I, _P,
                              _P, _P]),
    "hb_resample_emit_cap": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P, _I, _I,
                                  _P, _P, _P]),
    "hb_clamp_starts": (_I, [_P, _I64, _I64, _P, _P]),
    "hb_probe": (_I, [_P, _I, _I, _P, _I64, _P, _P, _P]),
    "hb_point_span": (_I, [_P, _I64, _P, _P, _P]),
    "hb_exact_check": (_I, [_P, _P, _I, _I, _I, _D, _P, _P]),
    "hb_hits_workspace_bytes": (_SZ, [_I64]),
    "hb_hits_count": (_I, [_P, _P, _I64, _I64, _P, _P, _SZ, _P]),
    "hb_ordered_workspace_bytes": (_SZ, [_I64, _I, _I, _I]),
    "hb_accumulate_ordered": (_I, [_P, _P, _I64, _P, _I64, _I64, _I, _I64, _I64, _P, _P, _P,
                                   _I, _I, _I, _P, _P, _P, _SZ, _P]),
    "hb_hits_sorted_workspace_bytes": (_SZ, [_I64]),
    "hb_hits_fill_sorted": (_I, [_P, _P, _I64, _P, _I64, _I, _I64, _I64, _I, _I, _P, _P, _P,
                                 _P, _SZ, _P]),
    "hb_ordered_fold_workspace_bytes": (_SZ, [_I64, _I64]),
    "hb_ordered_fold": (_I, [_P, _P, _I64, _I, _I, _I64, _I64, _P, _P, _P, _I, _P, _P, _SZ,
                             _P]),
}

class HbTiles(ctypes.Structure):
    """Mirror of ``hb_tiles`` (include/histobundle_b200.h)."""

    _fields_ = [("tile", ctypes.c_int), ("halo", ctypes.c_int), ("ntx", ctypes.c_int),
                ("nty", ctypes.c_int), ("nbins", ctypes.c_int), ("ntiles", ctypes.c_int),
                ("off", ctypes.c_void_p), ("cap", ctypes.c_void_p), ("fill", ctypes.c_void_p),
                ("work", ctypes.c_void_p), ("rec", ctypes.c_void_p),
                ("rec_capacity", ctypes.c_int64), ("mode", ctypes.c_int),
                ("tab", ctypes.c_void_p)]


_lib = None


def load_library(path: str | None = None):
    """dlopen the library and bind every declared symbol (no device needed).
    ``HB_B200_LIB`` points tools at a tuning variant built by ``build(out=...)``."""
    path = path or os.environ.get("HB_B200_LIB") or LIB_PATH
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load_library()


def call(name: str, *args) -> None:
    """Invoke an hb_* entry point and raise NativeError on a non-zero status."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().hb_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")
