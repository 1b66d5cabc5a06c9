"""Bundled-polyline export / import (reference ``io.py:136-171``), in bulk.

``export_polylines(result, sink)`` writes exactly the reference's text:

    # histobundle polylines v1
    # edges <E>
    <edge_index> <bin> <weight:.9g> <n> <x0:.9g> <y0:.9g> ... (one line per edge)

but formats the numbers natively (``csrc_host/hb_io.cpp``: ``std::to_chars``
with 9 significant digits, identical to ``format(x, ".9g")``), in parallel
over edge ranges, straight into the sink's file descriptor when it has one.
``read_polylines(source)`` parses an export back into ``PolylineRecord``s with
a native two-pass parser; inputs using spellings only Python accepts (``+1``,
``1_000``, ``Infinity``) go through a Python restatement of the reference
loop, so errors carry the reference's messages.
"""

from __future__ import annotations

import ctypes
import io as _stdio
import os
from dataclasses import dataclass
from typing import Iterable, TextIO

import numpy as np

from . import _native

__all__ = ["GraphFormatError", "PolylineRecord", "export_polylines", "read_polylines"]

_HEADER = "# histobundle polylines v1"
_CHUNK_BYTES = 64 << 20


class GraphFormatError(ValueError):
    """Raised for malformed input (reference ``io.py:31-32``)."""


@dataclass
class PolylineRecord:
    """One parsed line of a polyline export (reference ``io.py:126-133``)."""

    edge_index: int
    bin: int
    weight: float
    points: np.ndarray


_lib = None


def _io_lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_native.HOST_IO_LIB):
            _native.build_host_io()
        L = ctypes.CDLL(_native.HOST_IO_LIB)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.hb_io_format.argtypes = [P, P, P, P, P, I64, I64, P, I64, P]
        L.hb_io_format.restype = I64
        L.hb_io_export_fd.argtypes = [I, P, P, P, P, P, I64, I]
        L.hb_io_export_fd.restype = I
        L.hb_io_parse.argtypes = [P, I64, I, P, P, P, P, P, P, P, P, P, P]
        L.hb_io_parse.restype = I
        _lib = L
    return _lib


def _p(a) -> ctypes.c_void_p | None:
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _packed(result):
    """(world (N,2) f64, starts (E+1) i64, edge index or None) of a result."""
    se = result.sampled_edges
    world = getattr(se, "world", None)
    starts = getattr(se, "starts", None)
    if world is not None and starts is not None:  # PackedPolylines: edge k is graph edge k
        return (np.ascontiguousarray(world, dtype=np.float64),
                np.ascontiguousarray(starts, dtype=np.int64), None)
    pts = [np.asarray(s.points, dtype=np.float64).reshape(-1, 2) for s in se]
    starts = np.zeros(len(pts) + 1, dtype=np.int64)
    np.cumsum([len(p) for p in pts], out=starts[1:])
    world = np.concatenate(pts) if pts else np.zeros((0, 2))
    index = np.array([s.edge_index for s in se], dtype=np.int64)
    return np.ascontiguousarray(world), starts, index


def _sink_fd(sink) -> int | None:
    try:
        fd = sink.fileno()
    except (AttributeError, OSError, _stdio.UnsupportedOperation):
        return None
    return fd if isinstance(fd, int) and fd >= 0 else None


def export_polylines(result, sink: TextIO) -> None:
    """Write one record per edge: index, bin, weight, and sample points
    (reference ``io.py:136-145``; same bytes)."""
    graph = result.graph
    world, starts, index = _packed(result)
    n_edges = starts.size - 1
    bins = np.ascontiguousarray(graph.bins, dtype=np.int64)
    weights = np.ascontiguousarray(graph.weights, dtype=np.float64)
    L = _io_lib()
    fd = _sink_fd(sink)
    if fd is not None:
        sink.flush()
        rc = L.hb_io_export_fd(fd, _p(world), _p(starts), _p(bins), _p(weights), _p(index),
                               n_edges, max(1, min(32, os.cpu_count() or 1)))
        if rc:
            raise OSError(-rc, os.strerror(-rc))
        return
    sink.write(_HEADER + "\n")
    sink.write(f"# edges {n_edges}\n")
    buf = ctypes.create_string_buffer(_CHUNK_BYTES)
    used = ctypes.c_int64(0)
    e = 0
    while e < n_edges:
        done = L.hb_io_format(_p(world), _p(starts), _p(bins), _p(weights), _p(index), e,
                              n_edges, buf, _CHUNK_BYTES, ctypes.byref(used))
        if done == 0:  # a single record larger than the chunk
            big = ctypes.create_string_buffer(64 * int(starts[e + 1] - starts[e]) + 4096)
            done = L.hb_io_format(_p(world), _p(starts), _p(bins), _p(weights), _p(index), e,
                                  e + 1, big, len(big), ctypes.byref(used))
            sink.write(big.raw[:used.value].decode("ascii"))
        else:
            sink.write(buf.raw[:used.value].decode("ascii"))
        e += done


def _read_python(lines: Iterable[str]) -> list[PolylineRecord]:
    """The reference loop (io.py:148-171), for inputs the native parser defers."""
    records = []
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        try:
            edge_index = int(parts[0])
            bin_ = int(parts[1])
            weight = float(parts[2])
            n = int(parts[3])
            coords = np.array(parts[4:], dtype=np.float64)
        except (ValueError, IndexError):
            raise GraphFormatError(f"polyline line {lineno}: malformed record") from None
        if coords.size != 2 * n:
            raise GraphFormatError(
                f"polyline line {lineno}: expected {2 * n} coordinates, got {coords.size}")
        records.append(PolylineRecord(edge_index, bin_, weight, coords.reshape(n, 2)))
    return records


def read_polylines(source: Iterable[str]) -> list[PolylineRecord]:
    """Parse a polyline export back into records (reference ``io.py:148-171``)."""
    if hasattr(source, "read"):
        text = source.read()
    else:
        text = "".join(l if l.endswith("\n") else l + "\n" for l in source)
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    L = _io_lib()
    nrec, ncoord = ctypes.c_int64(0), ctypes.c_int64(0)
    err_line, err_a, err_b = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    rc = L.hb_io_parse(data, len(data), 0, ctypes.byref(nrec), ctypes.byref(ncoord), None, None,
                       None, None, None, ctypes.byref(err_line), ctypes.byref(err_a),
                       ctypes.byref(err_b))
    if rc == 1:
        return _read_python(data.decode("utf-8").split("\n"))
    if rc == -1:
        raise GraphFormatError(f"polyline line {err_line.value}: malformed record")
    if rc == -2:
        raise GraphFormatError(f"polyline line {err_line.value}: expected {err_a.value} "
                               f"coordinates, got {err_b.value}")
    n = nrec.value
    edge_index = np.empty(n, dtype=np.int64)
    bins = np.empty(n, dtype=np.int64)
    weights = np.empty(n, dtype=np.float64)
    starts = np.empty(n + 1, dtype=np.int64)
    coords = np.empty(ncoord.value, dtype=np.float64)
    rc = L.hb_io_parse(data, len(data), 1, ctypes.byref(nrec), ctypes.byref(ncoord),
                       _p(edge_index), _p(bins), _p(weights), _p(starts), _p(coords),
                       ctypes.byref(err_line), ctypes.byref(err_a), ctypes.byref(err_b))
    if rc != 0:  # pragma: no cover (the first pass saw the same bytes)
        raise GraphFormatError(f"polyline line {err_line.value}: malformed record")
    pts = coords.reshape(-1, 2)
    return [PolylineRecord(int(edge_index[k]), int(bins[k]), float(weights[k]),
                           pts[starts[k]:starts[k + 1]]) for k in range(n)]
