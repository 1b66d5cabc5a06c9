"""Device-resident bundling engine: buffers, the per-iteration kernel
sequence, metrics and timing.

One engine owns one shard of edges on one GPU (the whole graph at N=1). Per
iteration ``i`` (``bundler.py:351-376``) it launches, on the current CUDA
stream:

  i > 0: hb_scan_counts -> (1 host read: N_i)
         -> hb_resample_emit (+ fused splat into the int32 group counts)
  i = 0: hb_splat
  [world > 1: all-reduce of the int32 counts over NCCL]
  hb_smooth (mix + 3 exact box passes + layer peaks)
  hb_grad_field (packed rho/dX/dY), hb_advect_laplacian: advect + Laplacian
         in one streaming pass (+ per-block metric partials), then
         hb_resample_count for the NEXT iteration's resample
  hb_reduce_f64, hb_used_cells

Host reads per iteration: the new point total (needed to size the emit
buffer). Metrics stay on the device until the run ends unless an
``on_iteration`` callback asks for them each iteration.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .model import BundleConfig

__all__ = ["BundleEngine", "box_widths", "sample_counts", "IterationRecord", "WeightPlan",
           "weight_plan", "ordered_plan", "CapacityExceeded", "InexactHistogram"]

MIN_STEP = 0.25  # bundler.py:48


def box_widths(sigma: float, passes: int) -> list[int]:
    """Odd box widths for the n-box Gaussian approximation (raster.py:172-193)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    if passes < 1:
        raise ValueError("passes must be >= 1")
    ideal = math.sqrt(12.0 * sigma * sigma / passes + 1.0)
    lo = int(math.floor(ideal))
    if lo % 2 == 0:
        lo -= 1
    lo = max(lo, 1)
    m_ideal = ((12.0 * sigma * sigma - passes * lo * lo - 4.0 * passes * lo
                - 3.0 * passes) / (-4.0 * lo - 4.0))
    m = min(max(int(round(m_ideal)), 0), passes)
    return [lo] * m + [lo + 2] * (passes - m)


def sample_counts(src: np.ndarray, dst: np.ndarray, delta: float) -> np.ndarray:
    """Initial point counts max(ceil(|d|/delta), 1) + 1 (bundler.py:82-83),
    with the reference's numpy norm so the rounding is identical."""
    seg = np.linalg.norm(dst - src, axis=1)
    return np.maximum(np.ceil(seg / delta).astype(np.int64), 1) + 1


def smooth_counts_ok(radius: int, limit: float) -> bool:
    """Whether hb_smooth_counts takes this first pass (mirrors its checks in
    hb_field.cu: a shared-memory tile with >= 8 rows fits 220 KB, and the
    int32 vertical window sums (2r+1) x limit cannot overflow)."""
    if radius <= 0 or (2 * radius + 1) * limit >= 2 ** 31 - 1:
        return False
    pitch = (128 + 2 * radius) | 1
    return (4 * ((8 + 2 * radius) * pitch + 8 * pitch) <= 220 * 1024
            or radius > 32)  # (the separable pair: 4 padded rows of <= 8192 cells)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


# host<->device traffic of the public API, counted from the copied tensors
IO_BYTES = {"h2d": 0, "d2h": 0}


def upload(a: np.ndarray, dev) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    IO_BYTES["h2d"] += t.numel() * t.element_size()
    return t.to(dev)


def download(t: torch.Tensor) -> np.ndarray:
    IO_BYTES["d2h"] += t.numel() * t.element_size()
    return t.cpu().numpy()


def download_pinned(t: torch.Tensor) -> np.ndarray:
    """Device -> host into page-locked memory, returned as a numpy view.

    Copying a multi-GB result into fresh pageable memory is dominated by
    first-touch page faults (~2 s for config 4's 4.3 GB of polylines); a
    pinned destination takes the DMA path (~60 GB/s), and torch's pinned
    host allocator caches the block when the caller drops the result, so
    repeated bundle() calls reuse it instead of calling cudaHostAlloc.
    """
    IO_BYTES["d2h"] += t.numel() * t.element_size()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)
    return host.numpy()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class CapacityExceeded(RuntimeError):
    """A sync-free resample outgrew the point buffers (retried synchronously)."""

    def __init__(self, needed: int):
        super().__init__(f"resample needs {needed} points")
        self.needed = needed


@dataclass
class IterationRecord:
    iteration: int
    bandwidth: float
    n_points: int          # points entering splat/advect (this shard)
    n_edges: int
    moved_points: int = 0
    disp: float = 0.0
    used_cells: int = 0
    seconds: float = 0.0


class InexactHistogram(RuntimeError):
    """The integer fast path stopped equalling the reference's float32 sums
    (a cell's layer sum outgrew 2^24 quanta); the run is redone ordered."""


@dataclass
class WeightPlan:
    """How edge weights reach the histogram.

    The reference adds ``layer_w[e, l] = fl32(w_e) * M[l, b_e]`` into float32
    buffers one hit at a time (``bundler.py:345-346``, ``raster.py:70-94``).

    * ``"unit"`` / ``"int"``: every layer weight is an exact float32 multiple
      of ``quantum``, so while each cell's partial sums stay below
      ``limit = 2^24 * quantum`` the float32 sums are exact and order-free:
      per-group int32 counts mixed once (``hb_smooth``) equal them bit for bit.
      ``hb_exact_check`` guards the limit every iteration.
    * ``"ordered"``: anything else (repulsive -alpha/(B-1) matrices, fractional
      weights): the reference's own summation order, ``hb_accumulate_ordered``.

    Decided once from the WHOLE graph, so every rank of a sharded run takes
    the same path (``slice`` gives a rank its edges' arrays).
    """

    kind: str                      # "unit" | "int" | "ordered"
    int_w: np.ndarray | None = None
    f32_w: np.ndarray | None = None
    quantum: float = 1.0
    abs_matrix: np.ndarray | None = None   # (B,B) float64 |M|; None = identity

    @property
    def limit(self) -> float:
        return float(2 ** 24) * self.quantum

    def slice(self, lo: int, hi: int) -> "WeightPlan":
        return WeightPlan(self.kind,
                          None if self.int_w is None else self.int_w[lo:hi],
                          None if self.f32_w is None else self.f32_w[lo:hi],
                          self.quantum, self.abs_matrix)



def ordered_plan(weights: np.ndarray, unit: bool | None = None) -> WeightPlan:
    """The reference's summation order whatever the weights."""
    w32 = np.asarray(weights, dtype=np.float32)
    if unit is None:
        unit = bool(np.all(w32 == 1.0))
    return WeightPlan("ordered", f32_w=None if unit else w32)


def _lowest_bit(x: np.ndarray) -> float:
    """Largest power of two dividing every non-zero entry of ``x`` (floats)."""
    x = np.abs(np.asarray(x, dtype=np.float64))
    x = x[x > 0]
    if x.size == 0:
        return 1.0
    m, e = np.frexp(x)                      # x = m * 2^e, m in [0.5, 1)
    mi = (m * 2.0 ** 53).astype(np.int64)   # exact integer significand
    low = mi & -mi                          # lowest set bit of the significand
    tz = np.log2(low.astype(np.float64)).astype(np.int64)
    return float(2.0 ** int((e - 53 + tz).min()))


def _sig_bits(x: np.ndarray) -> int:
    """Most significand bits any non-zero entry of ``x`` needs."""
    x = np.abs(np.asarray(x, dtype=np.float64))
    x = x[x > 0]
    if x.size == 0:
        return 1
    m, _ = np.frexp(x)
    mi = (m * 2.0 ** 53).astype(np.int64)
    low = mi & -mi
    return int((53 - np.log2(low.astype(np.float64)).astype(np.int64)).max())


def weight_plan(weights: np.ndarray, matrix: np.ndarray | None = None,
                n_points: int = 0) -> WeightPlan:
    """Pick the histogram path for the whole graph (see :class:`WeightPlan`).

    ``n_points`` (initial sample points) bounds the hits per cell for the
    int32 overflow check of non-unit integer weights (the buffers hold at
    most ~4x that many points)."""
    w = np.asarray(weights)
    mat = (np.eye(1, dtype=np.float32) if matrix is None
           else np.ascontiguousarray(matrix, dtype=np.float32))
    nb = mat.shape[0]
    identity = np.array_equal(mat, np.eye(nb, dtype=np.float32))
    absm = None if identity else np.abs(mat.astype(np.float64))
    # all exactly 1.0 -> fl32 all 1.0 (then finite and nonnegative too): the
    # common case needs no float32 copy
    unit = bool(np.all(w == 1.0))
    w32 = w if unit else np.asarray(w, dtype=np.float32)  # (no copy when already float32)
    if not unit:
        unit = bool(np.all(w32 == 1.0))  # (weights that round to 1.0 in float32)
    if not unit and w32.size and (not np.all(np.isfinite(w32)) or np.any(w32 < 0)):
        return ordered_plan(w32, unit)
    if not unit and not (np.all(np.floor(w32) == w32) and np.all(w32 < 2 ** 24)):
        return ordered_plan(w32, unit)
    wmax = float(w32.max()) if w32.size else 1.0
    # every product fl32(w * M[l,b]) exact: the weights' bit span plus the
    # matrix entries' significand bits fit float32's 24
    qw = 1.0 if unit else _lowest_bit(w32)
    span_w = 1 if unit else int(math.floor(math.log2(max(wmax, qw) / qw))) + 1
    if span_w + _sig_bits(mat) > 24:
        return ordered_plan(w32, unit)
    if not unit and wmax * (4.0 * n_points + (1 << 20)) >= 2.0 ** 31:
        return ordered_plan(w32, unit)  # int32 counts could wrap
    q = qw * _lowest_bit(mat)
    if unit:
        return WeightPlan("unit", quantum=q, abs_matrix=absm)
    return WeightPlan("int", int_w=w32.astype(np.int32), quantum=q, abs_matrix=absm)


class BundleEngine:
    """Runs the bundling iterations for one edge shard on one CUDA device.

    ``src``/``dst`` are the shard's grid-space endpoints ((E,2) float64,
    ``transform.world_to_grid`` of the node positions), ``groups`` its bins.
    ``reduce_hist`` (optional) is called with the int32/float32 group
    histogram tensor after the splat; the distributed driver passes an
    all-reduce here.  ``reduce_flags`` (optional) takes a small int64
    tensor and returns its element-wise maximum over ranks, so every rank
    takes the same decision on the run's status (bounds, capacity retry,
    exactness) and raises together.  ``workers`` is the reference's
    partition count (``_parallel.partition_ranges``): it only changes results
    on the ordered path, exactly as it does in the reference.  ``shard``
    (multi-rank runs) describes this engine's place in the whole graph:
    ``rank, world, group, edge_base, edges_total`` and the global
    ``weights`` / ``bins`` arrays the ordered path indexes by global edge.
    """

    def __init__(self, src: np.ndarray, dst: np.ndarray, groups: np.ndarray,
                 weights: WeightPlan, matrix: np.ndarray, shape: tuple[int, int],
                 cfg: BundleConfig, *, fixed_step: bool = False,
                 offset_disp: np.ndarray | None = None, device=None,
                 reduce_hist=None, capacity_factor: float = 2.0,
                 starts: torch.Tensor | None = None, workers: int = 1,
                 reduce_flags=None, sync_free: bool = True, shard: dict | None = None):
        N.lib()  # fail loudly if the native library is missing
        if not torch.cuda.is_available():
            raise N.NativeError("paper_1504_02687_b200 needs a CUDA device (sm_100a); "
                                "there is no CPU path")
        self.dev = torch.device(device if device is not None else "cuda")
        self.cfg = cfg
        self.fixed_step = bool(fixed_step)
        self.reduce_hist = reduce_hist
        self.reduce_flags = reduce_flags
        self.nv, self.nu = int(shape[0]), int(shape[1])
        self.matrix = np.ascontiguousarray(matrix, dtype=np.float32)
        self.nbins = int(self.matrix.shape[0])
        self.n_edges = int(src.shape[0])
        self.radii = torch.tensor([(w - 1) // 2 for w in
                                   box_widths(cfg.sigma, cfg.smoothing_passes)],
                                  dtype=torch.int32)
        self.delta = float(cfg.delta)
        E, B = self.n_edges, self.nbins
        dev = self.dev

        on_device = isinstance(src, torch.Tensor)
        if on_device:
            # src/dst/starts were prepared on the device (hb_edge_prepare)
            self.n_pts = int(download(starts[E:E + 1])[0]) if E else 0
        else:
            counts = sample_counts(src, dst, self.delta)
            starts_h = np.zeros(E + 1, dtype=np.int64)
            np.cumsum(counts, out=starts_h[1:])
            self.n_pts = int(starts_h[-1])
        self.cap = max(int(self.n_pts * capacity_factor), 1024)
        self.pts = torch.empty((self.cap, 2), dtype=torch.float64, device=dev)
        self.alt = torch.empty((self.cap, 2), dtype=torch.float64, device=dev)
        self.pos = torch.empty(self.cap, dtype=torch.int32, device=dev)
        self.starts = starts if on_device else upload(starts_h, dev)
        self.starts_alt = torch.empty_like(self.starts)
        self.ecounts = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
        self.groups = upload(np.asarray(groups, dtype=np.int32), dev)
        self.plan = weights
        self.wkind = weights.kind
        self.wint = upload(weights.int_w, dev) if weights.kind == "int" else None
        self.wf32 = (upload(weights.f32_w, dev) if weights.kind == "ordered"
                     and weights.f32_w is not None else None)
        mat_is_identity = np.array_equal(self.matrix, np.eye(B, dtype=np.float32))
        self.mat_dev = None if mat_is_identity else upload(self.matrix, dev)
        self.absm_dev = (None if weights.abs_matrix is None
                         else upload(np.ascontiguousarray(weights.abs_matrix, np.float64), dev))
        # exact first smoothing pass from integer window sums (hb_smooth_counts):
        # H = scale * mix * G with an integer matrix, scale = the matrix quantum
        self.int_mix = None
        self.int_scale = 1.0
        self.smooth_int = (os.environ.get("HB_SMOOTH_INT", "1") != "0"
                           and weights.kind != "ordered")
        if self.smooth_int and not mat_is_identity:
            qm = _lowest_bit(self.matrix)
            mix = self.matrix.astype(np.float64) / qm
            if np.all(np.abs(mix) < 2 ** 31) and np.all(mix == np.round(mix)):
                self.int_mix = upload(mix.astype(np.int32), dev)
                self.int_scale = qm
            else:
                self.smooth_int = False
        self.smooth_int = self.smooth_int and smooth_counts_ok(
            int(self.radii[0]), weights.limit / self.int_scale)
        self.shard = shard
        e_total = E if shard is None else int(shard["edges_total"])
        self.nparts = max(1, min(int(workers), e_total)) if e_total else 1
        self.ord_w32 = self.ord_groups = None  # global arrays (sharded ordered path)
        if shard is not None and weights.kind == "ordered":
            self._upload_global_arrays()
        self.hoff = None         # ordered path: hit offsets + workspaces
        self.hits_ws = None
        self.ord_ws = None
        hdtype = torch.float32 if self.wkind == "ordered" else torch.int32
        self.hist = torch.empty((B, self.nv, self.nu), dtype=hdtype, device=dev)
        self.field = torch.empty((B, self.nv, self.nu), dtype=torch.float32, device=dev)
        # quad advection field (hb_grad_field), 48 B per cell, whenever memory
        # allows: it beats gathering rho even when it does not fit L2 (config
        # 5's 805 MB field cut its advect from 40.4 to 33.4 ms per iteration)
        quad_bytes = N.lib().hb_grad_field_bytes(B, self.nv, self.nu)
        quad_limit = min(int(float(os.environ.get("HB_QUAD_LIMIT_MB", "4096")) * (1 << 20)),
                         torch.cuda.mem_get_info(dev)[0] // 8)
        self.gfield = (torch.empty(quad_bytes // 4, dtype=torch.float32, device=dev)
                       if quad_bytes <= quad_limit else None)
        # resample count as its own launch after the advect pass (measured
        # faster than fusing it: the fused build's register footprint halves
        # the advect's occupancy)
        self.split_count = True
        # advection as a flat point stream (hb_advect_points) followed by the
        # Laplacian fused with the resample count; the per-edge fused pass
        # (hb_advect_laplacian with h >= 0) remains for very large fields
        self.flat_advect = (B * self.nv * self.nu < (1 << 31)
                            and os.environ.get("HB_FLAT_ADVECT", "1") != "0")
        self.peak = torch.empty(B, dtype=torch.float32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        sws = N.lib().hb_smooth_workspace_bytes(B, self.nv, self.nu)
        self.smooth_ws = torch.empty(sws, dtype=torch.uint8, device=dev)
        scw = N.lib().hb_scan_workspace_bytes(max(E, 1))
        self.scan_ws = torch.empty(scw, dtype=torch.uint8, device=dev)
        # Aggregated splatting (hb_splat.cu).  Resampled segments are at most
        # 1.5*delta long (delta before the first resample), so their cell
        # delta is at most floor(1.5*delta) + 1 per axis; longer ones simply
        # take the direct path.  Preferred: the segment-key table (one atomic
        # per segment, bundled duplicates collapse); else tile records.
        self.tiles = None
        self.tile_mode = -1
        # HB_SPLAT_MODE=auto|table|tiles|direct forces a path (tests cover all three)
        smode = os.environ.get("HB_SPLAT_MODE", "auto")
        if self.wkind != "ordered" and smode != "direct":
            geo = N.HbTiles()
            ent = ctypes.c_int64(0)
            budget = min(8 << 30, torch.cuda.mem_get_info(dev)[0] // 8)
            if (smode != "tiles"
                    and N.lib().hb_segtab_geometry(B, self.nv, self.nu, 1.5 * self.delta,
                                                   ctypes.byref(geo), ctypes.byref(ent)) == 0
                    and ent.value * 4 <= budget):
                self.t_tab = torch.zeros(ent.value, dtype=torch.int32, device=dev)
                self.t_keys = torch.zeros(1, dtype=torch.int64, device=dev)
                geo.tab = self.t_tab.data_ptr()
                self.tiles, self.tile_mode = geo, 1
            elif N.lib().hb_tiles_geometry(B, self.nv, self.nu, 1.5 * self.delta + 2.0,
                                           ctypes.byref(geo)) == 0:
                nt = geo.ntiles
                self.t_off = torch.zeros(nt + 1, dtype=torch.int64, device=dev)
                self.t_cap = torch.zeros(nt, dtype=torch.int32, device=dev)
                self.t_fill = torch.zeros(nt, dtype=torch.int32, device=dev)
                self.t_work = torch.zeros(nt + 2, dtype=torch.int32, device=dev)
                self.t_total = torch.zeros(1, dtype=torch.int64, device=dev)
                self.t_rec = torch.empty(max(int(self.n_pts * 1.5), 4096), dtype=torch.int64,
                                         device=dev)
                geo.off, geo.cap = self.t_off.data_ptr(), self.t_cap.data_ptr()
                geo.fill, geo.work = self.t_fill.data_ptr(), self.t_work.data_ptr()
                geo.rec, geo.rec_capacity = self.t_rec.data_ptr(), self.t_rec.numel()
                geo.mode = 0
                self.tiles, self.tile_mode = geo, 0
                self.tiles_census = N.HbTiles.from_buffer_copy(geo)
                self.tiles_census.rec = None
        # Sync-free iterations: the resample total stays on the device (the
        # kernels read it from `starts`, the emit checks it against the
        # buffer), so no host read separates the iterations.  The buffers get
        # headroom; a run that outgrows them is redone in the synchronous mode.
        self.async_n = (sync_free and self.tile_mode != 0 and self.wkind != "ordered"
                        and os.environ.get("HB_SYNC_FREE", "1") != "0")
        self._n_known = True
        self._init = None
        if self.async_n:
            # headroom for the sync-free resample: the kernels index points in
            # 32 bits (< 2^31) and the buffers must fit the device; without
            # room for 4x growth the run is synchronous instead
            f = float(os.environ.get("HB_ASYNC_CAP_FACTOR", "4"))  # (tests shrink it)
            want = int(f * self.n_pts) + (1 << 20 if f >= 1 else 0)
            free = torch.cuda.mem_get_info(dev)[0]
            extra = max(want - self.cap, 0) * (2 * 16 + 4) * 5 // 4
            if want * 5 // 4 >= (1 << 31) - 1 or extra > free * 0.6:
                self.async_n = False
            else:
                self._ensure_capacity(want)
        self.lap_passes = int(cfg.laplacian_passes)
        # one-pass advect + Laplacian + count (hb_advect_laplacian_count):
        # bit-identical, measured slower (config 4: 9.23 ms vs 5.29 + 2.41 ms)
        self.fused_field = os.environ.get("HB_FUSED_FIELD", "0") == "1"
        self._partials = torch.zeros(int(N.lib().hb_advect_partials()), dtype=torch.float64,
                                     device=dev)
        self.iters = int(cfg.iterations)
        # per-iteration device metrics: moved (u64 as int64), disp, used
        self.m_moved = torch.zeros(self.iters, dtype=torch.int64, device=dev)
        self.m_disp = torch.zeros(self.iters, dtype=torch.float64, device=dev)
        self.m_used = torch.zeros(self.iters, dtype=torch.int64, device=dev)
        self.m_ntot = torch.zeros(self.iters, dtype=torch.int64, device=dev)  # N_i (async)
        self.records: list[IterationRecord] = []
        self._ev: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        # optional per-kernel CUDA-event trace: name -> [(start, end, iteration)]
        self.trace: dict | None = None

        s = stream_ptr()
        srcd = src if on_device else upload(np.asarray(src, dtype=np.float64), dev)
        dstd = dst if on_device else upload(np.asarray(dst, dtype=np.float64), dev)
        N.call("hb_sample_fill", ptr(srcd), ptr(dstd), ptr(self.starts), E,
               ptr(self.pts), s)
        if offset_disp is not None:
            od = upload(offset_disp, dev)
            N.call("hb_offset", ptr(self.pts), ptr(self.starts), E, ptr(od), s)
        # _check_bounds (raster.py:57-67) of the first accumulate.  Later
        # iterations cannot leave the grid: advection clamps moved points to
        # [1, dim-2] and resampling / Laplacian smoothing only form convex
        # combinations, so the kernels' cell checks are a backstop.
        self._raise_if_out_of_bounds()
        self.iteration = 0
        self._tab_on = True       # segment-key table in use for the next emit
        self._tab_segments = 0    # segments the last table pass saw
        self.key_ratio: list[float] = []

    # ------------------------------------------------------------------
    def _ensure_capacity(self, n: int) -> None:
        if n <= self.cap:
            return
        cap = max(int(n * 1.25), self.cap * 3 // 2)
        new_pts = torch.empty((cap, 2), dtype=torch.float64, device=self.dev)
        new_pts[: self.n_pts].copy_(self.pts[: self.n_pts])
        self.pts = new_pts
        self.alt = torch.empty((cap, 2), dtype=torch.float64, device=self.dev)
        new_pos = torch.empty(cap, dtype=torch.int32, device=self.dev)
        new_pos[: self.n_pts].copy_(self.pos[: self.n_pts])
        self.pos = new_pos
        self.cap = cap

    def _k(self, name: str, *args) -> None:
        """Launch one C-ABI entry point, bracketed by events when tracing."""
        if self.trace is None:
            N.call(name, *args)
            return
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        N.call(name, *args)
        b.record()
        self.trace.setdefault(name, []).append((a, b, self.iteration))

    def _emit_groups(self):
        """Group ids for the emit's splat; NULL (= all group 0) for one group,
        which saves a gather per output."""
        return None if self.nbins == 1 else ptr(self.groups)

    def _splat(self, s) -> None:
        """Straight splat of the current points (iteration 0 / float weights);
        with tiles it also takes the per-tile census for the next plan."""
        E, B, nv, nu = self.n_edges, self.nbins, self.nv, self.nu
        if self.wkind == "ordered":
            self._accumulate_ordered(s)
            return
        # Straight initial polylines have no duplicate segments, so the key
        # table would only add its expansion: splat directly.  Tile mode
        # (long segments) bins them too: a census pass sizes the buckets,
        # the binned splat writes records, the flush rasterises them in
        # shared memory (the direct global atomics of ~28-cell segments were
        # L2-atomic-bound: config 5's iteration 0 took 91 ms)
        if self.tile_mode == 0 and os.environ.get("HB_ITER0_BINNED", "1") != "0":
            self.t_fill.zero_()
            census = N.HbTiles.from_buffer_copy(self.tiles_census)
            census.mode = 2
            self._k("hb_splat", ptr(self.pts), ptr(self.starts), E, self.n_pts,
                    ptr(self.groups), ptr(self.wint), ptr(self.hist), B, nv, nu,
                    ptr(self.status), ctypes.byref(census), s)
            self._k("hb_tiles_plan", ctypes.byref(self.tiles), ptr(self.t_total), s)
            self._ensure_records(int(download(self.t_total)[0]))
            self._k("hb_splat", ptr(self.pts), ptr(self.starts), E, self.n_pts,
                    ptr(self.groups), ptr(self.wint), ptr(self.hist), B, nv, nu,
                    ptr(self.status), ctypes.byref(self.tiles), s)
            self._k("hb_tiles_flush", ctypes.byref(self.tiles), ptr(self.hist), nv, nu, s)
            return
        sink = None
        if self.tile_mode == 0:
            self.t_fill.zero_()
            sink = ctypes.byref(self.tiles_census)
        self._k("hb_splat", ptr(self.pts), ptr(self.starts), E, self.n_pts, ptr(self.groups),
                ptr(self.wint), ptr(self.hist), B, nv, nu, ptr(self.status), sink, s)

    def _upload_global_arrays(self) -> None:
        sh = self.shard
        w32 = np.asarray(sh["weights"]).astype(np.float32)
        self.ord_w32 = None if np.all(w32 == 1.0) else upload(w32, self.dev)
        self.ord_groups = (None if self.nbins == 1 else
                           upload(np.asarray(sh["bins"], dtype=np.int32), self.dev))

    def _ws(self, attr: str, nbytes: int) -> torch.Tensor:
        t = getattr(self, attr, None)
        if t is None or t.numel() < nbytes:
            setattr(self, attr, None)
            t = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.dev)
            setattr(self, attr, t)
        return t

    def _accumulate_ordered(self, s) -> None:
        """The reference's float32 histogram in its own summation order
        (raster.py:70-94): hit offsets, one host read of the hit total to
        size the workspace, then records -> stable sort by cell -> fold."""
        E, B, nv, nu = self.n_edges, self.nbins, self.nv, self.nu
        n = self.n_pts
        if self.hoff is None or self.hoff.numel() < n + 1:
            self.hoff = torch.empty(int((n + 1) * 1.25) + 1024, dtype=torch.int64, device=self.dev)
        self.hits_ws = self._ws("hits_ws", int(N.lib().hb_hits_workspace_bytes(n)))
        self._k("hb_hits_count", ptr(self.pts), ptr(self.starts), E, n, ptr(self.hoff),
                ptr(self.hits_ws), self.hits_ws.numel(), s)
        n_hits = int(download(self.hoff[n:n + 1])[0])
        if self.shard is not None:
            self._accumulate_ordered_sharded(n, n_hits, s)
            return
        ob = int(N.lib().hb_ordered_workspace_bytes(n_hits, nv, nu, self.nparts))
        if self.ord_ws is None or self.ord_ws.numel() < ob:
            self.ord_ws = None
            self.ord_ws = torch.empty(int(ob * 1.25) + 4096, dtype=torch.uint8, device=self.dev)
        self._k("hb_accumulate_ordered", ptr(self.pts), ptr(self.starts), E, ptr(self.hoff), n,
                n_hits, self.nparts, 0, E, ptr(self.wf32), self._emit_groups(),
                ptr(self.mat_dev), B, nv, nu, ptr(self.hist), ptr(self.status),
                ptr(self.ord_ws), self.ord_ws.numel(), s)

    def _accumulate_ordered_sharded(self, n: int, n_hits: int, s) -> None:
        """Ordered histogram of an edge-sharded run: every rank sorts its own
        hit records by cell, the records travel to the rank owning their
        cell slab (all-to-all; rank order = global edge order, so each
        cell's hits arrive in the reference's order), each rank folds its
        slab and the slabs are all-gathered -- identical to one GPU."""
        from . import dist as D
        sh = self.shard
        rank, world, group = sh["rank"], sh["world"], sh["group"]
        E, B, nv, nu, P = self.n_edges, self.nbins, self.nv, self.nu, self.nparts
        plane = nv * nu
        keys = torch.empty(max(n_hits, 1), dtype=torch.int32, device=self.dev)
        vals = torch.empty(max(n_hits, 1), dtype=torch.int32, device=self.dev)
        ws = self._ws("ord_ws", int(N.lib().hb_hits_sorted_workspace_bytes(n_hits)))
        self._k("hb_hits_fill_sorted", ptr(self.pts), ptr(self.starts), E, ptr(self.hoff),
                n_hits, P, int(sh["edge_base"]), int(sh["edges_total"]), nv, nu, ptr(keys),
                ptr(vals), ptr(self.status), ptr(ws), ws.numel(), s)
        k64 = keys[:n_hits].to(torch.int64) & 0xFFFFFFFF  # keys are uint32
        bounds = torch.tensor([(r * plane // world) * P for r in range(world + 1)],
                              dtype=torch.int64, device=self.dev)
        cuts = torch.searchsorted(k64, bounds).cpu().tolist()  # out-of-grid keys sort last
        counts = [cuts[r + 1] - cuts[r] for r in range(world)]
        rk = D.all_to_all_var(keys[cuts[0]:cuts[-1]], counts, group)
        rv = D.all_to_all_var(vals[cuts[0]:cuts[-1]], counts, group)
        c0, c1 = rank * plane // world, (rank + 1) * plane // world
        m = int(rk.shape[0])
        slab = torch.empty((B, max(c1 - c0, 1)), dtype=torch.float32, device=self.dev)
        fws = self._ws("fold_ws", int(N.lib().hb_ordered_fold_workspace_bytes(m, max(c1 - c0, 1))))
        if c1 > c0:
            self._k("hb_ordered_fold", ptr(rk), ptr(rv), m, 1, P, c0, c1 - c0,
                    ptr(self.ord_w32), ptr(self.ord_groups), ptr(self.mat_dev), B, ptr(slab),
                    ptr(fws), fws.numel(), s)
        sizes = [(r + 1) * plane // world - r * plane // world for r in range(world)]
        full = D.all_gather_columns(slab[:, : c1 - c0], sizes, group)
        self.hist.view(B, plane).copy_(full)

    def _ensure_records(self, n: int) -> None:
        if n <= self.t_rec.numel():
            return
        self.t_rec = torch.empty(max(n, self.t_rec.numel() * 5 // 4), dtype=torch.int64,
                                 device=self.dev)
        self.tiles.rec = self.t_rec.data_ptr()
        self.tiles.rec_capacity = self.t_rec.numel()

    def step(self) -> IterationRecord:
        """One bundling iteration (bundler.py:351-376) on the device."""
        self.step_splat()
        if self.reduce_hist is not None and self.wkind != "ordered":
            # (a sharded ordered histogram is already global: slabs all-gathered)
            self.reduce_hist(self.hist)
        return self.step_field()

    def step_splat(self) -> None:
        """First half of an iteration: resample + histogram of this shard.

        Between the two halves ``self.hist`` holds this shard's int32 group
        counts; a multi-GPU run sums it over ranks (``reduce_hist``), and a
        single-GPU shard emulation may sum several engines' histograms here."""
        i = self.iteration
        if i >= self.iters:
            raise RuntimeError("all iterations done")
        s = stream_ptr()
        E, B, nv, nu = self.n_edges, self.nbins, self.nv, self.nu
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        self._ev_open = ev0
        self.hist.zero_()
        if i > 0:
            # resample (bundler.py:353-354): the counts/codes came out of the
            # previous iteration's fused advect pass; scan, size, then emit
            # fused with the splat (:355-356)
            fused = self.wkind != "ordered"
            tiles = None
            if fused and self.tile_mode == 0:
                self._k("hb_tiles_plan", ctypes.byref(self.tiles), ptr(self.t_total), s)
            self._k("hb_scan_counts", ptr(self.ecounts), E, ptr(self.starts_alt),
                    ptr(self.scan_ws), self.scan_ws.numel(), s)
            if self.async_n:
                self._resample_async(i, s)
                return
            n_new = int(download(self.starts_alt[E:E + 1])[0]) if E else 0
            self._ensure_capacity(n_new)
            if fused and self.tile_mode == 0:
                self._ensure_records(int(download(self.t_total)[0]))
            if fused and self.tile_mode == 1 and self._tab_on:
                # keys the last table pass produced vs segments it saw: the
                # table only pays off once bundles make segments repeat
                prev = int(download(self.t_keys)[0])
                if self._tab_segments:
                    self.key_ratio.append(prev / self._tab_segments)
                    self._tab_on = prev <= 0.5 * self._tab_segments
                self.t_keys.zero_()
            elif fused and self.tile_mode == 1:
                self._tab_on = True  # re-probe after one direct iteration
                self._tab_segments = 0
            use_tab = fused and self.tiles is not None and (self.tile_mode == 0 or self._tab_on)
            if use_tab:
                tiles = ctypes.byref(self.tiles)
                self._tab_segments = n_new - E
            self._k("hb_resample_emit", ptr(self.pts), ptr(self.starts), E, self.n_pts,
                    ptr(self.pos), ptr(self.starts_alt), ptr(self.alt), self._emit_groups(),
                    ptr(self.wint), ptr(self.hist) if fused else None, nv, nu,
                    ptr(self.status), tiles, s)
            if self.tile_mode == 0 and tiles is not None:
                self._k("hb_tiles_flush", tiles, ptr(self.hist), nv, nu, s)
            elif self.tile_mode == 1 and tiles is not None:
                self._k("hb_segtab_expand", tiles, ptr(self.hist), nv, nu, ptr(self.t_keys), s)
            self.pts, self.alt = self.alt, self.pts
            self.starts, self.starts_alt = self.starts_alt, self.starts
            self.n_pts = n_new
            if not fused:
                self._splat(s)
        else:
            self._splat(s)

    def _resample_async(self, i: int, s) -> None:
        """Emit + splat with the new total left on the device."""
        E, nv, nu = self.n_edges, self.nv, self.nu
        tiles = ctypes.byref(self.tiles) if self.tile_mode == 1 else None
        self._k("hb_resample_emit_cap", ptr(self.pts), ptr(self.starts), E, self.n_pts,
                ptr(self.pos), ptr(self.starts_alt), ptr(self.alt), self.cap, self._emit_groups(),
                ptr(self.wint), ptr(self.hist), nv, nu, ptr(self.status), tiles, s)
        # N_i on the device; starts clamped into the buffers if it did not fit
        self._k("hb_clamp_starts", ptr(self.starts_alt), E, self.cap,
                self.m_ntot.data_ptr() + 8 * i, s)
        if tiles is not None:
            self._k("hb_segtab_expand", tiles, ptr(self.hist), nv, nu, ptr(self.t_keys), s)
        self.pts, self.alt = self.alt, self.pts
        self.starts, self.starts_alt = self.starts_alt, self.starts
        self.n_pts = self.cap  # kernels read the count from `starts`
        self._n_known = False

    def sync_count(self) -> int:
        """Host copy of the current point count (one device read)."""
        if not self._n_known:
            self.n_pts = int(download(self.starts[self.n_edges:self.n_edges + 1])[0])
            self._n_known = True
        return self.n_pts

    def step_field(self) -> IterationRecord:
        """Second half: smoothing of the (global) histogram, advection,
        Laplacian, next resample count, metrics."""
        i = self.iteration
        cfg = self.cfg
        s = stream_ptr()
        E, B, nv, nu = self.n_edges, self.nbins, self.nv, self.nu
        ev0 = self._ev_open
        self._smooth(s)
        h_i = cfg.lambda_ ** i * cfg.h_max  # bundler.py:360, Python float power
        # advect -> Laplacian (-> next iteration's resample count), in place
        last = i == self.iters - 1
        if self.gfield is not None:
            self._k("hb_grad_field", ptr(self.field), B, nv, nu, ptr(self.gfield), s)
        if self.flat_advect:
            self._field_points(i, h_i, 0, E, last)
            self._k("hb_reduce_f64", ptr(self._partials), self._partials.numel(),
                    self.m_disp.data_ptr() + 8 * i, s)
            self._k("hb_used_cells", ptr(self.field), ptr(self.peak), B, nv, nu, 0.01,
                    self.m_used.data_ptr() + 8 * i, s)
            return self._close_iteration(ev0, h_i)
        fuse = not last and not self.split_count
        self._k("hb_advect_laplacian", ptr(self.pts), ptr(self.pts), ptr(self.starts), E,
                self.n_pts, ptr(self.groups), ptr(self.field), ptr(self.gfield), B, nv, nu,
                float(h_i), float(cfg.epsilon), MIN_STEP, int(self.fixed_step),
                float(cfg.laplacian_factor), self.lap_passes, self.delta,
                ptr(self.ecounts) if fuse else None, ptr(self.pos) if fuse else None,
                self.m_moved.data_ptr() + 8 * i, ptr(self._partials), s)
        if not last and self.split_count:
            self._k("hb_resample_count", ptr(self.pts), ptr(self.starts), E, self.delta,
                    ptr(self.ecounts), ptr(self.pos), s)
        self._k("hb_reduce_f64", ptr(self._partials), self._partials.numel(),
                self.m_disp.data_ptr() + 8 * i, s)
        self._k("hb_used_cells", ptr(self.field), ptr(self.peak), B, nv, nu, 0.01,
                self.m_used.data_ptr() + 8 * i, s)
        return self._close_iteration(ev0, h_i)

    def _field_points(self, i: int, h_i: float, e_lo: int, e_hi: int, last: bool) -> None:
        """Flat advection + Laplacian (+ next resample count) of edges
        [e_lo, e_hi), in place; disp partials left in self._partials."""
        cfg, s = self.cfg, stream_ptr()
        B, nv, nu = self.nbins, self.nv, self.nu
        ne = e_hi - e_lo
        st = self.starts.data_ptr() + 8 * e_lo
        if self.fused_field and self.lap_passes <= 1:
            # advect + Laplacian (+ next resample count) in one pass
            self._k("hb_advect_laplacian_count", ptr(self.pts), st, ne, self.n_pts,
                    self.groups.data_ptr() + 4 * e_lo, ptr(self.field), ptr(self.gfield), B,
                    nv, nu, float(h_i), float(cfg.epsilon), MIN_STEP, int(self.fixed_step),
                    float(cfg.laplacian_factor), self.lap_passes, self.delta,
                    None if last else self.ecounts.data_ptr() + 8 * e_lo,
                    None if last else ptr(self.pos), self.m_moved.data_ptr() + 8 * i,
                    ptr(self._partials), s)
            return
        self._k("hb_advect_points", ptr(self.pts), st, ne, self.n_pts,
                self.groups.data_ptr() + 4 * e_lo, ptr(self.field), ptr(self.gfield), B, nv, nu,
                float(h_i), float(cfg.epsilon), MIN_STEP, int(self.fixed_step),
                self.m_moved.data_ptr() + 8 * i, ptr(self._partials), s)
        if self.lap_passes > 0 or not last:
            # Laplacian sweep(s) fused with the next resample count, in place
            self._k("hb_laplacian_count", ptr(self.pts), ptr(self.pts), st, ne, self.n_pts,
                    float(cfg.laplacian_factor), self.lap_passes, self.delta,
                    None if last else self.ecounts.data_ptr() + 8 * e_lo,
                    None if last else ptr(self.pos), s)

    def run_streamed(self, origin, cell, node_pos: torch.Tensor, sources: torch.Tensor,
                     targets: torch.Tensor, chunks: int = 8):
        """run() + world_points_nodes() + the host copy, with the last
        iteration's advection, Laplacian and grid -> world conversion done
        in edge chunks whose device -> host copies (pinned, side stream)
        overlap the next chunk's kernels.  Returns (host world (N,2) numpy,
        records).  Results are those of run(): points are independent per
        edge (the displacement metric sums in chunk order)."""
        if not self.flat_advect or self.iters < 1 or self.n_edges < chunks:
            self.run()
            return download_pinned(self.world_points_nodes(origin, cell, node_pos, sources,
                                                           targets)), self.records
        if self._retryable() and self._init is None and self.iteration == 0:
            self.keep_initial_state()
        try:
            while self.iteration < self.iters - 1:
                self.step()
            out = self._last_iteration_streamed(origin, cell, node_pos, sources, targets, chunks)
            return out, self.finish_metrics()
        except (CapacityExceeded, InexactHistogram) as ex:
            if self._init is None:
                raise
            self._retry(ex)
            return self.run_streamed(origin, cell, node_pos, sources, targets, chunks)

    def _last_iteration_streamed(self, origin, cell, node_pos, sources, targets, chunks):
        E, B, nv, nu, s = self.n_edges, self.nbins, self.nv, self.nu, stream_ptr()
        self.step_splat()
        i, cfg = self.iteration, self.cfg
        ev0 = self._ev_open
        self._smooth(s)
        if self.gfield is not None:
            self._k("hb_grad_field", ptr(self.field), B, nv, nu, ptr(self.gfield), s)
        h_i = cfg.lambda_ ** i * cfg.h_max
        n = self.sync_count()  # one read: sizes the host buffer
        cuts = [E * k // chunks for k in range(chunks + 1)]
        bounds = download(self.starts[torch.tensor(cuts, device=self.dev)])
        world = torch.empty((n, 2), dtype=torch.float64, device=self.dev)
        host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
        IO_BYTES["d2h"] += n * 16
        disp = torch.zeros(chunks, dtype=torch.float64, device=self.dev)
        copy = torch.cuda.Stream(device=self.dev)
        cur = torch.cuda.current_stream()
        for k in range(chunks):
            e_lo, e_hi = cuts[k], cuts[k + 1]
            self._field_points(i, h_i, e_lo, e_hi, True)
            self._k("hb_reduce_f64", ptr(self._partials), self._partials.numel(),
                    disp.data_ptr() + 8 * k, s)
            self._k("hb_to_world_nodes", ptr(self.pts), self.starts.data_ptr() + 8 * e_lo,
                    e_hi - e_lo, float(origin[0]), float(origin[1]), float(cell), ptr(node_pos),
                    sources.data_ptr() + 8 * e_lo, targets.data_ptr() + 8 * e_lo, ptr(world), s)
            a, b = int(bounds[k]), int(bounds[k + 1])
            done = torch.cuda.Event()
            done.record(cur)
            copy.wait_event(done)
            with torch.cuda.stream(copy):
                host[a:b].copy_(world[a:b], non_blocking=True)
        self._k("hb_reduce_f64", ptr(disp), chunks, self.m_disp.data_ptr() + 8 * i, s)
        self._k("hb_used_cells", ptr(self.field), ptr(self.peak), B, nv, nu, 0.01,
                self.m_used.data_ptr() + 8 * i, s)
        self._close_iteration(ev0, h_i)
        cur.wait_stream(copy)  # the host buffer is complete once the stream is
        world.record_stream(copy)
        return host.numpy()

    def _smooth(self, s) -> None:
        """Exactness guard of the integer path (the global histogram), then
        mix + 3 box passes + layer peaks."""
        B, nv, nu = self.nbins, self.nv, self.nu
        if self.wkind == "ordered":  # layer weights already applied, float32
            self._k("hb_smooth", None, ptr(self.hist), None, B, nv, nu,
                    self.radii.data_ptr(), int(self.radii.numel()), ptr(self.field),
                    ptr(self.smooth_ws), self.smooth_ws.numel(), ptr(self.peak), s)
            return
        if self.smooth_int:
            # exact integer first pass + the guard in the same launch
            self._k("hb_smooth_counts", ptr(self.hist), ptr(self.int_mix), self.int_scale,
                    float(self.plan.limit / self.int_scale), B, nv, nu,
                    self.radii.data_ptr(), int(self.radii.numel()), ptr(self.field),
                    ptr(self.smooth_ws), self.smooth_ws.numel(), ptr(self.peak),
                    ptr(self.status), s)
            return
        self._k("hb_exact_check", ptr(self.hist), ptr(self.absm_dev), B, nv, nu,
                float(self.plan.limit), ptr(self.status), s)
        self._k("hb_smooth", ptr(self.hist), None, ptr(self.mat_dev), B, nv, nu,
                self.radii.data_ptr(), int(self.radii.numel()), ptr(self.field),
                ptr(self.smooth_ws), self.smooth_ws.numel(), ptr(self.peak), s)

    def _close_iteration(self, ev0, h_i: float) -> IterationRecord:
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        self._ev.append((ev0, ev1))
        rec = IterationRecord(self.iteration, h_i, self.n_pts if self._n_known else -1,
                              self.n_edges)
        self.records.append(rec)
        self.iteration += 1
        return rec

    def keep_initial_state(self) -> None:
        """Remember the sampled straight edges so :meth:`reset` can restart
        the run without re-sampling (bench: every step bundles from scratch)."""
        self._init = (self.pts[: self.n_pts].clone(), self.starts.clone(), self.n_pts)

    def reset(self) -> None:
        """Back to iteration 0 on the remembered initial points (device copies
        only, stream-ordered, no host sync)."""
        pts0, starts0, n0 = self._init
        self._cb_seen = -1
        self._ensure_capacity(n0)
        self.pts[:n0].copy_(pts0)
        self.starts.copy_(starts0)
        self.n_pts = n0
        self._n_known = True
        self.iteration = 0
        self._tab_on, self._tab_segments, self.key_ratio = True, 0, []
        self.records = []
        self._ev = []
        self.m_moved.zero_()
        self.m_disp.zero_()
        self.m_used.zero_()
        self.m_ntot.zero_()
        self.status.zero_()

    def _reduce_max(self, vals: list) -> list:
        """Element-wise maximum over ranks (identity on one rank)."""
        if self.reduce_flags is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        return [float(v) for v in self.reduce_flags(t)]

    def _raise_if_out_of_bounds(self) -> None:
        """The reference's bounds check on the current points, with its
        message (raster.py:57-67); the span is taken over all ranks."""
        n = self.sync_count()
        if self.n_edges == 0 or n == 0:
            span = [math.inf, math.inf, -math.inf, -math.inf]
        else:
            scratch = torch.empty(4, dtype=torch.int64, device=self.dev)
            out = torch.empty(4, dtype=torch.float64, device=self.dev)
            N.call("hb_point_span", ptr(self.pts), n, ptr(scratch), ptr(out), stream_ptr())
            span = [float(v) for v in download(out)]
        xmin, ymin, nxmax, nymax = self._reduce_max(
            [-span[0], -span[1], span[2], span[3]])
        xmin, ymin, xmax, ymax = -xmin, -ymin, nxmax, nymax
        if not math.isfinite(xmin):
            return  # no points anywhere
        width, height = self.nu, self.nv
        if xmin <= -0.5 or ymin <= -0.5 or xmax >= width - 0.5 or ymax >= height - 0.5:
            raise ValueError(
                f"sample out of bounds: points span ({xmin:.3f}, {ymin:.3f}) to "
                f"({xmax:.3f}, {ymax:.3f}) on a {width}x{height} grid")

    def _switch_to_ordered(self) -> None:
        """Leave the integer path for the reference's summation order."""
        p = self.plan
        w = None if p.kind == "unit" else p.int_w.astype(np.float32)
        self.plan = WeightPlan("ordered", f32_w=w)
        self.wkind = "ordered"
        self.wint = None
        self.wf32 = None if w is None else upload(w, self.dev)
        self.hist = torch.empty((self.nbins, self.nv, self.nu), dtype=torch.float32,
                                device=self.dev)
        if self.shard is not None:
            self._upload_global_arrays()
        self.tiles, self.tile_mode = None, -1
        self.t_tab = self.t_rec = None
        self.async_n = False

    def finish_metrics(self) -> list[IterationRecord]:
        """Synchronise once and fill moved/disp/used/seconds of all records.

        The status word is agreed over ranks first, so a retry (capacity,
        exactness) or a bounds error happens on every rank together."""
        torch.cuda.current_stream().synchronize()
        st = int(download(self.status)[0])
        oob, cap, inexact = self._reduce_max([st & 1, st & 4, st & 8])
        if oob:
            self._raise_if_out_of_bounds()
            raise ValueError("sample out of bounds: a polyline point left the grid")
        if cap:
            raise CapacityExceeded(int(download(self.m_ntot).max()))
        if inexact:
            raise InexactHistogram(
                "a histogram cell outgrew 2^24 weight quanta: the reference's float32 "
                "sums round there")
        if any(r.n_points < 0 for r in self.records):
            ntot = download(self.m_ntot)
            for r in self.records:
                if r.n_points < 0:
                    r.n_points = int(ntot[r.iteration])
        self.sync_count()
        moved = download(self.m_moved)
        disp = download(self.m_disp)
        used = download(self.m_used)
        for r, (a, b) in zip(self.records, self._ev):
            r.moved_points = int(moved[r.iteration])
            r.disp = float(disp[r.iteration])
            r.used_cells = int(used[r.iteration])
            r.seconds = a.elapsed_time(b) / 1e3
        return self.records

    def _retryable(self) -> bool:
        return self.async_n or self.wkind != "ordered"

    def _retry(self, ex) -> None:
        """Back to iteration 0 for a synchronous (capacity) or ordered
        (exactness) rerun; every rank gets here together."""
        seen = getattr(self, "_cb_seen", -1)
        self.status.zero_()
        if isinstance(ex, CapacityExceeded):
            # stay sync-free with room for what the run needed (the next
            # reset()+run() reuses it); after repeated overflows, or beyond
            # the 32-bit point index, run synchronously instead
            self._cap_retries = getattr(self, "_cap_retries", 0) + 1
            want = int(ex.needed * 1.25) + (1 << 20)
            if self._cap_retries > 2 or want * 5 // 4 >= (1 << 31) - 1:
                self.async_n = False
                want = int(ex.needed * 1.25)
            self.reset()
            self._ensure_capacity(want)
        else:
            self._switch_to_ordered()
            self.reset()
        self._cb_seen = seen

    def run(self, on_iteration=None) -> list[IterationRecord]:
        """All remaining iterations.  ``on_iteration(engine)`` runs after each
        one; after a retry it is called again only for iterations it has not
        seen (the rerun reproduces the earlier ones exactly)."""
        if self._retryable() and self._init is None and self.iteration == 0:
            self.keep_initial_state()  # for the (rare) capacity / exactness retry
        start = self.iteration
        seen = getattr(self, "_cb_seen", -1)
        try:
            while self.iteration < self.iters:
                self.step()
                if on_iteration is not None and self.iteration - 1 > seen:
                    on_iteration(self)
                    seen = self._cb_seen = self.iteration - 1
            return self.finish_metrics()
        except (CapacityExceeded, InexactHistogram) as ex:
            if start != 0 or self._init is None:
                raise
            self._retry(ex)
            return self.run(on_iteration)

    # ------------------------------------------------------------------
    def packed_points(self) -> tuple[torch.Tensor, torch.Tensor]:
        return self.pts[: self.sync_count()], self.starts

    def world_points_nodes(self, origin, cell, node_pos: torch.Tensor, sources: torch.Tensor,
                           targets: torch.Tensor) -> torch.Tensor:
        """grid -> world with the endpoint pins gathered on the device."""
        out = torch.empty((self.sync_count(), 2), dtype=torch.float64, device=self.dev)
        N.call("hb_to_world_nodes", ptr(self.pts), ptr(self.starts), self.n_edges,
               float(origin[0]), float(origin[1]), float(cell), ptr(node_pos), ptr(sources),
               ptr(targets), ptr(out), stream_ptr())
        return out

    def world_points(self, origin, cell, src_world=None, dst_world=None) -> torch.Tensor:
        out = torch.empty((self.sync_count(), 2), dtype=torch.float64, device=self.dev)
        sw = None if src_world is None else upload(np.asarray(src_world, np.float64), self.dev)
        dw = None if dst_world is None else upload(np.asarray(dst_world, np.float64), self.dev)
        N.call("hb_to_world", ptr(self.pts), ptr(self.starts), self.n_edges,
               float(origin[0]), float(origin[1]), float(cell), ptr(sw), ptr(dw),
               ptr(out), stream_ptr())
        return out
