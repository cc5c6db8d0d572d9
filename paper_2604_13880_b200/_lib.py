"""ctypes binding of the C-ABI in ``include/det_api.h`` (library ``_det.so``).

The product path has no fallback: if the CUDA library is missing or no CUDA
device is usable, :func:`lib` raises.  Build with ``__graft_entry__.build()``
or ``make -C paper_2604_13880_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DET_LIB") or os.path.join(_HERE, "_det.so")  # DET_LIB: A/B builds (diagnostics)

DET_OK, DET_E_ARG, DET_E_CUDA, DET_E_RASTER, DET_E_COLLAPSE, DET_E_NUMERIC, DET_E_VALUE, DET_E_STATE = range(8)
STOP_NAMES = {1: "converged", 2: "stagnation", 3: "max-iterations"}
STOP_COLLAPSED, STOP_BDV, STOP_NEGINDEX = 4, 5, 6
# field_dtype -> DET_PREC_* (include/det_api.h)
PRECISIONS = {"float32": 0, "float64": 1, "mixed": 2}

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int32_p = ctypes.POINTER(ctypes.c_int32)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)


class DetParams(ctypes.Structure):
    _fields_ = [("background_mass", ctypes.c_double), ("bdv_multiplier", ctypes.c_double),
                ("mean_density0", ctypes.c_double), ("total_statistic", ctypes.c_double),
                ("bdv_mode", ctypes.c_int32), ("pad", ctypes.c_int32)]


class DetCriteria(ctypes.Structure):
    _fields_ = [("error_threshold", ctypes.c_double), ("stagnation_window", ctypes.c_int32),
                ("max_iterations", ctypes.c_int32)]


class DetResult(ctypes.Structure):
    _fields_ = [("stop_reason", ctypes.c_int32), ("iteration", ctypes.c_int32),
                ("best_iteration", ctypes.c_int32), ("collapsed_region", ctypes.c_int32),
                ("clamp_events", ctypes.c_int64), ("epsilon", ctypes.c_double), ("xi", ctypes.c_double),
                ("bdv", ctypes.c_double), ("trace_len", ctypes.c_int32), ("status", ctypes.c_int32)]


EXPORTS = {
    "det_abi_version": (ctypes.c_int, []),
    "det_debug_guard_check": (ctypes.c_int, [ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]),
    "det_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "det_host_free": (ctypes.c_int, [ctypes.c_void_p]),
    "det_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "det_device_info": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_int]),
    "det_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "det_ctx_destroy": (None, [ctypes.c_void_p]),
    "det_set_band_height": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "det_set_groups": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "det_load_map": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, ctypes.c_int, _c_int32_p, ctypes.c_int,
                                     _c_int32_p, _c_int32_p, ctypes.c_int]),
    "det_set_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p, _c_double_p]),
    "det_rasterize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_int32_p, _c_int64_p]),
    "det_set_params": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DetParams), _c_double_p]),
    "det_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DetCriteria)]),
    "det_bench_iterations": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "det_bench_kernel_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]),
    "det_sync": (ctypes.c_int, [ctypes.c_void_p]),
    "det_progress": (ctypes.c_int, [ctypes.c_void_p, _c_int32_p, _c_int32_p]),
    "det_time_iterations": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]),
    "det_get_result": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(DetResult)]),
    "det_run_chain": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p, _c_double_p, _c_double_p,
                                      ctypes.POINTER(DetCriteria), _c_double_p, ctypes.POINTER(DetResult),
                                      _c_int64_p, _c_double_p]),
    "det_get_vertices": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p]),
    "det_get_labels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_int32_p]),
    "det_get_counts": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_int64_p]),
    "det_get_region_error": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p]),
    "det_get_trace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p]),
    "det_get_areas": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p]),
    "det_get_results": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_int64_p, _c_double_p, _c_double_p,
                                        ctypes.c_int]),
    "det_field": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p, _c_double_p, _c_double_p]),
    "det_mapping": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p]),
    "det_mapping_channels": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, ctypes.c_double, _c_double_p,
                                             _c_double_p]),
    "det_mapping_points": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, ctypes.c_double, _c_double_p,
                                           ctypes.c_int, _c_double_p]),
    "det_density": (ctypes.c_int, [ctypes.c_void_p, _c_int32_p, _c_double_p, ctypes.c_int, ctypes.c_double,
                                    _c_double_p, _c_int64_p]),
    "det_interpolate": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_longlong, _c_double_p,
                                        ctypes.c_int, _c_double_p]),
    "det_advect": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_int, _c_double_p, _c_int64_p]),
    "det_shape_metrics": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _c_double_p, ctypes.c_int, _c_int32_p,
                                          ctypes.c_int, _c_int32_p, _c_double_p, ctypes.c_int, _c_int32_p,
                                          ctypes.c_int, _c_int32_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          _c_double_p, _c_double_p, _c_double_p, _c_double_p, _c_int32_p]),
    "det_adjacency": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, ctypes.c_int, ctypes.c_int, _c_int32_p,
                                      ctypes.c_int, ctypes.c_double, _c_int32_p, ctypes.c_longlong,
                                      ctypes.POINTER(ctypes.c_longlong)]),
    "det_position_error": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_int, ctypes.c_int,
                                           _c_double_p, ctypes.POINTER(ctypes.c_longlong)]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every exported signature (no CUDA call)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(f"DET CUDA library not built: {path} missing "
                                   "(run __graft_entry__.build() or make -C paper_2604_13880_b200/csrc)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _p(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype)) if a is not None else None


class _PinnedBlock:
    """One page-locked host allocation (det_host_alloc); freed when the last user is gone."""

    def __init__(self, lib, nbytes):
        ptr = ctypes.c_void_p()
        if lib.det_host_alloc(nbytes, ctypes.byref(ptr)) != DET_OK or not ptr.value:
            raise MemoryError(f"det_host_alloc({nbytes}) failed")
        self.lib, self.ptr, self.nbytes = lib, ptr.value, nbytes

    def __del__(self):
        try:
            self.lib.det_host_free(self.ptr)
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


class PinnedPool:
    """Numpy arrays backed by page-locked host memory, recycled when their last view dies.

    Device->host result copies into these run as DMA at full link speed, without the
    staging copy and page faults of a fresh pageable array.
    """

    def __init__(self, lib):
        self.lib = lib
        self.free = {}
        self.lock = threading.Lock()
        self.misses = 0  # allocations the pool could not serve (diagnostics)

    def reserve(self, nbytes):
        with self.lock:
            if not self.free.get(nbytes):
                self.free.setdefault(nbytes, []).append(_PinnedBlock(self.lib, nbytes))

    def _release(self, blk):
        with self.lock:
            self.free.setdefault(blk.nbytes, []).append(blk)

    def empty(self, shape, dtype=np.float64) -> np.ndarray:
        dt = np.dtype(dtype)
        count = int(np.prod(shape))
        nbytes = max(count * dt.itemsize, 1)
        with self.lock:
            lst = self.free.get(nbytes)
            blk = lst.pop() if lst else None
        if blk is None:
            self.misses += 1
            blk = _PinnedBlock(self.lib, nbytes)
        buf = (ctypes.c_char * nbytes).from_address(blk.ptr)
        buf._blk = blk  # the block lives as long as any view of this buffer
        weakref.finalize(buf, self._release, blk)
        return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


class DetError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"det error {code}: {msg}")
        self.code = code
        self.msg = msg


class Context:
    """One device context (CUDA stream + buffers) of the DET engine."""

    def __init__(self, k: int, device: int = 0, precision: str = "float32"):
        if precision not in PRECISIONS:
            raise ValueError(f"field_dtype must be one of {sorted(PRECISIONS)}")
        self.lib = load_library()
        self.k, self.n, self.device, self.precision = k, 1 << k, device, precision
        self.field_f64 = precision == "float64"
        h = ctypes.c_void_p()
        rc = self.lib.det_ctx_create(device, k, PRECISIONS[precision], ctypes.byref(h))
        if rc != DET_OK:
            raise DetError(rc, "det_ctx_create failed (no usable CUDA device?)")
        self.h = h
        self.B = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.det_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc != DET_OK:
            raise DetError(rc, self.lib.det_last_error(self.h).decode(errors="replace"))

    # --- topology / batch ---
    def load_map(self, xy, ring_start, ring_region, region_rank):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        rs = np.ascontiguousarray(ring_start, dtype=np.int32)
        rr = np.ascontiguousarray(ring_region, dtype=np.int32)
        rk = np.ascontiguousarray(region_rank, dtype=np.int32)
        self.n_rows, self.R = xy.shape[0], rk.shape[0]
        self.check(self.lib.det_load_map(self.h, _p(xy, ctypes.c_double), xy.shape[0], _p(rs, ctypes.c_int32),
                                         rs.shape[0] - 1, _p(rr, ctypes.c_int32), _p(rk, ctypes.c_int32), rk.shape[0]))
        self.B = 0
        self._owner_token = None  # engines re-load their map when they see another owner

    def set_batch(self, stats, xy=None):
        self.generation = getattr(self, "generation", 0) + 1
        st = np.ascontiguousarray(np.atleast_2d(stats), dtype=np.float64)
        b = st.shape[0]
        x = None if xy is None else np.ascontiguousarray(xy, dtype=np.float64).reshape(b, self.n_rows, 2)
        self.check(self.lib.det_set_batch(self.h, b, _p(x, ctypes.c_double), _p(st, ctypes.c_double)))
        self.B = b

    def set_groups(self, g):
        self.check(self.lib.det_set_groups(self.h, int(g)))

    def set_band_height(self, h):
        self.check(self.lib.det_set_band_height(self.h, int(h)))

    def rasterize(self, b=0, want_labels=True):
        self.generation = getattr(self, "generation", 0) + 1
        lab = np.empty((self.n, self.n), dtype=np.int32) if want_labels else None
        cnt = np.empty(self.R + 1, dtype=np.int64)
        self.check(self.lib.det_rasterize(self.h, b, _p(lab, ctypes.c_int32), _p(cnt, ctypes.c_int64)))
        return lab, cnt

    def set_params(self, params, weights):
        arr = (DetParams * len(params))()
        for i, p in enumerate(params):
            arr[i] = DetParams(p["background_mass"], p["bdv_multiplier"], p["mean_density0"],
                               p["total_statistic"], p["bdv_mode"], 0)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        self.check(self.lib.det_set_params(self.h, arr, _p(w, ctypes.c_double)))

    def run(self, error_threshold, stagnation_window, max_iterations):
        c = DetCriteria(float(error_threshold), int(stagnation_window), int(max_iterations))
        self.generation = getattr(self, "generation", 0) + 1
        self.check(self.lib.det_run(self.h, ctypes.byref(c)))

    def run_chain(self, stats, totals, masses, error_threshold, stagnation_window, max_iterations):
        """Cumulative chain of T frames on the device (see det_run_chain)."""
        stats = np.ascontiguousarray(stats, dtype=np.float64)
        T = stats.shape[0]
        tot = np.ascontiguousarray(totals, dtype=np.float64)
        mb = np.ascontiguousarray(masses, dtype=np.float64)
        c = DetCriteria(float(error_threshold), int(stagnation_window), int(max_iterations))
        xy = np.zeros((T, self.n_rows, 2), dtype=np.float64)
        res = (DetResult * T)()
        cnt = np.zeros((T, self.R + 1), dtype=np.int64)
        tr = np.zeros((T, int(max_iterations) + 1, 4), dtype=np.float64)
        self.generation = getattr(self, "generation", 0) + 1
        self.check(self.lib.det_run_chain(self.h, T, _p(stats, ctypes.c_double), _p(tot, ctypes.c_double),
                                          _p(mb, ctypes.c_double), ctypes.byref(c), _p(xy, ctypes.c_double), res,
                                          _p(cnt, ctypes.c_int64), _p(tr, ctypes.c_double)))
        return xy, list(res), cnt, tr

    def bench_iterations(self, iters):
        self.generation = getattr(self, "generation", 0) + 1
        self.check(self.lib.det_bench_iterations(self.h, int(iters)))

    def kernel_times(self, iters):
        out = (ctypes.c_float * 4)()
        self.check(self.lib.det_bench_kernel_times(self.h, int(iters), out))
        return list(out)

    def time_iterations(self, iters):
        ms = ctypes.c_float(0.0)
        self.check(self.lib.det_time_iterations(self.h, int(iters), ctypes.byref(ms)))
        return float(ms.value)

    def progress(self):
        it = np.empty(self.B, dtype=np.int32)
        ac = np.empty(self.B, dtype=np.int32)
        self.check(self.lib.det_progress(self.h, _p(it, ctypes.c_int32), _p(ac, ctypes.c_int32)))
        return it, ac

    def sync(self):
        self.check(self.lib.det_sync(self.h))

    # --- results ---
    def result(self, b=0) -> DetResult:
        r = DetResult()
        self.check(self.lib.det_get_result(self.h, b, ctypes.byref(r)))
        return r

    def results_all(self, xy_out, trace_rows):
        """Vertices (into xy_out, B x rows x 2), counts, per-region errors and traces of every cartogram."""
        counts = np.empty((self.B, self.R + 1), dtype=np.int64)
        errs = np.empty((self.B, self.R), dtype=np.float64)
        trace = np.empty((self.B, max(int(trace_rows), 0), 4), dtype=np.float64)
        self.check(self.lib.det_get_results(self.h, _p(xy_out, ctypes.c_double), _p(counts, ctypes.c_int64),
                                            _p(errs, ctypes.c_double), _p(trace, ctypes.c_double),
                                            int(trace_rows)))
        return counts, errs, trace

    def vertices(self, b=0, out=None):
        if out is None:
            out = np.empty((self.n_rows, 2), dtype=np.float64)
        self.check(self.lib.det_get_vertices(self.h, b, _p(out, ctypes.c_double)))
        return out

    @property
    def pinned(self) -> PinnedPool:
        pool = getattr(self, "_pinned", None)
        if pool is None:
            pool = self._pinned = PinnedPool(self.lib)
        return pool

    def labels(self, b=0):
        out = np.empty((self.n, self.n), dtype=np.int32)
        self.check(self.lib.det_get_labels(self.h, b, _p(out, ctypes.c_int32)))
        return out

    def counts(self, b=0):
        out = np.empty(self.R + 1, dtype=np.int64)
        self.check(self.lib.det_get_counts(self.h, b, _p(out, ctypes.c_int64)))
        return out

    def region_error(self, b=0):
        out = np.empty(self.R, dtype=np.float64)
        self.check(self.lib.det_get_region_error(self.h, b, _p(out, ctypes.c_double)))
        return out

    def trace(self, b=0, length=None):
        if length is None:
            length = self.result(b).trace_len
        out = np.empty((max(length, 0), 4), dtype=np.float64)
        if length > 0:
            self.check(self.lib.det_get_trace(self.h, b, _p(out, ctypes.c_double)))
        return out

    def areas(self, b=0):
        out = np.empty(self.R, dtype=np.float64)
        self.check(self.lib.det_get_areas(self.h, b, _p(out, ctypes.c_double)))
        return out

    # --- stage level ---
    def field(self, d, channels=False):
        d = np.ascontiguousarray(d, dtype=np.float64)
        u = np.empty((self.n, self.n, 2), dtype=np.float64)
        ch = np.empty((8, self.n, self.n), dtype=np.float64) if channels else None
        tot = ctypes.c_double(0.0)
        self.check(self.lib.det_field(self.h, _p(d, ctypes.c_double), _p(u, ctypes.c_double),
                                      _p(ch, ctypes.c_double), ctypes.byref(tot)))
        return u, ch, tot.value

    def channels(self, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        ch = np.empty((8, self.n, self.n), dtype=np.float64)
        tot = ctypes.c_double(0.0)
        self.check(self.lib.det_field(self.h, _p(d, ctypes.c_double), None, _p(ch, ctypes.c_double),
                                      ctypes.byref(tot)))
        return ch, tot.value

    def mapping(self, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        t = np.empty((self.n, self.n, 2), dtype=np.float64)
        self.check(self.lib.det_mapping(self.h, _p(d, ctypes.c_double), _p(t, ctypes.c_double)))
        return t

    def mapping_channels(self, channels, total, base=None):
        """mapping_grid of a channel set (8, n, n), minus `base` (n, n, 2) when given."""
        ch = np.ascontiguousarray(channels, dtype=np.float64)
        bs = None if base is None else np.ascontiguousarray(base, dtype=np.float64)
        t = np.empty((self.n, self.n, 2), dtype=np.float64)
        self.check(self.lib.det_mapping_channels(self.h, _p(ch, ctypes.c_double), float(total),
                                                 _p(bs, ctypes.c_double), _p(t, ctypes.c_double)))
        return t

    def mapping_points(self, channels, total, xy):
        """mapping_point at (N, 2) points of a channel set (8, n, n)."""
        ch = np.ascontiguousarray(channels, dtype=np.float64)
        pts = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(pts)
        self.check(self.lib.det_mapping_points(self.h, _p(ch, ctypes.c_double), float(total),
                                               _p(pts, ctypes.c_double), pts.shape[0], _p(out, ctypes.c_double)))
        return out

    def interpolate(self, a, b, fracs):
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        b = np.ascontiguousarray(b, dtype=np.float64).ravel()
        fr = np.ascontiguousarray(fracs, dtype=np.float64)
        out = np.empty((fr.shape[0], a.shape[0]), dtype=np.float64)
        self.check(self.lib.det_interpolate(self.h, _p(a, ctypes.c_double), _p(b, ctypes.c_double), a.shape[0],
                                            _p(fr, ctypes.c_double), fr.shape[0], _p(out, ctypes.c_double)))
        return out

    def shape_metrics(self, layout_a, layout_b, raster_k, rescale=True):
        """Per (frame, region) Hamming distortion, carto area/centroid and status (k_shape).

        ``layout_*`` = (xy, ring_start, ring_region, n_regions); layout_b's xy may stack frames.
        """
        xa, rsa, rra, r = layout_a
        xb, rsb, rrb, rb = layout_b
        if r != rb:
            raise ValueError("region count mismatch")
        xa = np.ascontiguousarray(xa, dtype=np.float64)
        rsa = np.ascontiguousarray(rsa, dtype=np.int32)
        rra = np.ascontiguousarray(rra, dtype=np.int32)
        rsb = np.ascontiguousarray(rsb, dtype=np.int32)
        rrb = np.ascontiguousarray(rrb, dtype=np.int32)
        rows_a, rows_b = int(rsa[-1]), int(rsb[-1])
        xb = np.ascontiguousarray(xb, dtype=np.float64).reshape(-1, rows_b, 2)
        f = xb.shape[0]
        ham = np.empty((f, r))
        area = np.empty((f, r))
        ca = np.empty((r, 2))
        cb = np.empty((f, r, 2))
        st = np.empty((f, r), dtype=np.int32)
        self.check(self.lib.det_shape_metrics(
            self.h, r, _p(xa, ctypes.c_double), rows_a, _p(rsa, ctypes.c_int32), rsa.shape[0] - 1,
            _p(rra, ctypes.c_int32), _p(xb, ctypes.c_double), rows_b, _p(rsb, ctypes.c_int32), rsb.shape[0] - 1,
            _p(rrb, ctypes.c_int32), f, int(raster_k), int(bool(rescale)), _p(ham, ctypes.c_double),
            _p(area, ctypes.c_double), _p(ca, ctypes.c_double), _p(cb, ctypes.c_double), _p(st, ctypes.c_int32)))
        return ham, area, ca, cb, st

    def adjacency(self, xy, row_region, n_regions, epsilon):
        """(frame, a, b) region index triples, a < b sharing >= 2 epsilon-cells (k_adj_*).

        ``xy`` is (rows, 2) or (frames, rows, 2) in one layout.
        """
        rr = np.ascontiguousarray(row_region, dtype=np.int32)
        x = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, rr.shape[0], 2)
        cap = 4 * int(n_regions) * x.shape[0] + 64
        for _ in range(2):
            out = np.empty((cap, 3), dtype=np.int32)
            cnt = ctypes.c_longlong(0)
            self.check(self.lib.det_adjacency(self.h, _p(x, ctypes.c_double), x.shape[0], rr.shape[0],
                                              _p(rr, ctypes.c_int32), int(n_regions), float(epsilon),
                                              _p(out, ctypes.c_int32), cap, ctypes.byref(cnt)))
            if cnt.value <= cap:
                return out[: cnt.value]
            cap = int(cnt.value)
        raise RuntimeError("adjacency pair count changed between calls")

    def position_error(self, cent_m, cent_c):
        """Sum of |angle change| over ordered barycenter pairs, and degenerate pair counts (k_poserr)."""
        cm = np.ascontiguousarray(cent_m, dtype=np.float64).reshape(-1, 2)
        r = cm.shape[0]
        cc = np.ascontiguousarray(cent_c, dtype=np.float64).reshape(-1, r, 2)
        f = cc.shape[0]
        sums = np.empty(f)
        dg = (ctypes.c_longlong * f)()
        self.check(self.lib.det_position_error(self.h, _p(cm, ctypes.c_double), _p(cc, ctypes.c_double), f, r,
                                               _p(sums, ctypes.c_double), dg))
        return sums, np.array(list(dg), dtype=np.int64)

    def advect(self, u, xy):
        u = np.ascontiguousarray(u, dtype=np.float64)
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.empty_like(xy)
        cl = ctypes.c_int64(0)
        self.check(self.lib.det_advect(self.h, _p(u, ctypes.c_double), _p(xy, ctypes.c_double), xy.shape[0],
                                       _p(out, ctypes.c_double), ctypes.byref(cl)))
        return out, int(cl.value)


def device_info(device: int = 0) -> str:
    lib = load_library()
    buf = ctypes.create_string_buffer(256)
    lib.det_device_info(device, buf, 256)
    return buf.value.decode()
