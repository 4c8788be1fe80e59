"""Host-side mirror of the reference's library interface for the DGS path.

Same names, argument meaning and error behaviour as the reference C++ API in
/root/reference/proj/include/mrf (sequence.hpp, bloch.hpp, dictionary.hpp,
zoom.hpp), over the C ABI of include/mrfg.h:

=========================  ===============================================
reference                  here
=========================  ===============================================
Schedule / build_schedule  Schedule, reference_schedule, baseline_schedule
grid_from_ranges           grid_from_ranges (endpoint-exclusive) / grid()
BlochSimulator::simulate   Context.simulate (precision 64 or 32)
generate                   Context.generate
scan_grid                  Context.scan_grid (+ scan_grid_device)
brute_force_search         Context.brute_force_search
cc_map                     Context.cc_map (precision 64 exact / 32 fused FP32)
cc_map_to_file             Context.cc_map_to_file (.mrfc)
save_generated             Context.save_generated (.mrfd, GPU-generated)
save / load (Dictionary)   save_dictionary / load_dictionary / read_header
quantify / quantify_slice  Context.quantify / Context.quantify_slice
add_noise / rng            add_noise / rng_at / uniform01 / gaussian
calibrate_noise            calibrate_noise / make_calibrated_noise
smooth                     smooth
=========================  ===============================================
"""
from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import (STAGE_NAMES, TRACE_MAX, Axis, Grid, Match, Quant, ScanOpts, ScanStats, Stage, ZoomConfig,
                      ZoomIo, check)

METRIC = {"cc": 0, "euclidean": 1}


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# --------------------------------------------------------------- schedule
@dataclass
class Schedule:
    """Schedule (sequence.hpp:14-31): per-TR flip/phase in degrees, TR/TE in ms."""
    flip_deg: np.ndarray
    phase_deg: np.ndarray
    tr_ms: np.ndarray
    te_ms: np.ndarray

    def __post_init__(self):
        for k in ("flip_deg", "phase_deg", "tr_ms", "te_ms"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.float64))

    @property
    def n(self) -> int:
        return len(self.flip_deg)

    def to_csv(self) -> str:
        """Canonical CSV bytes (sequence.cpp:94-103); also the digest input."""
        rows = ["idx,flip_deg,phase_deg,tr_ms,te_ms\n"]
        rows += [f"{k},{self.flip_deg[k]:.9g},{self.phase_deg[k]:.9g},{self.tr_ms[k]:.9g},"
                 f"{self.te_ms[k]:.9g}\n" for k in range(self.n)]
        return "".join(rows)

    def digest(self) -> str:
        """schedule_digest (dictionary.cpp:163-171), hex."""
        return hashlib.sha256(self.to_csv().encode()).hexdigest()


def _schedule(fn, n: int, seed: int) -> Schedule:
    arrs = [np.zeros(n) for _ in range(4)]
    check(fn(n, seed, *[_dp(a) for a in arrs]))
    return Schedule(*arrs)


def reference_schedule(n: int, seed: int) -> Schedule:
    """build_schedule (sequence.hpp:51)."""
    return _schedule(N.load().mrfg_reference_schedule, n, seed)


def baseline_schedule(n: int, seed: int = 1) -> Schedule:
    """BASELINE.json generator: FA 10+50|sin(2 pi j/250)|+N(0,2) deg, 0/180 phase,
    TR ~ U[10.5,14] ms, TE = TR/2."""
    return _schedule(N.load().mrfg_baseline_schedule, n, seed)


# ------------------------------------------------------------------ grids
def grid(t1, t2, df) -> Grid:
    """Grid from per-axis (min, step, count)."""
    return Grid(Axis(*t1), Axis(*t2), Axis(*df))


def grid_values(t1_ms, t2_ms, df) -> Grid:
    """Grid with EXPLICIT T1 and T2 values [ms] (e.g. log-spaced, BASELINE
    configs[2]) and an evenly spaced df axis (min, step, count).  The arrays are
    kept alive by the returned Grid.  generate / scan_grid / cc_map accept it;
    the reference builds such dictionaries from explicit TissueParams."""
    t1 = np.ascontiguousarray(t1_ms, dtype=np.float64)
    t2 = np.ascontiguousarray(t2_ms, dtype=np.float64)
    dp = C.POINTER(C.c_double)
    g = Grid(Axis(float(t1[0]), 0.0, len(t1), t1.ctypes.data_as(dp)),
             Axis(float(t2[0]), 0.0, len(t2), t2.ctypes.data_as(dp)), Axis(*df))
    g._keep = (t1, t2)
    return g


def axis_values(ax: Axis) -> np.ndarray:
    """AxisSpec::value over the axis (or its explicit values)."""
    if ax.values:
        return np.ctypeslib.as_array(ax.values, shape=(ax.count,)).copy()
    return ax.min + np.arange(ax.count, dtype=np.float64) * ax.step


def axis_count(lo: float, hi: float, step: float) -> int:
    c = C.c_int64()
    rc = N.load().mrfg_axis_count(lo, hi, step, C.byref(c))
    if rc:
        raise N.InvalidArgument(rc, "axis: need step > 0 and max > min")
    return c.value


def grid_from_ranges(t1, t2, df) -> Grid:
    """grid_from_ranges (dictionary.cpp:154-161): half-open (min, max, step) per axis."""
    return grid(*[(r[0], r[2], axis_count(*r)) for r in (t1, t2, df)])


def grid_inclusive(t1, t2, df) -> Grid:
    """Endpoint-INCLUSIVE axes (BASELINE.json's convention)."""
    return grid_from_ranges(*[(lo, hi + st, st) for lo, hi, st in (t1, t2, df)])


def grid_total(g: Grid) -> int:
    return g.t1_ms.count * g.t2_ms.count * g.df_hz.count


def unflatten(g: Grid, flat):
    """ParameterGrid::unflatten (dictionary.hpp:45-49)."""
    flat = np.asarray(flat, dtype=np.int64)
    idf = flat % g.df_hz.count
    rest = flat // g.df_hz.count
    return rest // g.t2_ms.count, rest % g.t2_ms.count, idf


def params_at(g: Grid, i1, i2, idf):
    """ParameterGrid::params_at (dictionary.hpp:51-53): seconds, seconds, Hz."""
    def val(ax, i):
        i = np.asarray(i)
        if ax.values:
            return axis_values(ax)[i.astype(np.int64)]
        return ax.min + i.astype(np.float64) * ax.step
    return val(g.t1_ms, i1) * 1e-3, val(g.t2_ms, i2) * 1e-3, val(g.df_hz, idf)


# -------------------------------------------------------------------- rng
def rng_at(seed: int, stream: int, index: int) -> int:
    return N.load().mrfg_rng_at(seed, stream, index)


def uniform01(seed: int, stream: int, index: int) -> float:
    return N.load().mrfg_rng_uniform01(seed, stream, index)


def gaussian(seed: int, stream: int, index: int) -> float:
    return N.load().mrfg_rng_gaussian(seed, stream, index)


def add_noise(fp: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """add_noise (fingerprint.cpp:68-78)."""
    fp = np.ascontiguousarray(fp, dtype=np.complex128)
    out = np.empty_like(fp)
    check(N.load().mrfg_add_noise(_dp(fp.view(np.float64)), len(fp), sigma, seed,
                                  _dp(out.view(np.float64))))
    return out


def calibrate_noise(fp: np.ndarray, target_cc: float, seed: int) -> float:
    """calibrate_noise (fingerprint.cpp:80-105): sigma with cc(fp, noisy) within 0.02 of target."""
    fp = np.ascontiguousarray(fp, dtype=np.complex128)
    sigma = C.c_double()
    check(N.load().mrfg_calibrate_noise(_dp(fp.view(np.float64)), len(fp), target_cc, seed,
                                        C.byref(sigma)))
    return sigma.value


def make_calibrated_noise(fp: np.ndarray, target_cc: float, seed: int):
    """make_calibrated_noise (fingerprint.cpp:107-120) -> (sigma, seed_used, noisy)."""
    fp = np.ascontiguousarray(fp, dtype=np.complex128)
    sigma, used = C.c_double(), C.c_uint64()
    out = np.empty_like(fp)
    check(N.load().mrfg_make_calibrated_noise(_dp(fp.view(np.float64)), len(fp), target_cc, seed,
                                              C.byref(sigma), C.byref(used), _dp(out.view(np.float64))))
    return sigma.value, used.value, out


def smooth(fp: np.ndarray, k: int) -> np.ndarray:
    """smooth (fingerprint.cpp:122-145): Gaussian k = 3 / 5 taps, edge-truncated."""
    fp = np.ascontiguousarray(fp, dtype=np.complex128)
    out = np.empty_like(fp)
    check(N.load().mrfg_smooth(_dp(fp.view(np.float64)), len(fp), k, _dp(out.view(np.float64))))
    return out


MAGIC_DICT, MAGIC_MAP = b"MRFD", b"MRFC"


def _digest_bytes(digest) -> "C.Array":
    d = bytes.fromhex(digest) if isinstance(digest, str) else bytes(digest)
    if len(d) != 32:
        raise ValueError("digest must be 32 bytes")
    return (C.c_uint8 * 32).from_buffer_copy(d)


def read_header(path: str, magic: bytes = MAGIC_DICT):
    """read_header (dictionary.cpp:90-112) -> (grid, digest hex, entry_len, payload offset)."""
    g, dg = Grid(), (C.c_uint8 * 32)()
    el, off = C.c_int64(), C.c_int64()
    check(N.load().mrfg_read_header(str(path).encode(), magic, C.byref(g), dg, C.byref(el),
                                    C.byref(off)))
    return g, bytes(dg).hex(), el.value, off.value


def save_dictionary(path: str, g: Grid, digest, entries: np.ndarray) -> None:
    """save (dictionary.cpp:196-203): header + float32 (re, im) entries in flat order."""
    entries = np.ascontiguousarray(entries, dtype=np.float32)
    if entries.ndim != 2 or entries.shape[0] != grid_total(g) or entries.shape[1] % 2:
        raise ValueError("save: entries must be (grid total, 2N) float32")
    check(N.load().mrfg_write_header(str(path).encode(), MAGIC_DICT, C.byref(g), _digest_bytes(digest),
                                     entries.shape[1] // 2))
    with open(path, "ab") as f:
        entries.tofile(f)


def load_dictionary(path: str):
    """load (dictionary.cpp:205-220) -> (grid, digest hex, entries (total, 2N) float32)."""
    g, dg, el, off = read_header(path, MAGIC_DICT)
    want = grid_total(g) * 2 * el
    data = np.fromfile(path, dtype=np.float32, offset=off)
    if data.size < want:
        raise N.MrfgError(-3, f"truncated payload in {path}")  # MRFG_E_RUNTIME
    return g, dg, data[:want].reshape(grid_total(g), 2 * el)


def load_cc_map(path: str):
    """An .mrfc file (cc_map_to_file, dictionary.cpp:333-347) -> (grid, digest hex, scores)."""
    g, dg, el, off = read_header(path, MAGIC_MAP)
    data = np.fromfile(path, dtype=np.float32, offset=off)
    if data.size < grid_total(g):
        raise N.MrfgError(-3, f"truncated payload in {path}")
    return g, dg, data[:grid_total(g)]


def zoom_config(**kw) -> ZoomConfig:
    """ZoomConfig with the reference defaults (zoom.hpp:23-52), overridable."""
    c = ZoomConfig()
    N.load().mrfg_zoom_config_default(C.byref(c))
    for k, v in kw.items():
        if k in ("metric", "final_metric") and isinstance(v, str):
            v = METRIC[v]
        if k == "t1t2_2d_steps_ms":
            c.n2d = len(v)
            for i, x in enumerate(v):
                c.t1t2_2d_steps_ms[i] = x
        elif k == "t1t2_1d_steps_ms":
            c.n1d = len(v)
            for i, x in enumerate(v):
                c.t1t2_1d_steps_ms[i] = x
        else:
            setattr(c, k, v)
    return c


# ---------------------------------------------------------------- context
class Context:
    """One schedule on one sm_100 device: BlochSimulator plus the search paths."""

    def __init__(self, sched: Schedule, device: int = 0):
        self.lib = N.load()
        self.sched = sched
        self.n = sched.n
        h = C.c_void_p()
        check(self.lib.mrfg_create(_dp(sched.flip_deg), _dp(sched.phase_deg), _dp(sched.tr_ms),
                                   _dp(sched.te_ms), sched.n, device, C.byref(h)))
        self.h = h

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.mrfg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_stream(self, stream_handle: int) -> None:
        check(self.lib.mrfg_set_stream(self.h, C.c_void_p(stream_handle)))

    def synchronize(self) -> None:
        check(self.lib.mrfg_synchronize(self.h))

    # -- K1
    def simulate(self, params, precision: int = 64, normalize: bool = False) -> np.ndarray:
        """params: (k, 3) of (t1_s, t2_s, df_hz) -> (k, N) complex128."""
        p = np.ascontiguousarray(np.atleast_2d(params), dtype=np.float64)
        out = np.empty((p.shape[0], self.n), dtype=np.complex128)
        check(self.lib.mrfg_simulate(self.h, _dp(p), p.shape[0], precision, int(normalize),
                                     _dp(out.view(np.float64))))
        return out

    def simulate_device(self, d_params_ptr: int, count: int, d_out_ptr: int, precision: int = 64,
                        normalize: bool = False) -> None:
        """Device form of simulate: d_params (count, 3) float64 -> d_out (count, 2N) float64."""
        check(self.lib.mrfg_simulate_dev(self.h, C.c_void_p(d_params_ptr), count, precision,
                                         int(normalize), C.c_void_p(d_out_ptr)))

    def generate(self, g: Grid, first: int = 0, count: int | None = None,
                 precision: int = 64) -> np.ndarray:
        """generate (dictionary.cpp:184-194): unit-norm float32 entries, (count, 2N)."""
        if count is None:
            count = grid_total(g) - first
        out = np.empty((count, 2 * self.n), dtype=np.float32)
        check(self.lib.mrfg_generate(self.h, C.byref(g), first, count, precision,
                                     out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def generate_device(self, g: Grid, first: int, count: int, d_out_ptr: int, precision: int = 64) -> None:
        """generate into device memory: (count, 2N) float32 at d_out_ptr."""
        check(self.lib.mrfg_generate_dev(self.h, C.byref(g), first, count, precision, C.c_void_p(d_out_ptr)))

    # -- K2/K3
    @staticmethod
    def _unit_opts(opts, unit_norm, nq):
        """Attach Fingerprint::unit_norm flags (bool or per-query array) to the options."""
        if unit_norm is None or unit_norm is False:
            return opts, None
        flags = np.ascontiguousarray(np.broadcast_to(np.asarray(unit_norm, dtype=np.uint8), (nq,)))
        o = ScanOpts() if opts is None else ScanOpts.from_buffer_copy(opts)
        o.unit_queries = flags.ctypes.data_as(C.POINTER(C.c_uint8))
        return o, flags

    def scan_grid(self, g: Grid, queries, metric="cc", flat_range=(0, 0), opts: ScanOpts = None,
                  unit_norm=None):
        """scan_grid (dictionary.cpp:257-308) -> (best_flat, best_score, stats).
        unit_norm: queries flagged Fingerprint::unit_norm are scored as given."""
        q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.complex128)
        if q.shape[-1] != self.n:
            raise N.InvalidArgument(-1, "query length does not match dictionary entries")
        opts, _flags = self._unit_opts(opts, unit_norm, q.shape[0])
        out = (Match * q.shape[0])()
        st = ScanStats()
        check(self.lib.mrfg_scan_grid(self.h, C.byref(g), flat_range[0], flat_range[1],
                                      _dp(q.view(np.float64)), q.shape[0],
                                      METRIC.get(metric, metric),
                                      C.byref(opts) if opts is not None else None, out,
                                      C.byref(st)))
        arr = np.frombuffer(out, dtype=np.dtype([("flat", np.int64), ("score", np.float64)]))
        return arr["flat"].copy(), arr["score"].copy(), st

    def scan_grid_device(self, g: Grid, d_queries_ptr: int, nq: int, d_out_ptr: int,
                         metric="cc", flat_range=(0, 0), opts: ScanOpts = None) -> ScanStats:
        """Device-resident variant (async on the context stream; pointers from torch)."""
        st = ScanStats()
        check(self.lib.mrfg_scan_grid_dev(self.h, C.byref(g), flat_range[0], flat_range[1],
                                          C.c_void_p(d_queries_ptr), nq,
                                          METRIC.get(metric, metric),
                                          C.byref(opts) if opts is not None else None,
                                          C.c_void_p(d_out_ptr), C.byref(st)))
        return st

    def scan_seed_device(self, g: Grid, d_queries_ptr: int, nq: int, d_seed_ptr: int, metric="cc",
                         flat_range=(0, 0), opts: ScanOpts = None, d_dict_ptr: int = 0,
                         natoms: int = 0) -> ScanStats:
        """Seed pass only: float screening maxima (nq) of a strided sample of the
        flat range (lattice g, or a device dictionary when d_dict_ptr is given)."""
        st = ScanStats()
        check(self.lib.mrfg_scan_seed_dev(self.h, None if d_dict_ptr else C.byref(g),
                                          C.c_void_p(d_dict_ptr) if d_dict_ptr else None, natoms,
                                          flat_range[0], flat_range[1], C.c_void_p(d_queries_ptr), nq,
                                          METRIC.get(metric, metric),
                                          C.byref(opts) if opts is not None else None,
                                          C.c_void_p(d_seed_ptr), C.byref(st)))
        return st

    def merge_matches_device(self, d_in_ptr: int, nranks: int, nq: int, d_out_ptr: int) -> None:
        check(self.lib.mrfg_merge_matches_dev(self.h, C.c_void_p(d_in_ptr), nranks, nq,
                                              C.c_void_p(d_out_ptr)))

    def bloch_norms_device(self, g: Grid, first: int, count: int, d_out_ptr: int) -> None:
        check(self.lib.mrfg_bloch_norms_dev(self.h, C.byref(g), first, count,
                                            C.c_void_p(d_out_ptr)))

    def brute_force_search(self, queries, dictionary: np.ndarray, metric="cc",
                           opts: ScanOpts = None, unit_norm=None):
        """brute_force_search (dictionary.cpp:241-255) over a STORED dictionary.

        dictionary: (atoms, 2N) float32 unit entries in flat order (generate()'s
        layout).  Returns (best_flat, best_score, stats) per query."""
        q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.complex128)
        d = np.ascontiguousarray(dictionary, dtype=np.float32)
        if q.shape[-1] != self.n or d.shape[-1] != 2 * self.n:
            raise N.InvalidArgument(-1, "query length does not match dictionary entries")
        opts, _flags = self._unit_opts(opts, unit_norm, q.shape[0])
        out = (Match * q.shape[0])()
        st = ScanStats()
        check(self.lib.mrfg_scan_dict(self.h, d.ctypes.data_as(C.POINTER(C.c_float)), d.shape[0],
                                      _dp(q.view(np.float64)), q.shape[0], METRIC.get(metric, metric),
                                      C.byref(opts) if opts is not None else None, out, C.byref(st)))
        arr = np.frombuffer(out, dtype=np.dtype([("flat", np.int64), ("score", np.float64)]))
        return arr["flat"].copy(), arr["score"].copy(), st

    def scan_dict_device(self, d_dict_ptr: int, natoms: int, d_queries_ptr: int, nq: int,
                         d_out_ptr: int, metric="cc", flat_range=(0, 0),
                         opts: ScanOpts = None) -> ScanStats:
        st = ScanStats()
        check(self.lib.mrfg_scan_dict_dev(self.h, C.c_void_p(d_dict_ptr), natoms, flat_range[0],
                                          flat_range[1], C.c_void_p(d_queries_ptr), nq,
                                          METRIC.get(metric, metric),
                                          C.byref(opts) if opts is not None else None,
                                          C.c_void_p(d_out_ptr), C.byref(st)))
        return st

    def screen_scores(self, g: Grid, queries, first: int, count: int, metric="cc",
                      use_simt: bool = False, producer: str = "table") -> np.ndarray:
        """Dense K2 screening scores (count, nq) -- test support.

        producer "table": the per-atom table producer; "rows": the production
        K1 row producer used by scan_grid (MRFG_K1 selects its variant)."""
        q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.complex128)
        out = np.empty((count, q.shape[0]), dtype=np.float32)
        check(self.lib.mrfg_screen_scores(self.h, C.byref(g), first, count, _dp(q.view(np.float64)),
                                          q.shape[0], METRIC.get(metric, metric),
                                          int(use_simt) | (2 if producer == "rows" else 0),
                                          out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def cc_map(self, fp, g: Grid, first: int = 0, count: int | None = None,
               precision: int = 64) -> np.ndarray:
        """cc_map (dictionary.cpp:310-331): float32 CC of fp vs flats [first, first+count).

        precision 64: the reference pipeline (bit-identical); 32: fused FP32 kernel."""
        if count is None:
            count = grid_total(g) - first
        q = np.ascontiguousarray(fp, dtype=np.complex128)
        out = np.empty(count, dtype=np.float32)
        check(self.lib.mrfg_cc_map_ex(self.h, C.byref(g), _dp(q.view(np.float64)), first, count,
                                      precision, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def cc_map_to_file(self, fp, g: Grid, path: str, precision: int = 64) -> None:
        """cc_map_to_file (dictionary.cpp:333-347): the lattice's cc_map as an .mrfc file."""
        q = np.ascontiguousarray(fp, dtype=np.complex128)
        check(self.lib.mrfg_cc_map_to_file(self.h, C.byref(g), _dp(q.view(np.float64)),
                                           _digest_bytes(self.sched.digest()), str(path).encode(),
                                           precision))

    def save_generated(self, g: Grid, path: str, chunk_entries: int = 1 << 15,
                       precision: int = 64) -> None:
        """save_generated (dictionary.cpp:216-239): the GPU-generated dictionary as .mrfd."""
        check(self.lib.mrfg_save_generated(self.h, C.byref(g), _digest_bytes(self.sched.digest()),
                                           str(path).encode(), chunk_entries, precision))

    # -- K5
    def _zoom_io(self, nvox: int, dictionary, trace: bool):
        """mrfg_zoom_io for a dictionary payload (float32 (entries, 2N) or
        complex64 (entries, N), or None) and/or the StageLog outputs."""
        if dictionary is None and not trace:
            return None, None
        io = ZoomIo()
        keep = []
        if dictionary is not None:
            d = np.ascontiguousarray(dictionary)
            d = d.view(np.float32) if d.dtype == np.complex64 else np.ascontiguousarray(d, dtype=np.float32)
            d = d.reshape(-1, 2 * self.n)
            keep.append(d)
            io.dict = d.ctypes.data
            io.dict_entries = d.shape[0]
        bufs = None
        if trace:
            rec = (Stage * (TRACE_MAX * nvox))()
            ln = np.zeros(nvox, dtype=np.int32)
            io.trace = C.addressof(rec)
            io.trace_len = ln.ctypes.data
            bufs = (rec, ln)
        return io, (keep, bufs)

    @staticmethod
    def _traces(bufs, idx):
        rec, ln = bufs
        out = []
        for v in idx:
            k0 = int(v) * TRACE_MAX
            out.append([(STAGE_NAMES[rec[k0 + k].stage], rec[k0 + k].evaluations, rec[k0 + k].best,
                         rec[k0 + k].t1_ms, rec[k0 + k].t2_ms, rec[k0 + k].df_hz)
                        for k in range(min(int(ln[v]), TRACE_MAX))])
        return out

    def quantify(self, fps, lattice: Grid, cfg: ZoomConfig = None, dictionary=None, trace: bool = False):
        """quantify (zoom.cpp:533-539) for a batch of fingerprints -> Quant records.

        dictionary: the df slab (cfg.dict_mode 1) or full lattice dictionary
        (dict_mode 2) payload, scored as given (zoom.cpp:101-113).  trace=True
        also returns each voxel's StageLog list (zoom.cpp:441-451) as
        (stage, evaluations, best, t1_ms, t2_ms, df_hz) tuples."""
        q = np.ascontiguousarray(np.atleast_2d(fps), dtype=np.complex128)
        cfg = cfg or zoom_config()
        out = (Quant * q.shape[0])()
        io, keep = self._zoom_io(q.shape[0], dictionary, trace)
        check(self.lib.mrfg_quantify_ex(self.h, C.byref(lattice), C.byref(cfg), _dp(q.view(np.float64)),
                                        q.shape[0], None, None, None if io is None else C.byref(io), out))
        res = quant_array(out)
        return (res, self._traces(keep[1], range(q.shape[0]))) if trace else res

    def quantify_device(self, d_fps_ptr: int, nvox: int, lattice: Grid, cfg: ZoomConfig,
                        d_out_ptr: int) -> None:
        """quantify on device buffers (nvox x 2N float64 in, nvox Quant records out)."""
        check(self.lib.mrfg_quantify_dev(self.h, C.byref(lattice), C.byref(cfg),
                                         C.c_void_p(d_fps_ptr), nvox, C.c_void_p(d_out_ptr)))

    def quantify_bounded(self, fps, lattice: Grid, cfg: ZoomConfig = None, bounds=None,
                         init_ms=None, dictionary=None, trace: bool = False):
        """quantify_impl with per-voxel index bounds (V,6) and initial T1/T2 ms (V,2)."""
        q = np.ascontiguousarray(np.atleast_2d(fps), dtype=np.complex128)
        cfg = cfg or zoom_config()
        out = (Quant * q.shape[0])()
        b = None if bounds is None else np.ascontiguousarray(bounds, dtype=np.int64)
        i = None if init_ms is None else np.ascontiguousarray(init_ms, dtype=np.float64)
        io, keep = self._zoom_io(q.shape[0], dictionary, trace)
        check(self.lib.mrfg_quantify_ex(
            self.h, C.byref(lattice), C.byref(cfg), _dp(q.view(np.float64)), q.shape[0],
            None if b is None else b.ctypes.data_as(C.POINTER(C.c_int64)),
            None if i is None else _dp(i), None if io is None else C.byref(io), out))
        res = quant_array(out)
        return (res, self._traces(keep[1], range(q.shape[0]))) if trace else res

    def quantify_slice(self, fps, mask, nx: int, ny: int, lattice: Grid,
                       cfg: ZoomConfig = None, use_prior: int = 0, dictionary=None, trace: bool = False):
        """quantify_slice (zoom.cpp:555-629).  use_prior: 0/False none, 1/True the
        reference's raster order, 2 the row-wavefront relaxation.
        Returns (Quant records, seconds) [+ per-voxel StageLog lists with trace]."""
        q = np.ascontiguousarray(fps, dtype=np.complex128)
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        cfg = cfg or zoom_config()
        out = (Quant * (nx * ny))()
        secs = C.c_double()
        io, keep = self._zoom_io(nx * ny, dictionary, trace)
        check(self.lib.mrfg_quantify_slice_ex(self.h, C.byref(lattice), C.byref(cfg),
                                              _dp(q.view(np.float64)),
                                              m.ctypes.data_as(C.POINTER(C.c_uint8)), nx, ny,
                                              int(use_prior), None if io is None else C.byref(io), out,
                                              C.byref(secs)))
        res = quant_array(out)
        if trace:
            return res, secs.value, self._traces(keep[1], range(nx * ny))
        return res, secs.value


def quantify_b1(contexts, fps, lattice: Grid, cfg: ZoomConfig = None, steps=(4, 1), init_ib: int = 0):
    """Four-parameter MRF-ZOOM (BASELINE configs[4]): contexts[ib] holds the
    schedule with flips scaled by the ib-th B1 value; an outer zoom_1d over
    the B1 index (steps in index units) of the three-parameter quantify
    (mrfg_quantify_b1).  Returns (Quant records, chosen B1 indices)."""
    q = np.ascontiguousarray(np.atleast_2d(fps), dtype=np.complex128)
    cfg = cfg or zoom_config()
    hs = (C.c_void_p * len(contexts))(*[c.h for c in contexts])
    st = np.ascontiguousarray(steps, dtype=np.int64)
    out = (Quant * q.shape[0])()
    ib = np.zeros(q.shape[0], dtype=np.int64)
    check(N.load().mrfg_quantify_b1(hs, len(contexts), C.byref(lattice), C.byref(cfg),
                                    st.ctypes.data_as(C.POINTER(C.c_int64)), len(st), int(init_ib),
                                    _dp(q.view(np.float64)), q.shape[0], out,
                                    ib.ctypes.data_as(C.POINTER(C.c_int64))))
    return quant_array(out), ib


QUANT_DTYPE = np.dtype([("i1", np.int64), ("i2", np.int64), ("idf", np.int64),
                        ("t1_ms", np.float64), ("t2_ms", np.float64), ("df_hz", np.float64),
                        ("pd", np.float64), ("score", np.float64), ("evaluations", np.int64)])


def quant_array(buf) -> np.ndarray:
    return np.frombuffer(buf, dtype=QUANT_DTYPE).copy()
