"""CPU oracles -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/oracle_api.h`` for:

* ``Oracle("restatement")`` -> ``oracle/liboracle.so``: the plain-C restatement of
  the reference algorithm (``oracle/mrf_oracle.c``);
* ``Oracle("reference")``   -> ``oracle/_ref/libmrf_ref.so``: the reference library
  compiled from ``/root/reference/proj/src`` (only where it was built).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libmrf_ref.so"),
}


class Axis(C.Structure):
    _fields_ = [("min", C.c_double), ("step", C.c_double), ("count", C.c_int64)]


class Grid(C.Structure):
    _fields_ = [("t1_ms", Axis), ("t2_ms", Axis), ("df_hz", Axis)]


class Sched(C.Structure):
    _fields_ = [("n", C.c_int64), ("flip_deg", C.POINTER(C.c_double)),
                ("phase_deg", C.POINTER(C.c_double)), ("tr_ms", C.POINTER(C.c_double)),
                ("te_ms", C.POINTER(C.c_double))]


class ZoomCfg(C.Structure):
    _fields_ = [("metric", C.c_int32), ("final_metric", C.c_int32), ("smooth_k", C.c_int32),
                ("n2d", C.c_int32), ("n1d", C.c_int32), ("dict_mode", C.c_int32),
                ("omega_hz", C.c_double), ("df_coarse_hz", C.c_double),
                ("df_refine_hz", C.c_double), ("df_window_hz", C.c_double),
                ("plateau_eps", C.c_double), ("heavy_noise_cc", C.c_double),
                ("fallback_coarse_hz", C.c_double), ("fallback_window_hz", C.c_double),
                ("t1t2_2d_steps_ms", C.c_double * 8), ("t1t2_1d_steps_ms", C.c_double * 8),
                ("final_2d_step_ms", C.c_double), ("init_t1_ms", C.c_double),
                ("init_t2_ms", C.c_double), ("prior_window_t1_ms", C.c_double),
                ("prior_window_t2_ms", C.c_double), ("prior_window_df_hz", C.c_double)]


class Stage(C.Structure):
    """StageLog (zoom.hpp:54-59); stage codes in STAGE_NAMES order."""
    _fields_ = [("stage", C.c_int32), ("pad", C.c_int32), ("evaluations", C.c_int64), ("best", C.c_double),
                ("t1_ms", C.c_double), ("t2_ms", C.c_double), ("df_hz", C.c_double)]


STAGE_NAMES = ("df.coarse", "df.refine", "df.translate", "df.rerefine", "df.plateau_stop", "df.finest",
               "df.fallback", "t1t2.2d", "df.sweep", "t1.1d", "t2.1d", "t1t2.final")


class Quant(C.Structure):
    _fields_ = [("i1", C.c_int64), ("i2", C.c_int64), ("idf", C.c_int64),
                ("t1_ms", C.c_double), ("t2_ms", C.c_double), ("df_hz", C.c_double),
                ("pd", C.c_double), ("score", C.c_double), ("evaluations", C.c_int64)]


@dataclass
class Schedule:
    flip_deg: np.ndarray
    phase_deg: np.ndarray
    tr_ms: np.ndarray
    te_ms: np.ndarray

    @property
    def n(self) -> int:
        return len(self.flip_deg)

    def c(self) -> Sched:
        for a in (self.flip_deg, self.phase_deg, self.tr_ms, self.te_ms):
            assert a.dtype == np.float64 and a.flags.c_contiguous
        dp = C.POINTER(C.c_double)
        return Sched(self.n, self.flip_deg.ctypes.data_as(dp), self.phase_deg.ctypes.data_as(dp),
                     self.tr_ms.ctypes.data_as(dp), self.te_ms.ctypes.data_as(dp))


def make_grid(t1, t2, df) -> Grid:
    """Each axis is (min, step, count)."""
    return Grid(Axis(*t1), Axis(*t2), Axis(*df))


def zoom_cfg(**kw) -> ZoomCfg:
    """ZoomConfig defaults (zoom.hpp:23-52), overridable by keyword."""
    d = dict(metric=0, final_metric=0, smooth_k=0, omega_hz=70.0, df_coarse_hz=60.0,
             df_refine_hz=3.0, df_window_hz=150.0, plateau_eps=1e-7, heavy_noise_cc=0.1,
             fallback_coarse_hz=30.0, fallback_window_hz=300.0,
             t1t2_2d_steps_ms=[200.0, 100.0], t1t2_1d_steps_ms=[100.0, 50.0, 20.0, 10.0],
             final_2d_step_ms=1.0, init_t1_ms=1000.0, init_t2_ms=500.0,
             prior_window_t1_ms=3000.0, prior_window_t2_ms=800.0, prior_window_df_hz=150.0)
    d.update(kw)
    c = ZoomCfg()
    for k, v in d.items():
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


def build(quiet: bool = True) -> None:
    """Compile the oracles (restatement always; reference when its sources exist)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    # the CLI parity harness needs the drop-in libraries (built by the
    # package's build.py); skipped until they exist
    pkg = os.path.join(os.path.dirname(HERE), "paper_1506_05393_b200")
    if os.path.exists(os.path.join(pkg, "libmrf_b200.so")):
        subprocess.run(["make", "-C", HERE, "cli"], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)


def available(which: str) -> bool:
    return os.path.exists(LIBS[which])


class Oracle:
    def __init__(self, which: str = "restatement"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.which = which
        L = self.lib = C.CDLL(path)
        dp, i64 = C.POINTER(C.c_double), C.c_int64
        L.orc_last_error.restype = C.c_char_p
        L.orc_impl_name.restype = C.c_char_p
        L.orc_cc.restype = C.c_double
        for name in ("orc_build_schedule", "orc_baseline_schedule"):
            getattr(L, name).argtypes = [i64, C.c_uint64, dp, dp, dp, dp]
        L.orc_simulate.argtypes = [C.POINTER(Sched), C.c_double, C.c_double, C.c_double, dp]
        L.orc_add_noise.argtypes = [dp, i64, C.c_double, C.c_uint64, dp]
        L.orc_cc.argtypes = [dp, dp, i64]
        L.orc_cc_unit.restype = C.c_double
        L.orc_cc_unit.argtypes = [dp, dp, i64]
        L.orc_generate.argtypes = [C.POINTER(Sched), C.POINTER(Grid), i64, i64,
                                   C.POINTER(C.c_float)]
        L.orc_scan_grid.argtypes = [C.POINTER(Sched), C.POINTER(Grid), dp, i64, C.c_int,
                                    C.c_int, C.POINTER(i64), dp, dp]
        L.orc_scan_grid_ex.argtypes = [C.POINTER(Sched), C.POINTER(Grid), dp, C.POINTER(C.c_uint8), i64,
                                       C.c_int, C.c_int, C.POINTER(i64), dp, dp]
        L.orc_quantify.argtypes = [C.POINTER(Sched), C.POINTER(Grid), C.POINTER(ZoomCfg), dp,
                                   C.POINTER(Quant)]
        L.orc_quantify_b1.argtypes = [C.POINTER(Sched), C.c_int, C.POINTER(Grid), C.POINTER(ZoomCfg),
                                      C.POINTER(C.c_int64), C.c_int, C.c_int64, dp, C.POINTER(Quant),
                                      C.POINTER(C.c_int64)]
        L.orc_quantify_ex.argtypes = [C.POINTER(Sched), C.POINTER(Grid), C.POINTER(ZoomCfg), dp,
                                      C.POINTER(C.c_float), i64, C.POINTER(Stage), C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(Quant)]
        L.orc_quantify_slice.argtypes = [C.POINTER(Sched), C.POINTER(Grid),
                                         C.POINTER(ZoomCfg), dp, C.POINTER(C.c_uint8),
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Quant)]

        u64 = C.c_uint64
        L.orc_calibrate_noise.argtypes = [dp, i64, C.c_double, u64, dp]
        L.orc_make_calibrated_noise.argtypes = [dp, i64, C.c_double, u64, dp, C.POINTER(u64), dp]
        L.orc_smooth.argtypes = [dp, i64, C.c_int, dp]
        if which == "reference":
            L.orc_ref_save_generated.argtypes = [C.POINTER(Sched), C.POINTER(Grid), C.c_char_p]
            L.orc_ref_cc_map_to_file.argtypes = [C.POINTER(Sched), C.POINTER(Grid), dp, C.c_char_p]
            L.orc_ref_scan_rows.argtypes = [C.POINTER(Sched), dp, i64, dp, i64, C.POINTER(Axis), dp, i64,
                                            C.c_int, C.c_int, C.POINTER(i64), dp]

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise RuntimeError(f"{self.which} oracle: {self.lib.orc_last_error().decode()}")

    @staticmethod
    def _dp(a: np.ndarray):
        return a.ctypes.data_as(C.POINTER(C.c_double))

    def _sched(self, fn, n: int, seed: int) -> Schedule:
        arrs = [np.zeros(n) for _ in range(4)]
        self._check(fn(n, seed, *[self._dp(a) for a in arrs]))
        return Schedule(*arrs)

    def build_schedule(self, n: int, seed: int) -> Schedule:
        return self._sched(self.lib.orc_build_schedule, n, seed)

    def baseline_schedule(self, n: int, seed: int = 1) -> Schedule:
        return self._sched(self.lib.orc_baseline_schedule, n, seed)

    def simulate(self, s: Schedule, t1_s: float, t2_s: float, df_hz: float) -> np.ndarray:
        out = np.zeros(2 * s.n)
        cs = s.c()
        self._check(self.lib.orc_simulate(C.byref(cs), t1_s, t2_s, df_hz, self._dp(out)))
        return out.view(np.complex128)

    def add_noise(self, fp: np.ndarray, sigma: float, seed: int) -> np.ndarray:
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        out = np.zeros_like(fp)
        self._check(self.lib.orc_add_noise(self._dp(fp.view(np.float64)), len(fp), sigma, seed,
                                           self._dp(out.view(np.float64))))
        return out

    def cc(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        return self.lib.orc_cc(self._dp(a.view(np.float64)), self._dp(b.view(np.float64)), len(a))

    def cc_unit(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        return self.lib.orc_cc_unit(self._dp(a.view(np.float64)), self._dp(b.view(np.float64)), len(a))

    def calibrate_noise(self, fp: np.ndarray, target: float, seed: int):
        """-> sigma, or None when the reference throws runtime_error (code -3)."""
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        sg = C.c_double()
        rc = self.lib.orc_calibrate_noise(self._dp(fp.view(np.float64)), len(fp), target, seed, C.byref(sg))
        if rc == -3:
            return None
        self._check(rc)
        return sg.value

    def make_calibrated_noise(self, fp: np.ndarray, target: float, seed: int):
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        sg, used = C.c_double(), C.c_uint64()
        out = np.zeros_like(fp)
        rc = self.lib.orc_make_calibrated_noise(self._dp(fp.view(np.float64)), len(fp), target, seed,
                                                C.byref(sg), C.byref(used), self._dp(out.view(np.float64)))
        if rc == -3:
            return None
        self._check(rc)
        return sg.value, used.value, out

    def smooth(self, fp: np.ndarray, k: int) -> np.ndarray:
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        out = np.zeros_like(fp)
        self._check(self.lib.orc_smooth(self._dp(fp.view(np.float64)), len(fp), k,
                                        self._dp(out.view(np.float64))))
        return out

    def save_generated(self, s: Schedule, g: Grid, path: str) -> None:
        """Reference library only: mrf::save_generated (dictionary.cpp:216-239)."""
        cs = s.c()
        self._check(self.lib.orc_ref_save_generated(C.byref(cs), C.byref(g), str(path).encode()))

    def cc_map_to_file(self, s: Schedule, g: Grid, fp: np.ndarray, path: str) -> None:
        """Reference library only: mrf::cc_map_to_file (dictionary.cpp:333-347)."""
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        cs = s.c()
        self._check(self.lib.orc_ref_cc_map_to_file(C.byref(cs), C.byref(g), self._dp(fp.view(np.float64)),
                                                    str(path).encode()))

    def scan_rows(self, s: Schedule, t1_ms: np.ndarray, t2_ms: np.ndarray, df: tuple,
                  queries: np.ndarray, metric: int = 0, threads: int = 0):
        """Reference library only: argmax over explicit T1 x T2 values x a linear
        df axis (min, step, count) with mrf::generate rows + mrf::brute_force_search
        (ref_capi.cpp orc_ref_scan_rows).  -> (flat, score)."""
        q = np.ascontiguousarray(queries, dtype=np.complex128)
        t1 = np.ascontiguousarray(t1_ms, dtype=np.float64)
        t2 = np.ascontiguousarray(t2_ms, dtype=np.float64)
        nq = q.shape[0]
        flat = np.zeros(nq, dtype=np.int64)
        score = np.zeros(nq)
        cs = s.c()
        ax = Axis(*df)
        self._check(self.lib.orc_ref_scan_rows(
            C.byref(cs), self._dp(t1), len(t1), self._dp(t2), len(t2), C.byref(ax),
            self._dp(q.view(np.float64)), nq, metric, threads or os.cpu_count() or 1,
            flat.ctypes.data_as(C.POINTER(C.c_int64)), self._dp(score)))
        return flat, score

    def generate(self, s: Schedule, g: Grid, first: int, count: int) -> np.ndarray:
        out = np.zeros((count, 2 * s.n), dtype=np.float32)
        cs = s.c()
        self._check(self.lib.orc_generate(C.byref(cs), C.byref(g), first, count,
                                          out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def scan_grid(self, s: Schedule, g: Grid, queries: np.ndarray, metric: int = 0,
                  threads: int = 0, unit_norm=None):
        """unit_norm: None, or per-query flags (Fingerprint::unit_norm: used as given)."""
        q = np.ascontiguousarray(queries, dtype=np.complex128)
        nq = q.shape[0]
        flat = np.zeros(nq, dtype=np.int64)
        score = np.zeros(nq)
        second = np.zeros(nq)
        cs = s.c()
        threads = threads or os.cpu_count() or 1
        unit = None
        if unit_norm is not None:
            unit = np.ascontiguousarray(np.broadcast_to(np.asarray(unit_norm, dtype=np.uint8), (nq,)))
        self._check(self.lib.orc_scan_grid_ex(C.byref(cs), C.byref(g), self._dp(q.view(np.float64)),
                                              None if unit is None else unit.ctypes.data_as(C.POINTER(C.c_uint8)),
                                              nq, metric, threads,
                                              flat.ctypes.data_as(C.POINTER(C.c_int64)),
                                              self._dp(score), self._dp(second)))
        return flat, score, second

    def quantify(self, s: Schedule, g: Grid, cfg: ZoomCfg, fp: np.ndarray) -> Quant:
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        out = Quant()
        cs = s.c()
        self._check(self.lib.orc_quantify(C.byref(cs), C.byref(g), C.byref(cfg),
                                          self._dp(fp.view(np.float64)), C.byref(out)))
        return out

    def quantify_ex(self, s: Schedule, g: Grid, cfg: ZoomCfg, fp: np.ndarray, dict_payload=None):
        """quantify with an explicit dictionary payload (float32 entries x 2N,
        or None) -> (Quant, list of (stage name, evaluations, best, t1_ms, t2_ms, df_hz))."""
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        out = Quant()
        cs = s.c()
        cap = 256
        tr = (Stage * cap)()
        ntr = C.c_int(0)
        d = None
        nd = 0
        if dict_payload is not None:
            d = np.ascontiguousarray(dict_payload, dtype=np.float32).reshape(-1, 2 * s.n)
            nd = d.shape[0]
        self._check(self.lib.orc_quantify_ex(
            C.byref(cs), C.byref(g), C.byref(cfg), self._dp(fp.view(np.float64)),
            None if d is None else d.ctypes.data_as(C.POINTER(C.c_float)), nd, tr, cap, C.byref(ntr),
            C.byref(out)))
        trace = [(STAGE_NAMES[tr[k].stage], tr[k].evaluations, tr[k].best, tr[k].t1_ms, tr[k].t2_ms,
                  tr[k].df_hz) for k in range(min(ntr.value, cap))]
        return out, trace

    def quantify_b1(self, scheds, g: Grid, cfg: ZoomCfg, fp: np.ndarray, steps, init_ib: int):
        """Four-parameter ZOOM (oracle_api.h orc_quantify_b1) -> (Quant, ib)."""
        fp = np.ascontiguousarray(fp, dtype=np.complex128)
        cs = (Sched * len(scheds))(*[x.c() for x in scheds])
        st = np.ascontiguousarray(steps, dtype=np.int64)
        out = Quant()
        ib = C.c_int64(-1)
        self._check(self.lib.orc_quantify_b1(cs, len(scheds), C.byref(g), C.byref(cfg),
                                             st.ctypes.data_as(C.POINTER(C.c_int64)), len(st), init_ib,
                                             self._dp(fp.view(np.float64)), C.byref(out), C.byref(ib)))
        return out, ib.value

    def quantify_slice(self, s: Schedule, g: Grid, cfg: ZoomCfg, fps: np.ndarray,
                       mask: np.ndarray, nx: int, ny: int, use_prior: bool, threads: int = 0):
        fps = np.ascontiguousarray(fps, dtype=np.complex128)
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        out = (Quant * (nx * ny))()
        cs = s.c()
        threads = threads or os.cpu_count() or 1
        self._check(self.lib.orc_quantify_slice(
            C.byref(cs), C.byref(g), C.byref(cfg), self._dp(fps.view(np.float64)),
            mask.ctypes.data_as(C.POINTER(C.c_uint8)), nx, ny, int(use_prior), threads, out))
        return out
