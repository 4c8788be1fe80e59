"""ctypes binding of the C ABI in include/mrfg.h (paper_1506_05393_b200/libmrfg.so).

The extension is built in-tree by ``paper_1506_05393_b200/build.py`` (called by
``__graft_entry__.build()``).  Importing this module without the shared
library fails loudly: there is no CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmrfg.so")


class Axis(C.Structure):
    """AxisSpec (reference dictionary.hpp:17-24)."""
    _fields_ = [("min", C.c_double), ("step", C.c_double), ("count", C.c_int64),
                ("values", C.POINTER(C.c_double))]  # optional explicit values (log axes)


class Grid(C.Structure):
    """ParameterGrid (reference dictionary.hpp:34-56)."""
    _fields_ = [("t1_ms", Axis), ("t2_ms", Axis), ("df_hz", Axis)]


class Match(C.Structure):
    _fields_ = [("flat", C.c_int64), ("score", C.c_double)]


class ScanOpts(C.Structure):
    _fields_ = [("delta", C.c_double), ("chunk_atoms", C.c_int64), ("cand_capacity", C.c_int64),
                ("seed_atoms", C.c_int64), ("floor_matches", C.c_void_p),
                ("unit_queries", C.POINTER(C.c_uint8))]


class ScanStats(C.Structure):
    _fields_ = [("atoms", C.c_int64), ("voxels", C.c_int64), ("chunks", C.c_int64),
                ("candidates", C.c_int64), ("reranked", C.c_int64),
                ("overflow_passes", C.c_int64), ("bloch_ms", C.c_double),
                ("gemm_ms", C.c_double), ("rerank_ms", C.c_double), ("total_ms", C.c_double),
                ("gemm_kernel_ms_avg", C.c_double), ("gemm_launches", C.c_int64),
                ("screen_err_max", C.c_double), ("rescreened32", C.c_int64),
                ("screen_err_audit_max", C.c_double), ("rescreen_err_audit_max", C.c_double),
                ("delta_used", C.c_double), ("audit_samples", C.c_int64), ("rescans", C.c_int64),
                ("rescreen_err_max", C.c_double), ("chunk_atoms", C.c_int64),
                ("project_ms", C.c_double), ("subspace_rank", C.c_int64),
                ("subspace_residual_max", C.c_double), ("subspace_residual_device", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ZoomConfig(C.Structure):
    """ZoomConfig (reference zoom.hpp:23-52)."""
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


class Quant(C.Structure):
    """QuantResult (reference zoom.hpp:61-67) plus lattice indices."""
    _fields_ = [("i1", C.c_int64), ("i2", C.c_int64), ("idf", C.c_int64),
                ("t1_ms", C.c_double), ("t2_ms", C.c_double), ("df_hz", C.c_double),
                ("pd", C.c_double), ("score", C.c_double), ("evaluations", C.c_int64)]


class Stage(C.Structure):
    """StageLog (reference zoom.hpp:54-59); stage codes in STAGE_NAMES order."""
    _fields_ = [("stage", C.c_int32), ("pad", C.c_int32), ("evaluations", C.c_int64), ("best", C.c_double),
                ("t1_ms", C.c_double), ("t2_ms", C.c_double), ("df_hz", C.c_double)]


STAGE_NAMES = ("df.coarse", "df.refine", "df.translate", "df.rerefine", "df.plateau_stop", "df.finest",
               "df.fallback", "t1t2.2d", "df.sweep", "t1.1d", "t2.1d", "t1t2.final")
TRACE_MAX = 64  # MRFG_TRACE_MAX


class ZoomIo(C.Structure):
    """mrfg_zoom_io: dictionary payload and StageLog outputs."""
    _fields_ = [("dict", C.c_void_p), ("dict_entries", C.c_int64), ("dict_on_device", C.c_int32),
                ("pad", C.c_int32), ("trace", C.c_void_p), ("trace_len", C.c_void_p)]


EXPORTS = [
    "mrfg_last_error", "mrfg_version", "mrfg_zoom_config_default", "mrfg_reference_schedule",
    "mrfg_baseline_schedule", "mrfg_add_noise", "mrfg_rng_at", "mrfg_rng_uniform01",
    "mrfg_rng_gaussian", "mrfg_axis_count", "mrfg_create", "mrfg_destroy", "mrfg_length",
    "mrfg_set_stream", "mrfg_synchronize", "mrfg_simulate", "mrfg_simulate_dev", "mrfg_generate",
    "mrfg_generate_dev", "mrfg_bloch_norms_dev", "mrfg_scan_grid", "mrfg_scan_grid_dev",
    "mrfg_scan_dict", "mrfg_scan_dict_dev", "mrfg_scan_seed_dev",
    "mrfg_merge_matches_dev", "mrfg_screen_scores", "mrfg_cc_map", "mrfg_quantify", "mrfg_quantify_slice", "mrfg_quantify_bounded",
    "mrfg_quantify_dev", "mrfg_cc_map_ex", "mrfg_save_generated", "mrfg_cc_map_to_file",
    "mrfg_write_header", "mrfg_read_header", "mrfg_calibrate_noise", "mrfg_make_calibrated_noise",
    "mrfg_smooth", "mrfg_quantify_ex", "mrfg_quantify_slice_ex", "mrfg_quantify_b1",
]

_lib = None


def load() -> C.CDLL:
    """Load libmrfg.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1506_05393_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    dp, i64, u64, vp = C.POINTER(C.c_double), C.c_int64, C.c_uint64, C.c_void_p
    L.mrfg_last_error.restype = C.c_char_p
    L.mrfg_version.restype = C.c_char_p
    L.mrfg_zoom_config_default.argtypes = [C.POINTER(ZoomConfig)]
    L.mrfg_zoom_config_default.restype = None
    for name in ("mrfg_reference_schedule", "mrfg_baseline_schedule"):
        getattr(L, name).argtypes = [i64, u64, dp, dp, dp, dp]
    L.mrfg_add_noise.argtypes = [dp, i64, C.c_double, u64, dp]
    L.mrfg_rng_at.argtypes = [u64, u64, u64]
    L.mrfg_rng_at.restype = u64
    L.mrfg_rng_uniform01.argtypes = [u64, u64, u64]
    L.mrfg_rng_uniform01.restype = C.c_double
    L.mrfg_rng_gaussian.argtypes = [u64, u64, u64]
    L.mrfg_rng_gaussian.restype = C.c_double
    L.mrfg_axis_count.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(i64)]
    L.mrfg_create.argtypes = [dp, dp, dp, dp, i64, C.c_int, C.POINTER(vp)]
    L.mrfg_destroy.argtypes = [vp]
    L.mrfg_length.argtypes = [vp]
    L.mrfg_length.restype = i64
    L.mrfg_set_stream.argtypes = [vp, vp]
    L.mrfg_synchronize.argtypes = [vp]
    L.mrfg_simulate.argtypes = [vp, dp, i64, C.c_int, C.c_int, dp]
    L.mrfg_simulate_dev.argtypes = [vp, vp, i64, C.c_int, C.c_int, vp]
    L.mrfg_generate.argtypes = [vp, C.POINTER(Grid), i64, i64, C.c_int, C.POINTER(C.c_float)]
    L.mrfg_generate_dev.argtypes = [vp, C.POINTER(Grid), i64, i64, C.c_int, vp]
    L.mrfg_bloch_norms_dev.argtypes = [vp, C.POINTER(Grid), i64, i64, vp]
    L.mrfg_scan_grid.argtypes = [vp, C.POINTER(Grid), i64, i64, dp, i64, C.c_int,
                                 C.POINTER(ScanOpts), C.POINTER(Match), C.POINTER(ScanStats)]
    L.mrfg_scan_grid_dev.argtypes = [vp, C.POINTER(Grid), i64, i64, vp, i64, C.c_int,
                                     C.POINTER(ScanOpts), vp, C.POINTER(ScanStats)]
    L.mrfg_scan_dict.argtypes = [vp, C.POINTER(C.c_float), i64, dp, i64, C.c_int,
                                 C.POINTER(ScanOpts), C.POINTER(Match), C.POINTER(ScanStats)]
    L.mrfg_scan_dict_dev.argtypes = [vp, vp, i64, i64, i64, vp, i64, C.c_int,
                                     C.POINTER(ScanOpts), vp, C.POINTER(ScanStats)]
    L.mrfg_scan_seed_dev.argtypes = [vp, C.POINTER(Grid), vp, i64, i64, i64, vp, i64, C.c_int,
                                     C.POINTER(ScanOpts), vp, C.POINTER(ScanStats)]
    L.mrfg_merge_matches_dev.argtypes = [vp, vp, C.c_int, i64, vp]
    L.mrfg_screen_scores.argtypes = [vp, C.POINTER(Grid), i64, i64, dp, i64, C.c_int, C.c_int,
                                     C.POINTER(C.c_float)]
    L.mrfg_cc_map.argtypes = [vp, C.POINTER(Grid), dp, i64, i64, C.POINTER(C.c_float)]
    L.mrfg_cc_map_ex.argtypes = [vp, C.POINTER(Grid), dp, i64, i64, C.c_int, C.POINTER(C.c_float)]
    u8p, cp = C.POINTER(C.c_uint8), C.c_char_p
    L.mrfg_save_generated.argtypes = [vp, C.POINTER(Grid), u8p, cp, i64, C.c_int]
    L.mrfg_cc_map_to_file.argtypes = [vp, C.POINTER(Grid), dp, u8p, cp, C.c_int]
    L.mrfg_write_header.argtypes = [cp, cp, C.POINTER(Grid), u8p, i64]
    L.mrfg_read_header.argtypes = [cp, cp, C.POINTER(Grid), u8p, C.POINTER(i64), C.POINTER(i64)]
    L.mrfg_calibrate_noise.argtypes = [dp, i64, C.c_double, u64, dp]
    L.mrfg_make_calibrated_noise.argtypes = [dp, i64, C.c_double, u64, dp, C.POINTER(u64), dp]
    L.mrfg_smooth.argtypes = [dp, i64, C.c_int, dp]
    L.mrfg_quantify.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), dp, i64,
                                C.POINTER(Quant)]
    L.mrfg_quantify_dev.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), vp, i64, vp]
    L.mrfg_quantify_bounded.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), dp, i64,
                                        C.POINTER(i64), dp, C.POINTER(Quant)]
    L.mrfg_quantify_slice.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), dp,
                                      C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                      C.POINTER(Quant), dp]
    L.mrfg_quantify_b1.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(Grid), C.POINTER(ZoomConfig),
                                   C.POINTER(i64), C.c_int, i64, dp, i64, C.POINTER(Quant), C.POINTER(i64)]
    L.mrfg_quantify_ex.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), dp, i64,
                                   C.POINTER(i64), dp, C.POINTER(ZoomIo), C.POINTER(Quant)]
    L.mrfg_quantify_slice_ex.argtypes = [vp, C.POINTER(Grid), C.POINTER(ZoomConfig), dp,
                                         C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                         C.POINTER(ZoomIo), C.POINTER(Quant), dp]
    _lib = L
    return L


class MrfgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(MrfgError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(MrfgError, IndexError):
    """std::out_of_range in the reference."""


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().mrfg_last_error().decode()
    if rc == -1:
        raise InvalidArgument(rc, msg)
    if rc == -2:
        raise OutOfRange(rc, msg)
    raise MrfgError(rc, msg)
