"""B200-native MRF dictionary generating-and-searching (DGS) path.

sm_100a CUDA kernels behind the C ABI of include/mrfg.h (libmrfg.so, built
in-tree by ``paper_1506_05393_b200/build.py``), with a host-side mirror of the
reference library's interface in :mod:`paper_1506_05393_b200.dgs`.
"""
from . import dgs  # noqa: F401
from ._native import LIB_PATH, load  # noqa: F401
from .dgs import (Context, Schedule, add_noise, baseline_schedule, grid, grid_from_ranges,  # noqa: F401
                  grid_inclusive, grid_total, params_at, reference_schedule, unflatten,
                  zoom_config, calibrate_noise, make_calibrated_noise, smooth, read_header,
                  save_dictionary, load_dictionary, load_cc_map, grid_values, axis_values, quantify_b1)

__all__ = ["Context", "Schedule", "add_noise", "baseline_schedule", "grid", "grid_from_ranges",
           "grid_inclusive", "grid_total", "params_at", "reference_schedule", "unflatten",
           "zoom_config", "load", "LIB_PATH", "dgs", "calibrate_noise", "make_calibrated_noise",
           "smooth", "read_header", "save_dictionary", "load_dictionary", "load_cc_map",
           "grid_values", "axis_values", "quantify_b1"]
