"""CPU-side checks of the product boundary (no GPU compute).

* libmrfg.so loads and exports every function include/mrfg.h declares;
* the host-side input synthesis (schedules, rng, add_noise, axis rule) equals
  the oracle bit-for-bit;
* argument validation that happens before any device work matches the
  reference's error behaviour; without an sm_100 device every compute entry
  fails loudly (no CPU fallback).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import _native as N
from paper_1506_05393_b200._native import InvalidArgument, MrfgError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mrfg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mrfg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(N.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(N.EXPORTS)


def test_baseline_schedule_matches_oracle(orc):
    for n, seed in ((500, 1), (1000, 1), (3000, 1), (37, 9)):
        a, b = P.baseline_schedule(n, seed), orc.baseline_schedule(n, seed)
        for k in ("flip_deg", "phase_deg", "tr_ms", "te_ms"):
            assert np.array_equal(getattr(a, k), getattr(b, k))


def test_reference_schedule_and_digest(orc):
    s = P.reference_schedule(500, 1)
    o = orc.build_schedule(500, 1)
    assert np.array_equal(s.flip_deg, o.flip_deg) and np.array_equal(s.tr_ms, o.tr_ms)
    assert s.digest() == "99b129a4b97065d83595554534b6434b0c5cbe05b7223af5981b79ec6965bc8e"


def test_add_noise_matches_oracle(orc):
    fp = orc.simulate(orc.baseline_schedule(200, 1), 1.0, 0.2, 3.0)
    for sigma, seed in ((0.0, 1), (0.01, 5), (0.3, 1_000_123)):
        assert np.array_equal(P.add_noise(fp, sigma, seed), orc.add_noise(fp, sigma, seed))
    with pytest.raises(InvalidArgument):
        P.add_noise(fp, -1.0, 1)


def test_rng_streams():
    # rng.hpp: uniform in [0,1), deterministic per (seed, stream, index)
    u = [P.dgs.uniform01(7, 20, k) for k in range(1000)]
    assert min(u) >= 0 and max(u) < 1
    assert P.dgs.rng_at(7, 20, 3) == P.dgs.rng_at(7, 20, 3)
    assert P.dgs.rng_at(7, 20, 3) != P.dgs.rng_at(7, 21, 3)
    g = np.array([P.dgs.gaussian(1, 3, k) for k in range(4000)])
    assert abs(g.mean()) < 0.06 and abs(g.std() - 1) < 0.05


def test_axis_count_rule():
    """test_dictionary.cpp:37-55."""
    g = P.grid_from_ranges((100, 5500, 10), (50, 1200, 10), (-300, 300, 1))
    assert (g.t1_ms.count, g.t2_ms.count, g.df_hz.count) == (540, 115, 600)
    assert P.grid_total(g) == 37_260_000
    assert P.grid_total(P.grid_from_ranges((500, 2000, 10), (200, 800, 10), (-30, 450, 2))) == 2_160_000
    f = P.grid_from_ranges((0.1, 0.4, 0.1), (1, 2, 0.25), (0, 1, 0.2))
    assert (f.t1_ms.count, f.t2_ms.count, f.df_hz.count) == (3, 4, 5)
    with pytest.raises(InvalidArgument):
        P.grid_from_ranges((100, 100, 10), (50, 1200, 10), (-300, 300, 1))
    with pytest.raises(InvalidArgument):
        P.grid_from_ranges((100, 200, 0), (50, 1200, 10), (-300, 300, 1))
    # BASELINE configs (endpoint-inclusive)
    assert P.grid_total(P.grid_inclusive((100, 2000, 20), (20, 300, 10), (-50, 50, 5))) == 58_464
    assert P.grid_total(P.grid_inclusive((100, 5000, 10), (20, 2000, 5), (-250, 250, 1))) == 97_658_427


def test_flat_ordering():
    """test_dictionary.cpp:57-73: T1 outer, T2 middle, df inner."""
    g = P.grid((600, 100, 3), (80, 20, 3), (-10, 10, 3))
    flat = np.arange(27)
    i1, i2, idf = P.unflatten(g, flat)
    assert np.array_equal((i1 * 3 + i2) * 3 + idf, flat)
    t1, t2, df = P.params_at(g, 1, 2, 0)
    assert t1 == pytest.approx(0.7) and t2 == pytest.approx(0.12) and df == -10.0


def test_context_rejects_bad_timing_before_device_use():
    s = P.baseline_schedule(8, 1)
    s.te_ms[3] = s.tr_ms[3] + 1.0  # bloch.cpp:97-99
    with pytest.raises(InvalidArgument):
        P.Context(s)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(MrfgError) as e:
        P.Context(P.baseline_schedule(16, 1))
    assert e.value.code == -4


def test_zoom_config_defaults():
    c = P.zoom_config()
    assert (c.omega_hz, c.df_coarse_hz, c.df_refine_hz, c.df_window_hz) == (70, 60, 3, 150)
    assert list(c.t1t2_2d_steps_ms[:c.n2d]) == [200, 100]
    assert list(c.t1t2_1d_steps_ms[:c.n1d]) == [100, 50, 20, 10]
    assert (c.final_2d_step_ms, c.init_t1_ms, c.init_t2_ms) == (1, 1000, 500)
