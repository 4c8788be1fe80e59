"""Pin the CPU oracle (test infrastructure) before trusting it.

1. The C restatement (oracle/liboracle.so) is bit-identical to the reference
   library compiled from /root/reference (oracle/_ref) -- skipped where the
   reference was not built.
2. The restatement reproduces the reference's RECORDED outputs (committed
   fixtures under tests/golden/, made by tests/golden/make_golden.py):
   the build_schedule(500, 1) digest, runs/exp1 CC values at %.9g, runs/exp2
   MRF-ZOOM answers and evaluation counts, runs/exp3 64x64 slice maps and
   per-voxel evaluation counts.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def digest(s):
    csv = "idx,flip_deg,phase_deg,tr_ms,te_ms\n" + "".join(
        f"{k},{s.flip_deg[k]:.9g},{s.phase_deg[k]:.9g},{s.tr_ms[k]:.9g},{s.te_ms[k]:.9g}\n"
        for k in range(s.n))
    return hashlib.sha256(csv.encode()).hexdigest()


def test_schedule_digest_golden(orc):
    # build_schedule(500, 1) digest recorded by the reference
    assert digest(orc.build_schedule(500, 1)) == \
        "99b129a4b97065d83595554534b6434b0c5cbe05b7223af5981b79ec6965bc8e"


def test_schedule_ranges(orc):
    s = orc.build_schedule(1000, 3)  # sequence.hpp:33-48 ranges
    assert s.flip_deg.min() >= 0 and s.flip_deg.max() <= 79 + 1e-6
    assert set(np.unique(s.phase_deg)) <= {0.0, 90.0, 180.0}
    assert s.tr_ms.min() >= 14 - 1e-9 and s.tr_ms.max() <= 20 + 1e-6
    b = orc.baseline_schedule(1000, 1)
    assert b.tr_ms.min() >= 10.5 and b.tr_ms.max() < 14.0 + 1e-9
    assert set(np.unique(b.phase_deg)) == {0.0, 180.0}
    np.testing.assert_allclose(b.te_ms, b.tr_ms / 2, rtol=1e-8)


@pytest.mark.parametrize("fn", ["build_schedule", "baseline_schedule"])
def test_schedules_match_reference(orc, ref, fn):
    a, b = getattr(orc, fn)(777, 5), getattr(ref, fn)(777, 5)
    for k in ("flip_deg", "phase_deg", "tr_ms", "te_ms"):
        assert np.array_equal(getattr(a, k), getattr(b, k))


@pytest.mark.parametrize("p", [(1.4, 0.5, 100.0), (0.1, 0.02, -50.0), (5.0, 2.0, 249.0), (0.75, 0.12, 3.3)])
def test_simulate_bit_exact_vs_reference(orc, ref, p):
    s = orc.baseline_schedule(1000, 1)
    assert np.array_equal(orc.simulate(s, *p), ref.simulate(s, *p))


def test_noise_and_cc_vs_reference(orc, ref):
    s = orc.build_schedule(300, 2)
    fp = orc.simulate(s, 0.9, 0.1, 7.0)
    assert np.array_equal(orc.add_noise(fp, 0.01, 42), ref.add_noise(fp, 0.01, 42))
    g = orc.add_noise(fp, 0.05, 43)
    assert orc.cc(fp, g) == ref.cc(fp, g)
    assert orc.cc_unit(fp, g) == ref.cc_unit(fp, g)


def test_generate_vs_reference(orc, ref):
    s = orc.build_schedule(60, 3)
    g = oracle.make_grid((600, 100, 3), (80, 20, 3), (-10, 10, 3))
    assert np.array_equal(orc.generate(s, g, 0, 27), ref.generate(s, g, 0, 27))


def test_scan_grid_vs_reference(orc, ref):
    s = orc.build_schedule(48, 7)
    g = oracle.make_grid((600, 100, 5), (80, 20, 5), (-20, 10, 5))
    rng = np.random.default_rng(0)
    q = np.stack([orc.add_noise(orc.simulate(s, 0.55 + 0.6 * rng.random(), 0.07 + 0.12 * rng.random(),
                                             50 * rng.random() - 25), 0.002, 80 + k) for k in range(6)])
    for metric in (0, 1):
        a = orc.scan_grid(s, g, q, metric=metric)
        b = ref.scan_grid(s, g, q, metric=metric, threads=1)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.all(a[1] >= a[2])  # top-2 bookkeeping


def test_quantify_vs_reference(orc, ref):
    s = orc.build_schedule(60, 15)
    g = oracle.make_grid((600, 10, 40), (80, 5, 16), (-20, 2, 25))
    rng = np.random.default_rng(1)
    for cfg in (oracle.zoom_cfg(df_coarse_hz=2.0), oracle.zoom_cfg(df_coarse_hz=2.0, final_metric=1)):
        for k in range(4):
            fp = orc.add_noise(orc.simulate(s, 0.6 + 0.4 * rng.random(), 0.08 + 0.08 * rng.random(),
                                            -20 + 50 * rng.random()), 0.003, 9 + k)
            a, b = orc.quantify(s, g, cfg, fp), ref.quantify(s, g, cfg, fp)
            assert (a.i1, a.i2, a.idf, a.score, a.pd, a.evaluations) == \
                   (b.i1, b.i2, b.idf, b.score, b.pd, b.evaluations)


@pytest.mark.parametrize("mode", [1, 2])
def test_quantify_dictionary_modes_vs_reference(orc, ref, mode):
    """zoom.cpp:94-123: df-dictionary (stage-1 acquisitions) and full-dictionary
    lookups read float entries; the reference wrapper passes the reference's
    own make_df_dictionary / generate dictionaries, the restatement
    synthesizes float(normalize(simulate)).  Answers usually equal the plain
    objective's (test_zoom.cpp:384-400); scores read from float entries differ."""
    s = orc.baseline_schedule(300, 1)
    g = oracle.make_grid((300.0, 20.0, 60), (40.0, 5.0, 40), (-50.0, 1.0, 101))
    cfg = oracle.zoom_cfg(df_coarse_hz=10, df_refine_hz=2, df_window_hz=10, omega_hz=82,
                          t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20)
    cfg.dict_mode = mode
    plain = oracle.zoom_cfg(df_coarse_hz=10, df_refine_hz=2, df_window_hz=10, omega_hz=82,
                            t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20)
    rng = np.random.default_rng(3)
    changed = 0
    for k in range(6):
        fp = orc.simulate(s, rng.uniform(0.4, 1.4), rng.uniform(0.06, 0.22), rng.uniform(-40, 40))
        fp = orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(300) / 20, 100 + k)
        a, b = orc.quantify(s, g, cfg, fp), ref.quantify(s, g, cfg, fp)
        assert (a.i1, a.i2, a.idf, a.score, a.pd, a.evaluations) == \
               (b.i1, b.i2, b.idf, b.score, b.pd, b.evaluations)
        c = ref.quantify(s, g, plain, fp)
        changed += c.score != b.score
    if mode == 2:
        assert changed > 0  # every score comes from a float entry


@pytest.mark.parametrize("k,mode", [(3, 0), (5, 0), (3, 1), (3, 2)])
def test_quantify_smoothing_vs_reference(orc, ref, k, mode):
    """smooth_k with and without dictionary entries (zoom.cpp:49-50, 106-118)."""
    s = orc.baseline_schedule(300, 1)
    g = oracle.make_grid((300.0, 20.0, 60), (40.0, 5.0, 40), (-50.0, 1.0, 101))
    cfg = oracle.zoom_cfg(smooth_k=k, df_coarse_hz=10, df_refine_hz=2, df_window_hz=10, omega_hz=82,
                          t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20)
    cfg.dict_mode = mode
    rng = np.random.default_rng(5)
    for j in range(3):
        fp = orc.simulate(s, rng.uniform(0.4, 1.4), rng.uniform(0.06, 0.22), rng.uniform(-40, 40))
        fp = orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(300) / 15, 300 + j)
        a, b = orc.quantify(s, g, cfg, fp), ref.quantify(s, g, cfg, fp)
        assert (a.i1, a.i2, a.idf, a.score, a.pd, a.evaluations) == \
               (b.i1, b.i2, b.idf, b.score, b.pd, b.evaluations)


def _perturbed_payload(orc, s, g, cfg, mode, seed):
    """A dictionary payload that is NOT the recomputation: the generated
    entries with seeded noise (a dictionary written on another machine, or
    edited before save) -- quantify must score these bytes (zoom.cpp:101-113)."""
    n = s.n
    if mode == 2:
        payload = orc.generate(s, g, 0, g.t1_ms.count * g.t2_ms.count * g.df_hz.count)
    else:
        i1 = min(max(int(round((cfg.init_t1_ms - g.t1_ms.min) / g.t1_ms.step)), 0), g.t1_ms.count - 1)
        i2 = min(max(int(round((cfg.init_t2_ms - g.t2_ms.min) / g.t2_ms.step)), 0), g.t2_ms.count - 1)
        first = (i1 * g.t2_ms.count + i2) * g.df_hz.count
        payload = orc.generate(s, g, first, g.df_hz.count)
    payload = payload.reshape(-1, 2 * n).astype(np.float32)
    rng = np.random.default_rng(seed)
    payload += (rng.standard_normal(payload.shape) * 2e-3).astype(np.float32)
    return payload


@pytest.mark.parametrize("mode,smooth,edge", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 3, 0), (2, 5, 0), (0, 0, 1),
                                               (1, 0, 1)])
def test_quantify_trace_and_payload_vs_reference(orc, ref, mode, smooth, edge):
    """QuantResult::trace (zoom.cpp:441-451, test_zoom.cpp:334-336) and
    dictionary payloads that differ from the recomputation: answers, scores,
    PD, evaluation counts and every StageLog record equal the reference's.
    `edge` reaches every stage name: the heavy-noise fallback rerun, the
    omega-translate rerefinements and the plateau stop (zoom.cpp:189-249)."""
    s = orc.baseline_schedule(200, 1)
    if edge:
        g = oracle.make_grid((300.0, 20.0, 50), (40.0, 5.0, 30), (-250.0, 2.0, 251))
        cfg = oracle.zoom_cfg(smooth_k=smooth, df_coarse_hz=40, df_refine_hz=4, df_window_hz=30, omega_hz=82,
                              t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20,
                              heavy_noise_cc=0.6, plateau_eps=0.05)
    else:
        g = oracle.make_grid((300.0, 20.0, 50), (40.0, 5.0, 30), (-50.0, 1.0, 101))
        cfg = oracle.zoom_cfg(smooth_k=smooth, df_coarse_hz=10, df_refine_hz=2, df_window_hz=10, omega_hz=82,
                              t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20)
    cfg.dict_mode = mode
    payload = _perturbed_payload(orc, s, g, cfg, mode, 7) if mode else None
    rng = np.random.default_rng(11)
    dfr = 200.0 if edge else 40.0
    seen = set()
    for k in range(6 if edge else 4):
        fp = orc.simulate(s, rng.uniform(0.4, 1.2), rng.uniform(0.06, 0.16), rng.uniform(-dfr, dfr))
        snr = (20 if k % 2 else 0.5) if edge else (20 if k else 0.5)
        fp = orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(200) / snr, 500 + k)
        a, ta = orc.quantify_ex(s, g, cfg, fp, payload)
        b, tb = ref.quantify_ex(s, g, cfg, fp, payload)
        assert (a.i1, a.i2, a.idf, a.score, a.pd, a.evaluations) == \
               (b.i1, b.i2, b.idf, b.score, b.pd, b.evaluations)
        assert ta == tb
        assert sum(t[1] for t in ta) == a.evaluations
        names = [t[0] for t in ta]
        assert names[0] == "df.coarse" and names[-1] == "t1t2.final"
        seen |= set(names)
    if edge:
        assert set(oracle.STAGE_NAMES) == seen


def test_quantify_slice_prior_vs_reference(orc, ref):
    s = orc.build_schedule(60, 15)
    g = oracle.make_grid((600, 10, 40), (80, 5, 16), (-20, 2, 25))
    cfg = oracle.zoom_cfg(df_coarse_hz=2.0)
    nx, ny = 4, 3
    mask = np.ones(nx * ny, dtype=np.uint8)
    mask[0] = mask[11] = 0
    fps = np.zeros((nx * ny, 60), dtype=np.complex128)
    for v in range(nx * ny):
        if mask[v]:
            fps[v] = orc.simulate(s, (600 + 10 * (20 + v % 2)) * 1e-3, (80 + 5 * (8 + v % 3)) * 1e-3, 0.0)
    for prior in (False, True):
        a = orc.quantify_slice(s, g, cfg, fps, mask, nx, ny, prior)
        b = ref.quantify_slice(s, g, cfg, fps, mask, nx, ny, prior, threads=1)
        for v in range(nx * ny):
            assert (a[v].i1, a[v].i2, a[v].idf, a[v].evaluations) == (b[v].i1, b[v].i2, b[v].idf, b[v].evaluations)


def test_golden_exp1_cc_vs_df(orc):
    """runs/exp1/cc_vs_df.csv: cc(normalize(target), normalize(entry)) at %.9g."""
    d = np.load(os.path.join(GOLD, "exp1_ccdf.npz"))
    s = orc.build_schedule(500, 1)
    target = orc.simulate(s, 1.4, 0.5, 100.0)
    idx = np.arange(0, len(d["df_hz"]), 7)
    for i in idx:
        e = orc.simulate(s, d["t1_ms"][i] * 1e-3, d["t2_ms"][i] * 1e-3, d["df_hz"][i])
        assert f"{orc.cc_unit(target, e):.9g}" == str(d["cc_text"][i]), i


def test_golden_exp2_zoom(orc):
    gold = json.load(open(os.path.join(GOLD, "exp2.json")))
    s = orc.build_schedule(500, 1)
    g = oracle.make_grid((500, 10, 150), (200, 10, 60), (-30, 2, 240))
    cfg = oracle.zoom_cfg(df_coarse_hz=2.0)
    for (t1, t2, df), (z1, z2, zdf, pd, score, evals) in zip(gold["targets"], gold["zoom"]):
        q = orc.quantify(s, g, cfg, orc.simulate(s, t1 * 1e-3, t2 * 1e-3, df))
        assert (q.t1_ms, q.t2_ms, q.df_hz, q.evaluations) == (z1, z2, zdf, evals)
        assert float(f"{q.score:.9g}") == score and float(f"{q.pd:.9g}") == pd


def test_golden_exp3_slice(orc):
    """runs/exp3: 64x64 phantom (data/slice64.csv), 1 ms/1 Hz lattice, no prior."""
    d = np.load(os.path.join(GOLD, "exp3_slice.npz"))
    s = orc.build_schedule(500, 1)
    g = oracle.make_grid((800, 1, 2401), (50, 1, 551), (-48, 1, 133))
    cfg = oracle.zoom_cfg(df_coarse_hz=1.0)
    mask = d["mask"]
    fps = np.zeros((4096, 500), dtype=np.complex128)
    for v in np.nonzero(mask)[0]:
        fps[v] = orc.simulate(s, d["t1_ms"][v] * 1e-3, d["t2_ms"][v] * 1e-3, d["df_hz"][v]) * d["pd"][v]
    res = orc.quantify_slice(s, g, cfg, fps, mask, 64, 64, False)
    got_evals = np.array([r.evaluations for r in res])
    assert np.array_equal(got_evals, d["evals_noprior"])
    for v in np.nonzero(mask)[0]:
        assert float(f"{res[v].t1_ms:.9g}") == pytest.approx(d["t1_map"][v], abs=1e-9)
        assert float(f"{res[v].t2_ms:.9g}") == pytest.approx(d["t2_map"][v], abs=1e-9)
        assert float(f"{res[v].df_hz:.9g}") == pytest.approx(d["df_map"][v], abs=1e-9)


def test_quantify_b1_vs_reference(orc, ref):
    """Four-parameter ZOOM (BASELINE configs[4]): the restatement's outer B1
    zoom_1d over memoized three-parameter quantify equals the composition of
    the reference's OWN zoom_1d and quantify (oracle/ref_capi.cpp), answer,
    B1 index, score, PD and summed evaluations."""
    base = orc.baseline_schedule(200, 1)
    b1 = [0.7 + 0.1 * k for k in range(7)]
    scheds = [oracle.Schedule(base.flip_deg * b, base.phase_deg, base.tr_ms, base.te_ms) for b in b1]
    g = oracle.make_grid((300.0, 25.0, 40), (20.0, 10.0, 30), (-50.0, 5.0, 21))
    cfg = oracle.zoom_cfg(df_coarse_hz=5, df_refine_hz=5, df_window_hz=20, omega_hz=82,
                          t1t2_2d_steps_ms=[200, 100], t1t2_1d_steps_ms=[50, 25], final_2d_step_ms=10,
                          init_t2_ms=100)
    rng = np.random.default_rng(21)
    hits = 0
    for k in range(6):
        kb = int(rng.integers(0, len(b1)))
        fp = orc.simulate(scheds[kb], rng.uniform(0.4, 1.2), rng.uniform(0.03, 0.25), rng.uniform(-40, 40))
        fp = orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(200) / 25, 700 + k)
        a, ia = orc.quantify_b1(scheds, g, cfg, fp, [2, 1], 3)
        b, ib = ref.quantify_b1(scheds, g, cfg, fp, [2, 1], 3)
        assert (ia, a.i1, a.i2, a.idf, a.score, a.pd, a.evaluations) == \
               (ib, b.i1, b.i2, b.idf, b.score, b.pd, b.evaluations)
        per_b1 = [orc.quantify(x, g, cfg, fp).score for x in scheds]
        hits += a.score == max(per_b1)
    assert hits >= 5  # the outer walk reaches the best B1 of the inner searches
