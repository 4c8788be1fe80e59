"""K5 MRF-ZOOM parity on the GPU against the CPU oracle (reference restatement).

The GPU kernel evaluates the reference's FP64 objective bit-exactly and runs
the reference's decision logic, so lattice answers, scores, proton density
and the unique-evaluation counts must all match; the BASELINE exemption
(top-2 gap < 1e-5) is not needed here and not applied.
"""
import numpy as np
import pytest

import oracle
import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads
from conftest import to_oracle_grid, to_oracle_sched

pytestmark = pytest.mark.gpu


def ocfg(c):
    """product ZoomConfig -> oracle ZoomCfg (same POD layout)."""
    o = oracle.ZoomCfg()
    for name, _ in oracle.ZoomCfg._fields_:
        v = getattr(c, name)
        if name.startswith("t1t2"):
            for i in range(8):
                getattr(o, name)[i] = v[i]
        else:
            setattr(o, name, v)
    return o


def check_same(got, orc, sched, g, cfg, fps):
    os_, og, oc = to_oracle_sched(sched), to_oracle_grid(g), ocfg(cfg)
    for v, fp in enumerate(fps):
        w = orc.quantify(os_, og, oc, fp)
        assert (got["i1"][v], got["i2"][v], got["idf"][v]) == (w.i1, w.i2, w.idf), v
        assert got["score"][v] == w.score, v
        assert got["evaluations"][v] == w.evaluations, v
        assert got["pd"][v] == pytest.approx(w.pd, rel=1e-12), v


def test_zoom_mini_lattice_targets(orc):
    """test_zoom.cpp:317-345 setup: build_schedule(60, 15), 40x16x25 lattice."""
    s = P.reference_schedule(60, 15)
    g = P.grid_from_ranges((600, 1000, 10), (80, 160, 5), (-20, 30, 2))
    cfg = P.zoom_config(df_coarse_hz=2.0)
    truth = [(P.dgs.rng_at(92, 0, k) % 40, P.dgs.rng_at(92, 1, k) % 16, P.dgs.rng_at(92, 2, k) % 25)
             for k in range(5)]
    fps = np.stack([orc.simulate(to_oracle_sched(s), *[float(x) for x in P.params_at(g, *t)])
                    for t in truth])
    with P.Context(s) as c:
        got = c.quantify(fps, g, cfg)
        np.testing.assert_array_equal(np.stack([got["i1"], got["i2"], got["idf"]], 1), np.array(truth))
        check_same(got, orc, s, g, cfg, fps)
        # final metric euclidean (test_zoom.cpp:339-344)
        cfge = P.zoom_config(df_coarse_hz=2.0, final_metric="euclidean")
        got_e = c.quantify(fps, g, cfge)
        check_same(got_e, orc, s, g, cfge, fps)


def test_zoom_exp2_golden_rows(orc):
    """runs/exp2/zoom.csv: 25 targets on the 2.16M lattice, N=500 seed 1, df_coarse=2."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "exp2.json")))
    s = P.reference_schedule(500, 1)
    g = P.grid_from_ranges((500, 2000, 10), (200, 800, 10), (-30, 450, 2))
    cfg = P.zoom_config(df_coarse_hz=2.0)
    tg = gold["targets"]
    fps = np.stack([orc.simulate(to_oracle_sched(s), t[0] * 1e-3, t[1] * 1e-3, float(t[2])) for t in tg])
    with P.Context(s) as c:
        got = c.quantify(fps, g, cfg)
    for k, row in enumerate(gold["zoom"]):
        t1, t2, df, pd, score, evals = row
        assert got["t1_ms"][k] == pytest.approx(t1, abs=1e-9)
        assert got["t2_ms"][k] == pytest.approx(t2, abs=1e-9)
        assert got["df_hz"][k] == pytest.approx(df, abs=1e-9)
        assert got["evaluations"][k] == evals
        assert got["score"][k] == pytest.approx(score, abs=5e-9)


def test_zoom_config1_noisy(orc):
    def sim(sc, params):
        os_ = to_oracle_sched(sc)
        return np.stack([orc.simulate(os_, *p) for p in params])
    wl = workloads.make(1, sim, nvox=48)
    cfg = P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0)
    with P.Context(wl.schedule) as c:
        got = c.quantify(wl.fps, wl.grid, cfg)
    check_same(got, orc, wl.schedule, wl.grid, cfg, wl.fps)


def test_zoom_fine_lattice_config4_like(orc):
    """Config-4 pitch (1 ms / 0.5 ms / 0.1 Hz) on a reduced lattice."""
    s = P.baseline_schedule(200, 1)
    g = P.grid((600, 1, 600), (40, 0.5, 400), (-40, 0.1, 801))
    cfg = P.zoom_config(df_coarse_hz=10, df_refine_hz=1, df_window_hz=20, omega_hz=82,
                        t1t2_2d_steps_ms=[100, 10], t1t2_1d_steps_ms=[50, 5, 1], final_2d_step_ms=0.5,
                        init_t1_ms=900, init_t2_ms=120)
    rng = np.random.default_rng(3)
    params = [(0.6 + 0.5 * rng.random(), 0.04 + 0.15 * rng.random(), -35 + 70 * rng.random())
              for _ in range(6)]
    os_ = to_oracle_sched(s)
    fps = np.stack([orc.add_noise(orc.simulate(os_, *p), 0.002, 500 + k) for k, p in enumerate(params)])
    with P.Context(s) as c:
        got = c.quantify(fps, g, cfg)
    check_same(got, orc, s, g, cfg, fps)


def test_zoom_slice_noprior_matches_quantify(orc):
    s = P.reference_schedule(60, 15)
    g = P.grid_from_ranges((600, 1000, 10), (80, 160, 5), (-20, 30, 2))
    cfg = P.zoom_config(df_coarse_hz=2.0)
    nx, ny = 4, 3
    mask = np.ones(nx * ny, dtype=np.uint8)
    mask[0] = mask[11] = 0
    fps = np.zeros((nx * ny, 60), dtype=np.complex128)
    for v in range(nx * ny):
        if mask[v]:
            fps[v] = orc.simulate(to_oracle_sched(s), *[float(x) for x in P.params_at(g, 20 + v % 2, 8 + v % 3, 10)])
    with P.Context(s) as c:
        res, secs = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=False)
    w = orc.quantify_slice(to_oracle_sched(s), to_oracle_grid(g), ocfg(cfg), fps, mask, nx, ny, False)
    for v in range(nx * ny):
        if not mask[v]:
            assert res["evaluations"][v] == 0
            continue
        assert (res["i1"][v], res["i2"][v], res["idf"][v]) == (w[v].i1, w[v].i2, w[v].idf)
        assert res["evaluations"][v] == w[v].evaluations


def test_zoom_errors():
    s = P.reference_schedule(32, 2)
    g = P.grid((600, 10, 10), (80, 5, 10), (-20, 2, 10))
    with P.Context(s) as c:
        with pytest.raises(ValueError):
            c.quantify(np.zeros((1, 32), dtype=np.complex128), g)
        with pytest.raises(ValueError):
            c.quantify(np.ones((1, 32), dtype=np.complex128), g, P.zoom_config(smooth_k=4))  # fingerprint.cpp:123


def _slice_problem(orc):
    s = P.reference_schedule(60, 15)
    g = P.grid_from_ranges((600, 1000, 10), (80, 160, 5), (-20, 30, 2))
    cfg = P.zoom_config(df_coarse_hz=2.0, prior_window_t1_ms=60, prior_window_t2_ms=30,
                        prior_window_df_hz=10)
    nx, ny = 6, 5
    mask = np.ones(nx * ny, dtype=np.uint8)
    mask[[0, 7, 29]] = 0
    fps = np.zeros((nx * ny, 60), dtype=np.complex128)
    for v in range(nx * ny):
        if mask[v]:
            x, y = v % nx, v // nx
            t = (18 + x // 2, 7 + y // 2, 9 + (x + y) % 3)
            fps[v] = orc.add_noise(orc.simulate(to_oracle_sched(s), *[float(u) for u in P.params_at(g, *t)]),
                                   0.001, 70 + v)
    return s, g, cfg, nx, ny, mask, fps


def test_zoom_slice_raster_prior_matches_reference(orc):
    """use_prior=1: the reference's sequential raster semantics, evals included."""
    s, g, cfg, nx, ny, mask, fps = _slice_problem(orc)
    with P.Context(s) as c:
        res, _ = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=1)
    w = orc.quantify_slice(to_oracle_sched(s), to_oracle_grid(g), ocfg(cfg), fps, mask, nx, ny, True)
    for v in range(nx * ny):
        assert (res["i1"][v], res["i2"][v], res["idf"][v], res["evaluations"][v]) == \
               (w[v].i1, w[v].i2, w[v].idf, w[v].evaluations), v


def test_zoom_slice_wavefront_prior(orc):
    """use_prior=2 (SPEC.md:449 relaxation): same maps as without priors, fewer evals."""
    s, g, cfg, nx, ny, mask, fps = _slice_problem(orc)
    with P.Context(s) as c:
        a, _ = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=0)
        b, _ = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=2)
    m = mask.astype(bool)
    for k in ("i1", "i2", "idf"):
        np.testing.assert_array_equal(a[k][m], b[k][m])
    assert b["evaluations"].sum() < a["evaluations"].sum()


@pytest.mark.parametrize("mode", [1, 2])
def test_zoom_dictionary_modes(orc, mode):
    """dict_mode 1 (df dictionary, zoom.cpp:101-113 in stage 1) and 2 (full
    dictionary): float dictionary entries, reproduced on the GPU, give the
    oracle's answers, scores, PD and evaluation counts; the certified path and
    the all-FP64 path agree."""
    import os
    s = P.baseline_schedule(300, 1)
    g = P.grid_from_ranges((300.0, 1500.0, 20.0), (40.0, 240.0, 5.0), (-50.0, 51.0, 1.0))
    kw = dict(df_coarse_hz=10, df_refine_hz=2, df_window_hz=10, omega_hz=82,
              t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20], final_2d_step_ms=20)
    cfg = P.zoom_config(dict_mode=mode, **kw)
    rng = np.random.default_rng(3)
    os_ = to_oracle_sched(s)
    fps = []
    for k in range(6):
        fp = orc.simulate(os_, rng.uniform(0.4, 1.4), rng.uniform(0.06, 0.22), rng.uniform(-40, 40))
        fps.append(orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(300) / 20, 100 + k))
    fps = np.stack(fps)
    with P.Context(s) as c:
        got = c.quantify(fps, g, cfg)
        check_same(got, orc, s, g, cfg, fps)
        old = os.environ.get("MRFG_ZOOM_EPS")
        os.environ["MRFG_ZOOM_EPS"] = "-1"
        try:
            exact = c.quantify(fps, g, cfg)
        finally:
            if old is None:
                del os.environ["MRFG_ZOOM_EPS"]
            else:
                os.environ["MRFG_ZOOM_EPS"] = old
        for k in ("i1", "i2", "idf", "score", "pd", "evaluations"):
            np.testing.assert_array_equal(got[k], exact[k])


@pytest.mark.parametrize("k,mode", [(3, 0), (5, 0), (3, 1), (3, 2)])
def test_zoom_smoothing(orc, k, mode):
    """smooth_k (fingerprint.cpp:122-145; zoom.cpp:49-50, 106-118): smoothed
    query and entries (dictionary entries float-cast before smoothing), PD from
    the raw fingerprints; oracle answers, scores, PD and counts."""
    s = P.baseline_schedule(300, 1)
    g = P.grid_from_ranges((300.0, 1500.0, 20.0), (40.0, 240.0, 5.0), (-50.0, 51.0, 1.0))
    cfg = P.zoom_config(smooth_k=k, dict_mode=mode, df_coarse_hz=10, df_refine_hz=2, df_window_hz=10,
                        omega_hz=82, t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20],
                        final_2d_step_ms=20)
    rng = np.random.default_rng(5)
    os_ = to_oracle_sched(s)
    fps = []
    for j in range(5):
        fp = orc.simulate(os_, rng.uniform(0.4, 1.4), rng.uniform(0.06, 0.22), rng.uniform(-40, 40))
        fps.append(orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(300) / 15, 300 + j))
    fps = np.stack(fps)
    with P.Context(s) as c:
        check_same(c.quantify(fps, g, cfg), orc, s, g, cfg, fps)


def _lround(x):  # std::lround: half away from zero
    import math
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def _prior_of(g, cfg, r):
    """Host restatement of the prior window (zoom.cpp:595-610)."""
    t1 = (g.t1_ms.min + float(r["i1"]) * g.t1_ms.step) * 1e-3 * 1e3
    t2 = (g.t2_ms.min + float(r["i2"]) * g.t2_ms.step) * 1e-3 * 1e3
    df = g.df_hz.min + float(r["idf"]) * g.df_hz.step
    units = lambda s, fine: max(1, _lround(s / fine))  # noqa: E731
    p1, p2, pd = (_lround((t1 - g.t1_ms.min) / g.t1_ms.step), _lround((t2 - g.t2_ms.min) / g.t2_ms.step),
                  _lround((df - g.df_hz.min) / g.df_hz.step))
    w1, w2, wd = (units(cfg.prior_window_t1_ms, g.t1_ms.step), units(cfg.prior_window_t2_ms, g.t2_ms.step),
                  units(cfg.prior_window_df_hz, g.df_hz.step))
    b = [max(0, p1 - w1), min(g.t1_ms.count - 1, p1 + w1), max(0, p2 - w2), min(g.t2_ms.count - 1, p2 + w2),
         max(0, pd - wd), min(g.df_hz.count - 1, pd + wd)]
    return b, [t1, t2]


def test_zoom_slice_row_relaxation_exact(orc):
    """use_prior=2 runs the SPEC.md:449 row relaxation in one launch (device
    seeding and completion flags); it must equal the same relaxation driven
    voxel by voxel from the host through quantify_bounded (whose prior path is
    the one pinned against the reference's raster mode)."""
    s, g, cfg, nx, ny, mask, fps = _slice_problem(orc)
    with P.Context(s) as c:
        dev, _ = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=2)
        rows = [[y * nx + x for x in range(nx) if mask[y * nx + x]] for y in range(ny)]
        rows = [r for r in rows if r]
        host = {}
        for ri, r in enumerate(rows):
            for k, v in enumerate(r):
                prev = r[k - 1] if k > 0 else (rows[ri - 1][0] if ri > 0 else None)
                if prev is None:
                    res = c.quantify_bounded(fps[v:v + 1], g, cfg)
                else:
                    b, init = _prior_of(g, cfg, host[prev])
                    res = c.quantify_bounded(fps[v:v + 1], g, cfg, bounds=[b], init_ms=[init])
                host[v] = res[0]
    for v, h in host.items():
        for k in ("i1", "i2", "idf", "score", "pd", "evaluations"):
            assert dev[k][v] == h[k], (v, k)


@pytest.mark.parametrize("n", [1, 2, 33])
def test_zoom_tiny_shapes(orc, n):
    """ZOOM on degenerate lattices (single-valued axes, one voxel, 1-2 TR
    schedules): the oracle's answers, scores, PD and evaluation counts."""
    s = P.reference_schedule(n, 3)
    os_ = to_oracle_sched(s)
    rng = np.random.default_rng(n)
    for g in (P.grid((700.0, 10.0, 1), (90.0, 5.0, 1), (0.0, 1.0, 1)),
              P.grid((600.0, 50.0, 7), (80.0, 5.0, 1), (-10.0, 5.0, 5)),
              P.grid((600.0, 10.0, 30), (80.0, 5.0, 20), (0.0, 1.0, 1))):
        fps = np.stack([orc.add_noise(orc.simulate(os_, 0.5 + rng.random(), 0.05 + 0.1 * rng.random(),
                                                   10 * rng.random() - 5), 0.01, 60 + k) for k in range(2)])
        cfg = P.zoom_config(df_coarse_hz=5.0)
        with P.Context(s) as c:
            check_same(c.quantify(fps, g, cfg), orc, s, g, cfg, fps)


def _payload(orc, s, g, cfg, mode, seed):
    """A dictionary payload that is NOT the recomputation (generated entries
    plus seeded noise): K5 must score these bytes (zoom.cpp:101-113)."""
    os_, og = to_oracle_sched(s), to_oracle_grid(g)
    if mode == 2:
        payload = orc.generate(os_, og, 0, P.grid_total(g))
    else:
        i1 = min(max(_lround((cfg.init_t1_ms - g.t1_ms.min) / g.t1_ms.step), 0), g.t1_ms.count - 1)
        i2 = min(max(_lround((cfg.init_t2_ms - g.t2_ms.min) / g.t2_ms.step), 0), g.t2_ms.count - 1)
        payload = orc.generate(os_, og, (i1 * g.t2_ms.count + i2) * g.df_hz.count, g.df_hz.count)
    payload = payload.reshape(-1, 2 * s.n).astype(np.float32)
    rng = np.random.default_rng(seed)
    return payload + (rng.standard_normal(payload.shape) * 2e-3).astype(np.float32)


@pytest.mark.parametrize("mode,smooth,edge", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 3, 0), (2, 5, 0), (0, 0, 1),
                                               (1, 0, 1)])
def test_zoom_trace_and_payload(orc, mode, smooth, edge):
    """QuantResult::trace (zoom.cpp:441-451; test_zoom.cpp:334-336: the stage
    counts sum to evaluations) and dictionary payloads that differ from the
    recomputation, against the oracle (itself pinned to the reference on the
    same cases, tests/test_oracle.py): answer, score, PD, evaluations and
    every StageLog record (stage, evaluations, exact best, lattice point)."""
    s = P.baseline_schedule(200, 1)
    if edge:  # every stage name: fallback rerun, rerefinements, plateau stop
        g = P.grid((300.0, 20.0, 50), (40.0, 5.0, 30), (-250.0, 2.0, 251))
        cfg = P.zoom_config(smooth_k=smooth, dict_mode=mode, df_coarse_hz=40, df_refine_hz=4, df_window_hz=30,
                            omega_hz=82, t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20],
                            final_2d_step_ms=20, heavy_noise_cc=0.6, plateau_eps=0.05)
    else:
        g = P.grid((300.0, 20.0, 50), (40.0, 5.0, 30), (-50.0, 1.0, 101))
        cfg = P.zoom_config(smooth_k=smooth, dict_mode=mode, df_coarse_hz=10, df_refine_hz=2, df_window_hz=10,
                            omega_hz=82, t1t2_2d_steps_ms=[200, 40], t1t2_1d_steps_ms=[100, 20],
                            final_2d_step_ms=20)
    payload = _payload(orc, s, g, cfg, mode, 7) if mode else None
    os_, og, oc = to_oracle_sched(s), to_oracle_grid(g), ocfg(cfg)
    rng = np.random.default_rng(11)
    dfr = 200.0 if edge else 40.0
    fps = []
    for k in range(6 if edge else 4):
        fp = orc.simulate(os_, rng.uniform(0.4, 1.2), rng.uniform(0.06, 0.16), rng.uniform(-dfr, dfr))
        snr = (20 if k % 2 else 0.5) if edge else (20 if k else 0.5)
        fps.append(orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(200) / snr, 500 + k))
    fps = np.stack(fps)
    seen = set()
    with P.Context(s) as c:
        got, traces = c.quantify(fps, g, cfg, dictionary=payload, trace=True)
    for v, fp in enumerate(fps):
        w, tw = orc.quantify_ex(os_, og, oc, fp, payload)
        assert (got["i1"][v], got["i2"][v], got["idf"][v]) == (w.i1, w.i2, w.idf), v
        assert (got["score"][v], got["pd"][v], got["evaluations"][v]) == (w.score, w.pd, w.evaluations), v
        assert traces[v] == tw, v
        assert sum(t[1] for t in traces[v]) == got["evaluations"][v]
        seen |= {t[0] for t in traces[v]}
    if edge:
        assert seen == set(oracle.STAGE_NAMES)


@pytest.mark.parametrize("prior", [0, 1, 2])
def test_zoom_slice_traces(orc, prior):
    """quantify_slice traces: per voxel the stage counts sum to evaluations;
    without priors each voxel's trace equals quantify's; with the strict
    raster (one launch) the maps, evaluations and traces equal the same
    chain driven voxel by voxel from the host through quantify_bounded."""
    s, g, cfg, nx, ny, mask, fps = _slice_problem(orc)
    with P.Context(s) as c:
        res, _, tr = c.quantify_slice(fps, mask, nx, ny, g, cfg, use_prior=prior, trace=True)
        m = np.nonzero(mask)[0]
        for v in m:
            assert sum(t[1] for t in tr[v]) == res["evaluations"][v], v
        for v in np.nonzero(mask == 0)[0]:
            assert tr[v] == []
        if prior == 0:
            q, tq = c.quantify(fps[m], g, cfg, trace=True)
            for k, v in enumerate(m):
                assert tr[v] == tq[k]
        if prior == 1:
            prev = None
            for v in m:
                if prev is None:
                    h, th = c.quantify_bounded(fps[v:v + 1], g, cfg, trace=True)
                else:
                    b, init = _prior_of(g, cfg, res[prev])
                    h, th = c.quantify_bounded(fps[v:v + 1], g, cfg, bounds=[b], init_ms=[init], trace=True)
                for k in ("i1", "i2", "idf", "score", "pd", "evaluations"):
                    assert res[k][v] == h[k][0], (v, k)
                assert tr[v] == th[0]
                prev = v


def test_zoom_four_parameter_b1(orc):
    """Four-parameter ZOOM (mrfg_quantify_b1): the outer B1 walk over K5's
    three-parameter quantify equals the oracle restatement (itself pinned to
    the reference's zoom_1d + quantify): B1 index, point, score, PD,
    evaluations; with one B1 value it is plain quantify."""
    base = P.baseline_schedule(200, 1)
    b1 = [0.7 + 0.1 * k for k in range(7)]
    scheds = [P.Schedule(base.flip_deg * b, base.phase_deg, base.tr_ms, base.te_ms) for b in b1]
    g = P.grid((300.0, 25.0, 40), (20.0, 10.0, 30), (-50.0, 5.0, 21))
    kw = dict(df_coarse_hz=5, df_refine_hz=5, df_window_hz=20, omega_hz=82, t1t2_2d_steps_ms=[200, 100],
              t1t2_1d_steps_ms=[50, 25], final_2d_step_ms=10, init_t2_ms=100)
    cfg = P.zoom_config(**kw)
    rng = np.random.default_rng(21)
    fps = []
    for k in range(12):
        kb = int(rng.integers(0, len(b1)))
        fp = orc.simulate(to_oracle_sched(scheds[kb]), rng.uniform(0.4, 1.2), rng.uniform(0.03, 0.25),
                          rng.uniform(-40, 40))
        fps.append(orc.add_noise(fp, float(np.linalg.norm(fp)) / np.sqrt(200) / 25, 700 + k))
    fps = np.stack(fps)
    ctxs = [P.Context(s) for s in scheds]
    try:
        q, ib = P.quantify_b1(ctxs, fps, g, cfg, (2, 1), 3)
        q1, ib1 = P.quantify_b1(ctxs[2:3], fps, g, cfg, (2, 1), 0)
        plain = ctxs[2].quantify(fps, g, cfg)
    finally:
        for c in ctxs:
            c.close()
    os_ = [to_oracle_sched(s) for s in scheds]
    ocf = ocfg(cfg)
    og = to_oracle_grid(g)
    for v, fp in enumerate(fps):
        w, wb = orc.quantify_b1(os_, og, ocf, fp, [2, 1], 3)
        assert (ib[v], q["i1"][v], q["i2"][v], q["idf"][v]) == (wb, w.i1, w.i2, w.idf), v
        assert (q["score"][v], q["pd"][v], q["evaluations"][v]) == (w.score, w.pd, w.evaluations), v
    assert (ib1 == 0).all()
    for k in ("i1", "i2", "idf", "score", "pd", "evaluations"):
        np.testing.assert_array_equal(q1[k], plain[k])
