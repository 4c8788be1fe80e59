"""K2/K3 brute-force parity on the GPU against the CPU oracle.

The screening GEMM (fp16 tcgen05) only selects candidates; the re-rank scores
them through the reference's own FP64 pipeline, so best flats AND scores are
expected to be identical to the reference.  The exemption of BASELINE.json
(top-2 CC gap < 1e-5) is applied only if an index differs.
"""
import numpy as np
import pytest

import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads
from paper_1506_05393_b200._native import ScanOpts
from conftest import to_oracle_grid, to_oracle_sched

pytestmark = pytest.mark.gpu


def oracle_sim(orc):
    def sim(s, params):
        os_ = to_oracle_sched(s)
        return np.stack([orc.simulate(os_, *p) for p in params])
    return sim


def assert_parity(flat, score, oflat, oscore, osecond, tol_exempt=1e-5):
    bad = np.nonzero(flat != oflat)[0]
    for v in bad:
        assert oscore[v] - osecond[v] < tol_exempt, (v, flat[v], oflat[v], oscore[v], osecond[v])
    same = flat == oflat
    np.testing.assert_array_equal(score[same], oscore[same])


@pytest.fixture(scope="module")
def small(orc):
    # config-1 shapes (N=500, 96x29x21 grid) with 160 voxels
    return workloads.make(1, oracle_sim(orc), nvox=160)


@pytest.fixture(scope="module")
def small_ref(orc, small):
    return orc.scan_grid(to_oracle_sched(small.schedule), to_oracle_grid(small.grid), small.fps)


def test_screen_tcgen05_matches_simt(orc, small):
    with P.Context(small.schedule) as c:
        a = c.screen_scores(small.grid, small.fps[:200], 2000, 700, use_simt=False)
        b = c.screen_scores(small.grid, small.fps[:200], 2000, 700, use_simt=True)
    assert np.isfinite(a).all() and np.isfinite(b).all()
    np.testing.assert_allclose(a, b, rtol=2e-5, atol=2e-6)


def test_screen_close_to_exact_cc2(orc, small):
    with P.Context(small.schedule) as c:
        a = c.screen_scores(small.grid, small.fps[:64], 5000, 512)
    ent = orc.generate(to_oracle_sched(small.schedule), to_oracle_grid(small.grid), 5000, 512)
    e = ent[:, 0::2] + 1j * ent[:, 1::2]
    q = small.fps[:64] / np.linalg.norm(small.fps[:64], axis=1, keepdims=True)
    cc = np.abs(e @ q.conj().T)
    assert np.abs(np.sqrt(a) - cc).max() < 1e-3


@pytest.mark.parametrize("k1,apt", [("fold", "2"), ("fold", "4"), ("fold", "8"), ("rows", "4"), ("rows", "8"),
                                    ("rows2", "4"), ("rows2", "8"), ("pairs", "4"), ("pairs", "8"),
                                    ("pairs_nost", "4"), ("pairs_nost_hb4", "4"), ("pairs_hb4", "8"),
                                    ("pairs_minb3", "4")])
def test_screen_production_producer(orc, small, monkeypatch, k1, apt):
    """The GEMM operand of the production K1 (scan_grid's producer) screens
    within fp16 rounding of the exact CC; ranges start and end mid-row and
    cut T2 pencils."""
    monkeypatch.setenv("MRFG_K1", k1.split("_")[0])
    monkeypatch.setenv("MRFG_K1_HB", "4" if "_hb4" in k1 else "8")
    monkeypatch.setenv("MRFG_K1_ST", "0" if "_nost" in k1 else "1")
    monkeypatch.setenv("MRFG_K1_MINB", "3" if "_minb3" in k1 else "2")
    monkeypatch.setenv("MRFG_K1_APT", apt)
    first, count = 4999, 1777
    with P.Context(small.schedule) as c:
        a = c.screen_scores(small.grid, small.fps[:48], first, count, producer="rows")
        b = c.screen_scores(small.grid, small.fps[:48], first, count)
    ent = orc.generate(to_oracle_sched(small.schedule), to_oracle_grid(small.grid), first, count)
    e = ent[:, 0::2] + 1j * ent[:, 1::2]
    q = small.fps[:48] / np.linalg.norm(small.fps[:48], axis=1, keepdims=True)
    cc = np.abs(e @ q.conj().T)
    assert np.isfinite(a).all()
    assert np.abs(np.sqrt(a) - cc).max() < 1e-3
    assert np.abs(a - b).max() < 1e-3


@pytest.mark.parametrize("apt", ["4", "8"])
@pytest.mark.parametrize("xr", ["1", "0"])
def test_k1_symmetric_echo_identical(orc, monkeypatch, apt, xr):
    """BASELINE schedules have TE = TR/2, so te == rest at every TR and the
    packed K1 takes its symmetric-echo path (one E1/E2/phasor per step):
    the GEMM operand screens bit-identically to the two-stage path
    (MRFG_K1_SYM=0), and the fused FP32 cc_map is identical too.  (The
    default producer for such schedules, the atom-pair kernel, is checked
    against the exact scores in test_screen_production_producer and
    test_cc_map_fp32_close.)"""
    monkeypatch.setenv("MRFG_K1", "rows2")
    monkeypatch.setenv("MRFG_K1_APT", apt)
    monkeypatch.setenv("MRFG_K1_XR", xr)
    s = P.baseline_schedule(1000, 3)
    assert np.array_equal(s.te_ms, s.tr_ms / 2)
    g = P.grid((100, 20, 50), (20, 10, 40), (-250, 1, 501))
    fp = orc.add_noise(orc.simulate(to_oracle_sched(s), 0.9, 0.06, -3.0), 0.002, 5)
    q = np.stack([fp, fp * 1j, np.conj(fp)])
    out = {}
    with P.Context(s) as c:
        for sym in ("1", "0"):
            monkeypatch.setenv("MRFG_K1_SYM", sym)
            out[sym] = (c.screen_scores(g, q, 12345, 9 * 512 + 77, producer="rows"),
                        c.cc_map(fp, g, first=777, count=3333, precision=32))
    np.testing.assert_array_equal(out["1"][0], out["0"][0])
    np.testing.assert_array_equal(out["1"][1], out["0"][1])


@pytest.mark.parametrize("pair", ["1", "0"])
@pytest.mark.parametrize("group", ["3", "7", "64"])
def test_screen_grouped_raster(small, monkeypatch, pair, group):
    """K2's grouped tile raster (query operand larger than L2) visits every
    (atom tile, query tile) once: dense scores identical to atom-major order,
    including a short last group."""
    monkeypatch.setenv("MRFG_K2_PAIR", pair)
    q = np.concatenate([small.fps] * 4)  # 640 voxels: 5 query tiles
    with P.Context(small.schedule) as c:
        monkeypatch.setenv("MRFG_K2_GROUP", "1")
        a = c.screen_scores(small.grid, q, 1000, 9 * 256 + 17)
        monkeypatch.setenv("MRFG_K2_GROUP", group)
        b = c.screen_scores(small.grid, q, 1000, 9 * 256 + 17)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("walk", ["1", "2"])
@pytest.mark.parametrize("metric", ["cc", "euclidean"])
def test_rerank_walk_modes(small, orc, monkeypatch, walk, metric):
    """K3 with one walk + echo scratch (default) or two walks: identical bits."""
    monkeypatch.setenv("MRFG_RERANK_WALK", walk)
    with P.Context(small.schedule) as c:
        flat, score, _ = c.scan_grid(small.grid, small.fps[:96], metric=metric)
    oflat, oscore, osecond = orc.scan_grid(to_oracle_sched(small.schedule), to_oracle_grid(small.grid),
                                           small.fps[:96], metric=1 if metric == "euclidean" else 0)
    assert_parity(flat, score, oflat, oscore, osecond)


@pytest.mark.parametrize("fp32", ["1", "0"])
def test_rerank_fp32_rescreen(small, small_ref, monkeypatch, fp32):
    """The certified FP32 re-screen only thins the FP64 re-rank: answers and
    scores identical with and without it; near-ties still reach FP64."""
    monkeypatch.setenv("MRFG_RERANK_FP32", fp32)
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        flat, score, st = c.scan_grid(small.grid, small.fps)
    assert_parity(flat, score, oflat, oscore, osecond)
    if fp32 == "1":
        assert st.rescreened32 >= st.reranked >= len(flat)
        assert st.reranked < st.rescreened32
    else:
        assert st.rescreened32 == 0


@pytest.mark.parametrize("batch", ["128", "256"])
def test_scan_voxel_batches(small, small_ref, monkeypatch, batch):
    """Voxel-batched screening (query rows kept L2-resident): same answers."""
    monkeypatch.setenv("MRFG_VOX_BATCH", batch)
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        flat, score, st = c.scan_grid(small.grid, small.fps)
        dflat, dscore, _ = c.brute_force_search(small.fps, c.generate(small.grid, precision=64))
    assert_parity(flat, score, oflat, oscore, osecond)
    np.testing.assert_array_equal(dflat, flat)
    np.testing.assert_array_equal(dscore, score)


def test_scan_grid_config1_slice(small, small_ref):
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        flat, score, st = c.scan_grid(small.grid, small.fps)
    assert st.candidates >= len(flat) and st.reranked >= len(flat)
    assert_parity(flat, score, oflat, oscore, osecond)


@pytest.mark.parametrize("chunk", [128, 1000, 1 << 20])
def test_scan_chunk_invariance(small, small_ref, chunk):
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        flat, score, _ = c.scan_grid(small.grid, small.fps, opts=ScanOpts(0.0, chunk, 0, 0))
    assert_parity(flat, score, oflat, oscore, osecond)


def test_scan_sharded_ranges_merge(small, small_ref):
    """Atom sharding (8 contiguous ranges) + the C1 merge rule == one pass."""
    import torch
    oflat, oscore, osecond = small_ref
    total = P.grid_total(small.grid)
    cuts = np.linspace(0, total, 9).astype(np.int64)
    parts = []
    with P.Context(small.schedule) as c:
        for r in range(8):
            f, s, _ = c.scan_grid(small.grid, small.fps, flat_range=(int(cuts[r]), int(cuts[r + 1])))
            parts.append((f, s))
        rec = np.zeros((8, len(small.fps), 2), dtype=np.float64)
        packed = np.zeros((8, len(small.fps)), dtype=[("flat", np.int64), ("score", np.float64)])
        for r, (f, s) in enumerate(parts):
            packed[r]["flat"], packed[r]["score"] = f, s
        d_in = torch.from_numpy(packed.view(np.uint8).reshape(-1)).cuda()
        d_out = torch.empty(len(small.fps) * 16, dtype=torch.uint8, device="cuda")
        c.merge_matches_device(d_in.data_ptr(), 8, len(small.fps), d_out.data_ptr())
        c.synchronize()
        out = d_out.cpu().numpy().view([("flat", np.int64), ("score", np.float64)])
    assert_parity(out["flat"], out["score"], oflat, oscore, osecond)


def test_scan_euclidean_metric(orc, small):
    q = small.fps[:48]
    oflat, oscore, osecond = orc.scan_grid(to_oracle_sched(small.schedule), to_oracle_grid(small.grid),
                                           q, metric=1)
    with P.Context(small.schedule) as c:
        flat, score, _ = c.scan_grid(small.grid, q, metric="euclidean")
    assert_parity(flat, score, oflat, oscore, osecond)


def test_scan_on_lattice_noise_free_ties(orc):
    """Clamped CC = 1 ties resolve to the lowest flat (dictionary.cpp:291-294)."""
    s = P.baseline_schedule(64, 8)
    g = P.grid((600, 100, 3), (80, 20, 3), (-10, 10, 3))
    truth = [(2, 1, 0), (0, 0, 0), (1, 2, 2)]
    fps = np.stack([orc.simulate(to_oracle_sched(s), *[float(x) for x in P.params_at(g, *t)]) for t in truth])
    oflat, oscore, _ = orc.scan_grid(to_oracle_sched(s), to_oracle_grid(g), fps)
    with P.Context(s) as c:
        flat, score, _ = c.scan_grid(g, fps)
    np.testing.assert_array_equal(flat, oflat)
    np.testing.assert_array_equal(score, oscore)


def test_scan_errors():
    s = P.baseline_schedule(32, 2)
    g = P.grid((600, 100, 3), (80, 20, 3), (-10, 10, 3))
    with P.Context(s) as c:
        with pytest.raises(ValueError):
            c.scan_grid(g, np.zeros((0, 32), dtype=np.complex128))
        with pytest.raises(ValueError):
            c.scan_grid(g, np.zeros((2, 32), dtype=np.complex128))  # zero fingerprint
        with pytest.raises(ValueError):
            c.scan_grid(g, np.ones((1, 31), dtype=np.complex128))


def test_cc_map_bit_identical(orc):
    s = P.baseline_schedule(120, 3)
    g = P.grid((600, 50, 8), (80, 20, 6), (-30, 2, 31))
    fp = orc.add_noise(orc.simulate(to_oracle_sched(s), 0.72, 0.11, 4.0), 0.001, 99)
    with P.Context(s) as c:
        got = c.cc_map(fp, g)
    ent = orc.generate(to_oracle_sched(s), to_oracle_grid(g), 0, P.grid_total(g))
    e = ent[:, 0::2].astype(np.float64) + 1j * ent[:, 1::2].astype(np.float64)
    q = fp / np.linalg.norm(fp)
    want = np.minimum(np.abs(e @ q.conj()), 1.0).astype(np.float32)
    np.testing.assert_allclose(got, want, rtol=1e-6)


def test_brute_force_search_stored_dictionary(orc, small, small_ref):
    """K4: stored float32 dictionary (generate() layout) == lattice scan == reference."""
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        d = c.generate(small.grid, precision=64)  # bit-identical to the reference's entries
        flat, score, st = c.brute_force_search(small.fps, d)
    assert_parity(flat, score, oflat, oscore, osecond)
    assert st.candidates >= len(flat)


def test_brute_force_search_arbitrary_dictionary(orc):
    """Entries need not come from a lattice: random unit atoms vs a numpy FP64 scan."""
    rng = np.random.default_rng(5)
    n, atoms = 64, 3000
    e = rng.standard_normal((atoms, n)) + 1j * rng.standard_normal((atoms, n))
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    d = np.empty((atoms, 2 * n), dtype=np.float32)
    d[:, 0::2], d[:, 1::2] = e.real, e.imag
    q = e[[5, 17, 2999]] + 0.05 * (rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n)))
    s = P.baseline_schedule(n, 1)
    with P.Context(s) as c:
        flat, score, _ = c.brute_force_search(q, d)
    ed = d[:, 0::2].astype(np.float64) + 1j * d[:, 1::2].astype(np.float64)
    qn = q / np.linalg.norm(q, axis=1, keepdims=True)
    cc = np.minimum(np.abs(ed @ qn.conj().T), 1.0)
    np.testing.assert_array_equal(flat, cc.argmax(axis=0))
    np.testing.assert_allclose(score, cc.max(axis=0), rtol=1e-12)


@pytest.mark.parametrize("pair", ["1", "0"])
def test_screen_both_k2_variants_match_simt(small, pair, monkeypatch):
    """cta_group::2 (default) and cta_group::1 kernels vs the CUDA-core twin."""
    monkeypatch.setenv("MRFG_K2_PAIR", pair)
    with P.Context(small.schedule) as c:
        a = c.screen_scores(small.grid, small.fps, 3000, 1500, use_simt=False)
        b = c.screen_scores(small.grid, small.fps, 3000, 1500, use_simt=True)
    np.testing.assert_allclose(a, b, rtol=2e-5, atol=2e-6)


def test_scan_single_cta_kernel(small, small_ref, monkeypatch):
    monkeypatch.setenv("MRFG_K2_PAIR", "0")
    oflat, oscore, osecond = small_ref
    with P.Context(small.schedule) as c:
        flat, score, _ = c.scan_grid(small.grid, small.fps)
    assert_parity(flat, score, oflat, oscore, osecond)


def test_scan_floor_from_other_atoms(small, small_ref):
    """floor_matches: scanning the second half of the grid with the first half's
    matches as the screening floor, then merging (max score, lowest flat), gives
    the full scan's answer; voxels whose best lies in the first half may return
    flat -1 from the second scan (nothing above the floor)."""
    import torch
    g, fps = small.grid, small.fps
    total = P.grid_total(g)
    half = total // 2
    nq, n = fps.shape
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(np.ascontiguousarray(fps).view(np.float64).reshape(nq, 2 * n)).to(dev)
    d_all = torch.empty((2, nq, 2), dtype=torch.int64, device=dev)
    d_out = torch.empty((nq, 2), dtype=torch.int64, device=dev)
    with P.Context(small.schedule) as c:
        c.scan_grid_device(g, d_q.data_ptr(), nq, d_all[0].data_ptr(), flat_range=(0, half))
        opts = ScanOpts(0.0, 0, 0, 0, d_all[0].data_ptr())
        st = c.scan_grid_device(g, d_q.data_ptr(), nq, d_all[1].data_ptr(), flat_range=(half, total), opts=opts)
        c.merge_matches_device(d_all.data_ptr(), 2, nq, d_out.data_ptr())
        torch.cuda.synchronize()
        # without the floor, for comparison of re-rank work
        st0 = c.scan_grid_device(g, d_q.data_ptr(), nq, d_all[1].data_ptr(), flat_range=(half, total))
    out = d_out.cpu().numpy()
    flat, score = out[:, 0], out[:, 1].view(np.float64)
    assert_parity(flat, score, *small_ref)
    assert st.reranked <= st0.reranked


@pytest.mark.parametrize("n", [1, 2, 33])
def test_scan_tiny_shapes(orc, n):
    """Degenerate shapes: schedules of 1/2/33 TRs (K padded from 2N to 64),
    single-valued axes, a 1-point lattice, one voxel; the reference library's
    answers and scores (flat + score bit-identical)."""
    s = P.reference_schedule(n, 3)
    os_ = to_oracle_sched(s)
    grids = [P.grid((700.0, 10.0, 1), (90.0, 5.0, 1), (0.0, 1.0, 1)),
             P.grid((600.0, 50.0, 7), (80.0, 5.0, 1), (-10.0, 5.0, 5)),
             P.grid((600.0, 50.0, 1), (80.0, 5.0, 9), (0.0, 1.0, 1))]
    rng = np.random.default_rng(n)
    for g in grids:
        for nv in (1, 3):
            fps = np.stack([orc.add_noise(orc.simulate(os_, 0.5 + rng.random(), 0.05 + 0.1 * rng.random(),
                                                       10 * rng.random() - 5), 0.01, 40 + k) for k in range(nv)])
            with P.Context(s) as c:
                flat, score, _ = c.scan_grid(g, fps)
            of, osc, osec = orc.scan_grid(os_, to_oracle_grid(g), fps)
            assert_parity(flat, score, of, osc, osec)


# ---------------------------------------------------------------- round 2
def test_screen_audit_certifies_margin(small, small_ref):
    """The unbiased audit (hash sample of ALL screened pairs, scored exactly)
    reports the fp16 screening error; the default margin (2.5e-3) is at least
    twice it, and the FP32 re-screen error stays below half its margin."""
    with P.Context(small.schedule) as c:
        flat, score, st = c.scan_grid(small.grid, small.fps)
    assert_parity(flat, score, *small_ref)
    assert st.delta_used == 2.5e-3 and st.rescans == 0
    assert st.audit_samples > 1000
    assert 0 < st.screen_err_audit_max <= 0.5 * st.delta_used
    assert st.rescreen_err_audit_max <= 5e-6
    assert st.rescreen_err_max <= 5e-6


def test_screen_audit_widens_too_small_margin(small, small_ref):
    """A margin below twice the audited error is widened by a rescan: the
    answers stay the reference's."""
    with P.Context(small.schedule) as c:
        flat, score, st = c.scan_grid(small.grid, small.fps, opts=ScanOpts(1e-5, 0, 0, 0))
    assert_parity(flat, score, *small_ref)
    assert st.rescans >= 1 and st.delta_used > 1e-5
    assert st.screen_err_audit_max <= 0.5 * st.delta_used


def seq_normalize(fp):
    """normalize (fingerprint.cpp:28-37) with the reference's summation order."""
    acc = 0.0
    for v in fp:
        acc += v.real * v.real + v.imag * v.imag
    inv = 1.0 / np.sqrt(acc)
    return np.array([complex(v.real * inv, v.imag * inv) for v in fp])


@pytest.mark.parametrize("metric", ["cc", "euclidean"])
def test_scan_unit_norm_queries(orc, small, metric):
    """Fingerprint::unit_norm queries are used as given (prep_query,
    dictionary.cpp:145-150), in scan_grid and brute_force_search: scores
    equal the reference's for normalize()d queries, including exact on-grid ones."""
    os_ = to_oracle_sched(small.schedule)
    og = to_oracle_grid(small.grid)
    q = np.stack([seq_normalize(f) for f in small.fps[:24]])
    exact = orc.simulate(os_, *[float(x) for x in P.params_at(small.grid, 40, 11, 7)])
    q = np.concatenate([q, seq_normalize(exact)[None]])
    m = 1 if metric == "euclidean" else 0
    oflat, oscore, osecond = orc.scan_grid(os_, og, q, metric=m, unit_norm=True)
    with P.Context(small.schedule) as c:
        flat, score, _ = c.scan_grid(small.grid, q, metric=metric, unit_norm=True)
        dflat, dscore, _ = c.brute_force_search(q, c.generate(small.grid, precision=64), metric=metric,
                                                unit_norm=True)
    assert_parity(flat, score, oflat, oscore, osecond)
    np.testing.assert_array_equal(dflat, flat)
    np.testing.assert_array_equal(dscore, score)


def explicit_problem(orc):
    s = P.baseline_schedule(200, 1)
    t1 = np.geomspace(300.0, 2500.0, 23)
    t2 = np.geomspace(30.0, 400.0, 17)
    df = (-30.0, 5.0, 13)
    rng = np.random.default_rng(3)
    os_ = to_oracle_sched(s)
    q = np.stack([orc.add_noise(orc.simulate(os_, t1[rng.integers(23)] * 1e-3 * (1 + 0.01 * rng.random()),
                                             t2[rng.integers(17)] * 1e-3, -30 + 60 * rng.random()), 0.003, 500 + k)
                  for k in range(40)])
    return s, t1, t2, df, q


def oracle_rows_scan(orc, s, t1, t2, df, q):
    """Restatement oracle over explicit T1 x T2 values: one-row subgrids
    {t1, 1, 1} x {t2, 1, 1} x df in flat order, strict > across rows."""
    import oracle
    os_ = to_oracle_sched(s)
    best_f = np.zeros(len(q), np.int64)
    best_s = np.full(len(q), -np.inf)
    for i1, a in enumerate(t1):
        for i2, b in enumerate(t2):
            g = oracle.make_grid((a, 1.0, 1), (b, 1.0, 1), df)
            f, sc, _ = orc.scan_grid(os_, g, q, threads=8)
            better = sc > best_s
            best_f = np.where(better, (i1 * len(t2) + i2) * df[2] + f, best_f)
            best_s = np.where(better, sc, best_s)
    return best_f, best_s


def test_explicit_axes_generate_bit_identical(orc):
    """A lattice with explicit (log-spaced) T1/T2 values: FP64 generate equals
    the reference pipeline over the same TissueParams bit for bit."""
    import oracle
    s, t1, t2, df, _ = explicit_problem(orc)
    g = P.grid_values(t1, t2, df)
    os_ = to_oracle_sched(s)
    with P.Context(s) as c:
        ent = c.generate(g, precision=64)
    for i1 in (0, 7, 22):
        for i2 in (0, 9, 16):
            sub = oracle.make_grid((t1[i1], 1.0, 1), (t2[i2], 1.0, 1), df)
            want = orc.generate(os_, sub, 0, df[2])
            f0 = (i1 * len(t2) + i2) * df[2]
            np.testing.assert_array_equal(ent[f0:f0 + df[2]], want)


def test_explicit_axes_scan_and_dictionary(orc):
    """Streamed scan_grid over the explicit-axis lattice and K4 over its
    materialized dictionary: the reference's answers and scores."""
    s, t1, t2, df, q = explicit_problem(orc)
    g = P.grid_values(t1, t2, df)
    of, osc = oracle_rows_scan(orc, s, t1, t2, df, q)
    with P.Context(s) as c:
        flat, score, st = c.scan_grid(g, q)
        dflat, dscore, _ = c.brute_force_search(q, c.generate(g, precision=64))
        cm = c.cc_map(q[0], g, precision=64)
    np.testing.assert_array_equal(flat, of)
    np.testing.assert_array_equal(score, osc)
    np.testing.assert_array_equal(dflat, of)
    np.testing.assert_array_equal(dscore, osc)
    assert int(np.argmax(cm)) == of[0]


def test_explicit_axes_rejected_where_unsupported(orc):
    s, t1, t2, df, q = explicit_problem(orc)
    g = P.grid_values(t1, t2, df)
    with P.Context(s) as c:
        with pytest.raises(ValueError):
            c.quantify(q[:1], g)
        with pytest.raises(ValueError):
            c.save_generated(g, "/tmp/never.mrfd")


def test_seeded_shards_equal_single_scan(small, small_ref):
    """The multi-GPU protocol on one device: per-shard seed maxima, reduced by
    max, floor every shard's scan; merge == the single scan, and the seeded
    shards re-rank no more than unseeded ones."""
    import torch
    g, fps = small.grid, small.fps
    total = P.grid_total(g)
    nq, n = fps.shape
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(np.ascontiguousarray(fps).view(np.float64).reshape(nq, 2 * n)).to(dev)
    W = 3
    slab = g.t2_ms.count * g.df_hz.count
    cuts = [g.t1_ms.count * r // W * slab for r in range(W + 1)]
    with P.Context(small.schedule) as c:
        seeds = torch.full((W, nq), -3.0, dtype=torch.float32, device=dev)
        for r in range(W):
            c.scan_seed_device(g, d_q.data_ptr(), nq, seeds[r].data_ptr(), flat_range=(cuts[r], cuts[r + 1]))
        seed = seeds.max(dim=0).values
        floor = torch.zeros((nq, 2), dtype=torch.float64, device=dev)
        floor[:, 1] = seed.double()
        fl = floor.view(torch.int64)
        fl[:, 0] = 0
        d_all = torch.empty((W, nq, 2), dtype=torch.int64, device=dev)
        seeded, plain = 0, 0
        for r in range(W):
            st = c.scan_grid_device(g, d_q.data_ptr(), nq, d_all[r].data_ptr(), flat_range=(cuts[r], cuts[r + 1]),
                                    opts=ScanOpts(0.0, 0, 0, 0, fl.data_ptr()))
            seeded += st.reranked
        d_out = torch.empty((nq, 2), dtype=torch.int64, device=dev)
        c.merge_matches_device(d_all.data_ptr(), W, nq, d_out.data_ptr())
        torch.cuda.synchronize()
        tmp = torch.empty((nq, 2), dtype=torch.int64, device=dev)
        for r in range(W):
            plain += c.scan_grid_device(g, d_q.data_ptr(), nq, tmp.data_ptr(),
                                        flat_range=(cuts[r], cuts[r + 1])).reranked
    out = d_out.cpu().numpy()
    assert_parity(out[:, 0], out[:, 1].view(np.float64), *small_ref)
    assert seeded <= plain


def test_subspace_screening_same_answers(small, monkeypatch):
    """Experimental per-off-resonance subspace screening (MRFG_SUBSPACE, csrc/subspace.cu):
    the K1 off-resonance-major slabs, the projection and K2 on one K block only
    change WHICH atoms survive the screen; the audit-driven margin and the exact
    FP64 re-rank keep best atoms and scores identical to the default path
    (dictionary.cpp:257-308)."""
    with P.Context(small.schedule) as c:
        monkeypatch.delenv("MRFG_SUBSPACE", raising=False)
        f0, s0, st0 = c.scan_grid(small.grid, small.fps)
        monkeypatch.setenv("MRFG_SUBSPACE", "16")
        f1, s1, st1 = c.scan_grid(small.grid, small.fps)
    assert st0.subspace_rank == 0 and st1.subspace_rank == 16 and st1.project_ms > 0
    np.testing.assert_array_equal(f0, f1)
    np.testing.assert_array_equal(s0, s1)
