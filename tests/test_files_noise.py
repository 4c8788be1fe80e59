"""CPU tests of the §8(f) host pieces: .mrfd/.mrfc headers, noise calibration,
smoothing.  The product's host functions (libmrfg.so, no GPU needed) are
checked against the C restatement and, where oracle/_ref was built, against
the reference library itself -- bit-for-bit."""
import os

import numpy as np
import pytest

import paper_1506_05393_b200 as P
from paper_1506_05393_b200._native import MrfgError
from conftest import to_oracle_grid, to_oracle_sched


def _fp(orc, n=300, t1=0.9, t2=0.08, df=7.0, seed=2):
    s = P.baseline_schedule(n, seed)
    return s, orc.simulate(to_oracle_sched(s), t1, t2, df)


@pytest.mark.parametrize("k", [3, 5])
@pytest.mark.parametrize("n", [1, 2, 3, 300])
def test_smooth_matches_oracles(orc, k, n):
    _, fp = _fp(orc)
    fp = fp[:n]
    got = P.smooth(fp, k)
    np.testing.assert_array_equal(got, orc.smooth(fp, k))
    import oracle
    if oracle.available("reference"):
        np.testing.assert_array_equal(got, oracle.Oracle("reference").smooth(fp, k))


def test_smooth_errors():
    with pytest.raises(MrfgError) as e:
        P.smooth(np.ones(4, complex), 4)
    assert e.value.code == -1
    with pytest.raises(MrfgError) as e:
        P.smooth(np.ones(0, complex), 3)
    assert e.value.code == -1


TARGETS = [0.98, 0.9, 0.7, 0.4, 0.2, 0.1, 0.05]


@pytest.mark.parametrize("target", TARGETS)
def test_calibrate_noise_bit_identical(orc, target):
    """calibrate_noise (fingerprint.cpp:80-105): same sigma, or the same
    runtime_error, as the restatement and the reference (exp4's 13 levels
    span 0.98 .. 0.05)."""
    import oracle
    _, fp = _fp(orc)
    impls = [orc] + ([oracle.Oracle("reference")] if oracle.available("reference") else [])
    for seed in (1, 5, 11):
        want = [o.calibrate_noise(fp, target, seed) for o in impls]
        assert all(w == want[0] for w in want)
        if want[0] is None:
            with pytest.raises(MrfgError) as e:
                P.calibrate_noise(fp, target, seed)
            assert e.value.code == -3
        else:
            got = P.calibrate_noise(fp, target, seed)
            assert got == want[0]
            assert abs(orc.cc(fp, orc.add_noise(fp, got, seed)) - target) <= 0.02


@pytest.mark.parametrize("target", [0.95, 0.5, 0.08, 0.03])
def test_make_calibrated_noise_bit_identical(orc, target):
    import oracle
    _, fp = _fp(orc, n=200)
    impls = [orc] + ([oracle.Oracle("reference")] if oracle.available("reference") else [])
    want = [o.make_calibrated_noise(fp, target, 4) for o in impls]
    if want[0] is None:
        assert all(w is None for w in want)
        with pytest.raises(MrfgError):
            P.make_calibrated_noise(fp, target, 4)
        return
    sg, used, noisy = P.make_calibrated_noise(fp, target, 4)
    for w in want:
        assert (sg, used) == (w[0], w[1])
        np.testing.assert_array_equal(noisy, w[2])


def test_calibrate_noise_rejects_bad_target(orc):
    _, fp = _fp(orc, n=50)
    for t in (0.0, 1.0, -0.5, 1.5):
        with pytest.raises(MrfgError) as e:
            P.calibrate_noise(fp, t, 1)
        assert e.value.code == -1


def test_dictionary_file_bytes_match_reference(orc, ref, tmp_path):
    """save (header via mrfg_write_header + float32 payload) writes the
    reference's exact bytes: save_generated of the reference library on the
    same schedule and lattice."""
    s = P.baseline_schedule(60, 1)
    g = P.grid((300, 40, 5), (40, 15, 4), (-20, 5, 9))
    ent = orc.generate(to_oracle_sched(s), to_oracle_grid(g), 0, P.grid_total(g))
    mine, theirs = tmp_path / "mine.mrfd", tmp_path / "ref.mrfd"
    P.save_dictionary(str(mine), g, s.digest(), ent)
    ref.save_generated(to_oracle_sched(s), to_oracle_grid(g), str(theirs))
    assert mine.read_bytes() == theirs.read_bytes()
    g2, dg, data = P.load_dictionary(str(theirs))
    assert dg == s.digest() and P.grid_total(g2) == P.grid_total(g)
    assert (g2.t1_ms.min, g2.t1_ms.step, g2.t1_ms.count) == (300, 40, 5)
    np.testing.assert_array_equal(data, ent)


def test_cc_map_file_header_matches_reference(orc, ref, tmp_path):
    s = P.baseline_schedule(40, 2)
    g = P.grid((500, 100, 3), (50, 25, 3), (-4, 2, 5))
    fp = orc.simulate(to_oracle_sched(s), 0.61, 0.07, 1.0)
    theirs = tmp_path / "ref.mrfc"
    ref.cc_map_to_file(to_oracle_sched(s), to_oracle_grid(g), fp, str(theirs))
    mine = tmp_path / "hdr.mrfc"
    import ctypes as C
    from paper_1506_05393_b200 import dgs
    from paper_1506_05393_b200._native import check, load
    check(load().mrfg_write_header(str(mine).encode(), b"MRFC", C.byref(g), dgs._digest_bytes(s.digest()), 40))
    hdr = mine.read_bytes()
    assert theirs.read_bytes()[:len(hdr)] == hdr
    g2, dg, scores = P.load_cc_map(str(theirs))
    assert dg == s.digest() and scores.shape == (P.grid_total(g),)


def test_read_header_errors(tmp_path):
    g = P.grid((300, 40, 5), (40, 15, 4), (-20, 5, 9))
    good = tmp_path / "g.mrfd"
    P.save_dictionary(str(good), g, "00" * 32, np.zeros((P.grid_total(g), 4), np.float32))
    raw = good.read_bytes()
    cases = {
        "magic": b"XXXX" + raw[4:],
        "version": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "truncated": raw[:50],
        "degenerate": raw[:4 + 4 + 32 + 16] + (0).to_bytes(8, "little") + raw[4 + 4 + 32 + 24:],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.mrfd"
        p.write_bytes(data)
        with pytest.raises(MrfgError) as e:
            P.load_dictionary(str(p))
        assert e.value.code == -3, name
    with pytest.raises(MrfgError) as e:
        P.load_dictionary(str(tmp_path / "missing.mrfd"))
    assert e.value.code == -3
    (tmp_path / "short.mrfd").write_bytes(raw[:-8])
    with pytest.raises(MrfgError):
        P.load_dictionary(str(tmp_path / "short.mrfd"))
    with pytest.raises(MrfgError):  # a dictionary is not a correlation map
        P.load_cc_map(str(good))
