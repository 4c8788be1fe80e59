"""K1 Bloch parity on the GPU against the CPU oracle (reference restatement).

Bars: FP64 lattice entries bit-identical to the reference (generate, precision
64); FP64 free-parameter simulate within 1e-12 relative L2 (device libm vs
glibc); FP32 within 1e-4 relative L2 (north_star).
"""
import numpy as np
import pytest

import paper_1506_05393_b200 as P
from conftest import to_oracle_grid, to_oracle_sched

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def sched():
    return P.baseline_schedule(500, 1)


@pytest.fixture(scope="module")
def ctx(sched):
    c = P.Context(sched)
    yield c
    c.close()


PARAMS = [(0.1, 0.02, -50.0), (1.4, 0.5, 100.0), (2.0, 0.3, 49.5), (5.0, 2.0, -250.0),
          (0.75, 0.12, 3.0), (0.3, 0.3, 0.0)]


def test_simulate_fp64_matches_reference(ctx, sched, orc):
    got = ctx.simulate(np.array(PARAMS), precision=64)
    for k, p in enumerate(PARAMS):
        want = orc.simulate(to_oracle_sched(sched), *p)
        assert rel_l2(got[k], want) < 1e-12


def test_simulate_fp32_within_1e4(ctx, sched, orc):
    got = ctx.simulate(np.array(PARAMS), precision=32)
    for k, p in enumerate(PARAMS):
        want = orc.simulate(to_oracle_sched(sched), *p)
        assert rel_l2(got[k], want) < 1e-4


def test_simulate_normalized(ctx):
    got = ctx.simulate(np.array(PARAMS), precision=64, normalize=True)
    np.testing.assert_allclose(np.linalg.norm(got, axis=1), 1.0, rtol=1e-14)


def test_simulate_rejects_nonpositive_t1(ctx):
    with pytest.raises(ValueError):
        ctx.simulate(np.array([[0.0, 0.1, 0.0]]))


@pytest.mark.parametrize("grid_spec", [
    ((600, 100, 5), (80, 20, 5), (-20, 10, 5)),
    ((100, 20, 96), (20, 10, 29), (-50, 5, 21)),
])
def test_generate_fp64_bit_identical(ctx, sched, orc, grid_spec):
    g = P.grid(*grid_spec)
    total = P.grid_total(g)
    first, count = (0, total) if total < 400 else (total - 777, 777)
    got = ctx.generate(g, first, count, precision=64)
    want = orc.generate(to_oracle_sched(sched), to_oracle_grid(g), first, count)
    assert np.array_equal(got, want)


# K1 variants: the frame-folded producer (MRFG_K1=fold, 2/4/8 T2 rows per thread)
# and the phasor-ladder row producer (default, MRFG_K1=rows)
K1_VARIANTS = [("fold", "2"), ("fold", "4"), ("fold", "8"), ("rows", "4")]


@pytest.mark.parametrize("k1,apt", K1_VARIANTS)
def test_generate_fp32_close(ctx, sched, orc, monkeypatch, k1, apt):
    monkeypatch.setenv("MRFG_K1", k1)
    monkeypatch.setenv("MRFG_K1_APT", apt)
    g = P.grid((100, 20, 96), (20, 10, 29), (-50, 5, 21))
    # 29 T2 rows: partial pencils at every T1; the range starts mid-row
    got = ctx.generate(g, 1000, 1300, precision=32)
    want = orc.generate(to_oracle_sched(sched), to_oracle_grid(g), 1000, 1300)
    errs = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert errs.max() < 1e-4


@pytest.mark.parametrize("k1,apt", K1_VARIANTS)
def test_generate_n3000_fp32(orc, monkeypatch, k1, apt):
    monkeypatch.setenv("MRFG_K1", k1)
    monkeypatch.setenv("MRFG_K1_APT", apt)
    s = P.baseline_schedule(3000, 1)
    with P.Context(s) as c:
        g = P.grid((100, 25, 117), (20, 10, 49), (-100, 10, 21))
        got = c.generate(g, 5000, 64, precision=32)
        want = orc.generate(to_oracle_sched(s), to_oracle_grid(g), 5000, 64)
    errs = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert errs.max() < 1e-4
