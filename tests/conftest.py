import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) device")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (test infrastructure) and the product extension."""
    from paper_1506_05393_b200 import build as B
    B.build()
    import oracle
    oracle.build()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle("restatement")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("reference"):
        pytest.skip("reference library (oracle/_ref) not built on this host")
    return oracle.Oracle("reference")


def to_oracle_sched(s):
    import oracle
    return oracle.Schedule(s.flip_deg, s.phase_deg, s.tr_ms, s.te_ms)


def to_oracle_grid(g):
    import oracle
    return oracle.make_grid((g.t1_ms.min, g.t1_ms.step, g.t1_ms.count),
                            (g.t2_ms.min, g.t2_ms.step, g.t2_ms.count),
                            (g.df_hz.min, g.df_hz.step, g.df_hz.count))
