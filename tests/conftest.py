import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


def pytest_terminal_summary(terminalreporter):
    """Report the worst GPU-vs-oracle soft errors seen (whole-tensor rel-L2 and the largest
    per-subcarrier rel-L2), SURVEY 8(c)'s parity contract."""
    mod = sys.modules.get("tests.test_gpu_parity") or sys.modules.get("test_gpu_parity")
    worst = getattr(mod, "WORST", None)
    if worst and (worst["rel_l2"] or worst["max_subcarrier"]):
        terminalreporter.write_line(
            f"parity worst: rel-L2 {worst['rel_l2']:.3e}, max per-subcarrier rel-L2 {worst['max_subcarrier']:.3e} "
            f"(bar 1e-4)")
    dbp = sys.modules.get("paper_1702_04458_b200.dbp")
    if dbp is not None and getattr(dbp, "_lib", None) is not None:
        terminalreporter.write_line(f"libdbp loaded from {dbp.LIB_PATH}")
