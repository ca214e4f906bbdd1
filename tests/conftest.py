import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    # oracle C restatement (+ the reference, when its sources are present)
    import oracle_py
    if not oracle_py.available("orc") or (os.path.isdir("/root/reference/proj")
                                          and not oracle_py.available("ref")):
        target = "all" if os.path.isdir("/root/reference/proj") else "oracle"
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), target], check=True,
                       capture_output=True)
    from paper_2302_12454_b200 import build as b
    b.build()


_ensure_built()


@pytest.fixture(autouse=True)
def _reset_engine_tune():
    """Engine overrides (include/ssqa_tune.h) never leak from one test into the next.
    SSQA_TEST_TUNE="key=v,key=v" runs every test on top of those overrides (e.g.
    the whole GPU suite through an opt-in engine path)."""
    import paper_2302_12454_b200 as sq
    base = os.environ.get("SSQA_TEST_TUNE", "")
    if base:
        sq.tune(**{k: int(v) for k, v in (kv.split("=") for kv in base.split(","))})
    yield
    sq.tune()


@pytest.fixture(scope="session")
def orc():
    import oracle_py
    return oracle_py.Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    import oracle_py
    if not oracle_py.available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle_py.Oracle("ref")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        cases = {}
        for key in z.files:
            case, field = key.split("/", 1)
            cases.setdefault(case, {})[field] = z[key]
        return cases
    return load


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
