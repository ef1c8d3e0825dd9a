import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")
# the reference install (baseline/install_ref.sh): drop-in type identity + the reference arm
if os.path.isdir(os.path.join(REF_INSTALL, "ncstream")) and REF_INSTALL not in sys.path:
    sys.path.append(REF_INSTALL)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    g = np.load(GOLDEN, allow_pickle=False)
    return {k: g[k] for k in g.files}


def golden_cases(g, prefix=""):
    return [c for c in g["__cases__"].tolist() if c.startswith(prefix)]
