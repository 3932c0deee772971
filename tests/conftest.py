import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built libgeer.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def tiny():
    import workloads as W
    g, pairs, _ = W.load_config("tiny", with_lambda=True)
    return g, pairs


@pytest.fixture(scope="session")
def geer():
    """The built CUDA library (fails loudly without a device: there is no fallback)."""
    import importlib.util
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    spec = importlib.util.spec_from_file_location("geer_build", ROOT / "paper_2312_06123_b200" / "build.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.build()
    import paper_2312_06123_b200 as G
    return G


@pytest.fixture(scope="session")
def rmat20(geer):
    """BASELINE config 1 (R-MAT s20 ef5, 10k queries) with ARPACK's lambda (the paper's
    preprocessing), pinned for both the library and the oracle (R12)."""
    import workloads as W
    g, pairs, eps = W.load_config("rmat20", with_lambda=True)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    geer.er_graph_set_lambda(h, g.lam)
    return g, pairs, eps, h
