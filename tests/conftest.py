"""Shared test setup.

Markers: ``gpu`` tests need a B200 (run on the GPU box via gpurun / the
driver); everything else runs on CPU.  BLAS is pinned to one thread: the
multi-threaded OpenBLAS in this image is pathologically slow on small
LAPACK calls (measured 200x on 441^2 ?sygvx).
"""

import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import pytest  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

try:
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
except Exception:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def load_golden(name):
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
