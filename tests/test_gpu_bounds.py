"""Device-side bounds checks of the ring / halo / gather index arithmetic.

compute-sanitizer is closed on the GPU pool, so the library has its own
checked build: `make check` compiles every kernel with -DMS_BOUNDS_CHECK
(`MS_BCHECK` in common.cuh asserts chunk ranges of the bulk-copy rings, the
level-1 gathers, the cell loops, the SYMV tile ranges ... and traps with the
failing expression), into build/check/libmsgpu_check.so.  The cases below run
every level-1 layout (plain, twisted, one factor copy in both backward forms,
padded TMA ring, heat, dense inverses, Cholesky coarse solve), ragged meshes,
the generic PCG and the multi-rank strips through that library in a
subprocess; a trap fails the subprocess and its message is shown.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
CHECK_LIB = ROOT / "build" / "check" / "libmsgpu_check.so"

CASE = r"""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import scipy.sparse as sp
from paper_2006_13387_b200 import configs, pcg_solve, _lib
from paper_2006_13387_b200.solve import setup_spec
assert "libmsgpu_check" in str(_lib.LIB_PATH)
tag = os.environ.get("CASE_TAG", "EH+Rot")
kw = {}
if os.environ.get("CASE_DENSE"):
    kw["local_solver"] = "dense"
if os.environ.get("CASE_CHOL"):
    kw["coarse_solve"] = "cholesky"
shape = os.environ.get("CASE_SHAPE", "config1")
if shape == "config1":
    spec = configs.config1(seed=0, n=64, H=16, delta=2)
elif shape == "strip":
    spec = configs.config3(seed=0, n=128, ny=64)
else:
    spec = configs.config4(seed=0, nx=128, ny=64)
mesh, op, pre = setup_spec(spec, tag, **kw)
x, rep = pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=400)
r = np.random.default_rng(0).standard_normal(op.n_free)
z = pre.apply(r)
assert np.all(np.isfinite(x)) and np.all(np.isfinite(z))
A = sp.diags(np.linspace(1.0, 9.0, 50)).tocsr()
xg, repg = pcg_solve(A, np.ones(50), lambda v: v / A.diagonal(), tol=1e-10)
assert repg.converged
print("ok", tag, shape, rep.iterations, pre.info["level1_twisted"], pre.info["level1_copies"], pre.info["level1_unit"])
"""

CASES = [
    ("plain", {"MS_L1_TWIST": "0"}),
    ("twisted", {"MS_L1_TWIST": "1"}),
    ("twisted-deep-ring", {"MS_L1_TWIST": "1", "MS_L1_NST": "6"}),
    ("cholesky-factors", {"MS_L1_UNIT": "0", "MS_L1_TWIST": "1"}),
    ("one-copy-dot", {"MS_L1_COPIES": "1", "MS_L1_BWD": "dot", "MS_L1_TWIST": "0"}),
    ("one-copy-window", {"MS_L1_COPIES": "1", "MS_L1_TWIST": "0"}),
    ("one-copy-twisted", {"MS_L1_COPIES": "1", "MS_L1_TWIST": "1"}),
    ("padded-ring", {"MS_L1_PAD": "1", "MS_L1_TWIST": "0"}),
    ("register-sweeps", {"MS_L1_SWEEP": "reg", "MS_L1_TWIST": "0"}),
    ("heat-level1", {"CASE_TAG": "HH+Rot"}),
    ("heat-level1-twisted", {"CASE_TAG": "HH+Rot", "MS_L1_TWIST": "1"}),
    ("elasticity-eigs", {"CASE_TAG": "EE"}),
    ("dense-inverses", {"CASE_DENSE": "1"}),
    ("cholesky-coarse", {"CASE_CHOL": "1"}),
    ("combine-per-node", {"MS_COMBINE": "0"}),
    ("no-table-sharing", {"MS_CHI_DEDUP": "0", "MS_PSI0_CONST": "0"}),
    ("symv-register-tiles", {"MS_SYMV": "0"}),
    ("strip-mesh", {"CASE_SHAPE": "strip"}),
    ("mbb-mesh", {"CASE_SHAPE": "mbb"}),
]


def run_checked(args, extra_env, timeout=900):
    if not CHECK_LIB.exists():
        pytest.skip("bounds-checked library not built (make check)")
    env = dict(os.environ)
    env.update(extra_env)
    env["MSGPU_LIB"] = str(CHECK_LIB)
    p = subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    out = p.stdout + p.stderr
    assert "bounds check failed" not in out, out[-3000:]
    assert p.returncode == 0, out[-3000:]
    return out


@pytest.mark.parametrize("name,env", CASES, ids=[c[0] for c in CASES])
def test_level1_layouts_under_bounds_checks(name, env):
    out = run_checked([sys.executable, "-c", CASE], env)
    assert "ok " in out


def test_multi_rank_strips_under_bounds_checks():
    """2 / 4 / 8 callback ranks on one GPU (halo plans, boundary subdomain
    rows, restriction partials) through the checked library."""
    out = run_checked([sys.executable, "-m", "pytest", "tests/test_dist.py", "-m", "gpu", "-q", "-x", "-k",
                       "strip_ranks_on_one_gpu or two_ranks_on_one_gpu or operator_apply_before"], {}, timeout=1800)
    assert " passed" in out
