"""The reference's behavioural tests (test_schwarz.py, test_krylov.py)
restated for the GPU path (B200 only).  Coefficient fields are seeded
two-phase inclusions of the given contrast."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2006_13387_b200 as G  # noqa: E402
from paper_2006_13387_b200.krylov import estimate_condition  # noqa: E402


def setup_problem(nx, Nx, eta=1e4, seed=3):
    mesh = G.build_fine_mesh(nx, nx)
    part = G.build_coarse_partition(mesh, Nx, Nx)
    rng = np.random.default_rng(seed)
    E = np.where(rng.random(mesh.n_elements) < 0.25, 1.0, 1.0 / eta) if eta != 1.0 else np.ones(mesh.n_elements)
    coeff = G.CoefficientField(E, 0.3, float(E.min()), 1.0)
    dirichlet = mesh.boundary_nodes()
    op = G.assemble_elasticity(mesh, coeff, dirichlet)
    return mesh, part, coeff, dirichlet, op


def test_heat_level1_shares_scalar_factorization(rng):
    """test_schwarz.py:107-117."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=20, Nx=2)
    hh = G.build_preconditioner("HH", op, mesh, part, coeff, dirichlet, G.EigOptions(n_max=2))
    v, w = rng.standard_normal(op.n_free), rng.standard_normal(op.n_free)
    assert v @ hh.apply(w) == pytest.approx(w @ hh.apply(v), rel=1e-10)
    _, report = G.pcg_solve(op, v, hh, tol=1e-6)
    assert report.converged


def test_coarse_dims_and_iterations_match_at_contrast_one(rng):
    """test_schwarz.py:119-137: at contrast 1 EE (3 elasticity modes) and
    EH+Rot (constant heat mode x 2 + rotation) span 3 functions per node."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=40, Nx=4, eta=1.0)
    b = rng.standard_normal(op.n_free)
    iters = {}
    for tag in ("EE", "EH+Rot"):
        pre = G.build_preconditioner(tag, op, mesh, part, coeff, dirichlet, G.EigOptions(n_max=3))
        assert pre.coarse_dim == 3 * part.n_neighborhoods
        _, report = G.pcg_solve(op, b, pre, tol=1e-6)
        assert report.converged
        iters[tag] = report.iterations
    assert abs(iters["EE"] - iters["EH+Rot"]) <= 2


def test_snapshot_count_insensitivity(rng):
    """test_schwarz.py:139-152 (10 snapshots in a 16-column block, 15 in a
    32-column block)."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=40, Nx=4, eta=1e4)
    b = rng.standard_normal(op.n_free)
    iters = []
    for n_snap in (10, 15):
        pre = G.build_preconditioner("EE;Rand", op, mesh, part, coeff, dirichlet,
                                     G.EigOptions(n_max=6, n_snapshots=n_snap))
        _, report = G.pcg_solve(op, b, pre, tol=1e-6)
        assert report.converged
        iters.append(report.iterations)
    assert abs(iters[0] - iters[1]) <= 2


def test_too_many_snapshots_rejected():
    mesh, part, coeff, dirichlet, op = setup_problem(nx=20, Nx=2)
    with pytest.raises(ValueError):
        G.build_preconditioner("EE;Rand", op, mesh, part, coeff, dirichlet, G.EigOptions(n_snapshots=30))


def test_preconditioned_operator_positive_ritz(rng):
    """test_schwarz.py:154-163, for every variant the GPU builds."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=20, Nx=2, eta=1e4)
    b = rng.standard_normal(op.n_free)
    for tag in ("EE", "HH", "HH+Rot", "EH", "EH+Rot", "EE;Rand", "EH+Rot;Rand"):
        pre = G.build_preconditioner(tag, op, mesh, part, coeff, dirichlet, G.EigOptions(n_max=3))
        _, report = G.pcg_solve(op, b, pre, tol=1e-6, check_symmetry=True)
        assert report.converged and report.ritz_min > 0.0 and report.ritz_max > 0.0, tag


def test_build_info_records_metadata():
    """test_schwarz.py:165-174."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=20, Nx=2)
    pre = G.build_preconditioner("EH+Rot", op, mesh, part, coeff, dirichlet, G.EigOptions(n_max=3))
    info = pre.info
    assert info["coarse_dim"] == pre.coarse_dim
    assert info["selection_rule"] == "gap"
    assert len(info["mode_counts"]) == part.n_neighborhoods
    assert info["t_coarse"] >= 0.0


def test_krylov_report_behaviour(rng, tmp_path):
    """test_krylov.py:93-116: true residual, nondecreasing condition history,
    residual CSV export."""
    mesh, part, coeff, dirichlet, op = setup_problem(nx=40, Nx=4, eta=1e2)
    pre = G.build_preconditioner("EH+Rot", op, mesh, part, coeff, dirichlet)
    b = rng.standard_normal(op.n_free)
    x, report = G.pcg_solve(op, b, pre, tol=1e-10)
    assert report.converged
    assert np.linalg.norm(b - op @ x) <= 2e-10 * np.linalg.norm(b)
    assert report.residuals[-1] <= 1e-10
    history = [estimate_condition(report, upto=j) for j in range(1, report.iterations + 1)]
    assert all(hb >= ha - 1e-9 * ha for ha, hb in zip(history, history[1:]))
    path = tmp_path / "residuals.csv"
    report.write_residual_csv(path)
    rows = path.read_text().strip().splitlines()
    assert rows[0] == "iteration,relative_residual" and len(rows) == len(report.residuals) + 1


_OVERLAP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2006_13387_b200 as G
mesh = G.build_fine_mesh(64, 64)
part = G.build_coarse_partition(mesh, 4, 4)
rng = np.random.default_rng(7)
E = np.where(rng.random(mesh.n_elements) < 0.3, 1.0, 1e-4)
coeff = G.CoefficientField(E, 0.3, 1e-4, 1.0)
op = G.assemble_elasticity(mesh, coeff, mesh.boundary_nodes())
pre = G.build_preconditioner("EH+Rot", op, mesh, part, coeff, mesh.boundary_nodes())
b = rng.standard_normal(op.n_free)
x, rep = G.pcg_solve(op, b, pre, tol=1e-8)
np.save(sys.argv[2], np.concatenate([x, np.asarray(rep.residuals), pre.apply(b)]))
"""


def test_coarse_branch_overlap_is_bit_identical(tmp_path):
    """The coarse restriction + SYMV forked onto a second stream (opt-in,
    MS_OVERLAP=1) gives the same bits as the serial apply."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    script = tmp_path / "ov.py"
    script.write_text(_OVERLAP_SCRIPT)
    out = {}
    for ov in ("1", "0"):
        env = dict(os.environ, MS_OVERLAP=ov)
        subprocess.run([sys.executable, str(script), root, str(tmp_path / f"ov{ov}.npy")], check=True, env=env,
                       timeout=600)
        out[ov] = np.load(tmp_path / f"ov{ov}.npy")
    assert np.array_equal(out["0"], out["1"])


@pytest.mark.gpu
def test_block_cache_reuses_and_releases_device_memory():
    """Released C-ABI buffers are kept for reuse (a rebuild of the same
    preconditioner is served from the cache) and returned on request."""
    import paper_2006_13387_b200 as G
    from paper_2006_13387_b200 import _lib, configs
    from paper_2006_13387_b200.solve import setup_spec

    spec = configs.config1(seed=0, n=64, H=16, delta=1)
    G.release_cached_memory()
    assert _lib.cache_trim(False) == 0
    mesh, op, pre = setup_spec(spec)
    x1, r1 = G.pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=5000)
    del pre
    held = _lib.cache_trim(False)
    assert held > 0
    pre = G.build_preconditioner("EH+Rot", op, mesh, G.build_coarse_partition(mesh, spec.Nx, spec.Ny), op.coeff,
                                 spec.heat_dirichlet_nodes, G.EigOptions(), level1="blocks", delta=spec.delta)
    assert _lib.cache_trim(False) < held  # the rebuild took its buffers from the cache
    x2, r2 = G.pcg_solve(op, spec.rhs(), pre, tol=1e-8, maxit=5000)
    assert r1.iterations == r2.iterations and np.array_equal(x1, x2)
    del pre, op
    assert G.release_cached_memory() > 0
    assert _lib.cache_trim(False) == 0
