"""The duck-typed operands of ``pcg_solve`` (krylov.py:73-78, 90) on the GPU.

The reference's solver takes any sparse / dense matrix or callable as ``A``
and any ``.apply`` object, callable or ``None`` as ``M``; its own
tests/test_krylov.py exercises exactly these seams (diagonal systems, an exact
preconditioner, Lanczos condition estimates, maxit, symmetry check, the
elasticity operator's ``.matrix`` against a direct solve).  The same
behaviours are checked here through the drop-in: CSR operands run on the
device (ms_csr), callables through host callbacks, the recurrence itself in
ms_pcg_solve_generic.  The oracle's PCG (pinned to the reference) is the
checker for iteration counts and iterates.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2006_13387_b200 as G

    return G


@pytest.fixture(scope="module")
def O():
    from oracle import mselast_oracle as O

    return O


class Wrapped:
    """An object whose only interface is .apply (the reference's preconditioner duck type)."""

    def __init__(self, fn):
        self.apply = fn


def spd(n, seed, shift):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((n, n))
    return sp.csr_matrix(B @ B.T + shift * np.eye(n)), rng.standard_normal(n)


def test_diagonal_system_terminates_within_n(G):
    n = 14
    A = sp.diags(np.linspace(1.0, 9.0, n)).tocsr()
    x, rep = G.pcg_solve(A, np.ones(n), tol=1e-12, maxit=5 * n)
    assert rep.converged and rep.iterations <= n
    assert np.allclose(A @ x, np.ones(n), atol=1e-10)


def test_exact_preconditioner_object_converges_in_one_step(G):
    n = 33
    d = np.geomspace(1.0, 80.0, n)
    x, rep = G.pcg_solve(sp.diags(d).tocsr(), np.ones(n), Wrapped(lambda r: r / d), tol=1e-10)
    assert rep.iterations == 1
    assert G.estimate_condition(rep) == pytest.approx(1.0, abs=1e-8)
    assert np.allclose(x, 1.0 / d)


def test_callable_preconditioner_and_callable_operator(G, O):
    A, b = spd(70, 11, 400.0)  # well conditioned: converges long before n steps
    dinv = 1.0 / A.diagonal()
    x1, r1 = G.pcg_solve(A, b, lambda r: dinv * r, tol=1e-10)
    x2, r2 = G.pcg_solve(lambda v: A @ v, b, Wrapped(lambda r: dinv * r), tol=1e-10)
    xo, ro = O.pcg(A, b, Wrapped(lambda r: dinv * r), tol=1e-10, maxit=2000)
    assert r1.converged and r2.converged
    assert r1.iterations == r2.iterations == ro.iterations
    assert np.allclose(x1, xo, rtol=0, atol=1e-12 * np.linalg.norm(xo))
    assert np.allclose(x2, xo, rtol=0, atol=1e-12 * np.linalg.norm(xo))
    assert np.allclose(r1.residuals, ro.residuals, rtol=1e-4)


def test_dense_ndarray_operand_and_two_by_two_condition(G):
    _, rep = G.pcg_solve(np.diag([1.0, 4.0]), np.array([1.0, 1.0]), tol=1e-12)
    assert G.estimate_condition(rep) == pytest.approx(4.0, rel=1e-6)
    # the 'None' variant's IdentityPreconditioner is the same solve as M = None
    _, rep_id = G.pcg_solve(np.diag([1.0, 4.0]), np.array([1.0, 1.0]), G.IdentityPreconditioner(), tol=1e-12)
    assert rep_id.iterations == rep.iterations and rep_id.residuals == rep.residuals


def test_condition_estimate_scale_invariant_and_monotone(G):
    rng = np.random.default_rng(2)
    n = 48
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = sp.csr_matrix(Q @ np.diag(np.linspace(1, 25, n)) @ Q.T)
    b = rng.standard_normal(n)
    _, r1 = G.pcg_solve(A, b, tol=1e-10)
    _, r2 = G.pcg_solve(A, 3 * b, tol=1e-10)
    assert G.estimate_condition(r1) == pytest.approx(G.estimate_condition(r2), rel=1e-6)
    hist = [G.estimate_condition(r1, upto=j) for j in range(1, r1.iterations + 1)]
    assert all(b_ >= a_ - 1e-9 * a_ for a_, b_ in zip(hist, hist[1:]))
    assert hist[-1] <= 25.0 * (1 + 1e-6)


def test_deterministic_and_history_lengths(G, tmp_path):
    A, b = spd(60, 3, 5.0)
    x1, r1 = G.pcg_solve(A, b, tol=1e-8)
    x2, r2 = G.pcg_solve(A, b, tol=1e-8)
    assert np.array_equal(x1, x2) and r1.iterations == r2.iterations
    assert r1.converged and r1.residuals[0] == 1.0 and r1.residuals[-1] <= 1e-8
    assert len(r1.residuals) == r1.iterations + 1 and len(r1.alphas) == r1.iterations
    assert len(r1.betas) == r1.iterations - 1
    assert np.linalg.norm(b - A @ x1) <= 1e-8 * np.linalg.norm(b) * 1.01
    r1.write_residual_csv(tmp_path / "res.csv")
    rows = (tmp_path / "res.csv").read_text().strip().splitlines()
    assert rows[0] == "iteration,relative_residual" and len(rows) == len(r1.residuals) + 1


def test_maxit_stops_unconverged_with_k_betas(G):
    n = 50
    A = sp.diags(np.geomspace(1e-6, 1.0, n)).tocsr()
    _, rep = G.pcg_solve(A, np.ones(n), tol=1e-14, maxit=3)
    assert not rep.converged and rep.iterations == 3
    assert len(rep.betas) == 3  # krylov.py:123-127: beta recorded after every non-final iteration


def test_zero_right_hand_side_and_bad_arguments(G):
    A = sp.identity(5, format="csr")
    x, rep = G.pcg_solve(A, np.zeros(5))
    assert rep.converged and rep.iterations == 0 and np.array_equal(x, np.zeros(5)) and rep.residuals == [1.0]
    with pytest.raises(ValueError):
        G.pcg_solve(A, np.ones(5), tol=2.0)
    with pytest.raises(ValueError):
        G.pcg_solve(A, np.ones(4))
    with pytest.raises(TypeError):
        G.pcg_solve("not an operator", np.ones(5))


def test_nonsymmetric_preconditioner_detected(G):
    n = 12
    A = sp.diags(np.arange(1.0, n + 1)).tocsr()
    S = np.triu(np.ones((n, n)))
    with pytest.raises(ValueError):
        G.pcg_solve(A, np.ones(n), Wrapped(lambda r: S @ r), check_symmetry=True)


def test_exception_in_callable_operand_propagates(G):
    A = sp.identity(6, format="csr")

    def broken(r):
        raise ZeroDivisionError("boom")

    with pytest.raises(ZeroDivisionError):
        G.pcg_solve(A, np.ones(6), broken)


def test_elasticity_operator_matrix_against_direct_solve(G, O):
    """``pcg_solve(op.matrix, b)`` on the Q1 operator (the reference's
    TestAgainstDirectOracle), the operator's scipy export against the oracle's
    assembled CSR, and a foreign preconditioner object on the GPU operator."""
    mesh = G.build_fine_mesh(20, 20)
    rng = np.random.default_rng(5)
    E = rng.uniform(1e-4, 1.0, mesh.n_elements)
    coeff = G.CoefficientField(E, 0.3, 1e-4, 1.0)
    op = G.assemble_elasticity(mesh, coeff, mesh.boundary_nodes())
    b = rng.standard_normal(op.n_free)
    x, rep = G.pcg_solve(op.matrix, b, tol=1e-8, maxit=5000)
    assert rep.converged
    K = op.matrix.tocsc()
    xd = spla.spsolve(K, b)
    assert np.linalg.norm(x - xd) <= 1e-5 * np.linalg.norm(xd)
    omesh = O.mesh_for(20, 20)
    Ko = O.elasticity_operator(omesh, E, 0.3, O.whole_node_dofs(omesh, mesh.boundary_nodes())).matrix
    assert abs(K - Ko).max() <= 1e-13 * abs(Ko).max()
    assert (K != 0).sum() == (Ko != 0).sum()
    # Jacobi through the .apply seam on the GPU operator, and the exported CSR on the generic path
    dinv = 1.0 / K.diagonal()
    xj, rj = G.pcg_solve(op, b, Wrapped(lambda r: dinv * r), tol=1e-8, maxit=5000)
    xc, rc = G.pcg_solve(op.matrix.tocsr(), b, Wrapped(lambda r: dinv * r), tol=1e-8, maxit=5000)
    xo, ro = O.pcg(Ko, b, Wrapped(lambda r: dinv * r), tol=1e-8, maxit=5000)
    assert rj.converged and rc.converged
    assert abs(rj.iterations - ro.iterations) <= 1 and abs(rc.iterations - ro.iterations) <= 1
    assert np.linalg.norm(xj - xo) <= 1e-7 * np.linalg.norm(xo)
    assert np.linalg.norm(xc - xo) <= 1e-7 * np.linalg.norm(xo)


def test_two_level_preconditioner_on_a_foreign_matrix(G, O):
    """The GPU TwoLevelPreconditioner as M for a scipy CSR A (the reference's
    composition ``pcg_solve(op.matrix, b, pre)`` with a foreign matrix type):
    same iterates as the fused path."""
    mesh = G.build_fine_mesh(40, 40)
    rng = np.random.default_rng(9)
    E = np.where(rng.random(mesh.n_elements) < 0.3, 1.0, 1e-4)
    coeff = G.CoefficientField(E, 0.3, 1e-4, 1.0)
    dn = mesh.boundary_nodes()
    op = G.assemble_elasticity(mesh, coeff, dn)
    part = G.build_coarse_partition(mesh, 4, 4)
    pre = G.build_preconditioner("EH+Rot", op, mesh, part, coeff, dn)
    b = rng.standard_normal(op.n_free)
    xf, rf = G.pcg_solve(op, b, pre, tol=1e-8)
    xg, rg = G.pcg_solve(op.matrix.tocsr(), b, pre, tol=1e-8)
    xh, rh = G.pcg_solve(op, b, pre.apply, tol=1e-8)  # the bound method as a plain callable
    assert rf.converged and rg.converged and rh.converged
    assert abs(rg.iterations - rf.iterations) <= 1 and abs(rh.iterations - rf.iterations) <= 1
    assert np.linalg.norm(xg - xf) <= 1e-7 * np.linalg.norm(xf)
    assert np.linalg.norm(xh - xf) <= 1e-7 * np.linalg.norm(xf)


def test_device_tensors_through_the_generic_path(G):
    """b as a float64 CUDA tensor with a CSR operand: x comes back as a CUDA
    tensor (nothing but the callback operands crosses PCIe); the CSR operator
    itself applies to host and device vectors."""
    import torch

    from paper_2006_13387_b200.krylov import CsrOperator

    A, b = spd(80, 21, 300.0)
    op = CsrOperator(A)
    v = np.random.default_rng(4).standard_normal(80)
    assert np.allclose(op @ v, A @ v, rtol=0, atol=1e-12 * np.abs(A @ v).max())
    vd = torch.from_numpy(v).cuda()
    assert np.allclose((op @ vd).cpu().numpy(), A @ v, rtol=0, atol=1e-12 * np.abs(A @ v).max())
    xh, rh = G.pcg_solve(op, b, tol=1e-10)
    xd, rd = G.pcg_solve(op, torch.from_numpy(b).cuda(), tol=1e-10)
    assert isinstance(xd, torch.Tensor) and xd.is_cuda
    assert rd.iterations == rh.iterations and np.array_equal(xd.cpu().numpy(), xh)
    with pytest.raises(ValueError):
        CsrOperator(sp.csr_matrix(np.ones((3, 4))))
